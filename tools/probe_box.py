"""One-off probe of the GPU box: host RAM, cores, PCIe pinned H2D bandwidth."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["meminfo"] = open("/proc/meminfo").read().splitlines()[:5]
out["nvidia_smi"] = subprocess.run(["nvidia-smi"], capture_output=True, text=True).stdout[-2500:]
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[-2000:]
out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout[:1500]
dev = torch.device("cuda:0")
res = {}
for mb in (8, 64, 352):
    n = mb * 1024 * 1024
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3): d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): d.copy_(h, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    res[f"h2d_{mb}MB_GBs"] = 10 * n / (s.elapsed_time(e) / 1e3) / 1e9
    s.record()
    for _ in range(10): h.copy_(d, non_blocking=True)
    e.record(); torch.cuda.synchronize()
    res[f"d2h_{mb}MB_GBs"] = 10 * n / (s.elapsed_time(e) / 1e3) / 1e9
# two streams concurrently
n = 352 * 1024 * 1024
hs = [torch.empty(n, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
ds = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(2)]
sts = [torch.cuda.Stream() for _ in range(2)]
torch.cuda.synchronize()
t0 = time.perf_counter()
for it in range(5):
    for i in range(2):
        with torch.cuda.stream(sts[i]): ds[i].copy_(hs[i], non_blocking=True)
torch.cuda.synchronize()
res["h2d_2streams_GBs"] = 10 * n / (time.perf_counter() - t0) / 1e9
# big pinned alloc test: how much can we pin
t0 = time.perf_counter()
big = []
try:
    for i in range(40):
        big.append(torch.empty(4 * 1024**3, dtype=torch.uint8, pin_memory=True))
except Exception as ex:
    res["pin_err"] = str(ex)[:200]
res["pinned_GB_ok"] = 4 * len(big)
res["pin_time_s"] = time.perf_counter() - t0
out["bw"] = res
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
print(json.dumps(res))
