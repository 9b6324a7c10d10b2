"""Pinned host -> HBM copy throughput by concurrency and transfer size: is one
copy stream the link's ceiling, or do 2-4 concurrent copies (several copy
engines) or other transfer sizes move more bytes per second?

    python tools/h2d_probe.py  ->  JSON {case: GB/s}
"""
import json

import torch


def main():
    dev = torch.device("cuda:0")
    total = 1 << 31  # 2 GiB per measurement
    h = torch.empty(total, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(total, dtype=torch.uint8, device=dev)
    res = {}

    def run(n_streams, chunk):
        streams = [torch.cuda.Stream() for _ in range(n_streams)]
        for _ in range(2):
            d[:chunk].copy_(h[:chunk], non_blocking=True)
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        start = torch.cuda.Event()
        start.record()
        n = total // chunk
        for i in range(n):
            st = streams[i % n_streams]
            st.wait_event(start)
            with torch.cuda.stream(st):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for st in streams:
            ev = torch.cuda.Event()
            ev.record(st)
            torch.cuda.current_stream().wait_event(ev)
        e.record()
        torch.cuda.synchronize()
        return n * chunk / (s.elapsed_time(e) / 1e3) / 1e9

    for n_streams in (1, 2, 3, 4):
        for chunk_mb in (16, 64, 352, 512):
            chunk = chunk_mb << 20
            res[f"streams{n_streams}_chunk{chunk_mb}MB"] = round(max(run(n_streams, chunk) for _ in range(2)), 2)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
