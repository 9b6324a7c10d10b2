mkdir -p gpurun_out/kv
for r in 1 2; do
for v in 0 1; do
timeout 300 python tools/profile_kernels.py --only attnop --kv-evict-first $v > gpurun_out/kv/kv${v}_$r.txt 2>&1
done; done
