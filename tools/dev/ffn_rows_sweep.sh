mkdir -p gpurun_out/rows
for r in 16 32 64 96 128 160 192 256; do
  timeout 120 python tools/profile_kernels.py --only ffn --rows $r > gpurun_out/rows/r$r.txt 2>&1
  timeout 120 python tools/profile_kernels.py --only ffn --rows $r --debug 1 > gpurun_out/rows/r${r}_d1.txt 2>&1
done
