mkdir -p gpurun_out/l2a
for a in 0 2 4 8 16 32; do
  timeout 120 python tools/profile_kernels.py --only ffn --l2-ahead $a > gpurun_out/l2a/ffn_$a.txt 2>&1
done
for a in 0 8; do
  timeout 300 python tools/profile_kernels.py --only attnop --l2-ahead $a > gpurun_out/l2a/attnop_$a.txt 2>&1
done
timeout 120 python tools/profile_kernels.py --only ffn --l2-ahead 8 --rows 256 > gpurun_out/l2a/ffn256_8.txt 2>&1
timeout 120 python tools/profile_kernels.py --only ffn --l2-ahead 8 --rows 32 > gpurun_out/l2a/ffn32_8.txt 2>&1
