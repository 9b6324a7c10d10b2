mkdir -p gpurun_out/oe
for e in 0 4 8 12 16; do
  timeout 120 python tools/profile_kernels.py --only ffn --owner-extra $e > gpurun_out/oe/ffn_$e.txt 2>&1
  timeout 120 python tools/profile_kernels.py --only ffn --owner-extra $e --debug 128 > gpurun_out/oe/ffn_tr_$e.txt 2>&1
done
for e in 0 4 8; do
  timeout 300 python tools/profile_kernels.py --only attnop --split 2 --owner-extra $e > gpurun_out/oe/attnop_$e.txt 2>&1
done
