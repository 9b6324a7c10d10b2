mkdir -p gpurun_out/is
timeout 300 python tools/op_timing.py --steps 1 > gpurun_out/is/default.txt 2>&1
timeout 300 python tools/op_timing.py --steps 1 --tune 12=2 > gpurun_out/is/ks2.txt 2>&1
timeout 300 python tools/op_timing.py --steps 1 --tune 16=0 > gpurun_out/is/nofuse.txt 2>&1
timeout 300 python tools/op_timing.py --steps 1 --pdl 0 > gpurun_out/is/nopdl.txt 2>&1
for hg in 1 2 4 8; do timeout 120 python tools/profile_kernels.py --only attnop --decode-hg $hg > gpurun_out/is/attnop_hg$hg.txt 2>&1; done
