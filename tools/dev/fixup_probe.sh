mkdir -p gpurun_out/fx
timeout 900 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "weight_streaming or expert_ffn" > gpurun_out/fx/tests.log 2>&1; tail -2 gpurun_out/fx/tests.log
P="timeout 120 python tools/profile_kernels.py --only ffn"
$P > gpurun_out/fx/ffn.txt 2>&1
$P --debug 128 > gpurun_out/fx/ffn_tr.txt 2>&1
$P --bulk-publish 1 > gpurun_out/fx/ffn_bulk.txt 2>&1
$P --bulk-publish 1 --debug 128 > gpurun_out/fx/ffn_bulk_tr.txt 2>&1
$P --fused-fixup 0 > gpurun_out/fx/ffn_nofuse.txt 2>&1
timeout 300 python tools/profile_kernels.py --only attnop > gpurun_out/fx/attnop.txt 2>&1
timeout 300 python tools/profile_kernels.py --only attnop --bulk-publish 1 > gpurun_out/fx/attnop_bulk.txt 2>&1
