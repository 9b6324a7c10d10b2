mkdir -p gpurun_out/ffnp
P="timeout 300 python tools/profile_kernels.py --only ffn"
$P > gpurun_out/ffnp/base.txt 2>&1
$P --debug 3 > gpurun_out/ffnp/dbg3.txt 2>&1
$P --debug 1 > gpurun_out/ffnp/dbg1.txt 2>&1
$P --debug 128 > gpurun_out/ffnp/trace.txt 2>&1
$P --h2d > gpurun_out/ffnp/h2d.txt 2>&1
$P --h2d --debug 3 > gpurun_out/ffnp/h2d_dbg3.txt 2>&1
$P --h2d --debug 128 > gpurun_out/ffnp/h2d_trace.txt 2>&1
$P --kb 0 > gpurun_out/ffnp/rowmajor.txt 2>&1
