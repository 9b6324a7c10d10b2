mkdir -p gpurun_out/l2p
P="timeout 300 python tools/profile_kernels.py --only attnop"
$P > gpurun_out/l2p/base.txt 2>&1
$P --hint 2 > gpurun_out/l2p/w_last.txt 2>&1
$P --hint 2 --kv-evict-first 1 > gpurun_out/l2p/w_last_kv_first.txt 2>&1
$P --kv-evict-first 1 > gpurun_out/l2p/kv_first.txt 2>&1
$P --hint 0 > gpurun_out/l2p/nohint.txt 2>&1
