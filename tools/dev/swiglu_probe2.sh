mkdir -p gpurun_out/sw2
P="timeout 120 python tools/profile_kernels.py --only ffn"
$P --rows 128 --ks 3 > gpurun_out/sw2/m128_ks3.txt 2>&1
$P --rows 128 --ks 3 --debug 1 > gpurun_out/sw2/m128_ks3_d1.txt 2>&1
$P --rows 64 --ks 3 > gpurun_out/sw2/m64_ks3.txt 2>&1
$P --rows 160 --ks 3 > gpurun_out/sw2/m160_ks3.txt 2>&1
$P --rows 256 --ks 3 > gpurun_out/sw2/m256_ks3.txt 2>&1
