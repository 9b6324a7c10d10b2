mkdir -p gpurun_out/sw
P="timeout 120 python tools/profile_kernels.py --only ffn"
$P --rows 32 --ks 1 > gpurun_out/sw/m32_ks1.txt 2>&1
$P --rows 32 --ks 1 --debug 1 > gpurun_out/sw/m32_ks1_d1.txt 2>&1
$P --rows 128 --stages 3 > gpurun_out/sw/m128_st3.txt 2>&1
$P --rows 128 --stages 3 --debug 1 > gpurun_out/sw/m128_st3_d1.txt 2>&1
$P --rows 128 --debug 2 > gpurun_out/sw/m128_d2.txt 2>&1
$P --rows 128 --hint 0 > gpurun_out/sw/m128_hint0.txt 2>&1
$P --rows 128 --whole 0 > gpurun_out/sw/m128_whole0.txt 2>&1
$P --rows 128 --whole 0 --debug 1 > gpurun_out/sw/m128_whole0_d1.txt 2>&1
