mkdir -p gpurun_out/nm
for nm in 1 2; do
timeout 300 python tools/profile_kernels.py --only attnop --nmma $nm > gpurun_out/nm/attnop_$nm.txt 2>&1
timeout 300 python tools/profile_kernels.py --only ffn --nmma $nm > gpurun_out/nm/ffn_$nm.txt 2>&1
done
