mkdir -p gpurun_out/ds
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -q -x -k "decode or rope" > gpurun_out/ds/tests.log 2>&1; tail -2 gpurun_out/ds/tests.log
for st in 0 5; do
timeout 300 python tools/profile_kernels.py --only attnop --decode-stages $st > gpurun_out/ds/st$st.txt 2>&1
done
