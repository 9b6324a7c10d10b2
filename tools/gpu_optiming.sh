mkdir -p gpurun_out
timeout 300 python tools/profile_kernels.py --iters 20 --only attn --debug 128 2>&1 | grep -v '^ *"GBs\|^{\|^}\|},'
timeout 300 python tools/profile_kernels.py --iters 20 --only attn --no-stream 2>&1 | grep '"us"'
