mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -m gpu -x -q -k "gate" 2>&1 | tail -2
timeout 120 python tools/profile_kernels.py --only route --iters 30 --gap-ms 0.05 2>&1 | grep -A1 "gate_topk\|permute\|combine" | grep -E "gate|perm|comb|us"
timeout 120 python tools/profile_kernels.py --only route --iters 30 2>&1 | grep -A1 "gate_topk" | grep -E "us"
