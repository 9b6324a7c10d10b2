mkdir -p gpurun_out
KL_ENGINE_DIAG=1 timeout 600 python tools/op_timing.py --steps 2 2>&1 | grep -E "compute_|breakdown"
