timeout 600 python tools/op_timing.py --steps 2 2>&1 | grep -E "compute_expert|compute_attention|compute_gate"
