timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
timeout 600 python tools/op_timing.py --steps 2 2>&1 | grep -E "compute_expert|compute_attention|compute_gate"
