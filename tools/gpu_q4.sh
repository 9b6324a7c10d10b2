timeout 600 python tools/op_timing.py --steps 2 2>&1 | grep -E "compute_expert"
KL_FFN_NO_FIRST_PDL=1 timeout 600 python tools/op_timing.py --steps 2 2>&1 | grep -E "compute_expert"
