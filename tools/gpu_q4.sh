mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -1
for bs in 8 16; do timeout 900 python tools/prefill_run.py --bs $bs --n 8 --reps 1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($bs, round(d['tok_s']), d['ms_per_step'], round(d['bubble_fraction'],3), d['compute_ms_by_kind'])"; done
