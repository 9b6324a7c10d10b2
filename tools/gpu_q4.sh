mkdir -p gpurun_out
for bs in 16 32; do timeout 900 python tools/prefill_run.py --bs $bs --n 8 --reps 1 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print($bs, round(d['tok_s']), d['ms_per_step'], round(d['bubble_fraction'],3), d['compute_ms_by_kind'], d['resident_expert_layers'])"; done
