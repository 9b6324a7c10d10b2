# Op-timestamp overhead probe: all-resident decode with and without the
# per-op stamp kernels (KL_PROBE_NO_STAMPS: the timeline is then invalid,
# only `value` -- whole-step events -- is meaningful).
bash tools/dev/resident_quick.sh stamps
KL_PROBE_NO_STAMPS=1 timeout 400 python bench.py --hbm-cap 140e9 --no-cpu-baseline --no-q4 --no-prefill --no-resident \
  --no-x22b --sweep off --no-ablation > gpurun_out/res_nostamps.json 2> gpurun_out/res_nostamps.err
python -c "import json;d=json.load(open('gpurun_out/res_nostamps.json'));print('nostamps', d['value'])"
