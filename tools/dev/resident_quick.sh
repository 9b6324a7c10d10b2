# All-resident decode (compute-exposed) only: bench headline at a 140e9 B cap.
timeout 400 python bench.py --hbm-cap 140e9 --no-cpu-baseline --no-q4 --no-prefill --no-resident --no-x22b \
  --sweep off --no-ablation > gpurun_out/res_${1:-x}.json 2> gpurun_out/res_${1:-x}.err
python -c "import json;d=json.load(open('gpurun_out/res_${1:-x}.json'));print('${1:-x}', d['value'], d['pipeline']['bubble_fraction'], d['roofline']['expert_op_us_in_step'])"
