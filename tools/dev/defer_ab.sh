mkdir -p gpurun_out/ab
A="--no-prefill --no-q4 --no-ablation --no-cpu-baseline --no-x22b --sweep off --no-resident"
timeout 600 python bench.py $A > gpurun_out/ab/def.json 2>/dev/null
KL_NO_DEFER=1 timeout 600 python bench.py $A > gpurun_out/ab/nodef.json 2>/dev/null
timeout 600 python bench.py $A > gpurun_out/ab/def2.json 2>/dev/null
