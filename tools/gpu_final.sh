# End-of-round evidence on one B200: every GPU test, smoke, the default bench
# line, ncu launch lists of one headline and one all-resident decode step, and
# the --set full capture of one expert FFN (summarised by tools/ncu_ffn_traffic.py).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -2 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
N="ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 $N --log-file gpurun_out/final_launches_resident.csv python tools/step_profile.py --resident > gpurun_out/sp_res.log 2>&1
timeout 900 $N --log-file gpurun_out/final_launches_headline.csv python tools/step_profile.py > gpurun_out/sp_head.log 2>&1
bash tools/gpu_ffn_ncu.sh
timeout 300 python tools/op_timing.py --steps 1 > gpurun_out/op_timing.txt 2>&1
