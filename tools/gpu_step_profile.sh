# ncu launch lists of one headline decode step and one all-resident step
# (round 2), isolated decode-path kernel timings, and a --set full capture
# of the small routing kernels.
mkdir -p gpurun_out
N="ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv"
timeout 900 $N --log-file gpurun_out/r02_launches_resident.csv python tools/step_profile.py --resident > gpurun_out/sp_res.log 2>&1; tail -2 gpurun_out/sp_res.log
timeout 900 $N --log-file gpurun_out/r02_launches_headline.csv python tools/step_profile.py > gpurun_out/sp_head.log 2>&1; tail -2 gpurun_out/sp_head.log
timeout 300 python tools/profile_kernels.py --only attn > gpurun_out/pk_attn.txt 2>&1
timeout 300 python tools/profile_kernels.py --only route > gpurun_out/pk_route.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"combine|permute|gate_topk|rmsnorm|rope" -c 12 -o gpurun_out/r02_small_kernels -f python tools/profile_kernels.py --only route > gpurun_out/ncu_small.log 2>&1; tail -3 gpurun_out/ncu_small.log
