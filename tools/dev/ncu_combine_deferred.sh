# ncu --set full of the deferred combine (the block's down-projection split
# sums + weighted combine + residual) at T = 512, one launch after warm-up.
mkdir -p gpurun_out
timeout 300 ncu --set full --clock-control none --import-source on -k regex:combine_deferred -s 3 -c 1 \
  -o gpurun_out/r02_full_combine_deferred -f python tools/profile_kernels.py --only route > gpurun_out/ncu_cd.log 2>&1
ncu -i gpurun_out/r02_full_combine_deferred.ncu-rep --page raw --csv \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,launch__grid_size \
  > gpurun_out/ncu_cd_raw.csv 2>&1
tail -3 gpurun_out/ncu_cd_raw.csv
