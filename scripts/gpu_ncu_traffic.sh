# DRAM bytes of every rounding launch of one full-scale config-4 step (the
# flux phase is the third round_bin_kernel group of a step), plus a launch
# list and a full-set capture of the config-3 microbench's rounding launch.
mkdir -p gpurun_out
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size \
  --clock-control none -k regex:"round_" --csv --log-file gpurun_out/traffic4.csv \
  python scripts/probe_config4.py --scale 1.0 --steps 2 > gpurun_out/traffic4.log 2>&1; echo "rc=$?" >> gpurun_out/traffic4.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench3.csv \
  python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch3.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch3.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:round_gram -s 3 -c 1 \
  -o gpurun_out/prof_c3 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full3.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full3.log
