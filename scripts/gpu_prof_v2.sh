# ncu evidence for the committed kernel: bench launch list + full set on the rounding kernel
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_step.py --scale 0.25 --steps 2 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:round_sums -s 7 -c 7 -o gpurun_out/prof_round_v2 python scripts/profile_step.py --scale 0.25 --steps 2 > gpurun_out/ncu_full.log 2>&1
echo done
