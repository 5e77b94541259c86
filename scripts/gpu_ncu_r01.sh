# round-1 ncu evidence for the config-4 bench: launch list of the bench command
# (every kernel's duration, serialised) and a full-set capture of the rounding
# kernel's flux launches of one full-scale step
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch4.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch4.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:round_gram -s 2 -c 3 -o gpurun_out/prof_r01_round4 python scripts/probe_config4.py --scale 1.0 --steps 1 > gpurun_out/ncu_full4.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full4.log
