# Round-1 (session 5) ncu evidence on the current kernels: launch list of the
# bench command, then a full-set capture of flux/residual rounding launches
# with source-line stall attribution (scripts/ncu_box_round.sh).
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_bench4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch4.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch4.log
bash scripts/ncu_box_round.sh 0.5 30 12 > gpurun_out/ncu_box.log 2>&1
