mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 > gpurun_out/bench2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench2.log
python scripts/profile_step.py --scale 0.25 --steps 2 > gpurun_out/prof_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_small.csv python scripts/profile_step.py --scale 0.25 --steps 2 > gpurun_out/ncu_launch.log 2>&1
python scripts/profile_step.py --scale 0.25 --steps 2 > gpurun_out/prof_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:round_sums -s 5 -c 5 -o gpurun_out/prof_round python scripts/profile_step.py --scale 0.25 --steps 2 > gpurun_out/ncu_full.log 2>&1
echo done
