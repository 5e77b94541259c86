mkdir -p gpurun_out
python scripts/profile_step.py --scale 0.25 --steps 2 > gpurun_out/prof_plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:round_sums -s 6 -c 5 -o gpurun_out/prof_round_v3 python scripts/profile_step.py --scale 0.25 --steps 2 > gpurun_out/ncu_full3.log 2>&1
echo done
