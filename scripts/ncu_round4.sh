mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:round_gram -c 6 -o gpurun_out/prof_round4c python scripts/probe_config4.py --scale 0.25 --steps 1 > gpurun_out/ncu_round4.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_round4.log
