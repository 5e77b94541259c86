mkdir -p gpurun_out
ROUND_PROF=1 timeout 300 python scripts/profile_step.py --scale 0.25 --steps 3 > gpurun_out/prof_quick.log 2>&1
timeout 300 python scripts/profile_step.py --scale 0.25 --steps 3 >> gpurun_out/prof_quick.log 2>&1
