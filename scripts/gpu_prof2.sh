mkdir -p gpurun_out
ROUND_PROF=1 python scripts/profile_step.py --scale 0.5 --steps 3 > gpurun_out/prof_phases.log 2>&1
python scripts/profile_step.py --scale 0.5 --steps 3 >> gpurun_out/prof_phases.log 2>&1
