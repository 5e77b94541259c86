mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_obstacle.py -q -m gpu > gpurun_out/pytest_obst.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_obst.log
timeout 600 python scripts/probe_config4.py --scale 0.25 --steps 2 > gpurun_out/probe4_q.log 2>&1; echo "rc=$?" >> gpurun_out/probe4_q.log
