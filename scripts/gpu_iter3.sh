mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python scripts/probe_config4.py --scale 0.25 --steps 3 > gpurun_out/probe4_q.log 2>&1; echo "rc=$?" >> gpurun_out/probe4_q.log
timeout 1500 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
