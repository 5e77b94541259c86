mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 2000 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench5.log 2>&1; echo "rc=$?" >> gpurun_out/bench5.log
nvidia-smi --query-gpu=memory.used,memory.total --format=csv >> gpurun_out/bench5.log
