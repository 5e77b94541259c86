# A/B check after a kernel change: GPU parity suite, then the config-4 bench
# line (no CPU arm) and the config-3 microbench line.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench3.log 2>&1; echo "rc=$?" >> gpurun_out/bench3.log
