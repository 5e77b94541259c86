# build-measure iteration: parity tests, per-phase cycles, bench line
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
ROUND_PROF=1 timeout 300 python scripts/profile_step.py --scale 0.5 --steps 3 > gpurun_out/prof_phases.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_iter.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_iter.log
