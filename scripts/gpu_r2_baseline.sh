set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench0.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/r2_bench0.log
