# round-2 bench check: reduced scale first (fast failure), then the full default line
set -x
python bench.py --scale 0.2 --steps 4 --warmup 3 > gpurun_out/r2_bench_small.log 2>&1; echo "small rc=$?"
tail -c 2500 gpurun_out/r2_bench_small.log
python bench.py > gpurun_out/r2_bench_full.log 2>&1; echo "full rc=$?"
tail -c 6000 gpurun_out/r2_bench_full.log
