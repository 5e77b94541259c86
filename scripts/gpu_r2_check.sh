# parity suite + the default bench line (config 4, its own 20 steps) + config 3 line
python -m pytest tests -m gpu -q 2>&1 | tail -5
python bench.py > gpurun_out/r2_bench_full.log 2>gpurun_out/r2_bench_full.err; echo "bench rc=$?"
tail -c 1500 gpurun_out/r2_bench_full.log
python bench.py --config 3 --steps 5 --warmup 3 > gpurun_out/r2_bench_c3.log 2>&1; echo "c3 rc=$?"
tail -c 1200 gpurun_out/r2_bench_c3.log
python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1; echo "ref rc=$?"
tail -c 900 gpurun_out/r2_bench_ref.log
