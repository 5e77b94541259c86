# Config 5 at full size (1,048,576 cells, 64^3; blocked step via the
# out-of-memory fallback) on the final code, with arena events logged.
mkdir -p gpurun_out
TTDVM_ARENA_LOG=0 timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench5.log 2>&1; echo "bench5 rc=$?" >> gpurun_out/bench5.log
