mkdir -p gpurun_out
timeout 1500 python bench.py --steps 3 --warmup 3 > gpurun_out/bench4.log 2>&1; echo "rc=$?" >> gpurun_out/bench4.log
