# Config 5 at full size after limiting parked/headroom blocks to 4 GB, then
# the GPU suite and the default bench line.
mkdir -p gpurun_out
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/bench5.log 2>&1; echo "bench5 rc=$?" >> gpurun_out/bench5.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
