# Session 6: arena events on the config-4 half-scale probe, GPU suite, smoke,
# default bench line (config 4) and config-3 line on the current build.
mkdir -p gpurun_out
TTDVM_ARENA_LOG=1 timeout 600 python scripts/probe_config4.py --scale 0.5 --steps 6 > gpurun_out/probe_arena.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
TTDVM_ARENA_LOG=1 timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --config 3 > gpurun_out/bench3.log 2>&1; echo "bench3 rc=$?" >> gpurun_out/bench3.log
