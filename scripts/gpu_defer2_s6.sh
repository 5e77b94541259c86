# Deferred frees for every DevBuf regrowth (+1.5x headroom): config-4
# half-scale probe twice with arena / bin events, GPU suite, smoke, bench.
mkdir -p gpurun_out
for r in 1 2; do
  TTDVM_ARENA_LOG=1 timeout 600 python scripts/probe_config4.py --scale 0.5 --steps 7 > gpurun_out/probe_defer2_$r.log 2>&1
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 python bench.py --steps 8 > gpurun_out/bench8.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench8.log
