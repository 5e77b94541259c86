# Deferred frees of regrown arenas: config-4 half-scale probe with
# TTDVM_DEFER_FREE=0 / 1 (arena events logged), GPU suite, default bench line.
mkdir -p gpurun_out
for d in 0 1; do
  TTDVM_DEFER_FREE=$d TTDVM_ARENA_LOG=1 timeout 600 python scripts/probe_config4.py --scale 0.5 --steps 7 2>&1 | grep -v "ttdvm bin" > gpurun_out/probe_defer_$d.log
done
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
