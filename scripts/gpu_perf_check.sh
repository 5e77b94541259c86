# One GPU call: parity suite, per-phase rounding cycles, config-4 half-scale
# probe, config-3 microbench (short).
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests_rc=$?"; tail -3 gpurun_out/gpu_tests.log
python scripts/round_phases.py --config 4 --scale 0.25 > gpurun_out/phases.log 2>&1
python scripts/round_phases.py --config 3 >> gpurun_out/phases.log 2>&1
cat gpurun_out/phases.log
python scripts/probe_config4.py --scale 0.5 --steps 4 2>&1 | grep '"step": 3' | cut -c1-420
python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | cut -c1-200
