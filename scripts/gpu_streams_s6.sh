# Concurrent rank bins: same-box A/B (TTDVM_BIN_STREAMS=0/1) on the config-4
# half-scale probe, GPU suite, smoke, bench lines (config 4, config 3), the
# ncu launch list of the bench command, and a full-set capture of the
# rounding launches of one half-scale step (scripts/ncu_box_round.sh).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
for r in 1 2; do
  for s in 0 1; do
    echo "== streams $s" >> gpurun_out/ab_streams.log
    TTDVM_BIN_STREAMS=$s timeout 600 python scripts/probe_config4.py --scale 0.5 --steps 6 2>&1 | grep '"step": [2-5]' | cut -c1-330 >> gpurun_out/ab_streams.log
  done
done
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --config 3 > gpurun_out/bench3.log 2>&1; echo "bench3 rc=$?" >> gpurun_out/bench3.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/launches_bench4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch4.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_launch4.log
bash scripts/ncu_box_round.sh 0.5 30 12 > gpurun_out/ncu_box.log 2>&1
