# Per-bin device times of the rounding launches (TTDVM_ARENA_LOG=1) on the
# config-4 half-scale probe, twice, to locate the intermittent slow flux phase.
mkdir -p gpurun_out
for r in 1 2; do
  TTDVM_ARENA_LOG=1 timeout 600 python scripts/probe_config4.py --scale 0.5 --steps 7 > gpurun_out/probe_bins_$r.log 2>&1
done
