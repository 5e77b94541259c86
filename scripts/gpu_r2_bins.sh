# per-bin device times of config 4 at full size over 20 steps (TTDVM_ARENA_LOG serialises the bins)
TTDVM_ARENA_LOG=1 python scripts/probe_config4.py --scale 1.0 --steps 20 > gpurun_out/r2_bins.log 2> gpurun_out/r2_bins.err
echo rc=$?
grep "ttdvm bin" gpurun_out/r2_bins.err | tail -45
tail -3 gpurun_out/r2_bins.log | cut -c1-600
