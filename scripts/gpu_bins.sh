# Per-bin device times of the rounding launches (TTDVM_ARENA_LOG serialises the bins):
#   gpurun -- 'bash scripts/gpu_bins.sh 1.0 20'   -> gpurun_out/bins.err, last step's bins printed
TTDVM_ARENA_LOG=1 python scripts/probe_config4.py --scale ${1:-0.5} --steps ${2:-20} > gpurun_out/bins.log 2> gpurun_out/bins.err
grep "ttdvm bin" gpurun_out/bins.err | tail -45
tail -2 gpurun_out/bins.log | cut -c1-600
