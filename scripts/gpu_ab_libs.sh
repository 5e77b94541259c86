# Same-box A/B of two library builds on the config-4 half-scale probe
# (alternating A B A B): $1 = A lib path, $2 = B lib path.
mkdir -p gpurun_out
A=$1; B=$2
for r in 1 2; do
  for L in "$A" "$B"; do
    echo "== $L"
    TTDVM_LIB=$L timeout 600 python scripts/probe_config4.py --scale 0.5 --steps 5 2>&1 | grep "\"step\": [2-4]" | cut -c1-400
  done
done
