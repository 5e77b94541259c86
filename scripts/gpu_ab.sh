# A/B of an environment switch on the config-4 half-scale probe: $1 = VAR=value
for env in "$@"; do
  echo "== $env"
  env $env python scripts/probe_config4.py --scale 0.5 --steps 6 2>&1 | grep "\"step\": [2-5]" | cut -c1-200
done
