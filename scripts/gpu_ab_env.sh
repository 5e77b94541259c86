# Same-box A/B of environment switches on the config-4 probe (half scale, 20 steps by default):
#   gpurun -- 'bash scripts/gpu_ab_env.sh TTDVM_LEAN=0 TTDVM_LEAN=1 TTDVM_LEAN=0 TTDVM_LEAN=1'
# Each argument is one run: comma-separated VAR=value assignments ("A=0" = defaults).
# Prints the mean per-phase device ms per step.  SCALE / STEPS override the probe size.
SCALE=${SCALE:-0.5}
STEPS=${STEPS:-20}
for spec in "$@"; do
  echo "== $spec"
  env $(echo "$spec" | tr ',' ' ') python scripts/probe_config4.py --scale $SCALE --steps $STEPS 2>/dev/null | python -c "
import sys, json
tot = {}
n = 0
for l in sys.stdin:
    if not l.startswith('{'): continue
    d = json.loads(l); n += 1
    for k, v in d['phase_ms'].items(): tot[k] = tot.get(k, 0) + v
    tot['step'] = tot.get('step', 0) + d['ms']
print({k: round(v / max(n, 1), 1) for k, v in tot.items()})
"
done
