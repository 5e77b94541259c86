# LEAN rounding kernel: parity suite, then same-box A/B against TTDVM_LEAN=0 (config 4 half scale, 20 steps)
python -m pytest tests -m gpu -q -x 2>&1 | tail -6
run() {
  echo "== $*"
  env "$@" python scripts/probe_config4.py --scale 0.5 --steps 20 2>/dev/null | python -c "
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
}
run TTDVM_LEAN=0
run TTDVM_LEAN=1
run TTDVM_LEAN=0
run TTDVM_LEAN=1
