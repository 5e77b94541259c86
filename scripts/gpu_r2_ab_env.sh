# same-box A/B of launch-plan environment knobs on config 4 at half scale, 20 steps
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
run A=0
run TTDVM_WIDE_D=17
run TTDVM_WIDE_D=25
run TTDVM_NARROW_D=8
run TTDVM_NARROW_D=8 TTDVM_JB=2
run TTDVM_NARROW_D=12 TTDVM_JB=2
run A=1
