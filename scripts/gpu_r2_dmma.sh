# DMMA slice products: parity suite, then same-box A/B against TTDVM_DMMA=0 on config 3, config 5 (quarter scale) and config 4 (half scale)
python -m pytest tests -m gpu -q -x 2>&1 | tail -6
for v in 0 1 0 1; do
  echo "== config 3 TTDVM_DMMA=$v"
  TTDVM_DMMA=$v python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print(round(d['value']), 'tensors/s', round(d['roofline']['frac'], 4), 'of FP64 peak')"
done
for v in 0 1; do
  echo "== config 5 scale 0.25 TTDVM_DMMA=$v"
  TTDVM_DMMA=$v python bench.py --config 5 --scale 0.25 --steps 4 --warmup 3 --no-cpu-baseline --no-parity 2>&1 | tail -1 | python -c "
import sys, json
d = json.loads(sys.stdin.read()); print(round(d['value']), 'cell-steps/s', {k: v['ms_per_step'] for k, v in d['roofline']['per_kernel'].items()})"
done
for v in 0 1; do
  echo "== config 4 scale 0.5 TTDVM_DMMA=$v"
  TTDVM_DMMA=$v python scripts/probe_config4.py --scale 0.5 --steps 20 2>/dev/null | python -c "
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
