for v in 0 1 1; do
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
TTDVM_ARENA_LOG=1 python bench.py --config 5 --scale 0.25 --steps 2 --warmup 1 --no-cpu-baseline --no-parity 2>&1 | grep "ttdvm bin" | tail -12
python - <<'PY'
# per-phase cycle profile of config 3 (thread-0 clocks)
import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from bench import c3_inputs
from paper_1912_04582_b200.cuda import Context
b, go = c3_inputs(4096)
ctx = Context(0); ctx.set_grid(32, 1.0)
ctx.rounded(b, 1e-6, 0, group_off=go)
ctx.round_profile(True)
ms = ctx.round_resident(1e-6, 0, 1)
cyc = ctx.round_profile(False).astype(float)
names = ["load","qr_last","cut1(T loop)","chol1","Zj","svd1","cut2_X2_S","chol2","cut2_gram","svd2","output","stage"]
tot = cyc[:12].sum()
print("config 3: %.2f ms, %.0f kcycles/rounding" % (ms, tot/4096/1e3))
for n, c in zip(names, cyc[:12]): print("  %-14s %5.1f%%  %8.1f kcyc" % (n, 100*c/tot, c/4096/1e3))
PY
