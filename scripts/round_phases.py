"""Per-phase SM-cycle breakdown of the exact-Gram rounding kernel
(clock64 on thread 0 of every CTA, summed; diagnostics only).

    python scripts/round_phases.py --config 4 --scale 0.25   # step roundings
    python scripts/round_phases.py --config 3 --count 2048   # config-3 sums
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1912_04582_b200.cuda import Context  # noqa: E402

NAMES = {0: "load", 1: "qr_last", 11: "stage_slices", 4: "cut1_Zj", 2: "cut1_gram_acc",
         3: "chol1(+C)", 5: "svd1", 8: "cut2_X2_S", 6: "P+cut2_gram_acc", 7: "chol2", 9: "svd2",
         10: "output"}

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--scale", type=float, default=0.25)
ap.add_argument("--steps", type=int, default=1)
ap.add_argument("--warmup", type=int, default=2)
ap.add_argument("--count", type=int, default=2048)
a = ap.parse_args()
ctx = Context(0)
if a.config == 3:
    import bench
    b, go = bench.c3_inputs(a.count)
    ctx.set_grid(32, 1.0)
    ctx.rounded(b, 1e-6, 0, group_off=go)
    ctx.round_profile(True)
    ms = ctx.round_resident(1e-6, 0, 1)
    nround = a.count
else:
    from paper_1912_04582_b200.problems import config
    p = config(a.config, a.scale)
    ctx.setup(p)
    ctx.step(p.dt, p.eps, p.cap, a.warmup)
    ctx.round_profile(True)
    ms = ctx.timed_step(p.dt, p.eps, p.cap, a.steps)
    nround = None
cyc = ctx.round_profile(False).astype(float)
tot = sum(cyc[k] for k in NAMES)
nr = cyc[13] / 2 if nround is None else nround  # two SVDs per rounding
print(f"config {a.config}: {ms:.2f} ms, {int(nr)} roundings, jacobi mean sweeps "
      f"{cyc[12] / max(1, cyc[13]):.2f}")
for k, nm in NAMES.items():
    print(f"  {nm:12s} {100 * cyc[k] / tot:5.1f}%  {cyc[k] / nr / 1e3:8.1f} kcycles/rounding")
print(f"  total {tot / nr / 1e3:.1f} kcycles per rounding (thread-0 clock, CTA residency)")
ctx.close()
