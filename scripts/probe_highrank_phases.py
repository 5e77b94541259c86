"""Per-phase SM cycles of the ONE-KERNEL rounding launches (the high-rank bins
the pipeline leaves) inside a real config-4 step: advance to step K-1, switch
the in-kernel phase clocks on, run step K with the bins serialised and logged.
python scripts/probe_highrank_phases.py [--scale 0.5] [--steps 20]"""
import argparse
import os
import sys

os.environ.setdefault("TTDVM_ARENA_LOG", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1912_04582_b200.cuda import Context  # noqa: E402
from paper_1912_04582_b200.problems import config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=0.5)
ap.add_argument("--steps", type=int, default=20)
a = ap.parse_args()
p = config(4, a.scale)
ctx = Context(0)
ctx.setup(p)
ctx.step(p.dt, p.eps, p.cap, a.steps - 1)
sys.stderr.write("==== profiled step\n")
sys.stderr.flush()
ctx.round_profile(True)
ms = ctx.timed_step(p.dt, p.eps, p.cap, 1)
cyc = ctx.round_profile(False).astype(float)
names = ["load", "qr_last", "cut1 (T loop / Gram)", "chol1", "Zj", "svd1", "cut2_X2_S", "chol2",
         "cut2_gram", "svd2", "output", "stage"]
tot = cyc[:12].sum()
print(f"step {a.steps} at scale {a.scale}: {ms:.1f} ms; one-kernel launches: {tot/1e6:.0f} Mcycles of CTA residency")
for nm, c in zip(names, cyc[:12]):
    print("  %-28s %5.1f%%  %9.1f Mcyc" % (nm, 100 * c / tot, c / 1e6))
print("  jacobi sweeps total %d over %d calls, >=60: %d" % (cyc[12], cyc[13], cyc[14]))
