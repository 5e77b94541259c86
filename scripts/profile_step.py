"""Run a few explicit steps of a (scaled) config -- the short command that
ncu captures (the bench itself is too long for a full-set replay)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04582_b200.cuda import Context  # noqa: E402
from paper_1912_04582_b200.problems import config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--scale", type=float, default=0.25)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
p = config(a.config, a.scale)
ctx = Context(0)
ctx.setup(p)
ap2 = None
if os.environ.get("ROUND_PROF"):
    ctx.round_profile(True)
ms = ctx.timed_step(p.dt, p.eps, p.cap, a.steps)
if os.environ.get("ROUND_PROF"):
    cyc = ctx.round_profile(False).astype(float)
    names = ["load", "qr_last", "cut1_blocks", "cut1_qrupd", "C+norm", "jacobi1", "cut2_blocks",
             "cut2_qrupd", "P..", "jacobi2", "output"]
    tot = cyc.sum()
    tot = cyc[:11].sum()
    print("round phases (% of thread-0 cycles):",
          {names[i]: round(100 * cyc[i] / tot, 1) for i in range(11)})
    nr = max(1, cyc[13] / 2)
    print("mean kcycles per rounding:", {names[i]: round(cyc[i] / nr / 1e3, 1) for i in range(11)},
          "total", round(tot / nr / 1e3, 1))
    print("jacobi: %d svds, mean sweeps %.2f, hit cap %d" % (cyc[13], cyc[12] / max(1, cyc[13]), cyc[14]))
print(f"{p.name} scale {a.scale}: {p.mesh.ncell} cells, {a.steps} steps, {ms:.2f} ms, "
      f"launches {ctx.launch_count()}")
ctx.close()
