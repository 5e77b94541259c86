"""LU-SGS iteration cost against the explicit step on config 4 (SPEC.md:408:
"wall-time per LU-SGS iteration <= 2x explicit iteration")."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04582_b200.cuda import Context  # noqa: E402
from paper_1912_04582_b200.problems import config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=0.5)
ap.add_argument("--iters", type=int, default=5)
a = ap.parse_args()
p = config(4, a.scale)
ctx = Context(0)
ctx.setup(p)
ctx.step(p.dt, p.eps, p.cap, 0)
print("cells", p.mesh.ncell, "levels (forward, backward)", ctx.lusgs_levels(), flush=True)
import time  # noqa: E402
for name, fn in (("explicit", lambda: ctx.step(p.dt, p.eps, p.cap, 1)),
                 ("lusgs", lambda: ctx.lusgs_step(p.dt, p.eps, p.cap, 1))):
    ctx.upload_state(p.f0)
    fn()
    ctx.upload_state(p.f0)
    t = time.perf_counter()
    for _ in range(a.iters):
        fn()
    dt = (time.perf_counter() - t) / a.iters
    st = ctx.download_state()
    print(f"{name}: {1e3 * dt:.1f} ms per iteration, {p.mesh.ncell / dt:.0f} cell-iterations/s, "
          f"max rank {int(st.ranks.max())}", flush=True)
ctx.upload_state(p.f0)
ctx.lusgs_step(p.dt, p.eps, p.cap, 2)
ctx.set_profiling(True)
ctx.lusgs_step(p.dt, p.eps, p.cap, 1)
rep = ctx.phase_report()
print({k: (round(v[0], 1), v[3]) for k, v in rep.items()})
