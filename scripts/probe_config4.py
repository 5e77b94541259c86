"""Config-4 probe on one GPU: set-up cost (mesh, face factors), per-phase
step times, ranks and memory at a given spatial scale."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1912_04582_b200.cuda import Context  # noqa: E402
from paper_1912_04582_b200.problems import config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=float, default=0.25)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--nv", type=int, default=0)
a = ap.parse_args()
t = time.time()
p = config(4, a.scale)
if a.nv:
    from paper_1912_04582_b200.problems import obstacle_flow
    p = obstacle_flow(p.mesh.shape, hole=p.meta["hole"], nv=a.nv)
print(f"mesh {p.mesh.ncell} cells {p.mesh.nface} faces, host setup {time.time() - t:.1f}s", flush=True)
import torch  # noqa: E402
ctx = Context(0)
t = time.time()
ctx.setup(p)
print(f"upload {time.time() - t:.1f}s", flush=True)
t = time.time()
ctx.step(p.dt, p.eps, p.cap, 0)
print(f"prepare (face factors) {time.time() - t:.1f}s info {ctx.setup_info()}", flush=True)
names = ["moments", "shakhov", "round_fs", "round_col", "round_flux", "round_res", "round_upd", "book"]
ctx.set_profiling(True)
for k in range(a.steps):
    ms = ctx.timed_step(p.dt, p.eps, p.cap, 1)
    ph = ctx.phase_times()
    fl, by, la = ctx.phase_work()
    st = ctx.download_state()
    phi = ctx.stage("phi")
    print(json.dumps({"step": k, "ms": round(ms, 1), "cell_steps_per_s": p.mesh.ncell / ms * 1e3,
                      "phase_ms": {names[i]: round(float(ph[i]), 1) for i in range(8)},
                      "phase_tflops": {names[i]: round(float(fl[i] / max(ph[i], 1e-9) / 1e9), 3)
                                       for i in range(2, 7)},
                      "state_rank_max": int(st.ranks.max()),
                      "state_rank_mean": float(st.ranks.mean()),
                      "phi_rank_max": int(phi.ranks.max()), "phi_rank_mean": float(phi.ranks.mean()),
                      "state_gb": st.cores.nbytes / 1e9,
                      "mem_gb": torch.cuda.mem_get_info()[1] / 1e9 - torch.cuda.mem_get_info()[0] / 1e9}),
          flush=True)
m = ctx.macros()
print("macro n range", m[:, 0].min(), m[:, 0].max(), "T range", m[:, 4].min(), m[:, 4].max())
