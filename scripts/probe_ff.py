"""Face-factor kernel timing: abs_xi_estimate of N random oblique normals."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1912_04582_b200.cuda import Context
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
n = int(sys.argv[2]) if len(sys.argv) > 2 else 44
rng = np.random.default_rng(0)
v = rng.normal(size=(N, 3)); v /= np.linalg.norm(v, axis=1, keepdims=True)
ctx = Context(0)
ctx.set_grid(n, 7.0)
ctx.face_factors(v[:64], cap=4, mode="abs")
t = time.time()
out, dg = ctx.face_factors(v, cap=4, mode="abs", diag=True)
el = time.time() - t
print(f"{N} normals n={n}: {el:.3f}s, {el / N * 1e6:.1f} us/normal; ranks max {out.ranks.max()}, "
      f"choices {np.bincount(dg[:, 2].astype(int) + 1)}")
