"""Face-factor set-up A/B: time abs_xi_estimate / xi_n^+ / xi_n^- factors of N
normals (random oblique + nearly axis-aligned ones, as config 4's jittered
mesh has) with the library TTDVM_LIB names and dump the results; with a
second argument, compare against an earlier dump bitwise.
  TTDVM_LIB=... python scripts/ab_ff.py out.npz [ref.npz] [N]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1912_04582_b200.cuda import Context
out_path = sys.argv[1]
ref_path = sys.argv[2] if len(sys.argv) > 2 and sys.argv[2] != "-" else None
N = int(sys.argv[3]) if len(sys.argv) > 3 else 8192
n = 44
rng = np.random.default_rng(0)
v = rng.normal(size=(N, 3))
# half of them: a lattice direction jittered by ~10 %, like a jittered hex face
ax = np.eye(3)[rng.integers(0, 3, N // 2)] * rng.choice([-1.0, 1.0], (N // 2, 1))
v[: N // 2] = ax + 0.1 * rng.normal(size=(N // 2, 3))
v /= np.linalg.norm(v, axis=1, keepdims=True)
ctx = Context(0)
ctx.set_grid(n, 7.0)
ctx.face_factors(v[:64], cap=4, mode="abs")
res = {}
for mode, cap in (("abs", 4), ("pos", 6), ("neg", 6)):
    el = 1e9
    for rep in range(3):  # minimum of three
        t = time.time()
        if mode == "abs":
            o, dg = ctx.face_factors(v, cap=cap, mode=mode, diag=True)
            res["abs_diag"] = dg
        else:
            o = ctx.face_factors(v, cap=cap, mode=mode)
        el = min(el, time.time() - t)
    print(f"{os.environ.get('TTDVM_LIB', 'default')} {mode}: {N} normals {el:.3f}s {el / N * 1e6:.1f} us/normal", flush=True)
    res[mode + "_ranks"] = o.ranks
    res[mode + "_off"] = o.offsets
    res[mode + "_cores"] = o.cores
np.savez(out_path, **res)
if ref_path:
    ref = np.load(ref_path)
    for k in res:
        a, b = np.asarray(res[k]), ref[k]
        same = a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))
        print(f"{k}: {'bitwise equal' if same else 'DIFFERENT'}")
