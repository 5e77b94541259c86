"""Face-factor A/B: time abs/pos/neg factors of N seeded oblique normals with
the library named by TTDVM_LIB and save the results (cores, ranks, diag) to
argv[2] for a bitwise comparison between builds."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1912_04582_b200.cuda import Context
N = int(sys.argv[1]); out_path = sys.argv[2]
rng = np.random.default_rng(7)
v = rng.normal(size=(N, 3)); v /= np.linalg.norm(v, axis=1, keepdims=True)
v[: N // 8] = np.array([1.0, 1e-3, 2e-4]) + 1e-4 * rng.normal(size=(N // 8, 3))  # near axis-aligned
v /= np.linalg.norm(v, axis=1, keepdims=True)
ctx = Context(0)
ctx.set_grid(44, 7.0)
ctx.face_factors(v[:64], cap=4, mode="abs")
res = {}
for mode in ("abs", "pos", "neg"):
    t = time.time()
    if mode == "abs":
        o, dg = ctx.face_factors(v, cap=4, mode=mode, diag=True)
        res["diag"] = dg
    else:
        o = ctx.face_factors(v, cap=4, mode=mode)
    el = time.time() - t
    print(f"{os.path.basename(os.environ.get('TTDVM_LIB', 'default'))} {mode}: {N} normals {el:.3f}s "
          f"{el / N * 1e6:.1f} us/normal", flush=True)
    res[mode + "_cores"] = o.cores.copy()
    res[mode + "_ranks"] = np.asarray(o.ranks).copy()
np.savez(out_path, **res)
