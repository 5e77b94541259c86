"""Per-phase SM cycles of face_factor_kernel (a -DTTDVM_FF_PROF build, scripts/build_ff_variant.sh):
  TTDVM_LIB=paper_1912_04582_b200/ab/libttdvm_cuda_ffprof.so python scripts/ff_phases.py [N]"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1912_04582_b200 import cuda
from paper_1912_04582_b200.cuda import Context
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
LATTICE_ONLY = len(sys.argv) > 2 and sys.argv[2] == "lattice"  # config 4's kind: jittered hex faces only
rng = np.random.default_rng(0)
v = rng.normal(size=(N, 3))
ax = np.eye(3)[rng.integers(0, 3, N // 2)] * rng.choice([-1.0, 1.0], (N // 2, 1))
v[: N // 2] = ax + 0.1 * rng.normal(size=(N // 2, 3))
if LATTICE_ONLY:
    ax = np.eye(3)[rng.integers(0, 3, N)] * rng.choice([-1.0, 1.0], (N, 1))
    v = ax + 0.05 * rng.normal(size=(N, 3))
v /= np.linalg.norm(v, axis=1, keepdims=True)
ctx = Context(0)
ctx.set_grid(44, 7.0)
ctx.face_factors(v[:64], cap=4, mode="abs")
out = (C.c_ulonglong * 16)()
ctx.lib.ttdvm_cuda_ff_profile(out)
t = time.time()
ctx.face_factors(v, cap=4, mode="abs")
el = time.time() - t
ctx.lib.ttdvm_cuda_ff_profile(out)
cyc = np.array(list(out), dtype=float)
names = ["cut1 gen", "cut1 dd Gram", "svd1 (chol+jacobi)", "cut2 gen", "cut2 Bj", "cut2 dd Grams", "svd2 a+b",
         "pass3 gen", "pass3 Bj+C", "pass3 Y", "pass3 err", "select+keep"]
tot = cyc[:12].sum()
print(f"{N} normals {el:.3f}s {el / N * 1e6:.1f} us/normal; {tot / N / 1e6:.2f} Mcycles of CTA residency per normal")
for nm, c in zip(names, cyc[:12]):
    print("  %-20s %5.1f%%  %8.0f kcyc/normal" % (nm, 100 * c / tot, c / N / 1e3))
print("  inside the svd phases: pivoted dd Cholesky %.0f kcyc/normal, svd_from_r (Jacobi) %.0f kcyc/normal; "
      "mean Cholesky rank %.1f over %d factorizations per normal" %
      (cyc[12] / N / 1e3, cyc[13] / N / 1e3, cyc[14] / max(cyc[15], 1), cyc[15] / N))
