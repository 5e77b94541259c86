"""Per-phase SM cycles (thread-0 clocks) of the one-kernel rounding path on
config-4-like HIGH-RANK sums: n = 44, K summands of ranks (r, r), e.g. 8 x 12
= summed rank 96 (T route).  python scripts/round_phases_highrank.py [K] [r] [count]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1912_04582_b200.cuda import Context  # noqa: E402
from paper_1912_04582_b200.tt_batch import TtBatch  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
r = int(sys.argv[2]) if len(sys.argv) > 2 else 12
count = int(sys.argv[3]) if len(sys.argv) > 3 else 2048
n = 44
rng = np.random.default_rng(0)
w = 0.5 ** np.arange(r)
first = rng.standard_normal((count * K, n, r)) * w[None, None, :]
middle = rng.standard_normal((count * K, n, r, r)) * w[None, None, :, None]
last = rng.standard_normal((count * K, r, n))
b = TtBatch.uniform(count * K, n, n, n, r, r, first, middle, last)
go = np.arange(0, count * K + 1, K, dtype=np.int64)
ctx = Context(0)
ctx.set_grid(n, 1.0)
out = ctx.rounded(b, 1e-5, 0, group_off=go)
ctx.round_profile(True)
ms = ctx.round_resident(1e-5, 0, 1)
cyc = ctx.round_profile(False).astype(float)
names = ["load", "qr_last", "cut1 (T loop: GEMMs + dd Gram)", "chol1", "Zj", "svd1", "cut2_X2_S", "chol2",
         "cut2_gram", "svd2", "output", "stage"]
tot = cyc[:12].sum()
print(f"K={K} r={r} summed rank {K*r}, {count} outputs: {ms:.2f} ms, {1e3*ms/count:.2f} us/output, "
      f"{tot/count/1e3:.0f} kcycles/output (CTA residency); output ranks max {out.ranks.max(0)}")
for nm, c in zip(names, cyc[:12]):
    print("  %-34s %5.1f%%  %9.1f kcyc" % (nm, 100 * c / tot, c / count / 1e3))
