"""Small exercise of every kernel family for compute-sanitizer runs (memcheck /
racecheck / synccheck): batched rounding on all three CTA widths incl. the
DMMA and operand-cache paths, moments, collision, one explicit step with
oblique faces and a diffuse wall, one LU-SGS iteration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.tt import random_tt  # noqa: E402
from paper_1912_04582_b200.cuda import Context  # noqa: E402
from paper_1912_04582_b200.problems import obstacle_flow  # noqa: E402
from paper_1912_04582_b200.tt_batch import TtBatch  # noqa: E402

rng = np.random.default_rng(0)
ctx = Context(0)
n = 16
ctx.set_grid(n, 1.0)
for ranks, k in (((1, 2), 2), ((3, 4), 3), ((6, 6), 4), ((8, 9), 3)):  # g32, g128, g256 + T route / DMMA
    ts = [random_tt(rng, n, n, n, *ranks) for _ in range(4 * k)]
    got = ctx.rounded(TtBatch.from_list(ts), 1e-6, group_off=np.arange(0, 4 * k + 1, k))
    assert np.all(np.isfinite(got.cores))
p = obstacle_flow((4, 4, 4), hole=2, nv=12)
ctx.setup(p)
ctx.step(p.dt, p.eps, p.cap, 2)
ctx.lusgs_step(p.dt, p.eps, p.cap, 1)
st = ctx.download_state()
assert np.all(np.isfinite(st.cores))
print("sanitize_small ok: ranks up to", int(st.ranks.max()))
ctx.close()
