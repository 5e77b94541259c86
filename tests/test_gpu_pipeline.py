"""The phase pipeline (round_pipe.cuh) against the one-kernel path on the
same seeded sums: the six kernels call the same helpers and add every sum in
the same order within a warp, so ranks must be identical; the one-kernel
path reduces norms and dot products over four or eight warps, so the cores
differ by roundoff amplified through the truncated subspaces (observed
2e-5 eps) -- asserted within 1e-4 eps, far inside the parity bar of 10 eps.  Each path runs in its own process (the switches are read
once per process)."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
EPS = (1e-6, 1e-5, 1e-3)  # of the worker's cases
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import sys, numpy as np
sys.path.insert(0, %r)
from oracle.tt import random_tt
from paper_1912_04582_b200.cuda import Context
from paper_1912_04582_b200.tt_batch import TtBatch
rng = np.random.default_rng(5)
ctx = Context(0)
out = {}
for case, (n, count, kmax, rmax, eps, cap) in enumerate([(20, 2600, 4, 3, 1e-6, 0), (44, 2200, 3, 5, 1e-5, 0),
                                                          (16, 2100, 5, 3, 1e-3, 2)]):
    ctx.set_grid(n, 1.0)
    pool = [random_tt(rng, n, n, n, int(rng.integers(1, rmax + 1)), int(rng.integers(1, rmax + 1)))
            for _ in range(64)]
    flat, go, sc = [], [0], []
    for _ in range(count):
        k = int(rng.integers(1, kmax + 1))
        for _ in range(k):
            flat.append(pool[int(rng.integers(0, 64))])
            sc.append(float(rng.choice([1.0, -1.0, 0.5, 1e-4])))
        go.append(go[-1] + k)
    got, mg = ctx.rounded(TtBatch.from_list(flat), eps, cap, group_off=np.array(go), scale=np.array(sc),
                          margins=True)
    out["r%%d" %% case] = got.ranks
    out["o%%d" %% case] = got.offsets
    out["c%%d" %% case] = got.cores
    out["n%%d" %% case] = np.array([n])
    out["l%%d" %% case] = np.array([ctx.launch_count()])
np.savez(sys.argv[1], **out)
"""


def run(tmp_path, name, env):
    path = str(tmp_path / (name + ".npz"))
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-c", WORKER % ROOT, path], env=e, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(path))


def test_pipeline_matches_one_kernel_path(tmp_path):
    from paper_1912_04582_b200.tt_batch import TtBatch
    a = run(tmp_path, "one", {"TTDVM_PIPE": "0"})
    b = run(tmp_path, "pipe", {"TTDVM_PIPE": "1", "TTDVM_PIPE_MIN": "64"})
    for case in range(3):
        n = int(a["n%d" % case][0])
        assert int(b["l%d" % case][0]) > int(a["l%d" % case][0])  # six launches per chunk: the pipeline ran
        np.testing.assert_array_equal(a["r%d" % case], b["r%d" % case])
        ta = TtBatch(n, n, n, a["r%d" % case], a["o%d" % case], a["c%d" % case])
        tb = TtBatch(n, n, n, b["r%d" % case], b["o%d" % case], b["c%d" % case])
        worst = 0.0
        for o in range(0, ta.count, 37):
            fa, fb = ta.full(o), tb.full(o)
            worst = max(worst, float(np.linalg.norm(fa - fb) / max(np.linalg.norm(fa), 1e-300)))
        assert worst <= 1e-4 * EPS[case], (case, worst)
