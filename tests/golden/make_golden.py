"""Generate the committed golden fixtures under tests/golden/ (test
infrastructure only).

The reference (C++ over Eigen) does not build in this
image and ships no golden vectors, so these fixtures are produced by the
oracle restatement (oracle/), itself pinned by the reference's own
known-answer tests (tests/test_oracle_*.py).  They freeze the oracle's
outputs on seeded inputs so that (a) the CPU suite catches any drift of
the oracle and (b) the GPU suite can check the CUDA path against stored
vectors without re-running the oracle.

    python tests/golden/make_golden.py        # rewrites the .npz files
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle.step import OracleSolver  # noqa: E402
from oracle.tt import TtTensor, random_tt  # noqa: E402
from paper_1912_04582_b200.problems import config  # noqa: E402

SHOCK_STEPS = 5


def shock_tube_fixture():
    """Config 1 (64x1x1 shock tube, 16^3 velocity mesh, eps 1e-6):
    per-cell macroparameters of the states t^0 .. t^(SHOCK_STEPS-1) and the
    ranks and dense tensors of a few cells after SHOCK_STEPS steps."""
    p = config(1)
    solver = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = [TtTensor(*p.f0.get(i)) for i in range(p.mesh.ncell)]
    macros = []
    for _ in range(SHOCK_STEPS):
        f, m = solver.step(f, p.dt, p.eps, p.cap)
        macros.append(np.stack([x.as_array() for x in m]))
    cells = np.array([0, 30, 31, 32, 33, 63])
    return dict(steps=np.int64(SHOCK_STEPS), dt=np.float64(p.dt), eps=np.float64(p.eps),
                macros=np.stack(macros), ranks=np.array([f[i].ranks()[1:3] for i in range(len(f))]),
                cells=cells, full=np.stack([f[i].to_full() for i in cells]))


ROUND_CASES = ((1e-6, 0), (1e-4, 5))  # (eps, rank cap)


def rounding_fixture():
    """Seeded sums of random TTs (24^3, 2..5 summands of ranks 1..8,
    scales 1 / -0.5 / 1e-3) rounded per case of ROUND_CASES: the packed
    summands (TtBatch layout), and the oracle's output ranks and dense
    reconstructions."""
    from paper_1912_04582_b200.tt_batch import TtBatch

    rng = np.random.default_rng(11)
    n = 24
    out = {"n": np.int64(n)}
    for c, (eps, cap) in enumerate(ROUND_CASES):
        flat, groups, scales, fulls, oranks = [], [0], [], [], []
        for _ in range(6):
            k = int(rng.integers(2, 6))
            s = None
            for _ in range(k):
                t = random_tt(rng, n, n, n, int(rng.integers(1, 9)), int(rng.integers(1, 9)))
                sc = float(rng.choice([1.0, -0.5, 1e-3]))
                flat.append(t)
                scales.append(sc)
                s = t.scaled(sc) if s is None else s + t.scaled(sc)
            groups.append(groups[-1] + k)
            r = s.rounded(eps, cap)
            fulls.append(r.to_full())
            oranks.append(r.ranks()[1:3])
        b = TtBatch.from_list(flat)
        out.update({f"c{c}_eps": np.float64(eps), f"c{c}_cap": np.int64(cap),
                    f"c{c}_cores": b.cores, f"c{c}_ranks": b.ranks, f"c{c}_offsets": b.offsets,
                    f"c{c}_group_off": np.array(groups), f"c{c}_scales": np.array(scales),
                    f"c{c}_out_ranks": np.array(oranks), f"c{c}_out_full": np.stack(fulls)})
    return out


if __name__ == "__main__":
    np.savez_compressed(os.path.join(HERE, "shock_tube_c1.npz"), **shock_tube_fixture())
    np.savez_compressed(os.path.join(HERE, "rounding_24.npz"), **rounding_fixture())
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
