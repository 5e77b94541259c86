"""Golden fixtures (tests/golden/, made by tests/golden/make_golden.py from
the oracle, which tests/test_oracle_*.py pin to the reference's own
known-answer tests).

CPU: the oracle still reproduces the committed vectors (catches drift of
the checker).  GPU: the CUDA path, through the C ABI, against the stored
vectors -- no oracle run on the box."""
import os

import numpy as np
import pytest

from oracle.tt import rel_err
from paper_1912_04582_b200.tt_batch import TtBatch

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(HERE, name)))


def test_oracle_reproduces_shock_tube_golden():
    import sys
    sys.path.insert(0, HERE)
    from make_golden import shock_tube_fixture
    want = load("shock_tube_c1.npz")
    got = shock_tube_fixture()
    np.testing.assert_array_equal(got["ranks"], want["ranks"])
    np.testing.assert_allclose(got["macros"], want["macros"], rtol=1e-10, atol=1e-13)
    for a, b in zip(got["full"], want["full"]):
        assert rel_err(a, b) <= 1e-10


def test_oracle_reproduces_rounding_golden():
    import sys
    sys.path.insert(0, HERE)
    from make_golden import rounding_fixture
    want = load("rounding_24.npz")
    got = rounding_fixture()
    for c in range(2):
        np.testing.assert_array_equal(got[f"c{c}_out_ranks"], want[f"c{c}_out_ranks"])
        np.testing.assert_array_equal(got[f"c{c}_cores"], want[f"c{c}_cores"])
        for a, b in zip(got[f"c{c}_out_full"], want[f"c{c}_out_full"]):
            assert rel_err(a, b) <= 1e-10


@pytest.fixture(scope="module")
def ctx():
    from paper_1912_04582_b200.cuda import Context
    c = Context(0)
    yield c
    c.close()


@pytest.mark.gpu
def test_gpu_rounding_matches_golden(ctx):
    d = load("rounding_24.npz")
    n = int(d["n"])
    ctx.set_grid(n, 1.0)
    for c in range(2):
        eps, cap = float(d[f"c{c}_eps"]), int(d[f"c{c}_cap"])
        b = TtBatch(n, n, n, d[f"c{c}_ranks"], d[f"c{c}_offsets"], d[f"c{c}_cores"])
        got = ctx.rounded(b, eps, cap, group_off=d[f"c{c}_group_off"], scale=d[f"c{c}_scales"])
        np.testing.assert_array_equal(got.ranks, d[f"c{c}_out_ranks"])
        for o, want in enumerate(d[f"c{c}_out_full"]):
            assert rel_err(got.full(o), want) <= 10 * eps, (c, o)


@pytest.mark.gpu
def test_gpu_shock_tube_matches_golden(ctx):
    """Config 1 run free on the GPU for the fixture's steps: macroparameters
    of t^0 to 1e-8 (same input state), later ones and the final tensors
    within the accumulated rounding budget (10 eps per step)."""
    from paper_1912_04582_b200.problems import config
    d = load("shock_tube_c1.npz")
    p = config(1)
    steps, eps = int(d["steps"]), float(d["eps"])
    assert float(d["dt"]) == p.dt
    ctx.setup(p)
    for k in range(steps):
        ctx.step(p.dt, eps, p.cap, 1)
        m = ctx.macros()[:, :10]
        tol = 1e-8 if k == 0 else 10 * eps * k
        np.testing.assert_allclose(m[:, [0, 4, 6]], d["macros"][k][:, [0, 4, 6]], rtol=tol)
        np.testing.assert_allclose(m[:, 1:4], d["macros"][k][:, 1:4], rtol=tol, atol=tol)
    st = ctx.download_state()
    np.testing.assert_array_equal(st.ranks, d["ranks"])
    for i, want in zip(d["cells"], d["full"]):
        assert rel_err(st.full(int(i)), want) <= 10 * eps * steps
