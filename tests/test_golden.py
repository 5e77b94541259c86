"""Golden fixtures (tests/golden/, made by tests/golden/make_golden.py from
the COMPILED REFERENCE, oracle/_ref: the unmodified proj/src/*.cpp gated on
its own 50 doctest TEST_CASEs).

CPU: the numpy restatement (oracle/) reproduces the stored reference
outputs, and so does a rebuilt reference when /root/reference is present
(catches drift of either checker).  GPU: the CUDA path, through the C ABI,
against the stored vectors -- nothing on the box reads /root/reference."""
import os
import sys

import numpy as np
import pytest

from oracle import ref
from oracle.tt import rel_err
from paper_1912_04582_b200.tt_batch import TtBatch

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
sys.path.insert(0, HERE)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))


def load(name):
    return dict(np.load(os.path.join(HERE, name)))


def steppers():
    import make_golden as mg
    out = [pytest.param(mg.numpy_stepper, mg.numpy_rounder, id="numpy-oracle")]
    if ref.available():
        out.append(pytest.param(None, None, id="compiled-reference"))
    return out


@pytest.mark.parametrize("stepper,rounder", steppers())
def test_oracle_reproduces_shock_tube_golden(stepper, rounder):
    from make_golden import shock_tube_fixture
    want = load("shock_tube_c1.npz")
    got = shock_tube_fixture(stepper)
    np.testing.assert_array_equal(got["ranks"], want["ranks"])
    np.testing.assert_allclose(got["macros"], want["macros"], rtol=1e-10, atol=1e-13)
    for a, b in zip(got["full"], want["full"]):
        assert rel_err(a, b) <= 1e-10


@pytest.mark.parametrize("stepper,rounder", steppers())
def test_oracle_reproduces_rounding_golden(stepper, rounder):
    from make_golden import rounding_fixture
    want = load("rounding_24.npz")
    got = rounding_fixture(rounder)
    for c in range(2):
        np.testing.assert_array_equal(got[f"c{c}_out_ranks"], want[f"c{c}_out_ranks"])
        np.testing.assert_array_equal(got[f"c{c}_cores"], want[f"c{c}_cores"])
        for a, b in zip(got[f"c{c}_out_full"], want[f"c{c}_out_full"]):
            assert rel_err(a, b) <= 1e-10


def c4_state(d, k):
    nv = int(d["nv"])
    return TtBatch(nv, nv, nv, d[f"s{k}_ranks"], d[f"s{k}_offsets"], d[f"s{k}_cores"])


C4_NUMPY_CELLS = 4  # the numpy restatement's face factors at 44^3 cost ~1 s per normal


def test_numpy_oracle_reproduces_obstacle_golden():
    """Config-4-shaped fixture (44^3, eps 1e-5, Mach 3, oblique faces, walls):
    the numpy oracle steps a few cells -- one next to the wall -- from the
    stored state t^2 and lands on the stored reference state t^3."""
    from make_golden import c4_problem
    from oracle.step import OracleSolver
    from oracle.parity import oracle_list
    d = load("obstacle_c4_nv44.npz")
    p = c4_problem()
    assert float(d["dt"]) == p.dt and int(d["ncell"]) == p.mesh.ncell
    np.testing.assert_array_equal(d["face_normal"], p.mesh.face_normal)
    k = int(d["steps"]) - 1
    wall_faces = np.nonzero(p.mesh.face_group == 2)[0]
    cells = sorted({int(p.mesh.face_left[wall_faces[0]]), 0, 1, 2})[:C4_NUMPY_CELLS]
    s = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    prev, want = c4_state(d, k), c4_state(d, k + 1)
    f = dict(enumerate(oracle_list(prev)))
    out, macros = s.step(f, p.dt, p.eps, p.cap, cells=cells)
    for c, t, m in zip(cells, out, macros):
        assert t.ranks()[1:3] == tuple(want.ranks[c]), c
        assert rel_err(t.to_full(), want.full(c)) <= 1e-10, c
        np.testing.assert_allclose(m.as_array(), d["macros"][k][c, :10], rtol=1e-10, atol=1e-12)


@pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")
def test_compiled_reference_reproduces_obstacle_golden():
    from make_golden import obstacle_fixture
    d = load("obstacle_c4_nv44.npz")
    got = obstacle_fixture()
    for k in range(int(d["steps"]) + 1):
        np.testing.assert_array_equal(got[f"s{k}_ranks"], d[f"s{k}_ranks"])
        a, b = c4_state(got, k), c4_state(d, k)
        for c in range(0, a.count, 7):
            assert rel_err(a.full(c), b.full(c)) <= 1e-10
    np.testing.assert_allclose(got["macros"], d["macros"], rtol=1e-10, atol=1e-12)


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


@pytest.mark.gpu
def test_gpu_obstacle_c4_matches_golden(ctx):
    """The benchmarked configuration's shape (VelocityGrid(44, 7), eps 1e-5,
    Mach 3, jittered shuffled obstacle mesh with oblique faces, diffuse walls
    and in/out boundaries) in lock-step against stored outputs of the
    compiled reference: every step starts from the reference's state t^k and
    must land on its t^(k+1) -- reconstructions within 10 eps,
    macroparameters within 1e-8, ranks identical except inside the TIE
    window of an oracle decision on the cell's chain (oracle/parity.py)."""
    from make_golden import c4_problem
    from oracle.step import OracleSolver
    from oracle.parity import ChainMargins, macro_err, oracle_list, tie
    d = load("obstacle_c4_nv44.npz")
    p = c4_problem()
    assert float(d["dt"]) == p.dt
    np.testing.assert_array_equal(d["face_normal"], p.mesh.face_normal)
    eps = float(d["eps"])
    ctx.setup(p)
    for k in range(int(d["steps"])):
        prev, want = c4_state(d, k), c4_state(d, k + 1)
        ctx.upload_state(prev)
        ctx.step(p.dt, eps, p.cap, 1)
        got = ctx.download_state()
        assert macro_err(ctx.macros(), d["macros"][k]) <= 1e-8
        flips = []
        for c in range(p.mesh.ncell):
            assert rel_err(got.full(c), want.full(c)) <= 10 * eps, (k, c)
            if tuple(got.ranks[c]) != tuple(want.ranks[c]):
                flips.append(c)
        if flips:
            s = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
            cm = ChainMargins(s, oracle_list(prev), p.dt, eps, p.cap)
            for c in flips:
                mg = cm.cell(c)
                assert min(mg.values()) < tie(eps), (k, c, got.ranks[c], want.ranks[c], mg)
