"""LU-SGS implicit iteration on the GPU against the
oracle's composition of reference calls (oracle/step.py lusgs_step:
SPEC.md:399-407 with TtTensor::divided_by_rank_one, tt_tensor.cpp:247-261).
The GPU runs the sweeps level by level; the oracle runs them cell by cell in
index order -- same increments, same sums."""
import numpy as np
import pytest

from oracle import ref
from oracle.parity import macro_err, oracle_list
from oracle.step import OracleSolver
from oracle.tt import rel_err
from paper_1912_04582_b200.problems import config, obstacle_flow, shock_tube
from paper_1912_04582_b200.tt_batch import TtBatch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_1912_04582_b200.cuda import Context
    c = Context(0)
    yield c
    c.close()


def lockstep(ctx, p, iters):
    """Every iteration starts from the oracle's state on both sides; the
    oracle is the compiled reference's LU-SGS composition (oracle/ref_step.cpp)
    when its library is present, else the numpy one."""
    ctx.setup(p)
    r = ref.RefSolver.for_problem(p) if ref.available() else None
    s = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = p.f0
    for it in range(iters):
        ctx.upload_state(f)
        ctx.lusgs_step(p.dt, p.eps, p.cap, 1)
        got = ctx.download_state()
        if r is not None:
            r.set_state(f)
            r.lusgs_step(p.dt, p.eps, p.cap)
            want, wm = r.state(), r.macros(p.mesh.ncell)
        else:
            out, macros = s.lusgs_step(oracle_list(f), p.dt, p.eps, p.cap)
            want, wm = TtBatch.from_list(out), np.stack([m.as_array() for m in macros])
        assert macro_err(ctx.macros(), wm) <= 1e-8
        for i in range(p.mesh.ncell):
            assert rel_err(got.full(i), want.full(i)) <= 10 * p.eps, (it, i)
            assert tuple(got.ranks[i]) == tuple(want.ranks[i]), (it, i)
        f = want


def test_lusgs_shock_tube_lockstep(ctx):
    """Config 1's mesh in natural order: the forward sweep is one chain of
    64 levels (the worst case for level scheduling)."""
    p = config(1)
    lockstep(ctx, p, 3)
    assert ctx.lusgs_levels() == (64, 64)


def test_lusgs_periodic_box_lockstep(ctx):
    lockstep(ctx, config(2, scale=3 / 32), 2)


def test_lusgs_obstacle_lockstep(ctx):
    """Jittered, shuffled obstacle mesh (oblique faces: Hadamard off-diagonal
    terms with xi_n and |xi_n|; diffuse walls and free stream stay explicit)."""
    p = obstacle_flow((5, 4, 4), hole=2, nv=12)
    lockstep(ctx, p, 2)
    nf, nb = ctx.lusgs_levels()
    assert 1 < nf < p.mesh.ncell and 1 < nb < p.mesh.ncell


def test_lusgs_equilibrium_fixed_point(ctx):
    """one LU-SGS iteration on a global-Maxwellian state with
    compatible (specular) walls leaves it unchanged to eps_round."""
    q = shock_tube(nx=8)
    f = q.f0.subset(np.zeros(q.mesh.ncell, dtype=int))  # every cell = cell 0's Maxwellian
    ctx.setup(q)
    ctx.upload_state(f)
    ctx.lusgs_step(q.dt, q.eps, q.cap, 1)
    got = ctx.download_state()
    for i in range(q.mesh.ncell):
        assert rel_err(got.full(i), f.full(i)) <= q.eps


def test_lusgs_rejects_partitioned_mesh(ctx):
    p = config(2, scale=3 / 32)
    ctx.setup(p)
    ctx.set_owned(p.mesh.ncell - 1)
    with pytest.raises(ValueError, match="unpartitioned"):
        ctx.lusgs_step(p.dt, p.eps, p.cap, 1)
    ctx.set_owned(p.mesh.ncell)
