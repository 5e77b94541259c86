"""GPU parity: the CUDA C-ABI path against the CPU oracle on identical,
seeded inputs (BASELINE.json north_star bar):

* reconstructed per-tensor full tensors within 10 x the TT tolerance
  (relative Frobenius; for the step, relative to the oracle's tensor);
* macroparameters within 1e-8 relative (S and heat flux: 1e-8 absolute in
  the dimensionless S, which is O(1) or smaller);
* identical TT ranks except where the oracle's decision margin
  |tail + sigma^2 - budget| / budget is below TIE(eps) = max(1e-12,
  1e-14/eps) (oracle/parity.py derives the window from the SVD error
  model); every mismatch must be explained by such a margin on the
  tensor's own dependency chain -- no flip allowances.

The step oracle is the COMPILED REFERENCE (oracle/_ref, the unmodified
proj/src/*.cpp + the S1 composition of reference calls) when its library
travelled to the box, else the numpy restatement; margins come from the
numpy restatement's singular values on the same inputs.
"""
import math

import numpy as np
import pytest

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from oracle import ref
from oracle.physics import (GasParameters, Macroparameters, VelocityGrid, compute_collision,
                            compute_macro, maxwell_tt, shakhov_tt, shakhov_tt_raw)
from oracle.step import OracleSolver
from oracle.parity import ChainMargins, macro_err, oracle_list, oracle_margin, tie
from oracle.tt import TtTensor, random_tt, rel_err
from paper_1912_04582_b200.problems import config, gas_params
from paper_1912_04582_b200.tt_batch import TtBatch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    from paper_1912_04582_b200.cuda import Context
    c = Context(0)
    yield c
    c.close()


def sum_tt(terms):
    s = terms[0][0].scaled(terms[0][1])
    for t, sc in terms[1:]:
        s = s + t.scaled(sc)
    return s


def check_round(ctx, groups, eps, cap=0):
    """groups: list of lists of (TtTensor, scale)."""
    flat = [t for g in groups for t, _ in g]
    scales = np.array([sc for g in groups for _, sc in g])
    go = np.cumsum([0] + [len(g) for g in groups])
    n = flat[0].mode_sizes()[0]
    ctx.set_grid(n, 1.0)
    got, mg = ctx.rounded(TtBatch.from_list(flat), eps, cap, group_off=go, scale=scales,
                          margins=True)
    flips = 0
    for o, g in enumerate(groups):
        s = sum_tt(g)
        want = s.rounded(eps, cap)
        gf = got.full(o)
        full = s.to_full()
        if cap == 0:
            assert rel_err(gf, full) <= 10 * eps + 1e-14, (o, rel_err(gf, full))
        assert rel_err(gf, want.to_full()) <= 10 * eps + 1e-14
        gr = tuple(int(v) for v in got.ranks[o])
        if gr != want.ranks()[1:3]:
            m = oracle_margin(s, eps, cap)
            assert m < tie(eps), (o, gr, want.ranks(), m)
            flips += 1
    return got, flips


def test_round_random_sums(ctx):
    rng = np.random.default_rng(1)
    groups = []
    for _ in range(40):
        n = 12
        k = int(rng.integers(1, 6))
        groups.append([(random_tt(rng, n, n, n, int(rng.integers(1, 7)), int(rng.integers(1, 7))),
                        float(rng.standard_normal())) for _ in range(k)])
    for eps in (1e-2, 1e-6, 1e-12):
        check_round(ctx, groups, eps)


def test_round_t_route_and_cap(ctx):
    # summed ranks above n exercise the T route (R1 > n1) and the cap
    rng = np.random.default_rng(2)
    n = 8
    groups = [[(random_tt(rng, n, n, n, 5, 6), 1.0), (random_tt(rng, n, n, n, 6, 5), -0.5)]
              for _ in range(10)]
    check_round(ctx, groups, 1e-6)
    got, _ = check_round(ctx, groups, 1e-3, cap=3)
    assert got.ranks.max() <= 3


def decaying_tt(rng, n, r, decay=0.5):
    """N(0,1) cores with decay^a on the outer cores' rank indices (config 3 style)."""
    w = decay ** np.arange(r)
    return TtTensor(rng.standard_normal((n, r)) * w[None, :], rng.standard_normal((n, r, r)),
                    rng.standard_normal((r, n)) * w[:, None])


def test_round_spill_plan_n64_t_route_cap(ctx):
    """n = 64 with summed ranks 140 (config 5's cell residual at cap 20: six
    face fluxes + J): the working set exceeds shared memory, so the launch
    takes the spill plan (global scratch slices, persistent CTAs), T route."""
    rng = np.random.default_rng(64)
    n = 64
    groups = [[(random_tt(rng, n, n, n, 20, 20), float(rng.standard_normal())) for _ in range(7)]
              for _ in range(3)]
    got, _ = check_round(ctx, groups, 1e-5, cap=20)
    assert got.ranks.max() == 20


def test_round_spill_plan_n64_w_route(ctx):
    """n = 64, summed ranks 60 < n (W route) with decaying spectra, no cap:
    spill plan, rank decisions against the oracle's margins."""
    rng = np.random.default_rng(65)
    n = 64
    groups = [[(decaying_tt(rng, n, 20, 0.3), 1.0), (decaying_tt(rng, n, 20, 0.3), -0.7),
               (decaying_tt(rng, n, 20, 0.3), 0.4)] for _ in range(3)]
    check_round(ctx, groups, 1e-6)


def test_round_config3_shape(ctx):
    """Config 3 inputs (32^3, six rank-12 summands with 0.5 decay, rank 72
    summed) at a few tensors: every reading gives full ranks (32, 32)."""
    from paper_1912_04582_b200.problems import rounding_summands
    rng = np.random.default_rng(3)
    f, m, l = rounding_summands(rng, 3)
    groups = [[(TtTensor(f[6 * g + k], m[6 * g + k], l[6 * g + k]), 1.0) for k in range(6)]
              for g in range(3)]
    got, flips = check_round(ctx, groups, 1e-6)
    assert flips == 0
    assert all(tuple(r) == (32, 32) for r in got.ranks)


def test_round_reference_edge_cases(ctx):
    rng = np.random.default_rng(31)
    a = random_tt(rng, 8, 8, 8, 2, 3)
    z = TtTensor.constant(6, 6, 6, 0.0)
    ctx.set_grid(8, 1.0)
    got = ctx.rounded(TtBatch.from_list([a, a]), 1e-13, group_off=[0, 2])
    assert tuple(got.ranks[0]) == (2, 3)  # test_tt_tensor.cpp:129-138
    assert rel_err(got.full(0), 2 * a.to_full()) < 1e-12
    ctx.set_grid(6, 1.0)
    got = ctx.rounded(TtBatch.from_list([z, z]), 1e-10, group_off=[0, 2])
    assert tuple(got.ranks[0]) == (1, 1)  # :305-310 canonical zero
    assert np.linalg.norm(got.full(0)) == 0.0
    b = random_tt(rng, 8, 8, 8, 3, 3)
    ctx.set_grid(8, 1.0)
    got = ctx.rounded(TtBatch.from_list([b] * 5), 1e-12, group_off=[0, 5])
    assert tuple(got.ranks[0]) == (3, 3)  # :295-303 m-fold sum


def test_round_perturbed_maxwellian(ctx):  # test_tt_tensor.cpp:140-157 shape
    rng = np.random.default_rng(37)
    n = 16
    x = -3.0 + 6.0 * np.arange(n) / (n - 1)
    g = np.exp(-x * x)
    m = TtTensor.rank_one(g, g, g)
    groups = []
    for _ in range(8):
        p = random_tt(rng, n, n, n, 6, 6)
        groups.append([(m, 1.0), (p, 1e-4 * m.frobenius_norm() / p.frobenius_norm())])
    check_round(ctx, groups, 1e-7)


def mixture(grid, gas, rng):
    f = maxwell_tt(1.0 + 0.2 * rng.random(), 0.8 + 0.4 * rng.random(), rng.uniform(-0.5, 0.5, 3),
                   grid, gas)
    g = maxwell_tt(0.3 * rng.random() + 0.05, 0.6 + 0.8 * rng.random(), rng.uniform(-1, 1, 3),
                   grid, gas)
    return f + g


def test_macro_parity(ctx):
    gas_a = gas_params(0.1, 32.0)
    gas = GasParameters(*gas_a)
    grid = VelocityGrid(24, 6.0)
    rng = np.random.default_rng(5)
    fs = [mixture(grid, gas, rng) for _ in range(16)]
    ctx.set_grid(24, 6.0)
    ctx.set_gas(gas_a)
    got = ctx.compute_macro(TtBatch.from_list(fs))
    for i, f in enumerate(fs):
        m = compute_macro(f, grid, gas)
        want = m.as_array()
        np.testing.assert_allclose(got[i, [0, 4, 5, 6]], want[[0, 4, 5, 6]], rtol=1e-8)
        np.testing.assert_allclose(got[i, 1:4], want[1:4], rtol=1e-8, atol=1e-10)
        np.testing.assert_allclose(got[i, 7:10], want[7:10], rtol=1e-8, atol=1e-10)


def test_macro_rejects_zero(ctx):
    ctx.set_grid(8, 1.0)
    with pytest.raises(RuntimeError, match="nonpositive density"):
        ctx.compute_macro(TtBatch.from_list([TtTensor.constant(8, 8, 8, 0.0)]))


def test_collision_parity(ctx):
    """J = nu * round(round(f_S) - f) (physics.cpp:112-125).  When both
    roundings make the oracle's rank decisions the two J are the same
    truncated SVDs: they agree to 1e-9 ||J|| plus the singular-subspace
    perturbation of the kept part, ~u ||f|| / (sigma_r - sigma_r+1) with
    sigma ~ eps ||f|| at the cut, i.e. TIE(eps) nu ||f|| (1000 x tighter than
    the rounding budget).  A decision inside the TIE window may differ; then
    the difference is one truncated term, within the budget 10 eps nu ||f||."""
    gas_a = gas_params(0.1, 32.0)
    gas = GasParameters(*gas_a)
    grid = VelocityGrid(24, 6.0)
    rng = np.random.default_rng(7)
    fs = [mixture(grid, gas, rng) for _ in range(12)]
    fs.append(maxwell_tt(1.0, 1.0, np.zeros(3), grid, gas))  # equilibrium: J ~ 0
    ctx.set_grid(24, 6.0)
    ctx.set_gas(gas_a)
    eps = 1e-6
    jr, mac = ctx.compute_collision(TtBatch.from_list(fs), eps)
    for i, f in enumerate(fs):
        mo = []
        j = compute_collision(f, grid, gas, eps, mo)
        nu = mo[0].pressure / (gas.mu_ref * (mo[0].temperature / gas.t_ref) ** gas.omega)
        assert mac[i, 10] == pytest.approx(nu, rel=1e-8)
        got = jr.full(i) * mac[i, 10]
        want = j.to_full()
        nf = np.linalg.norm(f.to_full())
        err = np.linalg.norm(got - want)
        if tuple(jr.ranks[i]) == j.ranks()[1:3]:
            assert err <= 1e-9 * np.linalg.norm(want) + tie(eps) * nu * nf, (i, err)
        else:
            raw = shakhov_tt_raw(mo[0], grid, gas)
            mg = min(oracle_margin(raw, eps), oracle_margin(raw.rounded(eps) - f, eps))
            assert mg < tie(eps), (i, jr.ranks[i], j.ranks(), mg)
            assert err <= 10 * eps * nu * nf


def oracle_state(problem):
    return [TtTensor(*problem.f0.get(i)) for i in range(problem.mesh.ncell)]


def check_step(ctx, problem, nsteps, eps_mult=10.0):
    """Lock-step: every step starts from the oracle's state on both sides.
    Returns (worst reconstruction error, number of rank mismatches); every
    mismatch is asserted to sit inside the TIE window of an oracle decision
    on the cell's chain (fluxes of its faces, f_S, J_r, R, state)."""
    ctx.setup(problem)
    solver = OracleSolver(problem.mesh, problem.nv, problem.bound, problem.gas, problem.bcs)
    r = ref.RefSolver.for_problem(problem) if ref.available() else None
    f = problem.f0
    eps, ncell = problem.eps, problem.mesh.ncell
    worst, flips = 0.0, 0
    for it in range(nsteps):
        ctx.upload_state(f)
        ctx.step(problem.dt, eps, problem.cap, 1)
        got = ctx.download_state()
        gm = ctx.macros()
        if r is not None:
            r.set_state(f)
            r.step(problem.dt, eps, problem.cap)
            want, wm = r.state(), r.macros(ncell)
        else:
            f_new, macros = solver.step(oracle_list(f), problem.dt, eps, problem.cap)
            want, wm = TtBatch.from_list(f_new), np.stack([m.as_array() for m in macros])
        assert macro_err(gm, wm) <= 1e-8
        bad = []
        for i in range(ncell):
            e = rel_err(got.full(i), want.full(i))
            worst = max(worst, e)
            assert e <= eps_mult * eps, (it, i, e)
            if tuple(got.ranks[i]) != tuple(want.ranks[i]):
                bad.append(i)
        if bad:
            cm = ChainMargins(solver, oracle_list(f), problem.dt, eps, problem.cap)
            for i in bad:
                mg = cm.cell(i)
                assert min(mg.values()) < tie(eps), (it, i, got.ranks[i], want.ranks[i], mg)
        flips += len(bad)
        f = want
    if r is not None:
        r.close()
    return worst, flips


def test_step_config1_shock_tube(ctx):
    p = config(1)
    check_step(ctx, p, 3)


def test_step_config2_small(ctx):
    p = config(2, scale=3 / 32)
    check_step(ctx, p, 2)


def test_step_config5_small(ctx):
    """Config 5's velocity mesh (64^3 on [-8,8]^3, eps 1e-5, cap 20) on a
    2x2x2 periodic box: n = 64 through the whole step."""
    p = config(5, scale=2 / 128)
    assert p.nv == 64 and p.cap == 20
    check_step(ctx, p, 2)


def test_step_stages_config2(ctx):
    """Per-stage lock-step: fluxes, J and residual of one step."""
    p = config(2, scale=2 / 32)
    ctx.setup(p)
    ctx.step(p.dt, p.eps, p.cap, 1)
    solver = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = oracle_state(p)
    _, _, d = solver.step(f, p.dt, p.eps, p.cap, detail=True)
    phi = ctx.stage("phi")
    for j, want in d["phi"].items():
        assert rel_err(phi.full(j), want.to_full()) <= 10 * p.eps
    res = ctx.stage("res")
    for i, want in enumerate(d["R"]):
        assert rel_err(res.full(i), want.to_full()) <= 10 * p.eps


def test_step_many_steps_stable(ctx):
    """Free-running GPU steps stay finite with bounded ranks (SPEC.md
    explicit_step CFL smoke)."""
    p = config(1)
    ctx.setup(p)
    ctx.step(p.dt, p.eps, p.cap, 20)
    st = ctx.download_state()
    assert st.ranks.max() <= 16
    assert np.all(np.isfinite(st.cores))
    m = ctx.macros()
    assert np.all(m[:, 0] > 0) and np.all(m[:, 4] > 0)


def test_download_in_chunks_matches_one_gather(ctx, monkeypatch):
    """The state download gathers in bounded chunks (capi.cu download_set,
    2 GB by default so config 5's 19 GB state needs no full staging copy):
    forcing chunks of a few tensors gives bitwise the one-chunk result."""
    p = config(1)
    ctx.setup(p)
    ctx.step(p.dt, p.eps, p.cap, 3)
    whole = ctx.download_state()
    sizes = np.diff(whole.offsets)
    monkeypatch.setenv("TTDVM_DOWNLOAD_CHUNK", str(int(3 * sizes.max())))
    l0 = ctx.launch_count()
    parts = ctx.download_state()
    gathers = ctx.launch_count() - l0
    monkeypatch.delenv("TTDVM_DOWNLOAD_CHUNK")
    # chunks of <= 3 of the largest tensors: at least total / (3 max) gathers
    assert gathers >= max(2, math.ceil(whole.offsets[-1] / (3 * sizes.max()))), gathers
    assert np.array_equal(parts.ranks, whole.ranks)
    assert np.array_equal(parts.cores, whole.cores)


def test_partitioned_step_two_contexts():
    """Two library contexts on one GPU, each owning an x-slab of a periodic
    box with ghost cells, stepped one after the other with halo pack/unpack
    through device buffers (no kernel waits on another): must reproduce the
    single-rank oracle step."""
    import torch

    from paper_1912_04582_b200.cuda import Context
    from paper_1912_04582_b200.mesh import slab_partition
    from paper_1912_04582_b200.partition import build_part, local_state
    from paper_1912_04582_b200.problems import periodic_box

    p = periodic_box((4, 2, 2), steps=2)
    owner = slab_partition(p.mesh, 2)
    parts = [build_part(p.mesh, owner, r) for r in range(2)]
    ctxs = []
    for part in parts:
        c = Context(0)
        c.set_grid(p.nv, p.bound)
        c.set_gas(p.gas)
        c.set_mesh(part.mesh)
        c.set_bcs(p.bcs)
        c.set_owned(part.n_owned)
        c.upload_state(local_state(part, p.f0))
        ctxs.append(c)
    for _ in range(2):
        for c in ctxs:
            c.step(p.dt, p.eps, p.cap, 1)
        for r, part in enumerate(parts):
            for q, ids in part.send.items():
                need = ctxs[r].halo_size(ids)
                buf = torch.empty(max(1, need), dtype=torch.float64, device="cuda")
                torch.cuda.synchronize()
                ranks, offs = ctxs[r].halo_pack(ids, buf.data_ptr(), need)
                ctxs[q].halo_unpack(parts[q].recv[r], ranks, offs, buf.data_ptr())
    solver = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = oracle_state(p)
    for _ in range(2):
        f, _ = solver.step(f, p.dt, p.eps, p.cap)
    for part, c in zip(parts, ctxs):
        st = c.download_state()
        for lc in range(part.n_owned):
            g = int(part.owned[lc])
            assert rel_err(st.full(lc), f[g].to_full()) <= 10 * p.eps
        c.close()


def test_config2_full_size_conservation(ctx):
    """Config 2 at its full size (32^3 periodic cells, 24^3 velocity mesh):
    size-independent properties of the step -- interior fluxes telescope
    and the S-model collision conserves mass and momentum, so the totals
    sum_i n_i V_i and sum_i n_i u_i V_i stay put to the rounding budget
    (SPEC.md:415); states stay finite with ranks <= n."""
    p = config(2)
    assert p.mesh.ncell == 32768
    ctx.setup(p)
    vol = p.mesh.cell_volume
    ctx.step(p.dt, p.eps, p.cap, 1)
    m0 = ctx.macros()  # macroparameters of t^0
    k = 8
    ctx.step(p.dt, p.eps, p.cap, k)
    mk = ctx.macros()  # of t^k
    mass0, massk = np.sum(m0[:, 0] * vol), np.sum(mk[:, 0] * vol)
    assert abs(massk - mass0) <= 10 * p.eps * k * mass0
    mom0 = (m0[:, 0] * vol) @ m0[:, 1:4]
    momk = (mk[:, 0] * vol) @ mk[:, 1:4]
    assert np.all(np.abs(momk - mom0) <= 10 * p.eps * k * mass0)
    st = ctx.download_state()
    assert np.all(np.isfinite(st.cores)) and st.ranks.max() <= p.nv


def test_round_batch_edge_inputs(ctx):
    """Empty and ragged batches, bad arguments and non-finite data through
    the C ABI (the reference throws std::invalid_argument for argument and
    shape errors, proj/src/tt_tensor.cpp:139-145; a non-finite sum has no
    rounding)."""
    rng = np.random.default_rng(41)
    n = 10
    ctx.set_grid(n, 1.0)
    empty = TtBatch.from_list([], n=n)
    got = ctx.rounded(empty, 1e-8, group_off=[0])
    assert got.count == 0
    # ragged: every tensor its own ranks, groups of 1..4 summands
    ts = [random_tt(rng, n, n, n, int(rng.integers(1, 7)), int(rng.integers(1, 7)))
          for _ in range(10)]
    groups = [[(ts[0], 1.0)], [(ts[1], 1.0), (ts[2], -2.0)],
              [(ts[3], 1.0), (ts[4], 0.5), (ts[5], 1.0), (ts[6], 3.0)],
              [(ts[7], 1.0), (ts[8], 1.0), (ts[9], -1.0)]]
    check_round(ctx, groups, 1e-9)
    with pytest.raises(ValueError):
        ctx.rounded(TtBatch.from_list(ts[:2]), 0.0)  # eps must be > 0
    bad = TtBatch.from_list(ts[:2])
    bad.offsets[1] += 1
    with pytest.raises(ValueError):
        ctx.rounded(bad, 1e-8)  # offsets inconsistent with the ranks
    with pytest.raises(ValueError):
        ctx.rounded(TtBatch.from_list(ts[:2]), 1e-8, group_off=[0, 3])  # groups past the batch
    nanb = TtBatch.from_list(ts[:1])
    nanb.cores[5] = np.nan
    with pytest.raises(RuntimeError):
        ctx.rounded(nanb, 1e-8)
    # the context stays usable after the errors
    got = ctx.rounded(TtBatch.from_list(ts[:1]), 1e-12)
    assert rel_err(got.full(0), ts[0].to_full()) < 1e-11
    with pytest.raises(ValueError):
        ctx.rounded(TtBatch.from_list(ts[:2]), 1e-8, group_off=[0, 0, 2])  # an empty sum


@pytest.mark.parametrize("cfg,scale,blocks", [(2, 4 / 32, 3), (4, 0.1, 5)])
def test_blocked_step_matches_one_block(ctx, cfg, scale, blocks):
    """ttdvm_cuda_set_blocks: the bounded-memory step (fluxes, residuals and
    updates of contiguous cell blocks) forms the same sums as the one-block
    step, so states agree to roundoff with identical ranks."""
    p = config(cfg, scale)
    res = []
    for nb in (1, blocks):
        ctx.setup(p)
        ctx.set_blocks(nb)
        ctx.step(p.dt, p.eps, p.cap, 2)
        res.append((ctx.download_state(), ctx.macros()))
    ctx.set_blocks(0)
    (a, ma), (b, mb) = res
    np.testing.assert_array_equal(a.ranks, b.ranks)
    for i in range(p.mesh.ncell):
        assert rel_err(b.full(i), a.full(i)) <= 1e-12, i
    np.testing.assert_allclose(mb, ma, rtol=1e-12, atol=1e-14)
