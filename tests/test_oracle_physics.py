"""Pins oracle/physics.py against the reference's physics, velocity-grid and
boundary known-answer tests (proj/tests/test_physics.cpp,
test_velocity_grid.cpp, test_boundary.cpp; file:line per test).  Argon
fixture as in test_physics.cpp:13-22; tolerances are the reference's
(doctest::Approx default ~1.19e-5 relative where none is given)."""
import math

import numpy as np
import pytest

from oracle.physics import (BoundaryCondition, GasParameters, VelocityGrid, bc_kind_from_string,
                            compute_collision, compute_macro, maxwell_tt, shakhov_tt,
                            symmetry_ghost, viscosity, wall_ghost, Macroparameters)
from oracle.tt import TtTensor, hadamard, rel_err

APPROX = 100 * np.finfo(np.float32).eps  # doctest::Approx default epsilon
KRG = 208.13


def argon():
    return GasParameters(molecule_mass=6.6335e-26, gas_constant=208.13, prandtl=2.0 / 3.0,
                         mu_ref=2.117e-5, t_ref=273.0, omega=0.734)


def approx(v, eps=APPROX):
    return pytest.approx(v, rel=eps)


# ------------------------------------------------------------ physics tests
def test_viscosity_power_law():  # test_physics.cpp:26-34
    gas = argon()
    assert viscosity(gas.t_ref, gas) == gas.mu_ref
    assert viscosity(5.0 * gas.t_ref, gas) == approx(gas.mu_ref * 5.0 ** 0.734, 1e-14)
    gas.omega = 1.0
    assert viscosity(2.0 * gas.t_ref, gas) == approx(2.0 * gas.mu_ref, 1e-14)


def test_maxwell_pointwise():  # :36-55
    gas = argon()
    n0, t0 = 3.1e21, 350.0
    u0 = np.array([400.0, -150.0, 80.0])
    grid = VelocityGrid(16, abs(u0[0]) + 4.5 * math.sqrt(2 * gas.gas_constant * t0))
    fm = maxwell_tt(n0, t0, u0, grid, gas)
    assert fm.ranks() == (1, 1, 1, 1)
    d = fm.to_full()
    two_rt = 2.0 * gas.gas_constant * t0
    pref = n0 / (math.pi * two_rt) ** 1.5
    x = grid.nodes
    for i in range(0, 16, 3):
        for j in range(0, 16, 3):
            for k in range(0, 16, 3):
                v2 = (x[i] - u0[0]) ** 2 + (x[j] - u0[1]) ** 2 + (x[k] - u0[2]) ** 2
                assert d[i, j, k] == approx(pref * math.exp(-v2 / two_rt), 1e-13)


def test_macro_resting_gas():  # :57-75
    gas = argon()
    n0, t0 = 2e23, 200.0
    grid = VelocityGrid(64, 4.0 * math.sqrt(2 * gas.gas_constant * t0))
    m = compute_macro(maxwell_tt(n0, t0, np.zeros(3), grid, gas), grid, gas)
    assert m.number_density == approx(n0, 1e-3)
    assert m.temperature == approx(t0, 1e-3)
    assert np.linalg.norm(m.velocity) < 1e-8 * math.sqrt(gas.gas_constant * t0)
    assert np.linalg.norm(m.shakhov_s) < 1e-8
    assert np.linalg.norm(m.heat_flux) < 1e-3
    assert m.mass_density == approx(gas.molecule_mass * n0)
    assert m.pressure == approx(m.mass_density * gas.gas_constant * m.temperature)


def test_macro_freestream_state():  # :77-85
    gas = argon()
    n0, t0 = 2e23, 200.0
    u0 = np.array([2630.0, 0.0, 0.0])
    grid = VelocityGrid(48, 2630.0 + 4.5 * math.sqrt(2 * gas.gas_constant * t0))
    m = compute_macro(maxwell_tt(n0, t0, u0, grid, gas), grid, gas)
    assert m.number_density == approx(n0, 1e-3)
    assert m.temperature == approx(t0, 1e-3)
    assert m.velocity[0] == approx(2630.0, 1e-3)


def test_macro_zero_rejected():  # :87-91
    gas = argon()
    grid = VelocityGrid(8, 1000.0)
    with pytest.raises(RuntimeError):
        compute_macro(TtTensor.constant(8, 8, 8, 0.0), grid, gas)


def test_moment_idempotence():  # :94-108
    gas = argon()
    grid = VelocityGrid(32, 2800.0)
    f = (maxwell_tt(1e20, 220.0, np.array([300.0, 0, 0]), grid, gas)
         + maxwell_tt(4e19, 400.0, np.array([-200.0, 100, 0]), grid, gas))
    m1 = compute_macro(f, grid, gas)
    m2 = compute_macro(maxwell_tt(m1.number_density, m1.temperature, m1.velocity, grid, gas),
                       grid, gas)
    assert m2.number_density == approx(m1.number_density, 1e-6)
    assert m2.temperature == approx(m1.temperature, 1e-6)
    assert np.linalg.norm(m2.velocity - m1.velocity) < 1e-6 * (np.linalg.norm(m1.velocity) + 1)


def _macro(gas, n, t, u, s):
    m = Macroparameters()
    m.number_density, m.temperature = n, t
    m.velocity = np.asarray(u, dtype=np.float64)
    m.mass_density = gas.molecule_mass * n
    m.pressure = m.mass_density * gas.gas_constant * t
    m.shakhov_s = np.asarray(s, dtype=np.float64)
    return m


def test_shakhov_is_maxwellian_at_s0():  # :110-123
    gas = argon()
    grid = VelocityGrid(16, 1500.0)
    m = _macro(gas, 5e20, 300.0, [200, -100, 50], [0, 0, 0])
    fs = shakhov_tt(m, grid, gas, 1e-7)
    fm = maxwell_tt(m.number_density, m.temperature, m.velocity, grid, gas)
    assert (fs - fm).frobenius_norm() <= 1e-13 * fm.frobenius_norm()


def test_shakhov_pointwise_and_rank_bound():  # :125-168
    gas = argon()
    g = np.random.default_rng(17)
    for nv in (16, 32, 64):
        grid = VelocityGrid(nv, 2000.0)
        for _ in range(3):
            u = g.uniform(-1, 1, size=8)
            m = _macro(gas, 1e20 * (1.0 + 0.5 * u[0]), 260.0 + 120.0 * u[1],
                       300 * u[2:5], u[5:8])
            fs = shakhov_tt(m, grid, gas, 1e-7)
            assert fs.ranks()[1] <= 10 and fs.ranks()[2] <= 10
            if nv == 16:
                got = fs.to_full()
                s = math.sqrt(2 * gas.gas_constant * m.temperature)
                pref = m.number_density / (math.pi * s * s) ** 1.5
                c = [(grid.nodes - m.velocity[a]) / s for a in range(3)]
                C = np.meshgrid(*c, indexing="ij")
                c2 = C[0] ** 2 + C[1] ** 2 + C[2] ** 2
                sc = sum(m.shakhov_s[a] * C[a] for a in range(3))
                want = pref * np.exp(-c2) * (1.0 + 0.8 * (1.0 - gas.prandtl) * sc * (c2 - 2.5))
                assert np.sqrt(np.sum((got - want) ** 2) / np.sum(want ** 2)) <= 2e-7


def test_collision_vanishes_at_equilibrium():  # :170-179
    gas = argon()
    t0 = 300.0
    grid = VelocityGrid(32, 4.8 * math.sqrt(2 * gas.gas_constant * t0))
    fm = maxwell_tt(8e20, t0, np.zeros(3), grid, gas)
    mo = []
    j = compute_collision(fm, grid, gas, 1e-7, mo)
    nu = mo[0].pressure / viscosity(mo[0].temperature, gas)
    assert j.frobenius_norm() <= 1e-7 * nu * fm.frobenius_norm()


def test_collision_conserves():  # :181-203
    gas = argon()
    t_hot = 420.0
    grid = VelocityGrid(32, 600.0 + 5.5 * math.sqrt(2 * gas.gas_constant * t_hot))
    f = (maxwell_tt(6e20, 250.0, np.array([350.0, -120, 0]), grid, gas)
         + maxwell_tt(3e20, t_hot, np.array([-150.0, 200, 90]), grid, gas))
    j = compute_collision(f, grid, gas, 1e-9)
    w = grid.weights
    xw = grid.nodes * w
    x2w = grid.nodes * xw
    m = compute_macro(f, grid, gas)
    nu = m.pressure / viscosity(m.temperature, gas)
    scale = nu * m.number_density
    vref = math.sqrt(gas.gas_constant * m.temperature)
    assert abs(j.convolve(w, w, w)) / scale < 1e-8
    for u, v, ww in ((xw, w, w), (w, xw, w), (w, w, xw)):
        assert abs(j.convolve(u, v, ww)) / (scale * vref) < 1e-8
    e = j.convolve(x2w, w, w) + j.convolve(w, x2w, w) + j.convolve(w, w, x2w)
    assert abs(e) / (scale * vref * vref) < 1e-8


# ------------------------------------------------------- velocity grid tests
def _maxwell_factor(g, u, t):
    v = g.nodes - u
    return np.exp(-v * v / (2.0 * KRG * t)) / math.sqrt(2.0 * math.pi * KRG * t)


def test_grid_construction():  # test_velocity_grid.cpp:27-46
    tiny = VelocityGrid(2, 1.0)
    assert tiny.nodes[0] == -1.0 and tiny.nodes[1] == 1.0 and tiny.dxi == 2.0
    with pytest.raises(ValueError):
        VelocityGrid(1, 1.0)
    with pytest.raises(ValueError):
        VelocityGrid(8, 0.0)
    g = VelocityGrid(16, 3.0)
    box = 16 * g.dxi
    w = g.weights
    assert TtTensor.constant(16, 16, 16, 1.0).convolve(w, w, w) == approx(box ** 3, 1e-13)
    assert abs(g.xi_tensor(1).convolve(w, w, w)) < 1e-10 * box ** 3


def test_grid_maxwell_density():  # :48-65
    t0, u0, n0 = 200.0, 1200.0, 2e23
    g = VelocityGrid(64, abs(u0) + 4.0 * math.sqrt(2.0 * KRG * t0))
    fm = TtTensor.rank_one(_maxwell_factor(g, u0, t0), _maxwell_factor(g, 0, t0),
                           _maxwell_factor(g, 0, t0)).scaled(n0)
    w = g.weights
    assert abs(fm.convolve(w, w, w) - n0) / n0 < 1e-3
    assert hadamard(g.xi_tensor(1), fm).convolve(w, w, w) == approx(n0 * u0, 1e-3)


def test_xi_tensors():  # :67-82
    g = VelocityGrid(8, 2.0)
    for axis in (1, 2, 3):
        t = g.xi_tensor(axis)
        assert t.ranks() == (1, 1, 1, 1)
        d = t.to_full()
        idx = np.meshgrid(*(range(8),) * 3, indexing="ij")[axis - 1]
        assert np.array_equal(d, g.nodes[idx])
    with pytest.raises(ValueError):
        g.xi_tensor(4)


def test_xi_normal():  # :84-99
    g = VelocityGrid(16, 2.0)
    ax = g.xi_normal(np.array([1.0, 0, 0]))
    assert ax.ranks() == (1, 1, 1, 1)
    assert rel_err(ax.to_full(), g.xi_tensor(1).to_full()) < 1e-14
    ob = np.ones(3) / math.sqrt(3.0)
    t = g.xi_normal(ob)
    assert t.ranks()[1] <= 2 and t.ranks()[2] <= 2
    assert rel_err(t.to_full(), g.dense_xi_normal(ob)) < 1e-13
    with pytest.raises(ValueError):
        g.xi_normal(np.array([1.0, 1.0, 0.0]))


def test_abs_estimate_axis_exact():  # :101-118
    g = VelocityGrid(16, 2.0)
    for axis in range(3):
        n = np.zeros(3)
        n[axis] = 1.0
        e = g.abs_xi_estimate(n, 4)
        assert e.ranks()[1] == 1 and e.ranks()[2] == 1
        idx = np.meshgrid(*(range(16),) * 3, indexing="ij")[axis]
        np.testing.assert_allclose(e.to_full(), np.abs(g.nodes[idx]), rtol=1e-12, atol=1e-300)


def test_abs_estimate_dominates():  # :120-143
    g = VelocityGrid(32, 3.0)
    n = np.array([1.0, 1.0, 0.0]) / math.sqrt(2.0)
    e = g.abs_xi_estimate(n, 4)
    assert e.ranks()[1] <= 4 and e.ranks()[2] <= 4
    ax = np.abs(g.dense_xi_normal(n))
    d = e.to_full() - ax
    assert math.sqrt(np.sum(d * d) / np.sum(ax * ax)) <= 0.15
    assert d.min() >= -1e-12 * g.xi_max


def test_positive_part_axis_ramp():  # :145-155
    g = VelocityGrid(16, 2.0)
    p = g.xi_normal_positive(np.array([0.0, 0.0, 1.0]), 4)
    assert p.ranks()[1] == 1 and p.ranks()[2] == 1
    d = p.to_full()
    np.testing.assert_allclose(d[:, 0, :], np.broadcast_to(np.maximum(g.nodes, 0.0), (16, 16)),
                               rtol=1e-12, atol=1e-13)


def test_positive_plus_negative():  # :157-163
    g = VelocityGrid(32, 3.0)
    n = np.array([0.3, 0.9, 0.3])
    n = n / np.linalg.norm(n)
    s = g.xi_normal_positive(n, 4) + g.xi_normal_negative(n, 4)
    assert rel_err(s.to_full(), g.dense_xi_normal(n)) < 0.05


def test_half_range_integrals():  # :165-188
    t0 = 300.0
    g = VelocityGrid(32, 4.8 * math.sqrt(2.0 * KRG * t0))
    f1 = _maxwell_factor(g, 0, t0)
    fm = TtTensor.rank_one(f1, f1, f1)
    dfm = fm.to_full()
    w = g.weights
    for n in (np.array([1.0, 1, 0]), np.array([1.0, 1, 1]), np.array([0.3, 0.9, 0.3])):
        n = n / np.linalg.norm(n)
        xin = g.dense_xi_normal(n)
        exact = float(np.sum(np.where(xin > 0, xin * dfm, 0.0))) * g.dxi ** 3
        est = hadamard(g.xi_normal_positive(n, 4), fm).convolve(w, w, w)
        assert abs(est - exact) / exact < 0.02


def test_normal_tensors_deterministic():  # :190-197
    def build():
        g = VelocityGrid(24, 2.5)
        return g.abs_xi_estimate(np.array([0.6, 0.8, 0.0]), 4).to_full()
    assert np.array_equal(build(), build())


# ----------------------------------------------------------- boundary tests
def _dense_wall_density(f, mw, xin):
    out = float(np.sum(np.where(xin > 0, xin * f, 0.0)))
    inn = float(np.sum(np.where(xin > 0, 0.0, xin * mw)))
    return out / (-inn)


def test_bc_kind_strings():  # test_boundary.cpp:41-45
    for name in ("wall", "sym-x", "sym-y", "sym-z", "in", "out"):
        assert bc_kind_from_string(name) == name
    with pytest.raises(RuntimeError):
        bc_kind_from_string("periodic")


def test_wall_detailed_balance():  # :47-57
    gas = argon()
    t_wall, n0 = 500.0, 7e20
    grid = VelocityGrid(32, 4.8 * math.sqrt(2 * gas.gas_constant * t_wall))
    f = maxwell_tt(n0, t_wall, np.zeros(3), grid, gas)
    m = compute_macro(wall_ghost(f, t_wall, grid, gas, np.array([1.0, 0, 0]), 4), grid, gas)
    assert m.number_density == approx(n0, 1e-6)
    assert m.temperature == approx(t_wall, 1e-6)


def test_wall_density_dense_oracle():  # :59-85
    gas = argon()
    t_wall = 1000.0
    grid = VelocityGrid(32, 4.8 * math.sqrt(2 * gas.gas_constant * t_wall))
    f = maxwell_tt(5e20, 600.0, np.array([250.0, -80, 40]), grid, gas)
    mw = maxwell_tt(1.0, t_wall, np.zeros(3), grid, gas)
    df, dmw = f.to_full(), mw.to_full()
    n = np.array([1.0, 0, 0])
    want = _dense_wall_density(df, dmw, grid.dense_xi_normal(n))
    got = compute_macro(wall_ghost(f, t_wall, grid, gas, n, 4), grid, gas).number_density
    quad = compute_macro(mw.scaled(want), grid, gas).number_density
    assert got == approx(quad, 1e-10)
    n = np.array([1.0, 1.0, 0.0]) / math.sqrt(2.0)
    want = _dense_wall_density(df, dmw, grid.dense_xi_normal(n))
    got_nw = (compute_macro(wall_ghost(f, t_wall, grid, gas, n, 4), grid, gas).number_density
              / compute_macro(mw, grid, gas).number_density)
    assert abs(got_nw - want) / want < 0.02


def test_wall_impermeability():  # :87-106
    gas = argon()
    t_wall = 800.0
    grid = VelocityGrid(24, 4.8 * math.sqrt(2 * gas.gas_constant * t_wall))
    f = maxwell_tt(3e20, 400.0, np.array([150.0, 60, 0]), grid, gas)
    n = np.array([0.0, 1.0, 0.0])
    ghost = wall_ghost(f, t_wall, grid, gas, n, 4)
    xin = grid.dense_xi_normal(n)
    df, dg = f.to_full(), ghost.to_full()
    total = float(np.sum(np.where(xin > 0, xin * df, xin * dg)))
    incoming = float(np.sum(np.where(xin > 0, xin * df, 0.0)))
    assert abs(total) <= 1e-10 * incoming


def test_wall_rejects_zero_state():  # :108-114
    gas = argon()
    grid = VelocityGrid(16, 1000.0)
    with pytest.raises(RuntimeError):
        wall_ghost(TtTensor.constant(16, 16, 16, 0.0), 300.0, grid, gas, np.array([1.0, 0, 0]), 4)


def test_symmetry_ghost():  # :116-136
    gas = argon()
    grid = VelocityGrid(16, 1200.0)
    f = maxwell_tt(1e20, 300.0, np.array([200.0, -140, 90]), grid, gas)
    g = symmetry_ghost(f, 2)
    assert g.ranks() == f.ranks()
    mf, mg = compute_macro(f, grid, gas), compute_macro(g, grid, gas)
    assert mg.velocity[0] == approx(mf.velocity[0])
    assert mg.velocity[1] == approx(-mf.velocity[1])
    assert mg.velocity[2] == approx(mf.velocity[2])
    assert mg.number_density == approx(mf.number_density)
    assert mg.temperature == approx(mf.temperature)
    assert (symmetry_ghost(g, 2) - f).frobenius_norm() == 0.0
    even = maxwell_tt(1e20, 250.0, np.array([100.0, 0, 0]), grid, gas)
    assert (symmetry_ghost(even, 3) - even).frobenius_norm() < 1e-14 * even.frobenius_norm()


def test_freestream_ghost():  # :138-149
    gas = argon()
    grid = VelocityGrid(32, 2630.0 + 4.5 * math.sqrt(2 * gas.gas_constant * 200.0))
    bc = BoundaryCondition.freestream_in(2e23, 200.0, np.array([2630.0, 0, 0]), grid, gas)
    assert bc.freestream.ranks() == (1, 1, 1, 1)
    m = compute_macro(bc.freestream, grid, gas)
    assert m.number_density == approx(2e23, 1e-3)
    assert m.velocity[0] == approx(2630.0, 1e-3)
    assert m.temperature == approx(200.0, 1e-3)
