"""Pins the numpy oracle (oracle/tt.py) against every known-answer test of
the reference's TT suite, proj/tests/test_tt_tensor.cpp (file:line per
test).  numpy's PCG64 replaces std::mt19937, so the random draws differ;
each assertion and tolerance is the reference's own."""
import math

import numpy as np
import pytest

from oracle.tt import TtTensor, hadamard, random_tt, rel_err


def rng(seed):
    return np.random.default_rng(seed)


def dense_convolve(a, u, v, w):
    return float(np.einsum("ijk,i,j,k->", a, u, v, w))


def test_from_full_rank_one():  # test_tt_tensor.cpp:16-27
    g = rng(7)
    u, v, w = g.standard_normal(9), g.standard_normal(8), g.standard_normal(7)
    a = np.einsum("i,j,k->ijk", u, v, w)
    t = TtTensor.from_full(a, 1e-14)
    assert t.ranks() == (1, 1, 1, 1)
    assert rel_err(t.to_full(), a) < 1e-13


def test_from_full_maxwellian_rank_one():  # :29-45
    n = 16
    x = -2.0 + 4.0 * np.arange(n) / (n - 1)
    g = np.exp(-x * x)
    a = np.einsum("i,j,k->ijk", g, g, g)
    t = TtTensor.from_full(a, 1e-12)
    assert t.ranks()[1] == 1 and t.ranks()[2] == 1
    assert rel_err(t.to_full(), a) < 1e-12


def test_from_full_oblique_abs_needs_rank_above_4():  # :47-63
    n = 32
    s = 1.0 / math.sqrt(3.0)
    x = -1.0 + 2.0 * np.arange(n) / (n - 1)
    a = np.abs(s * (x[:, None, None] + x[None, :, None] + x[None, None, :]))
    t = TtTensor.from_full(a, 1e-7)
    assert t.ranks()[1] > 4 and t.ranks()[2] > 4
    assert rel_err(t.to_full(), a) <= 1e-7


def test_from_full_rejects_nonfinite():  # :65-69
    a = np.ones((2, 2, 2))
    a[1, 0, 1] = np.nan
    with pytest.raises(ValueError):
        TtTensor.from_full(a, 1e-10)


def test_to_full_rank_one_and_constant():  # :71-85
    g = rng(3)
    u, v, w = g.standard_normal(5), g.standard_normal(6), g.standard_normal(4)
    d = TtTensor.rank_one(u, v, w).to_full()
    np.testing.assert_allclose(d, np.einsum("i,j,k->ijk", u, v, w), rtol=1e-14)
    assert np.all(TtTensor.constant(3, 4, 5, 1.0).to_full() == 1.0)


def test_round_trip_random_dense():  # :87-92
    a = rng(11).standard_normal((8, 8, 8))
    assert rel_err(TtTensor.from_full(a, 1e-14).to_full(), a) < 1e-13


def test_add():  # :94-108
    g = rng(23)
    a, b = random_tt(g, 8, 8, 8, 2, 3), random_tt(g, 8, 8, 8, 4, 5)
    c = a + b
    assert c.ranks() == (1, 6, 8, 1)
    assert rel_err(c.to_full(), a.to_full() + b.to_full()) < 1e-13
    zero = TtTensor.constant(8, 8, 8, 0.0)
    assert rel_err((a + zero).to_full(), a.to_full()) < 1e-14
    with pytest.raises(ValueError):
        a + random_tt(g, 8, 7, 8, 2, 2)


def test_hadamard():  # :110-127
    g = rng(29)
    a, b = random_tt(g, 8, 8, 8, 2, 2), random_tt(g, 8, 8, 8, 3, 3)
    c = hadamard(a, b)
    assert c.ranks() == (1, 6, 6, 1)
    assert rel_err(c.to_full(), a.to_full() * b.to_full()) < 1e-13
    ones = TtTensor.constant(8, 8, 8, 1.0)
    assert rel_err(hadamard(a, ones).to_full(), a.to_full()) < 1e-14
    with pytest.raises(ValueError):
        hadamard(a, random_tt(g, 4, 8, 8, 2, 2))


def test_rounding_exact_ranks_of_duplicates():  # :129-138
    a = random_tt(rng(31), 8, 8, 8, 2, 3)
    d = (a + a).rounded(1e-13)
    assert d.ranks() == a.ranks()
    assert rel_err(d.to_full(), a.scaled(2.0).to_full()) < 1e-12
    assert a.rounded(1e-14).ranks() == a.ranks()


def test_rounding_perturbed_maxwellian():  # :140-157
    g = rng(37)
    n = 16
    x = -3.0 + 6.0 * np.arange(n) / (n - 1)
    m = TtTensor.rank_one(np.exp(-x * x), np.exp(-x * x), np.exp(-x * x))
    p = random_tt(g, n, n, n, 6, 6)
    p = p.scaled(1e-4 * m.frobenius_norm() / p.frobenius_norm())
    s = m + p
    r = s.rounded(1e-7)
    assert rel_err(r.to_full(), s.to_full()) <= 1e-7
    assert r.ranks()[1] <= s.ranks()[1] and r.ranks()[2] <= s.ranks()[2]


def test_convolve():  # :159-181
    g = rng(41)
    n = 8
    one = np.ones(n)
    assert TtTensor.constant(n, n, n, 1.0).convolve(one, one, one) == pytest.approx(n ** 3)
    u0, v0, w0, u, v, w = (g.standard_normal(n) for _ in range(6))
    r1 = TtTensor.rank_one(u0, v0, w0)
    assert r1.convolve(u, v, w) == pytest.approx(u @ u0 * (v @ v0) * (w @ w0), rel=1e-13)
    a = random_tt(g, n, n, n, 3, 4)
    assert a.convolve(u, v, w) == pytest.approx(dense_convolve(a.to_full(), u, v, w), rel=1e-13)
    with pytest.raises(ValueError):
        a.convolve(u, v, g.standard_normal(n + 1))


def test_rank_one_places_entries():  # :183-191
    e1 = np.zeros(4)
    e1[0] = 1.0
    d = TtTensor.rank_one(e1, e1, e1).to_full()
    want = np.zeros((4, 4, 4))
    want[0, 0, 0] = 1.0
    assert np.array_equal(d, want)


def test_scaled():  # :193-201
    a = random_tt(rng(43), 6, 6, 6, 2, 2)
    assert rel_err(a.scaled(1.0).to_full(), a.to_full()) == 0.0
    assert np.linalg.norm(a.scaled(0.0).to_full()) == 0.0
    assert rel_err(a.scaled(math.pi).to_full(), a.to_full() * math.pi) < 1e-14


def test_divided_by_rank_one():  # :203-228
    g = rng(47)
    n = 8
    a = random_tt(g, n, n, n, 3, 3)
    ones = np.ones(n)
    assert rel_err(a.divided_by_rank_one(ones, ones, ones).to_full(), a.to_full()) == 0.0
    u, v, w = (np.abs(g.uniform(-1, 1, n)) + 0.5 for _ in range(3))
    r1 = TtTensor.rank_one(u, v, w)
    assert rel_err(r1.divided_by_rank_one(u, v, w).to_full(), np.ones((n, n, n))) < 1e-14
    q = a.divided_by_rank_one(u, v, w)
    assert q.ranks() == a.ranks()
    want = a.to_full() / np.einsum("i,j,k->ijk", u, v, w)
    assert rel_err(q.to_full(), want) < 1e-13
    bad = u.copy()
    bad[2] = 0.0
    with pytest.raises(ValueError):
        a.divided_by_rank_one(bad, v, w)


def test_mode_reflection():  # :230-249
    a = random_tt(rng(53), 7, 6, 5, 3, 2)
    da = a.to_full()
    for axis in (1, 2, 3):
        r = a.mode_reflected(axis)
        assert r.ranks() == a.ranks()
        assert np.array_equal(r.to_full(), np.flip(da, axis=axis - 1))
        assert rel_err(r.mode_reflected(axis).to_full(), da) == 0.0
    with pytest.raises(ValueError):
        a.mode_reflected(0)


def test_frobenius_norm():  # :251-257
    a = random_tt(rng(59), 10, 9, 8, 4, 5)
    assert a.frobenius_norm() == pytest.approx(np.linalg.norm(a.to_full()), rel=1e-12)
    assert TtTensor.constant(4, 4, 4, 0.0).frobenius_norm() == 0.0


def test_homomorphism_property():  # :259-281
    g = rng(61)
    for trial in range(25):
        n = 8
        a = random_tt(g, n, n, n, 1 + trial % 4, 1 + (trial // 2) % 4)
        b = random_tt(g, n, n, n, 1 + (trial + 1) % 4, 1 + trial % 3)
        da, db = a.to_full(), b.to_full()
        assert rel_err((a + b).to_full(), da + db) < 1e-12
        assert rel_err(hadamard(a, b).to_full(), da * db) < 1e-12
        u, v, w = (g.standard_normal(n) for _ in range(3))
        want = dense_convolve(da, u, v, w)
        tol = 1e-12 if abs(want) > 1e-12 else 1.0
        assert a.convolve(u, v, w) == pytest.approx(want, rel=tol)


def test_rounding_nearly_idempotent():  # :283-293
    g = rng(67)
    for _ in range(10):
        a = random_tt(g, 8, 8, 8, 5, 5)
        r1 = a.rounded(1e-3)
        r2 = r1.rounded(1e-3)
        assert (r1 - r2).frobenius_norm() <= 1e-3 * a.frobenius_norm()


def test_rounded_m_fold_sum_storage():  # :295-303
    a = random_tt(rng(71), 8, 8, 8, 3, 3)
    s = a
    for _ in range(1, 5):
        s = s + a
    assert s.ranks()[1] == 15
    assert s.rounded(1e-12).storage_count() == a.storage_count()


def test_rounding_zero_is_canonical_zero():  # :305-310
    z = TtTensor.constant(6, 6, 6, 0.0)
    zz = (z + z).rounded(1e-10)
    assert zz.ranks() == (1, 1, 1, 1)
    assert np.linalg.norm(zz.to_full()) == 0.0
