"""CPU oracle: order-3 Tensor-Train algebra (numpy restatement).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library and
its host wrapper in ``paper_1912_04582_b200``) may import this module; only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg
use it, and only as the checker.

Restates ``proj/src/tt_tensor.cpp`` of the reference (file:line cited per
function).  Dense linear algebra: the reference uses Eigen ``HouseholderQR``
and ``BDCSVD`` (Eigen version unpinned, absent from the reference tree);
here numpy's LAPACK ``geqrf``/``gesdd`` stand in.  Both are backward stable;
QR/SVD signs are arbitrary so cores are compared through reconstructions,
never entry by entry.

Storage mirrors the reference's Eigen col-major cores:
  first  : (n1, r1)        A(i,j,k) = first[i,:] @ middle[j] @ last[:,k]
  middle : (n2, r1, r2)
  last   : (r2, n3)
"""
from __future__ import annotations

import numpy as np


def truncation_rank(sigma: np.ndarray, budget2: float, cap: int) -> int:
    """proj/src/tt_tensor.cpp:18-29 -- smallest leading rank whose dropped
    tail of squared singular values stays within budget2 (ties drop)."""
    r = int(sigma.shape[0])
    tail = 0.0
    while r > 1:
        s2 = float(sigma[r - 1]) * float(sigma[r - 1])
        if tail + s2 > budget2:
            break
        tail += s2
        r -= 1
    if cap > 0 and r > cap:
        r = cap
    return r


def thin_svd(m: np.ndarray):
    """proj/src/tt_tensor.cpp:37-40 (BDCSVD thin U, V)."""
    u, s, vt = np.linalg.svd(m, full_matrices=False)
    return u, s, vt.T


class TtTensor:
    """proj/include/ttdvm/tt_tensor.hpp:19-77; invariants tt_tensor.cpp:44-54."""

    __slots__ = ("first", "middle", "last")

    def __init__(self, first, middle, last):
        first = np.asarray(first, dtype=np.float64)
        middle = np.asarray(middle, dtype=np.float64)
        last = np.asarray(last, dtype=np.float64)
        if middle.ndim != 3 or middle.shape[0] == 0:
            raise ValueError("TtTensor: empty middle core")
        if first.ndim != 2 or last.ndim != 2:
            raise ValueError("TtTensor: core rank mismatch")
        if middle.shape[1] != first.shape[1] or middle.shape[2] != last.shape[0]:
            raise ValueError("TtTensor: core rank mismatch")
        self.first = first
        self.middle = middle
        self.last = last

    # -- construction ------------------------------------------------------
    @staticmethod
    def rank_one(u, v, w) -> "TtTensor":
        """tt_tensor.cpp:56-66."""
        u = np.asarray(u, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        w = np.asarray(w, dtype=np.float64)
        if u.size == 0 or v.size == 0 or w.size == 0:
            raise ValueError("rank_one: empty factor")
        return TtTensor(u.reshape(-1, 1).copy(), v.reshape(-1, 1, 1).copy(),
                        w.reshape(1, -1).copy())

    @staticmethod
    def constant(n1: int, n2: int, n3: int, value: float) -> "TtTensor":
        """tt_tensor.cpp:68-71."""
        return TtTensor.rank_one(np.full(n1, float(value)), np.ones(n2), np.ones(n3))

    @staticmethod
    def from_full(a: np.ndarray, eps: float, max_rank: int = 0) -> "TtTensor":
        """tt_tensor.cpp:104-137 (TT-SVD, budget eps^2||A||^2/2 per cut)."""
        if eps <= 0.0:
            raise ValueError("from_full: eps must be > 0")
        a = np.asarray(a, dtype=np.float64)
        if not np.all(np.isfinite(a)):
            raise ValueError("from_full: input contains non-finite values")
        n1, n2, n3 = a.shape
        norm = float(np.sqrt(np.sum(a * a)))
        budget2 = eps * eps * norm * norm / 2.0
        a1 = a.reshape(n1, n2 * n3)  # row-major (i, j*n3+k)
        u, s, v = thin_svd(a1)
        r1 = truncation_rank(s, budget2, max_rank)
        first = u[:, :r1].copy()
        m = s[:r1, None] * v[:, :r1].T  # r1 x (n2*n3)
        # b(j*r1 + a, k) = m(a, j*n3 + k)
        b = m.reshape(r1, n2, n3).transpose(1, 0, 2).reshape(n2 * r1, n3)
        u2, s2, v2 = thin_svd(b)
        r2 = truncation_rank(s2, budget2, max_rank)
        middle = u2[:, :r2].reshape(n2, r1, r2).copy()
        last = s2[:r2, None] * v2[:, :r2].T
        return TtTensor(first, middle, last)

    # -- queries -------------------------------------------------------------
    def mode_sizes(self):
        return (self.first.shape[0], self.middle.shape[0], self.last.shape[1])

    def ranks(self):
        return (1, self.first.shape[1], self.last.shape[0], 1)

    def storage_count(self) -> int:
        return int(self.first.size + self.middle.size + self.last.size)

    def value(self, i, j, k) -> float:
        return float(self.first[i] @ self.middle[j] @ self.last[:, k])

    def to_full(self) -> np.ndarray:
        """tt_tensor.cpp:93-102 (row-major, k fastest)."""
        return np.einsum("ia,jab,bk->ijk", self.first, self.middle, self.last,
                         optimize=True)

    # -- algebra ---------------------------------------------------------------
    def rounded(self, eps: float, max_rank: int = 0) -> "TtTensor":
        """tt_tensor.cpp:139-193: right-to-left QR orthogonalisation, then
        left-to-right truncated SVD with budget eps^2 ||A||^2 / 2 per cut."""
        if eps <= 0.0:
            raise ValueError("rounded: eps must be > 0")
        n1, n2, n3 = self.mode_sizes()
        r1 = self.first.shape[1]
        # :147-151 QR of last^T (n3 x r2)
        q3m, r3 = np.linalg.qr(self.last.T, mode="reduced")
        q3 = min(n3, self.last.shape[0])
        last_orth = q3m[:, :q3].T  # q3 x n3
        rfac3 = r3[:q3, :]
        # :153 mid_j = middle_j R3^T
        mid = np.einsum("jab,cb->jac", self.middle, rfac3)  # n2 x r1 x q3
        # :155-163 wide = [mid_0 ... mid_{n2-1}] (r1 x n2*q3); QR(wide^T)
        wide = mid.transpose(1, 0, 2).reshape(r1, n2 * q3)
        q2m, r2f = np.linalg.qr(wide.T, mode="reduced")
        q2 = min(n2 * q3, r1)
        mid_orth = q2m[:, :q2].T  # q2 x n2*q3
        rfac2 = r2f[:q2, :]
        first_carry = self.first @ rfac2.T  # n1 x q2
        # :167-169
        norm = float(np.linalg.norm(first_carry))
        if norm == 0.0:
            return TtTensor.constant(n1, n2, n3, 0.0)
        budget2 = eps * eps * norm * norm / 2.0
        # :172-175
        u1, s1, v1 = thin_svd(first_carry)
        t1 = truncation_rank(s1, budget2, max_rank)
        new_first = u1[:, :t1].copy()
        carry = s1[:t1, None] * v1[:, :t1].T  # t1 x q2
        # :178-181 stacked rows (j*t1 + a)
        mo = mid_orth.reshape(q2, n2, q3).transpose(1, 0, 2)  # n2 x q2 x q3
        stacked = np.einsum("ap,jpc->jac", carry, mo).reshape(n2 * t1, q3)
        # :183-189
        u2, s2, v2 = thin_svd(stacked)
        t2 = truncation_rank(s2, budget2, max_rank)
        new_middle = u2[:, :t2].reshape(n2, t1, t2).copy()
        new_last = (s2[:t2, None] * v2[:, :t2].T) @ last_orth
        return TtTensor(new_first, new_middle, new_last)

    def rounded_sigmas(self, eps: float, max_rank: int = 0):
        """Diagnostic twin of rounded(): returns (sigma1, sigma2, budget2) so
        parity tests can measure each rank decision's margin."""
        n1, n2, n3 = self.mode_sizes()
        r1 = self.first.shape[1]
        q3m, r3 = np.linalg.qr(self.last.T, mode="reduced")
        q3 = min(n3, self.last.shape[0])
        mid = np.einsum("jab,cb->jac", self.middle, r3[:q3, :])
        wide = mid.transpose(1, 0, 2).reshape(r1, n2 * q3)
        q2m, r2f = np.linalg.qr(wide.T, mode="reduced")
        q2 = min(n2 * q3, r1)
        first_carry = self.first @ r2f[:q2, :].T
        norm = float(np.linalg.norm(first_carry))
        if norm == 0.0:
            return np.zeros(1), np.zeros(1), 0.0
        budget2 = eps * eps * norm * norm / 2.0
        u1, s1, v1 = thin_svd(first_carry)
        t1 = truncation_rank(s1, budget2, max_rank)
        carry = s1[:t1, None] * v1[:, :t1].T
        mo = q2m[:, :q2].T.reshape(q2, n2, q3).transpose(1, 0, 2)
        stacked = np.einsum("ap,jpc->jac", carry, mo).reshape(n2 * t1, q3)
        s2 = np.linalg.svd(stacked, compute_uv=False)
        return s1, s2, budget2

    def convolve(self, u, v, w) -> float:
        """tt_tensor.cpp:195-204."""
        n1, n2, n3 = self.mode_sizes()
        u = np.asarray(u, dtype=np.float64)
        v = np.asarray(v, dtype=np.float64)
        w = np.asarray(w, dtype=np.float64)
        if u.size != n1 or v.size != n2 or w.size != n3:
            raise ValueError("convolve: weight length mismatch")
        acc1 = u @ self.first  # r1
        acc2 = np.zeros(self.last.shape[0])
        for j in range(n2):
            acc2 += v[j] * (acc1 @ self.middle[j])
        return float(acc2 @ (self.last @ w))

    def scaled(self, s: float) -> "TtTensor":
        """tt_tensor.cpp:206-210 (scale lands on the first core)."""
        return TtTensor(self.first * s, self.middle.copy(), self.last.copy())

    def hadamard(self, b: "TtTensor") -> "TtTensor":
        """tt_tensor.cpp:212-245 (slice-wise Kronecker, index p*rb + q)."""
        if self.mode_sizes() != b.mode_sizes():
            raise ValueError("hadamard: mode size mismatch")
        n1, n2, n3 = self.mode_sizes()
        ra1, rb1 = self.first.shape[1], b.first.shape[1]
        ra2, rb2 = self.last.shape[0], b.last.shape[0]
        first = (self.first[:, :, None] * b.first[:, None, :]).reshape(n1, ra1 * rb1)
        middle = np.einsum("jps,jqt->jpqst", self.middle, b.middle).reshape(
            n2, ra1 * rb1, ra2 * rb2)
        last = (self.last[:, None, :] * b.last[None, :, :]).reshape(ra2 * rb2, n3)
        return TtTensor(first, middle, last)

    def divided_by_rank_one(self, u1, u2, u3) -> "TtTensor":
        """tt_tensor.cpp:247-261."""
        n1, n2, n3 = self.mode_sizes()
        u1, u2, u3 = (np.asarray(x, dtype=np.float64) for x in (u1, u2, u3))
        if u1.size != n1 or u2.size != n2 or u3.size != n3:
            raise ValueError("divided_by_rank_one: length mismatch")
        if (u1 <= 0).any() or (u2 <= 0).any() or (u3 <= 0).any():
            raise ValueError("divided_by_rank_one: divisor entries must be strictly positive")
        return TtTensor(self.first / u1[:, None], self.middle / u2[:, None, None],
                        self.last / u3[None, :])

    def mode_reflected(self, axis: int) -> "TtTensor":
        """tt_tensor.cpp:263-280 (exact index reversal of one core)."""
        if axis == 1:
            return TtTensor(self.first[::-1].copy(), self.middle.copy(), self.last.copy())
        if axis == 2:
            return TtTensor(self.first.copy(), self.middle[::-1].copy(), self.last.copy())
        if axis == 3:
            return TtTensor(self.first.copy(), self.middle.copy(), self.last[:, ::-1].copy())
        raise ValueError("mode_reflected: axis must be 1, 2 or 3")

    def frobenius_norm(self) -> float:
        """tt_tensor.cpp:282-288 (Gram chain)."""
        # einsum (no BLAS/FMA contraction) keeps exact cancellations exact,
        # as the reference's symmetric A - A checks expect (test_boundary.cpp:133)
        w1 = np.einsum("ia,ib->ab", self.first, self.first)
        w2 = np.zeros((self.last.shape[0], self.last.shape[0]))
        for g in self.middle:
            w2 += np.einsum("ap,aq->pq", g, np.einsum("ab,bq->aq", w1, g))
        s = float(np.einsum("pk,pk->", self.last, np.einsum("pq,qk->pk", w2, self.last)))
        return float(np.sqrt(max(0.0, s)))

    def __add__(self, b: "TtTensor") -> "TtTensor":
        """tt_tensor.cpp:290-312 (block concat, block-diagonal middle)."""
        if self.mode_sizes() != b.mode_sizes():
            raise ValueError("tt add: mode size mismatch")
        n1, n2, n3 = self.mode_sizes()
        ra1, ra2 = self.first.shape[1], self.last.shape[0]
        rb1, rb2 = b.first.shape[1], b.last.shape[0]
        first = np.concatenate([self.first, b.first], axis=1)
        middle = np.zeros((n2, ra1 + rb1, ra2 + rb2))
        middle[:, :ra1, :ra2] = self.middle
        middle[:, ra1:, ra2:] = b.middle
        last = np.concatenate([self.last, b.last], axis=0)
        return TtTensor(first, middle, last)

    def __sub__(self, b: "TtTensor") -> "TtTensor":
        """tt_tensor.cpp:314-316."""
        return self + b.scaled(-1.0)


def hadamard(a: TtTensor, b: TtTensor) -> TtTensor:
    return a.hadamard(b)


def random_tt(rng: np.random.Generator, n1, n2, n3, r1, r2) -> TtTensor:
    """Fixture like proj/tests/support.hpp:20-35 (N(0,1) cores).  numpy's
    generator replaces std::mt19937, so draws differ from the C++ tests."""
    return TtTensor(rng.standard_normal((n1, r1)), rng.standard_normal((n2, r1, r2)),
                    rng.standard_normal((r2, n3)))


def rel_err(got: np.ndarray, want: np.ndarray) -> float:
    """proj/tests/support.hpp:46-49."""
    w = float(np.linalg.norm(want))
    return float(np.linalg.norm(got - want)) / (w if w > 0 else 1.0)
