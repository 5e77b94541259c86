"""CPU oracle: the explicit step S1, composed only of the
reference API restated in oracle/tt.py and oracle/physics.py.

TEST INFRASTRUCTURE ONLY (see oracle/tt.py header).

The step is not in the reference code; this is the
canonical composition of PAPER.md:165-182 (Algorithm 1, signs corrected to
upwinding) with SPEC.md:391-398's rounding cadence:

    xp = ((xi_normal(n) + abs_xi_estimate(n,4)) * 0.5).rounded(1e-14)
    xm = ((xi_normal(n) - abs_xi_estimate(n,4)) * 0.5).rounded(1e-14)
    Phi[j] = (xp o f_L + xm o f_R).rounded(eps, cap)
    J      = compute_collision(f_i, eps)                 (proj/src/physics.cpp:112-119)
    R_i    = (J + sum_j Phi[j] * (-s_ij A_j / V_i)).rounded(eps, cap)
    f_i'   = (f_i + R_i * dt).rounded(eps, cap)
"""
from __future__ import annotations

import numpy as np

from .physics import (GasParameters, VelocityGrid, compute_collision, maxwell_tt,
                      symmetry_axis, symmetry_ghost, wall_ghost)
from .tt import TtTensor, hadamard


def face_factors(grid: VelocityGrid, normal):
    """Recommended (xi.n)^{+/-} = (xi_n +- E)/2."""
    xn = grid.xi_normal(normal)
    e = grid.abs_xi_estimate(normal, 4)
    xp = (xn + e).scaled(0.5).rounded(1e-14)
    xm = (xn - e).scaled(0.5).rounded(1e-14)
    return xp, xm


class OracleSolver:
    """Holds grid, gas, mesh, BCs and the per-normal face-factor cache."""

    def __init__(self, mesh, nv, bound, gas_array, bcs):
        self.mesh = mesh
        self.grid = VelocityGrid(nv, bound)
        g = np.asarray(gas_array, dtype=np.float64)
        self.gas = GasParameters(molecule_mass=g[0], gas_constant=g[1], prandtl=g[2],
                                 mu_ref=g[3], t_ref=g[4], omega=g[5])
        self.bcs = bcs
        self._factors = {}
        self._freestream = {}

    def factors(self, normal):
        key = tuple(np.round(np.asarray(normal) / 1e-12).astype(np.int64).tolist())
        if key not in self._factors:
            self._factors[key] = face_factors(self.grid, normal)
        return self._factors[key]

    def ghost(self, face: int, f_left: TtTensor) -> TtTensor:
        m = self.mesh
        bc = self.bcs[int(m.face_group[face])]
        kind = bc["kind"]
        if kind.startswith("sym"):
            return symmetry_ghost(f_left, symmetry_axis(kind))
        if kind in ("in", "out"):
            g = int(m.face_group[face])
            if g not in self._freestream:
                self._freestream[g] = maxwell_tt(bc["n"], bc["t"], np.asarray(bc["u"]),
                                                 self.grid, self.gas)
            return self._freestream[g]
        if kind == "wall":
            return wall_ghost(f_left, bc["t_wall"], self.grid, self.gas, m.face_normal[face], 4)
        raise RuntimeError("unknown boundary condition kind: " + kind)

    def face_flux(self, f, face: int, eps: float, cap: int) -> TtTensor:
        m = self.mesh
        left, right = int(m.face_left[face]), int(m.face_right[face])
        fl = f[left]
        fr = f[right] if right >= 0 else self.ghost(face, fl)
        xp, xm = self.factors(m.face_normal[face])
        return (hadamard(xp, fl) + hadamard(xm, fr)).rounded(eps, cap)

    def step(self, f, dt: float, eps: float, cap: int = 0, detail: bool = False,
             cells=None):
        """One explicit step.  ``cells`` restricts the cell loop (the fluxes
        of the faces those cells touch are still computed); returns the list
        of new tensors for those cells, the macros, and, with ``detail``,
        the intermediate Phi / J / R tensors."""
        m = self.mesh
        cells = range(m.ncell) if cells is None else cells
        need = sorted({fid for c in cells for fid, _ in m.cell_faces(c)})
        phi = {j: self.face_flux(f, j, eps, cap) for j in need}
        out, macros, js, rs = [], [], [], []
        for i in cells:
            mo = []
            jt = compute_collision(f[i], self.grid, self.gas, eps, mo)
            acc = jt
            for fid, s in m.cell_faces(i):
                acc = acc + phi[fid].scaled(-s * m.face_area[fid] / m.cell_volume[i])
            r = acc.rounded(eps, cap)
            out.append((f[i] + r.scaled(dt)).rounded(eps, cap))
            macros.append(mo[0])
            if detail:
                js.append(jt)
                rs.append(r)
        if detail:
            return out, macros, dict(phi=phi, J=js, R=rs)
        return out, macros


# ----------------------------------------------------------------- LU-SGS (N4)
def lusgs_diagonal(solver: "OracleSolver", i: int, dt: float, nu: float) -> float:
    """SPEC.md:402 / DESIGN DECISIONS "D-hat-est construction": the constant
    rank-1 bound d_i = 1/dt + nu_i + (1/2)(1/V_i) sum_j A_j xi_abs_max with
    xi_abs_max = sqrt(3) xi_box_max (>= D-hat_i pointwise)."""
    m = solver.mesh
    xi_abs_max = np.sqrt(3.0) * solver.grid.bound
    s = 0.0
    for fid, _ in m.cell_faces(i):
        s += m.face_area[fid]
    return 1.0 / dt + nu + 0.5 * s * xi_abs_max / m.cell_volume[i]


def lusgs_step(solver: "OracleSolver", f, dt: float, eps: float, cap: int = 0, detail: bool = False):
    """One LU-SGS iteration, composed of reference API
    calls only.  The reference has no solver code;
    this is the canonical composition of SPEC.md:399-407 -- forward and
    backward Gauss-Seidel sweeps over the cells in index order with the
    first-order upwind Jacobian splitting, the diagonal replaced by the
    constant rank-1 over-estimate divided out exactly by
    TtTensor::divided_by_rank_one (tt_tensor.cpp:247-261):

        R_i   = the explicit residual of S1 (J_i + sum_j -s A_j/V_i Phi_j, rounded)
        c_ik  = (A_j/V_i) (xi.n_out)^-   = (A_j/V_i) xm   if i is the face's left cell
                                         = -(A_j/V_i) xp  if i is its right cell
        B*_i  = (R_i - sum_{k<i} c_ik o df*_k).rounded(eps, cap),  df*_i = B*_i / d_i
        B_i   = (B*_i - sum_{k>i} c_ik o df_k).rounded(eps, cap),  df_i  = B_i / d_i
        f_i'  = (f_i + df_i).rounded(eps, cap)

    (k: the neighbour behind an interior face of cell i; boundary ghosts
    stay explicit).  Returns the new tensors and the macroparameters of f."""
    m = solver.mesh
    ncell = m.ncell
    ones = np.ones(solver.grid.n)
    phi = {j: solver.face_flux(f, j, eps, cap) for j in range(m.nface)}
    res, macros, diag = [], [], []
    for i in range(ncell):
        mo = []
        acc = compute_collision(f[i], solver.grid, solver.gas, eps, mo)
        for fid, s in m.cell_faces(i):
            acc = acc + phi[fid].scaled(-s * m.face_area[fid] / m.cell_volume[i])
        res.append(acc.rounded(eps, cap))
        macros.append(mo[0])
        nu = mo[0].pressure / (solver.gas.mu_ref * (mo[0].temperature / solver.gas.t_ref) ** solver.gas.omega)
        diag.append(lusgs_diagonal(solver, i, dt, nu))

    def offdiag(i, k_of, df):
        """sum over interior faces of cell i whose neighbour k satisfies k_of(k): -c_ik o df_k"""
        out = []
        for fid, s in m.cell_faces(i):
            left, right = int(m.face_left[fid]), int(m.face_right[fid])
            if right < 0:
                continue
            k = right if left == i else left
            if not k_of(k):
                continue
            xp, xm = solver.factors(m.face_normal[fid])
            w = m.face_area[fid] / m.cell_volume[i]
            # i left: c = w xm ; i right: c = -w xp.  The term entering the bracket is -c o df_k.
            fac, sc = (xm, -w) if left == i else (xp, w)
            out.append(hadamard(fac, df[k]).scaled(sc))
        return out

    dstar = [None] * ncell
    bstar = [None] * ncell
    for i in range(ncell):  # forward sweep
        acc = res[i]
        for t in offdiag(i, lambda k: k < i, dstar):
            acc = acc + t
        bstar[i] = acc.rounded(eps, cap)
        dstar[i] = bstar[i].divided_by_rank_one(diag[i] * ones, ones, ones)
    delta = [None] * ncell
    for i in range(ncell - 1, -1, -1):  # backward sweep
        acc = bstar[i]
        for t in offdiag(i, lambda k: k > i, delta):
            acc = acc + t
        delta[i] = acc.rounded(eps, cap).divided_by_rank_one(diag[i] * ones, ones, ones)
    out = [(f[i] + delta[i]).rounded(eps, cap) for i in range(ncell)]
    if detail:
        return out, macros, dict(R=res, dstar=dstar, delta=delta, diag=np.array(diag))
    return out, macros


OracleSolver.lusgs_step = lusgs_step
