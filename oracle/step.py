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
