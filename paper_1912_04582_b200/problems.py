"""Synthetic problem set-ups for BASELINE.json's configs (host side).

All inputs are synthetic and seeded (no dataset is involved).  Units are
non-dimensional: molecule mass m = 1 and gas constant R = 1/2, so the thermal
speed sqrt(2RT) is 1 at T = 1.  The viscosity law is the reference's power
law mu = mu_ref (T/T_ref)^omega (proj/src/physics.cpp:11-15) with T_ref = 1;
mu_ref follows from the Knudsen number through the hard-sphere mean free
path lambda = (mu/p) sqrt(pi R T / 2) (SURVEY.md §7 step 2 asks for this
mapping to be fixed and recorded):

    mu_ref = Kn * L_ref * p0 / sqrt(pi R T0 / 2),  p0 = n0 m R T0.

The time step follows SPEC.md's CFL rule with the sum of per-axis maximum
speeds (first-order upwind stability in 3-D): dt = cfl * h_min / (3 B).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .mesh import Mesh, obstacle_mesh, structured_box
from .tt_batch import TtBatch

GAS_M = 1.0
GAS_R = 0.5
PRANDTL = 2.0 / 3.0


def gas_params(kn: float, l_ref: float, omega: float = 0.5, n0: float = 1.0,
               t0: float = 1.0) -> np.ndarray:
    """[molecule_mass, gas_constant, prandtl, mu_ref, t_ref, omega]
    (proj/include/ttdvm/physics.hpp:11-18 field order)."""
    p0 = n0 * GAS_M * GAS_R * t0
    mu_ref = kn * l_ref * p0 / math.sqrt(math.pi * GAS_R * t0 / 2.0)
    return np.array([GAS_M, GAS_R, PRANDTL, mu_ref, 1.0, omega], dtype=np.float64)


def maxwell_factors(nodes: np.ndarray, n: np.ndarray, t: np.ndarray, u: np.ndarray):
    """Per-cell rank-1 Maxwellian factors, same arithmetic as maxwell_tt
    (proj/src/physics.cpp:69-87): returns three [ncell, nv] arrays, density
    folded into the first."""
    two_rt = 2.0 * GAS_R * t
    norm1d = 1.0 / np.sqrt(math.pi * two_rt)
    f = []
    for a in range(3):
        v = nodes[None, :] - u[:, a:a + 1]
        f.append(norm1d[:, None] * np.exp(-v * v / two_rt[:, None]))
    f[0] = f[0] * n[:, None]
    return f


@dataclass
class Problem:
    name: str
    mesh: Mesh
    nv: int
    bound: float
    gas: np.ndarray
    bcs: list                     # per group: dict(kind=..., ...)
    f0: TtBatch
    dt: float
    eps: float
    cap: int
    steps: int
    meta: dict = field(default_factory=dict)

    @property
    def nodes(self) -> np.ndarray:
        dxi = 2.0 * self.bound / (self.nv - 1)
        return np.array([-self.bound + i * dxi for i in range(self.nv)])


def cfl_dt(mesh: Mesh, bound: float, cfl: float = 0.9) -> float:
    return cfl * mesh.min_cell_size() / (3.0 * bound)


def shock_tube(nx: int = 64, nv: int = 16, bound: float = 5.0, kn: float = 0.1,
               eps: float = 1e-6, steps: int = 100) -> Problem:
    """Config 1: 64x1x1 unit hexes, periodic y/z, specular (sym-x) x-walls,
    (n, T) = (1, 1) | (0.125, 0.8) split at x = nx/2, u = 0."""
    mesh = structured_box(nx, 1, 1, periodic=(False, True, True))
    dxi = 2.0 * bound / (nv - 1)
    nodes = np.array([-bound + i * dxi for i in range(nv)])
    x = mesh.cell_ijk[:, 0]
    n = np.where(x < nx // 2, 1.0, 0.125)
    t = np.where(x < nx // 2, 1.0, 0.8)
    u = np.zeros((mesh.ncell, 3))
    f1, f2, f3 = maxwell_factors(nodes, n, t, u)
    f0 = TtBatch.from_rank_one(f1, f2, f3)
    bcs = [dict(kind="sym-x"), dict(kind="sym-x")]
    return Problem("config1-shock-tube", mesh, nv, bound, gas_params(kn, float(nx)), bcs, f0,
                   cfl_dt(mesh, bound), eps, 0, steps)


def smooth_fields(mesh: Mesh, seed: int):
    """Seeded smooth per-cell (n, u, T) of configs 2 and 5: density
    1 + 0.2 * mean of three phased sines, u_a in +-0.3, T in [0.7, 1.3]."""
    rng = np.random.default_rng(seed)
    ph = rng.uniform(0.0, 2.0 * math.pi, size=(3, 3))
    dims = np.array(mesh.shape, dtype=np.float64)
    x = 2.0 * math.pi * (mesh.cell_ijk + 0.5) / dims[None, :]
    n = 1.0 + 0.2 * np.mean(np.sin(x + ph[0][None, :]), axis=1)
    u = 0.3 * np.sin(np.roll(x, 1, axis=1) + ph[1][None, :])
    t = 1.0 + 0.3 * np.sin(x[:, 0] + x[:, 1] - x[:, 2] + ph[2][0])
    return n, u, t


def periodic_box(shape=(32, 32, 32), nv: int = 24, bound: float = 6.0, kn: float = 0.1,
                 eps: float = 1e-6, steps: int = 50, cap: int = 0, seed: int = 2,
                 pert: float = 1e-3, pert_rank: int = 2, name="config2-periodic-box") -> Problem:
    """Config 2 (32^3 cells, 24^3 velocity mesh on [-6,6]^3) and, with other
    arguments, config 5.  Initial f = Maxwellian + pert * ||f_M|| * P/||P||
    with P one seeded N(0,1) rank-(pert_rank) TT for all cells (the sum is kept
    unrounded, ranks (1 + pert_rank) -- the first step rounds it)."""
    mesh = structured_box(*shape, periodic=(True, True, True))
    dxi = 2.0 * bound / (nv - 1)
    nodes = np.array([-bound + i * dxi for i in range(nv)])
    n, u, t = smooth_fields(mesh, seed)
    f1, f2, f3 = maxwell_factors(nodes, n, t, u)
    fm = TtBatch.from_rank_one(f1, f2, f3)
    if pert > 0.0:
        # ONE seeded N(0,1) rank-(pert_rank) TT shared by every cell, scaled
        # per cell to pert * ||f_M,i||: "a seeded 1e-3 random rank-2 TT
        # perturbation" (BASELINE.json config 2).  DESIGN.md records this
        # reading; independent per-cell noise would saturate every rank.
        rng = np.random.default_rng(seed + 1000)
        p1 = TtBatch.random_uniform_rank(rng, 1, nv, pert_rank, pert_rank)
        pf, pm, pl = p1.uniform_cores()
        c = mesh.ncell
        p = TtBatch.uniform(c, nv, nv, nv, pert_rank, pert_rank, np.repeat(pf, c, 0),
                            np.repeat(pm, c, 0), np.repeat(pl, c, 0))
        scale = pert * fm.norms() / p1.norms()[0]
        f0 = TtBatch.add(fm, p.scaled(scale))
    else:
        f0 = fm
    l_ref = float(shape[0])
    return Problem(name, mesh, nv, bound, gas_params(kn, l_ref), [], f0,
                   cfl_dt(mesh, bound), eps, cap, steps)


def obstacle_flow(shape=(100, 80, 64), hole: int = 8, nv: int = 44, bound: float = 7.0,
                  kn: float = 0.05, eps: float = 1e-5, mach: float = 3.0, steps: int = 20,
                  seed: int = 4, jitter: float = 0.1, t_wall: float = 1.0,
                  name="config4-obstacle-mach3") -> Problem:
    """Config 4: jittered, shuffled hex mesh around a hole^3 rigid box
    (mesh.obstacle_mesh), free-stream Maxwellian at Mach ``mach`` along +x
    (u = mach * sqrt(5/3 R T), T = 1, n = 1) on the outer faces, diffuse
    walls at T_w on the obstacle, impulsive start (the free stream in every
    cell).  Kn is referred to the obstacle edge (L_ref = hole * h)."""
    mesh = obstacle_mesh(shape, hole=hole, jitter=jitter, seed=seed)
    dxi = 2.0 * bound / (nv - 1)
    nodes = np.array([-bound + i * dxi for i in range(nv)])
    u0 = mach * math.sqrt(5.0 / 3.0 * GAS_R * 1.0)
    u = np.zeros((mesh.ncell, 3))
    u[:, 0] = u0
    f1, f2, f3 = maxwell_factors(nodes, np.ones(mesh.ncell), np.ones(mesh.ncell), u)
    f0 = TtBatch.from_rank_one(f1, f2, f3)
    free = dict(n=1.0, t=1.0, u=(u0, 0.0, 0.0))
    bcs = [dict(kind="in", **free), dict(kind="out", **free), dict(kind="wall", t_wall=t_wall)]
    return Problem(name, mesh, nv, bound, gas_params(kn, float(hole)), bcs, f0,
                   cfl_dt(mesh, bound), eps, 0, steps, meta=dict(mach=mach, jitter=jitter,
                                                                 hole=hole, seed=seed))


def rounding_summands(rng: np.random.Generator, count: int, n: int = 32, terms: int = 6,
                      rank: int = 12, decay: float = 0.5):
    """Config 3 inputs: ``count`` independent sums of ``terms`` seeded TT
    tensors of ranks (1, rank, rank, 1) on n^3.  Core entries are N(0,1);
    the "geometric singular-value decay of 0.5 per index" is put on the
    rank indices of the outer cores: column a of the first core is scaled by
    decay^a and row b of the last core by decay^b (the middle core stays
    N(0,1)).  DESIGN.md records this reading.  Returns (first, middle, last)
    arrays of shapes (count*terms, n, rank), (count*terms, n, rank, rank),
    (count*terms, rank, n) in the reference's index order (first[t, i, a],
    middle[t, j, a, b], last[t, b, k])."""
    m = count * terms
    w = decay ** np.arange(rank)
    first = rng.standard_normal((m, n, rank)) * w[None, None, :]
    middle = rng.standard_normal((m, n, rank, rank))
    last = rng.standard_normal((m, rank, n)) * w[None, :, None]
    return first, middle, last


def config(idx: int, scale: float = 1.0) -> Problem:
    """BASELINE.json configs by 1-based index; ``scale`` < 1 shrinks the
    spatial mesh for parity tests (velocity mesh unchanged)."""
    if idx == 1:
        return shock_tube()
    if idx == 2:
        s = max(2, int(round(32 * scale)))
        return periodic_box((s, s, s))
    if idx == 4:
        if scale >= 1.0:
            return obstacle_flow()
        sx, sy, sz = (max(4, int(round(v * scale))) for v in (100, 80, 64))
        hole = max(2, int(round(8 * scale)))
        return obstacle_flow((sx, sy, sz), hole=hole)
    if idx == 5:
        sx, sy, sz = (max(2, int(round(v * scale))) for v in (128, 128, 64))
        return periodic_box((sx, sy, sz), nv=64, bound=8.0, kn=0.1, eps=1e-5, steps=10,
                            cap=20, seed=5, name="config5-weak-scaling-box")
    raise ValueError(f"config {idx} not available")
