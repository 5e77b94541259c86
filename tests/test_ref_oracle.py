"""The oracle pinned to the reference itself.

oracle/_ref holds the UNMODIFIED reference C++ (proj/src/*.cpp) compiled by
oracle/build_ref.py against the repo's Eigen/doctest subsets:
* its own 50 doctest TEST_CASEs pass (the gate);
* the S1 step composed of reference API calls (oracle/ref_step.cpp) agrees
  with the numpy restatement (oracle/step.py) in lock-step on configs 1, 2
  and a small config-4 obstacle mesh -- so the numpy oracle, the golden
  fixtures and the GPU parity tests all stand on the reference's own code.
"""
import os
import subprocess

import numpy as np
import pytest

from oracle import ref
from oracle.step import OracleSolver
from oracle.tt import TtTensor, rel_err
from paper_1912_04582_b200.problems import config
from paper_1912_04582_b200.tt_batch import TtBatch

pytestmark = pytest.mark.skipif(not ref.available(), reason="oracle/_ref not built")


def test_reference_unit_tests_pass():
    """proj/tests/*.cpp: 50 TEST_CASEs, every assertion green."""
    from oracle import build_ref
    if os.path.isdir(build_ref.PROJ):
        build_ref.build()
    if not os.path.exists(build_ref.UNIT):
        pytest.skip("unit_tests binary not built")
    r = subprocess.run([build_ref.UNIT], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-4000:]
    assert "test cases: 50 | 50 passed | 0 failed" in r.stdout, r.stdout


@pytest.mark.parametrize("cfg,scale,steps", [(1, 1.0, 3), (2, 3 / 32, 2), (4, 0.06, 1)])
def test_numpy_oracle_matches_compiled_reference_step(cfg, scale, steps):
    """Lock-step S1: every step both start from the compiled reference's
    state; reconstructions agree to 1e-12, ranks identical, moments 1e-10."""
    p = config(cfg, scale)
    r = ref.RefSolver.for_problem(p)
    o = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = [TtTensor(*p.f0.get(i)) for i in range(p.mesh.ncell)]
    for _ in range(steps):
        r.step(p.dt, p.eps, p.cap)
        got = r.state()
        want, macros = o.step(f, p.dt, p.eps, p.cap)
        for i in range(p.mesh.ncell):
            assert tuple(got.ranks[i]) == want[i].ranks()[1:3], i
            assert rel_err(got.full(i), want[i].to_full()) < 1e-12, i
        m = r.macros(p.mesh.ncell)
        w = np.array([x.as_array() for x in macros])
        scale_ = np.maximum(np.abs(w), 1.0)  # u, S are O(1) or zero
        assert np.max(np.abs(m[:, :10] - w) / scale_) < 1e-10
        f = [TtTensor(*got.get(i)) for i in range(p.mesh.ncell)]


def test_round_sums_match_numpy_oracle():
    from oracle.tt import random_tt
    rng = np.random.default_rng(3)
    groups = [[(random_tt(rng, 10, 10, 10, int(rng.integers(1, 6)), int(rng.integers(1, 6))),
                float(rng.standard_normal())) for _ in range(int(rng.integers(1, 5)))]
              for _ in range(12)]
    flat = [t for g in groups for t, _ in g]
    sc = np.array([s for g in groups for _, s in g])
    go = np.cumsum([0] + [len(g) for g in groups])
    r = ref.RefSolver(10, 1.0, [1, 0.5, 2 / 3, 1, 1, 0.5])
    for eps, cap in ((1e-6, 0), (1e-2, 0), (1e-8, 3)):
        got = r.round_sums(TtBatch.from_list(flat), eps, cap, group_off=go, scale=sc)
        for o, g in enumerate(groups):
            s = g[0][0].scaled(g[0][1])
            for t, x in g[1:]:
                s = s + t.scaled(x)
            w = s.rounded(eps, cap)
            assert tuple(got.ranks[o]) == w.ranks()[1:3]
            assert rel_err(got.full(o), w.to_full()) < 1e-12


def test_face_factors_match_numpy_oracle():
    """abs_xi_estimate / xi_normal_positive of oblique normals
    (velocity_grid.cpp:61-146): same h choice, same tensors."""
    from oracle.physics import VelocityGrid
    rng = np.random.default_rng(9)
    nrm = rng.standard_normal((4, 3))
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    r = ref.RefSolver(16, 5.0, [1, 0.5, 2 / 3, 1, 1, 0.5])
    g = VelocityGrid(16, 5.0)
    for mode, fn in ((0, g.abs_xi_estimate), (1, g.xi_normal_positive)):
        got = r.face_factors(nrm, 4, mode)
        for i in range(len(nrm)):
            w = fn(nrm[i], 4)
            assert tuple(got.ranks[i]) == w.ranks()[1:3]
            assert rel_err(got.full(i), w.to_full()) < 1e-9


@pytest.mark.parametrize("kind", ["shock-tube", "obstacle"])
def test_numpy_lusgs_matches_compiled_reference(kind):
    """LU-SGS (N4): the numpy composition and the one written from the
    compiled reference's API agree in lock-step (ranks identical)."""
    from paper_1912_04582_b200.problems import obstacle_flow
    p = config(1) if kind == "shock-tube" else obstacle_flow((5, 4, 4), hole=2, nv=12)
    r = ref.RefSolver.for_problem(p)
    o = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = [TtTensor(*p.f0.get(i)) for i in range(p.mesh.ncell)]
    for _ in range(2):
        r.lusgs_step(p.dt, p.eps, p.cap)
        got = r.state()
        want, _ = o.lusgs_step(f, p.dt, p.eps, p.cap)
        for i in range(p.mesh.ncell):
            assert tuple(got.ranks[i]) == want[i].ranks()[1:3], i
            assert rel_err(got.full(i), want[i].to_full()) < 1e-11, i
        f = [TtTensor(*got.get(i)) for i in range(p.mesh.ncell)]
