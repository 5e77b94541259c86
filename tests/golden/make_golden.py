"""Generate the committed golden fixtures under tests/golden/ (test
infrastructure only).

Every vector here is an output of the REFERENCE ITSELF: the unmodified
proj/src/*.cpp compiled by oracle/build_ref.py (oracle/_ref/libttdvm_ref.so,
gated on the reference's own 50 doctest TEST_CASEs), driven through
oracle/ref.py -- TtTensor::rounded for the rounding cases, and the S1 step
composed of reference API calls (oracle/ref_step.cpp) for the step cases.
The fixtures freeze those outputs on seeded inputs so that (a) the CPU suite
checks the numpy restatement (oracle/) and a rebuilt reference against them,
and (b) the GPU suite checks the CUDA path against stored reference outputs
on a box where /root/reference does not exist.

    python tests/golden/make_golden.py        # rewrites the .npz files
                                              # (needs /root/reference or a built oracle/_ref)
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

from oracle.tt import random_tt  # noqa: E402
from paper_1912_04582_b200.problems import config, obstacle_flow  # noqa: E402
from paper_1912_04582_b200.tt_batch import TtBatch  # noqa: E402

SHOCK_STEPS = 5
C4_SHAPE, C4_HOLE, C4_STEPS = (6, 5, 4), 2, 3


def _ref():
    from oracle import ref
    if not ref.available():
        raise SystemExit("oracle/_ref is not built (python oracle/build_ref.py)")
    return ref


def shock_tube_fixture(stepper=None):
    """Config 1 (64x1x1 shock tube, 16^3 velocity mesh, eps 1e-6), run free
    for SHOCK_STEPS steps: per-cell macroparameters of t^0 .. t^(SHOCK_STEPS-1)
    and the ranks and dense tensors of a few cells after SHOCK_STEPS steps.
    ``stepper(p)`` yields (state TtBatch, macros) per step; default: the
    compiled reference."""
    p = config(1)
    macros, st = [], None
    for st, m in (stepper or ref_stepper)(p, SHOCK_STEPS):
        macros.append(np.asarray(m)[:, :10])
    cells = np.array([0, 30, 31, 32, 33, 63])
    return dict(steps=np.int64(SHOCK_STEPS), dt=np.float64(p.dt), eps=np.float64(p.eps),
                macros=np.stack(macros), ranks=st.ranks.copy(),
                cells=cells, full=np.stack([st.full(int(i)) for i in cells]))


def ref_stepper(p, steps):
    r = _ref().RefSolver.for_problem(p)
    for _ in range(steps):
        r.step(p.dt, p.eps, p.cap)
        yield r.state(), r.macros(p.mesh.ncell)
    r.close()


def numpy_stepper(p, steps):
    from oracle.step import OracleSolver
    from oracle.tt import TtTensor
    s = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = [TtTensor(*p.f0.get(i)) for i in range(p.mesh.ncell)]
    for _ in range(steps):
        f, m = s.step(f, p.dt, p.eps, p.cap)
        yield TtBatch.from_list(f), np.stack([x.as_array() for x in m])


ROUND_CASES = ((1e-6, 0), (1e-4, 5))  # (eps, rank cap)


def rounding_inputs():
    """Seeded sums of random TTs (24^3, 2..5 summands of ranks 1..8,
    scales 1 / -0.5 / 1e-3), one set per case of ROUND_CASES."""
    rng = np.random.default_rng(11)
    n = 24
    cases = []
    for eps, cap in ROUND_CASES:
        flat, groups, scales = [], [0], []
        for _ in range(6):
            k = int(rng.integers(2, 6))
            for _ in range(k):
                flat.append(random_tt(rng, n, n, n, int(rng.integers(1, 9)), int(rng.integers(1, 9))))
                scales.append(float(rng.choice([1.0, -0.5, 1e-3])))
            groups.append(groups[-1] + k)
        cases.append((eps, cap, TtBatch.from_list(flat), np.array(groups), np.array(scales)))
    return n, cases


def rounding_fixture(rounder=None):
    """The packed summands (TtBatch layout) and the reference's output ranks
    and dense reconstructions.  ``rounder(batch, eps, cap, group_off, scale)``
    returns a TtBatch; default: the compiled reference's TtTensor::rounded."""
    n, cases = rounding_inputs()
    if rounder is None:
        r = _ref().RefSolver(n, 1.0, [1, 0.5, 2 / 3, 1, 1, 0.5])
        rounder = lambda b, eps, cap, go, sc: r.round_sums(b, eps, cap, group_off=go, scale=sc)  # noqa: E731
    out = {"n": np.int64(n)}
    for c, (eps, cap, b, groups, scales) in enumerate(cases):
        res = rounder(b, eps, cap, groups, scales)
        out.update({f"c{c}_eps": np.float64(eps), f"c{c}_cap": np.int64(cap),
                    f"c{c}_cores": b.cores, f"c{c}_ranks": b.ranks, f"c{c}_offsets": b.offsets,
                    f"c{c}_group_off": groups, f"c{c}_scales": scales,
                    f"c{c}_out_ranks": res.ranks.copy(),
                    f"c{c}_out_full": np.stack([res.full(o) for o in range(res.count)])})
    return out


def numpy_rounder(b, eps, cap, go, sc):
    from oracle.tt import TtTensor
    outs = []
    for g in range(len(go) - 1):
        s = None
        for t in range(int(go[g]), int(go[g + 1])):
            x = TtTensor(*b.get(t)).scaled(float(sc[t]))
            s = x if s is None else s + x
        outs.append(s.rounded(eps, cap))
    return TtBatch.from_list(outs)


def c4_problem():
    """The benchmarked configuration's shape at oracle size: config 4's
    velocity mesh VelocityGrid(44, 7), eps 1e-5, Mach-3 free stream, diffuse
    walls, on a jittered, shuffled 6x5x4 hex mesh around a 2^3 obstacle (112
    cells, 422 faces: oblique interior faces, 24 wall faces, in/out boundary
    faces)."""
    return obstacle_flow(C4_SHAPE, hole=C4_HOLE)


def obstacle_fixture():
    """C4_STEPS free-running reference steps of c4_problem(): the packed
    state before every step and after the last (lock-step inputs / expected
    outputs), the macroparameters of every step, and the last step's face-flux
    and residual ranks."""
    ref = _ref()
    p = c4_problem()
    r = ref.RefSolver.for_problem(p)
    out = dict(steps=np.int64(C4_STEPS), dt=np.float64(p.dt), eps=np.float64(p.eps),
               nv=np.int64(p.nv), ncell=np.int64(p.mesh.ncell), nface=np.int64(p.mesh.nface),
               face_left=p.mesh.face_left.astype(np.int32), face_normal=p.mesh.face_normal)
    states = [p.f0]
    macros = []
    for _ in range(C4_STEPS):
        r.step(p.dt, p.eps, p.cap)
        states.append(r.state())
        macros.append(r.macros(p.mesh.ncell)[:, :11].copy())
    for k, s in enumerate(states):
        out[f"s{k}_ranks"], out[f"s{k}_offsets"], out[f"s{k}_cores"] = s.ranks, s.offsets, s.cores
    out["macros"] = np.stack(macros)
    out["phi_ranks"] = r.fetch(r.PHI).ranks.copy()
    out["res_ranks"] = r.fetch(r.R).ranks.copy()
    r.close()
    return out


if __name__ == "__main__":
    np.savez_compressed(os.path.join(HERE, "shock_tube_c1.npz"), **shock_tube_fixture())
    np.savez_compressed(os.path.join(HERE, "rounding_24.npz"), **rounding_fixture())
    np.savez_compressed(os.path.join(HERE, "obstacle_c4_nv44.npz"), **obstacle_fixture())
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))
