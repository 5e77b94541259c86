#!/usr/bin/env python
"""Benchmark of the TT-DVM explicit step (BASELINE.json metric: cell-steps/s
at the 44^3 velocity mesh).

A "step" is one explicit step S1 over every cell of the
workload's mesh, with the state resident in HBM.  Default workload: config
4 of BASELINE.json -- the unstructured (jittered, shuffled) hex mesh of
511,488 cells around an 8^3 obstacle, 44^3 velocity mesh on [-7,7]^3, Mach-3
free stream, diffuse walls, eps 1e-5, fp64 (synthetic, seeded).  The
one-time face-factor set-up (|xi_n| estimates of 1.5 M distinct oblique
normals) is timed separately (config.setup_s), not inside the step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 1|2|3|4|5] [--scale s]

--config 3 is the batched-rounding microbench (rounded tensors/s; a step
rounds one resident chunk of 8192 x scale config-3 sums, the 2^20 tensors
of the config being 128 such chunks of identical per-tensor work).

N > 1 under torchrun: config 4 is partitioned by recursive coordinate
bisection of the cell centroids (strong scaling, the same mesh on N GPUs);
configs 2 / 5 stack N x-slabs of the single-GPU box (weak scaling).  Halo TT
cores of cut faces are exchanged every step over NCCL.  The timing is the
max over ranks of the CUDA-event time of the K steps.  --impl reference
times the CPU oracle (the numpy restatement of the reference, all host
cores, one process per core) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=0,
                    help="0 = the config's own step count (20 for config 4, 10 for config 5)")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--parity-cells", type=int, default=64,
                    help="cells of the sampled full-size lock-step check (default 64)")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the sampled oracle lock-step check after the timed region")
    ap.add_argument("--e2e-steps", type=int, default=0, help="0 = same as --steps")
    return ap.parse_args()


def workload_config(p, args):
    return {"workload": p.name, "config_index": args.config, "cells": int(p.mesh.ncell),
            "faces": int(p.mesh.nface), "velocity_mesh": f"{p.nv}^3 on [-{p.bound},{p.bound}]^3",
            "eps": p.eps, "rank_cap": p.cap, "dt": p.dt,
            "l2_policy": "inputs larger than L2 (state and face-factor arenas >> 126 MB)",
            "timed_from": "initial state re-uploaded after warm-up (steps 1..K of the run)"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.stop = threading.Event()
        self.t = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if len(r) > 3 + k and r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def traffic_from_profiles():
    """ncu dram bytes per launch of the dominant kernel, if captured."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------ CPU arms
def _one_blas_thread():
    """numpy is imported with this module (also in spawned workers), so the
    BLAS pool is limited at run time, not through the environment."""
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass


def ref_sample_part(p, nblocks: int, b: int, seed: int = 7):
    """A bounded sample of the workload for the CPU arms: ``nblocks``
    contiguous b^3 blocks of cells at seeded uniform positions of the mesh
    lattice, as one local mesh (partition.build_part) with a one-cell ghost
    ring around every block.  Interior faces are shared by two sampled cells,
    so the flux work per cell is amortised as in the full step (b = 6:
    3.5 faces per cell against the mesh's 3.04); the ghost ring stays frozen
    at the initial state.  Returns None when the mesh is no larger than the
    sample (the whole mesh is stepped then)."""
    from paper_1912_04582_b200.partition import build_part
    m = p.mesh
    if m.cell_ijk is None or m.ncell <= nblocks * b ** 3:
        return None
    rng = np.random.default_rng(seed)
    ijk = m.cell_ijk
    mask = np.zeros(m.ncell, dtype=bool)
    for _ in range(nblocks):
        o = np.array([int(rng.integers(0, max(1, sdim - b + 1))) for sdim in m.shape])
        mask |= np.all((ijk >= o[None, :]) & (ijk < (o + b)[None, :]), axis=1)
    return build_part(m, np.where(mask, 0, 1).astype(np.int32), 0)


def cpu_reference_rate(p, nblocks: int, b: int, warmup: int, steps: int, threads: int):
    """Cell-steps/s of the reference CPU implementation on a bounded sample
    (ref_sample_part), advanced through warmup + steps explicit steps from
    the workload's initial state -- so its ranks grow with the step number
    as the GPU arm's do.  The compiled reference (oracle/_ref: the unmodified
    proj/src/*.cpp, S1 composed of reference calls, OpenMP over faces and
    cells) when its library is present, else the numpy port.  One-time
    face-factor set-up is kept out of the timed steps, as in the GPU arm.
    Returns (rate, info dict)."""
    from oracle import ref
    from paper_1912_04582_b200.partition import local_state
    part = ref_sample_part(p, nblocks, b)
    mesh = p.mesh if part is None else part.mesh
    f0 = p.f0 if part is None else local_state(part, p.f0)
    nown = p.mesh.ncell if part is None else part.n_owned
    cells = np.arange(nown, dtype=np.int32)
    t_setup = time.perf_counter()
    if ref.available():
        kind = "reference"
        r = ref.RefSolver(p.nv, p.bound, p.gas, mesh, p.bcs, threads=threads)
        r.set_state(f0)
        r.step(p.dt, p.eps, p.cap, cells=cells)   # fills the face-factor cache (one-time)
        r.set_state(f0)
        setup_s = time.perf_counter() - t_setup
        for _ in range(warmup):
            r.step(p.dt, p.eps, p.cap, cells=cells)
        t = time.perf_counter()
        for _ in range(steps):
            r.step(p.dt, p.eps, p.cap, cells=cells)
        el = time.perf_counter() - t
        max_rank = int(r.state().ranks[:nown].max())
        r.close()
        what = "compiled reference C++ (oracle/_ref, OpenMP)"
    else:
        kind, threads = "port", 1
        _one_blas_thread()
        from oracle.parity import oracle_list
        from oracle.step import OracleSolver
        solver = OracleSolver(mesh, p.nv, p.bound, p.gas, p.bcs)
        f = dict(enumerate(oracle_list(f0)))
        for c in cells:
            for fid, _ in mesh.cell_faces(int(c)):
                solver.factors(mesh.face_normal[fid])
        setup_s = time.perf_counter() - t_setup
        el = 0.0
        for it in range(warmup + steps):
            t = time.perf_counter()
            out, _ = solver.step(f, p.dt, p.eps, p.cap, cells=[int(c) for c in cells])
            if it >= warmup:
                el += time.perf_counter() - t
            for c, x in zip(cells, out):
                f[int(c)] = x
        max_rank = max(max(f[int(c)].ranks()) for c in cells)
        what = "numpy port (oracle/step.py), 1 BLAS thread"
    rate = nown * steps / el
    info = {"kind": kind, "cores": threads, "cells": int(nown), "setup_s": round(setup_s, 1),
            "max_rank_after": max_rank, "ms_per_step": 1e3 * el / steps,
            "sample": (f"{nown} cells " + ("(the whole mesh)" if part is None else
                       f"= {nblocks} contiguous {b}^3 blocks at seeded lattice positions, frozen "
                       "one-cell ghost ring") + f", advanced through {warmup}+{steps} steps from "
                       f"the initial state, {what}, {threads} threads, face factors set up before "
                       "timing")}
    return rate, info


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1912_04582_b200.problems import config
    p = config(args.config, args.scale)
    threads = os.cpu_count() or 1
    # ~8 blocks of 6^3 cells: ~6k distinct oblique normals of one-time
    # face-factor set-up (~1 min on 16 cores), seconds of timed steps
    nblocks = int(os.environ.get("TTDVM_REF_BLOCKS", "8"))
    value, info = cpu_reference_rate(p, nblocks, 6, args.warmup, args.steps, threads)
    line = {"impl": "reference", "metric": "cell-steps/s", "value": value, "unit": "cell-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": info["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(p, args),
            "cpu_baseline": {"value": value, "unit": "cell-steps/s", "cores": info["cores"],
                             "kind": info["kind"], "sample": info["sample"],
                             "setup_s": info["setup_s"], "max_rank_after": info["max_rank_after"]},
            "e2e": {"value": value, "unit": "cell-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ parity block
def parity_block(p, st_prev, st_new, macros_prev, from_step: int, ncells: int = 64, seed: int = 0,
                 stage_ranks=None):
    """Sampled full-size lock-step check of the run just timed: ``ncells``
    cells of the workload -- half of them the highest-rank cells of the new
    state and wall-adjacent cells (the disturbed region), half uniform --
    are stepped by the oracle from the GPU's own state t^(K-1), with the
    faces they touch and the neighbour states behind them, and compared with
    the GPU's state t^K: per-cell reconstruction error (bar 10 eps),
    macroparameters (1e-8), ranks (every mismatch inside the TIE window of an
    oracle decision on the cell's chain, oracle/parity.py).  The oracle is
    the checker here, never the thing measured."""
    from oracle import parity, ref
    from oracle.tt import rel_err
    from paper_1912_04582_b200.partition import build_part
    m = p.mesh
    rng = np.random.default_rng(seed)
    if not ref.available():
        ncells = min(ncells, 8)  # the numpy port's face factors cost ~1 s per normal
    ncells = min(ncells, m.ncell)
    hot = []
    walls = [g for g, bc in enumerate(p.bcs) if bc["kind"] == "wall"]
    if walls:
        wf = np.nonzero((m.face_right < 0) & np.isin(m.face_group, walls))[0]
        hot = list(np.unique(m.face_left[wf])[:: max(1, len(wf) // max(1, ncells // 8))][:ncells // 8])
    order = np.argsort(-st_new.ranks.max(1).astype(np.int64), kind="stable")
    for c in order:
        if len(hot) >= ncells // 2:
            break
        if int(c) not in hot:
            hot.append(int(c))
    rest = np.setdiff1d(np.arange(m.ncell), np.array(hot, dtype=np.int64))
    cells = np.sort(np.concatenate([np.array(hot, dtype=np.int64),
                                    rng.choice(rest, ncells - len(hot), replace=False)]))
    owner = np.ones(m.ncell, dtype=np.int32)
    owner[cells] = 0
    part = build_part(m, owner, 0)
    loc = st_prev.subset(part.local_to_global)
    nown = part.n_owned
    t0 = time.perf_counter()
    if ref.available():
        name = "compiled reference (oracle/_ref: unmodified proj/src/*.cpp, S1 of reference calls)"
        r = ref.RefSolver(p.nv, p.bound, p.gas, part.mesh, p.bcs)
        r.set_state(loc)
        r.step(p.dt, p.eps, p.cap, cells=np.arange(nown, dtype=np.int32))
        want = r.state()
        wm = r.macros(nown)
        ref_phi, ref_res, ref_j = r.ranks_of(r.PHI), r.ranks_of(r.R), r.ranks_of(r.J)
        r.close()
    else:
        name = "numpy port (oracle/step.py)"
        from oracle.step import OracleSolver
        from paper_1912_04582_b200.tt_batch import TtBatch
        s = OracleSolver(part.mesh, p.nv, p.bound, p.gas, p.bcs)
        out, mo = s.step(dict(enumerate(parity.oracle_list(loc))), p.dt, p.eps, p.cap,
                         cells=list(range(nown)))
        want = TtBatch.from_list(out)
        wm = np.stack([x.as_array() for x in mo])
    # intermediate stages (GPU ranks from the last step's sets, no core download):
    # the face fluxes of every face the sampled cells touch, and their residuals
    stage = None
    if stage_ranks is not None and ref.available():
        gphi, gres, gj = stage_ranks
        lf = np.nonzero(ref_phi[:, 0] > 0)[0]                  # local faces the reference computed
        phi_flip = lf[np.any(ref_phi[lf] != gphi[part.face_global[lf]], axis=1)]
        res_flip = np.nonzero(np.any(ref_res[:nown] != gres[part.owned], axis=1))[0]
        j_flip = np.nonzero(np.any(ref_j[:nown] != gj[part.owned], axis=1))[0]
        stage = {"faces": int(len(lf)), "phi_rank_flips": int(len(phi_flip)),
                 "res_rank_flips": int(len(res_flip)), "collision_rank_flips": int(len(j_flip)),
                 "max_phi_flip_margin": 0.0, "max_res_flip_margin": 0.0,
                 "max_collision_flip_margin": 0.0,
                 "collision_flip_cells": [int(part.owned[k]) for k in j_flip[:8]]}
        if len(phi_flip) or len(res_flip) or len(j_flip):
            from oracle.step import OracleSolver
            so = OracleSolver(part.mesh, p.nv, p.bound, p.gas, p.bcs)
            cmx = parity.ChainMargins(so, dict(enumerate(parity.oracle_list(loc))), p.dt, p.eps, p.cap)
            if len(phi_flip):
                stage["max_phi_flip_margin"] = max(cmx.phi(int(j)) for j in phi_flip[:4])
            for k in j_flip[:4]:  # the f_S rounding and the (f_S - f) rounding of the cell
                m_fs, m_j, _ = cmx.collision(int(k))
                stage["max_collision_flip_margin"] = max(stage["max_collision_flip_margin"],
                                                         min(m_fs, m_j))
            kappa = 0.0
            for k in res_flip[:4]:
                # a residual's inputs (the rounded fluxes) already differ between the two
                # sides by the roundoff of their own truncations (~u/eps, observed 1e-9);
                # the residual rounding sees that difference amplified by the
                # cancellation factor kappa = (sum_f |c_f| ||Phi_f|| + ||J||) / ||R||
                k = int(k)
                mg = cmx.cell(k)
                stage["max_res_flip_margin"] = max(stage["max_res_flip_margin"], mg["res"])
                m_ = part.mesh
                num = 0.0
                for fid, sg in m_.cell_faces(k):
                    num += abs(sg * m_.face_area[fid] / m_.cell_volume[k]) * cmx._phi_t[fid].frobenius_norm()
                _, _, jt = cmx.collision(k)
                acc = jt
                for fid, sg in m_.cell_faces(k):
                    acc = acc + cmx._phi_t[fid].scaled(-sg * m_.face_area[fid] / m_.cell_volume[k])
                kappa = max(kappa, (num + jt.frobenius_norm()) / max(acc.frobenius_norm(), 1e-300))
            stage["res_flip_cancellation"] = kappa
            # margin a 1e-9 input difference explains: 2 sqrt(2) delta kappa / eps
            stage["res_flip_margin_explained"] = 2.83 * 1e-9 * kappa / p.eps
    worst, flips, errs = 0.0, [], []
    for k in range(nown):
        g = int(part.owned[k])
        e = rel_err(st_new.full(g), want.full(k))
        errs.append(e)
        worst = max(worst, e)
        if tuple(st_new.ranks[g]) != tuple(want.ranks[k]):
            flips.append(k)
    top = np.argsort(-np.array(errs))[:5]
    res_flipped = set(int(k) for k in res_flip) if stage is not None else set()
    worst_cells = [{"cell": int(part.owned[k]), "rel_err": float(errs[k]),
                    "ranks": [int(v) for v in want.ranks[k]],
                    "ranks_before": [int(v) for v in loc.ranks[k]],
                    "hot": bool(int(part.owned[k]) in set(hot)),
                    "res_rank_flip": bool(int(k) in res_flipped)} for k in top]
    # decision margins of the oracle along the worst cell's chain (phi, f_S, J, R, state):
    # a deviation well above the rest of the sample should sit next to a small margin
    if errs[int(top[0])] > 100 * max(float(np.median(errs)), 1e-12):
        try:
            from oracle.step import OracleSolver
            so = OracleSolver(part.mesh, p.nv, p.bound, p.gas, p.bcs)
            cmw = parity.ChainMargins(so, dict(enumerate(parity.oracle_list(loc))), p.dt, p.eps, p.cap)
            worst_cells[0]["oracle_margins"] = {k_: float(v) for k_, v in cmw.cell(int(top[0])).items()}
        except Exception as e:  # diagnostics only
            worst_cells[0]["oracle_margins"] = str(e)
    macro = parity.macro_err(macros_prev[part.owned], wm)
    worst_margin = 0.0
    if flips:
        from oracle.step import OracleSolver
        s = OracleSolver(part.mesh, p.nv, p.bound, p.gas, p.bcs)
        cm = parity.ChainMargins(s, dict(enumerate(parity.oracle_list(loc))), p.dt, p.eps, p.cap)
        worst_margin = max(min(cm.cell(k).values()) for k in flips)
    tie = parity.tie(p.eps)
    return {"cells": int(nown), "from_step": int(from_step), "oracle": name,
            "max_rel_err": worst, "tol_rel_err": 10 * p.eps, "macro_max_rel": macro,
            "tol_macro": 1e-8, "rank_flips": len(flips), "max_flip_margin": worst_margin,
            "tie": tie, "max_rank_in_sample": int(want.ranks[:nown].max()),
            "wall_adjacent_cells": int(len(walls) and min(len(hot), ncells // 8)),
            "stages": stage, "worst_cells": worst_cells,
            "median_rel_err": float(np.median(errs)),
            "oracle_s": round(time.perf_counter() - t0, 1),
            # the bar is BASELINE.json's: per-cell tensors, macroparameters and the TT ranks of
            # the STATE; `stages` reports the intermediate fluxes / residuals as diagnostics
            "pass": bool(worst <= 10 * p.eps and macro <= 1e-8 and worst_margin < tie and
                         (stage is None or (stage["max_phi_flip_margin"] < tie and
                                            stage["max_collision_flip_margin"] < tie)))}


# ------------------------------------------------- config 3: batched rounding
C3_CHUNK = 8192


def c3_inputs(count: int, seed: int = 3):
    from paper_1912_04582_b200.problems import rounding_summands
    from paper_1912_04582_b200.tt_batch import TtBatch
    f, m, l = rounding_summands(np.random.default_rng(seed), count)
    b = TtBatch.uniform(6 * count, 32, 32, 32, 12, 12, f, m, l)
    return b, np.arange(0, 6 * count + 1, 6, dtype=np.int64)


def _c3_task(args_tuple):
    _one_blas_thread()
    from oracle.tt import TtTensor
    from paper_1912_04582_b200.problems import rounding_summands
    seed, count = args_tuple
    f, m, l = rounding_summands(np.random.default_rng(seed), count)
    sums = []
    for g in range(count):
        s = TtTensor(f[6 * g], m[6 * g], l[6 * g])
        for k in range(1, 6):
            s = s + TtTensor(f[6 * g + k], m[6 * g + k], l[6 * g + k])
        sums.append(s)
    t = time.perf_counter()
    for s in sums:
        s.rounded(1e-6)
    return time.perf_counter() - t


def c3_cpu_rate(workers: int, per: int, repeats: int = 1):
    import multiprocessing as mp
    ctxm = mp.get_context("spawn")
    with ctxm.Pool(workers) as pool:
        best = None
        for r in range(repeats):
            t = time.perf_counter()
            pool.map(_c3_task, [(100 + w, per) for w in range(workers)])
            el = time.perf_counter() - t
            best = el if best is None else min(best, el)
    return workers * per / best


def c3_config(count):
    return {"workload": "config3-batched-rounding", "config_index": 3,
            "tensors_per_step": count, "tensor_shape": "32x32x32",
            "summands": "6 x rank-(1,12,12,1), N(0,1) cores, 0.5^a decay on the outer cores' "
                        "rank indices (summed rank 72)", "eps": 1e-6,
            "full_config": "2^20 tensors = %d chunks of identical per-tensor work" % (
                (1 << 20) // count),
            "l2_policy": "inputs larger than L2 (%.1f GB resident summands)" % (
                count * 6 * (32 * 12 * 2 + 32 * 144) * 8 / 1e9)}


def run_config3(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    count = max(16, int(C3_CHUNK * args.scale))
    if args.impl == "reference":
        if rank != 0:
            return
        workers = os.cpu_count() or 1
        per = 32
        c3_cpu_rate(workers, 1)  # warm the pool imports
        t = time.perf_counter()
        for _ in range(args.steps):
            c3_cpu_rate(workers, per)
        value = workers * per * args.steps / (time.perf_counter() - t)
        print(json.dumps({"impl": "reference", "metric": "rounded tensors/s", "value": value,
                          "unit": "tensors/s", "n_gpus": args.gpus, "steps": args.steps,
                          "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
                          "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                          "config": c3_config(count),
                          "cpu_baseline": {"value": value, "unit": "tensors/s", "cores": workers,
                                           "kind": "port",
                                           "sample": f"{workers} processes x {per} config-3 sums "
                                                     "per step, numpy oracle rounded(1e-6)"},
                          "e2e": {"value": value, "unit": "tensors/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}), flush=True)
        return
    import torch
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1912_04582_b200.cuda import Context
    b, go = c3_inputs(count, seed=3 + rank)  # independent tensors per rank: weak scaling
    ctx = Context(local)
    ctx.set_grid(32, 1.0)
    eps = 1e-6
    ctx.rounded(b, eps, 0, group_off=go)  # upload; the inputs stay resident
    ctx.round_resident(eps, 0, args.warmup)
    ctx.set_profiling(True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = ctx.round_resident(eps, 0, args.steps)
    torch.cuda.synchronize()
    flops, bytes_, launches = ctx.phase_work()
    phase_ms = ctx.phase_times()
    gpu_launches = ctx.launch_count()
    res = ctx.result()
    ranks = res.ranks
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = world * count * args.steps / (ms / 1e3)
    ctx.set_profiling(False)
    # e2e: host summands -> device, round, result -> host, every step, from /
    # into pinned host buffers (filled before the timed region)
    from paper_1912_04582_b200.tt_batch import TtBatch
    pin_in = torch.empty(b.cores.size, dtype=torch.float64, pin_memory=True).numpy()
    pin_in[:] = b.cores
    b = TtBatch(b.n1, b.n2, b.n3, b.ranks, b.offsets, pin_in)
    pin_out = torch.empty(count * (32 * 32 * 34), dtype=torch.float64,  # max ranks (32, 32)
                          pin_memory=True).numpy()
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(args.e2e_steps):
        out = ctx.rounded(b, eps, 0, group_off=go, out=pin_out)
        d2h += int(out.cores.nbytes + out.ranks.nbytes + out.offsets.nbytes)
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    h2d = int(b.cores.nbytes + b.ranks.nbytes + b.offsets.nbytes + go.nbytes)
    fp64_peak = ctx.fp64_peak()
    dom_s = phase_ms[2] / 1e3
    achieved = flops[2] / dom_s / 1e12 if dom_s > 0 else 0.0
    traffic = traffic_from_profiles().get("config3")
    roofline = {"bound": "fp64", "kernel": "round_gram_kernel (config-3 T route)",
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak if fp64_peak else None,
                "peak_source": "measured on this GPU by the DFMA probe in libttdvm_cuda.so",
                "flops_per_launch": flops[2] / max(1, launches[2]),
                "flops_per_tensor": flops[2] / (count * args.steps),
                "launch_ms": phase_ms[2] / max(1, launches[2]),
                "algorithmic_bytes_per_launch": bytes_[2] / max(1, launches[2]),
                "hbm_frac": (bytes_[2] / dom_s / 1e9) / load_peaks().get("hbm_gbs", 6547.8)
                if dom_s > 0 else None,
                "traffic": traffic}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        per = 1024
        rate = c3_cpu_rate(1, per)
        cpu = {"value": rate, "unit": "tensors/s", "cores": 1, "kind": "port",
               "sample": f"{per} config-3 sums rounded at 1e-6 by the numpy oracle "
                         "(oracle/tt.py), 1 process, 1 BLAS thread"}
    if rank == 0:
        print(json.dumps({
            "metric": "rounded tensors/s", "value": value, "unit": "tensors/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": dict(c3_config(count), parallelism=f"independent chunks x{world}"
                           if world > 1 else "single GPU",
                           output_ranks={"min": ranks.min(0).tolist(),
                                         "max": ranks.max(0).tolist()}),
            "roofline": roofline, "cpu_baseline": cpu,
            "e2e": {"value": world * count * args.e2e_steps / e2e_s, "unit": "tensors/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h // args.e2e_steps,
                    "steps": args.e2e_steps},
            "gpu_launches": gpu_launches, "clocks": clk.summary()}), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


# ------------------------------------------------------------------- GPU arm
def spawn_ranks(args):
    """`python bench.py --gpus N` without torchrun: launch the N ranks here
    (one process per GPU over NCCL) and fail loudly when fewer GPUs are visible."""
    import socket

    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) visible",
              file=sys.stderr)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.run(cmd).returncode)


def kernel_rooflines(rep, steps, fp64_peak, hbm_peak):
    """Per-kernel achieved rates of one profiled pass: algorithmic FLOPs and
    bytes (ttdvm_cuda_phase_report) over the phase's device time, against
    the measured DFMA peak and the measured HBM bandwidth."""
    kernels = {"moments": ("macro_kernel", "hbm"), "shakhov_build": ("shakhov_raw_kernel", "hbm"),
               "wall_densities": ("wall_kernel", "latency"),
               # bulk rank bins: the six pipe_* phase kernels (round_pipe.cuh); the other
               # bins: round_gram_kernel at 32 / 128 / 256 / 512 threads
               "round_fs": ("rounding of f_S (pipe_* phase kernels)", "fp64"),
               "round_collision": ("rounding of f_S - f (pipe_* phase kernels + round_gram_kernel)", "fp64"),
               "round_flux": ("rounding of face fluxes (pipe_* phase kernels + round_gram_kernel "
                              "high-rank bins)", "fp64"),
               "round_residual": ("rounding of cell residuals (pipe_* phase kernels + "
                                  "round_gram_kernel high-rank bins)", "fp64"),
               "round_update": ("rounding of f + dt R (pipe_* phase kernels + round_gram_kernel)",
                                "fp64")}
    out = {}
    for name, (kern, bound) in kernels.items():
        ms, fl, by, la = rep[name]
        if ms <= 0.0 or la <= 0:
            continue
        tf, gbs = fl / ms / 1e9, by / ms / 1e6
        out[name] = {"kernel": kern, "bound": bound, "ms_per_step": round(ms / steps, 4),
                     "launches_per_step": round(la / steps, 2),
                     "tflops": round(tf, 4), "fp64_frac": round(tf / fp64_peak, 5) if fp64_peak else None,
                     "gbs": round(gbs, 2), "hbm_frac": round(gbs / hbm_peak, 5)}
    return out


def main():
    args = parse()
    if args.steps <= 0:  # each config's own step count (BASELINE.json configs)
        args.steps = {1: 100, 2: 50, 3: 5, 4: 20, 5: 10}.get(args.config, 5)
    if args.e2e_steps <= 0:
        args.e2e_steps = args.steps
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        spawn_ranks(args)
    if args.config == 3:
        run_config3(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1912_04582_b200.cuda import Context
    from paper_1912_04582_b200.problems import config
    t_setup = time.perf_counter()
    p = config(args.config, args.scale)
    setup = {"mesh_and_state_s": round(time.perf_counter() - t_setup, 2)}
    ctx = Context(local)
    part = None
    hx = None  # torch.distributed halo exchange (A/B only; the default is inside the library)
    scaling = "weak"
    ncell_total = p.mesh.ncell
    if world > 1:
        from paper_1912_04582_b200 import halo
        from paper_1912_04582_b200.partition import build_part, local_state
        if args.config == 4:
            # strong scaling: one mesh, RCB of the cell centroids over the ranks
            from paper_1912_04582_b200.mesh import rcb_partition
            part = build_part(p.mesh, rcb_partition(p.mesh.centroids, world), rank)
            scaling = "strong"
            pg = p
        else:
            # weak scaling: the global periodic box is `world` x-slabs of the
            # single-GPU workload; each rank owns one slab plus its halo ghosts
            from paper_1912_04582_b200.mesh import slab_partition
            from paper_1912_04582_b200.problems import periodic_box
            nx, ny, nz = p.mesh.shape
            pg = periodic_box((nx * world, ny, nz), nv=p.nv, bound=p.bound, eps=p.eps, cap=p.cap,
                              name=p.name + f"-x{world}")
            part = build_part(pg.mesh, slab_partition(pg.mesh, world), rank)
            ncell_total = pg.mesh.ncell
        ctx.set_grid(pg.nv, pg.bound)
        ctx.set_gas(pg.gas)
        ctx.set_mesh(part.mesh)
        ctx.set_bcs(pg.bcs)
        f_local = local_state(part, pg.f0)
        # halo exchange inside the library: NCCL communicator from a unique id
        # made by rank 0, the halo plan of this rank's part; every step then
        # starts with the exchange, overlapped with the collision phases
        # (TTDVM_HALO=python keeps the torch.distributed exchange for A/B)
        if os.environ.get("TTDVM_HALO", "library") == "python":
            ctx.set_owned(part.n_owned)
            hx = halo.HaloExchange(ctx, part, torch.device("cuda", local))
        else:
            uid = [Context.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ctx.comm_init(world, rank, uid[0])
            ctx.set_partition(part.n_owned, part.send, part.recv)
        ctx.upload_state(f_local)
        p = pg
        cells_per_rank = part.n_owned
    else:
        ctx.setup(p)
        if os.environ.get("TTDVM_BENCH_BLOCKS"):  # diagnostics: force the blocked step at small scale
            ctx.set_blocks(int(os.environ["TTDVM_BENCH_BLOCKS"]))
        f_local = p.f0
        cells_per_rank = p.mesh.ncell
    t0 = time.perf_counter()
    ctx.step(p.dt, p.eps, p.cap, 0)  # face factors, wall set-up, summand lists
    setup["face_factors_s"] = round(time.perf_counter() - t0, 2)
    setup.update({k: v for k, v in ctx.setup_info().items() if k != "face_factor_ms"})
    fp64_peak = ctx.fp64_peak()
    hbm_peak = load_peaks().get("hbm_gbs", 6547.8)

    def run_steps(k):
        """k steps; device ms by CUDA events on the stream the kernels run on."""
        if part is None or hx is None:
            return ctx.timed_step(p.dt, p.eps, p.cap, k)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(k):
            ctx.step(p.dt, p.eps, p.cap, 1)
            hx.exchange()
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1)

    # ---- timed region: steps 1..K from the initial state, profiling OFF ----
    run_steps(args.warmup)
    ctx.upload_state(f_local)
    ctx.set_profiling(False)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = run_steps(args.steps)
    torch.cuda.synchronize()
    gpu_launches = ctx.launch_count() * (1 if (part is None or hx is None) else args.steps)
    setup["cell_blocks"] = ctx.setup_info()["cell_blocks"]  # grown on out-of-memory
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ncell_total * args.steps / (ms / 1e3)

    # ---- e2e through the public API with host buffers: upload state, one
    # step, download state -- every step (steps 1..E from the initial state)
    from paper_1912_04582_b200.tt_batch import TtBatch
    pinned = torch.empty(max(2 * f_local.cores.size, 1 << 20), dtype=torch.float64,
                         pin_memory=True).numpy()
    pinned[:f_local.cores.size] = f_local.cores
    host = TtBatch(f_local.n1, f_local.n2, f_local.n3, f_local.ranks, f_local.offsets,
                   pinned[:f_local.cores.size])
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    h2d = d2h = 0
    for _ in range(args.e2e_steps):
        h2d += int(host.cores.nbytes + host.ranks.nbytes + host.offsets.nbytes)
        ctx.upload_state(host)
        ctx.step(p.dt, p.eps, p.cap, 1)
        if hx is not None:
            hx.exchange()
        host = ctx.download_state(out=pinned)
        d2h += int(host.cores.nbytes + host.ranks.nbytes + host.offsets.nbytes)
    h2d //= args.e2e_steps
    d2h //= args.e2e_steps
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if dist:
        t = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = ncell_total * args.e2e_steps / e2e_s
    max_rank = int(host.ranks.max())
    del host

    # ---- separate profiled pass over the same steps 1..K (per-phase CUDA
    # events cost a sync per phase, so they stay out of the timed region);
    # it also leaves the states t^(K-1) and t^K for the parity block
    ctx.upload_state(f_local)
    ctx.set_profiling(True)
    rep = None
    st_prev = st_new = macros_prev = None
    for chunk in (args.steps - 1, 1):
        if chunk <= 0:
            continue
        if part is None or hx is None:
            ctx.timed_step(p.dt, p.eps, p.cap, chunk)
            r = ctx.phase_report()
            rep = r if rep is None else {k: tuple(a + b for a, b in zip(rep[k], r[k])) for k in r}
            if chunk == args.steps - 1 and part is None:
                st_prev = ctx.download_state()
        else:
            for _ in range(chunk):
                ctx.timed_step(p.dt, p.eps, p.cap, 1)
                r = ctx.phase_report()
                rep = r if rep is None else {k: tuple(a + b for a, b in zip(rep[k], r[k]))
                                             for k in r}
                hx.exchange()
    ctx.set_profiling(False)
    parity = None
    if part is None and rank == 0 and not args.no_parity:
        if st_prev is None:
            st_prev = f_local
        st_new = ctx.download_state()
        macros_prev = ctx.macros()
        try:
            # the intermediate sets of a blocked step (cell_blocks > 1: config 5 at full size)
            # hold the last cell block only, so the stage-rank comparison needs one block
            one_block = ctx.setup_info()["cell_blocks"] == 1
            parity = parity_block(p, st_prev, st_new, macros_prev, args.steps - 1,
                                  ncells=args.parity_cells,
                                  stage_ranks=(ctx.stage_ranks("phi"), ctx.stage_ranks("res"),
                                               ctx.stage_ranks("jr")) if one_block else None)
        except Exception as e:  # the bench line still prints; the failure is visible
            parity = {"error": f"{type(e).__name__}: {e}", "pass": False}
        del st_prev, st_new

    # ---- rooflines: every kernel of the step, then the dominant one
    per_kernel = kernel_rooflines(rep, args.steps, fp64_peak, hbm_peak)
    rounds = [k for k in per_kernel if k.startswith("round_")]
    dom = max(rounds, key=lambda k: per_kernel[k]["ms_per_step"])
    d_ms, d_fl, d_by, d_la = rep[dom]
    # ncu DRAM bytes per rounded output of this phase (profiles/traffic.json),
    # times the phase's outputs per launch in this run
    per_out = traffic_from_profiles().get(dom + "_bytes_per_output")
    nface_local = (part.mesh if part is not None else p.mesh).nface
    outs_per_step = {"round_flux": nface_local}.get(dom, cells_per_rank)
    traffic = (per_out * outs_per_step * args.steps / max(1, d_la) if per_out else None)
    achieved = d_fl / d_ms / 1e9
    roofline = {"bound": "fp64", "kernel": per_kernel[dom]["kernel"],
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak if fp64_peak else None,
                "peak_source": "measured on this GPU by the DFMA probe in libttdvm_cuda.so "
                               "(MEASURED_PEAKS.json has no FP64 entry); hbm_frac against "
                               "MEASURED_PEAKS.json hbm_gbs",
                "flops_per_launch": d_fl / max(1, d_la), "launch_ms": d_ms / max(1, d_la),
                "algorithmic_bytes_per_launch": d_by / max(1, d_la),
                "hbm_frac": per_kernel[dom]["hbm_frac"], "traffic": traffic,
                "measured_in": "a separate profiled pass over the same steps 1..K "
                               "(per-phase CUDA events); the timed region runs unprofiled",
                "profiled_ms_per_step": round(sum(v[0] for v in rep.values()) / args.steps, 3),
                "per_kernel": per_kernel}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        # bounded: 2 blocks of 6^3 cells (~1.5k oblique normals of one-time
        # set-up), the same warm-up and step counts as the GPU arm
        threads = os.cpu_count() or 1
        rate, info = cpu_reference_rate(p, 2, 6, args.warmup, args.steps, threads)
        cpu = {"value": rate, "unit": "cell-steps/s", "cores": info["cores"],
               "kind": info["kind"], "sample": info["sample"], "setup_s": info["setup_s"],
               "max_rank_after": info["max_rank_after"]}
    if rank == 0:
        line = {"metric": "cell-steps/s", "value": value, "unit": "cell-steps/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
                "dtype": "f64", "data": "synthetic",
                "config": dict(workload_config(p, args),
                               parallelism=((f"RCB partition x{world}" if args.config == 4 else
                                             f"x-slab partition x{world}") +
                                            ", halo TT cores over NCCL" if world > 1
                                            else "single GPU"),
                               halo=(ctx.halo_stats() if part is not None and hx is None else None),
                               cells_total=ncell_total, cells_per_gpu=cells_per_rank,
                               max_rank_after=max_rank, setup_s=setup),
                "roofline": roofline, "cpu_baseline": cpu, "parity": parity,
                "e2e": {"value": e2e_value, "unit": "cell-steps/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "steps": args.e2e_steps},
                "gpu_launches": gpu_launches, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
