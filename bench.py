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
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
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


def _ref_worker_init(args_tuple):
    """Per worker: the problem, an oracle solver, and its face-factor cache
    filled for every face of ``warm_cells`` -- the one-time set-up the GPU
    arm also keeps out of its timed steps (pool.map hands a strip to
    whichever worker is free, so every worker warms every strip)."""
    _one_blas_thread()
    global _W
    cfg, scale, warm_cells = args_tuple
    from oracle.step import OracleSolver
    from oracle.tt import TtTensor
    from paper_1912_04582_b200.problems import config
    p = config(cfg, scale)
    solver = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    for c in warm_cells:
        for fid, _ in p.mesh.cell_faces(c):
            solver.factors(p.mesh.face_normal[fid])
    _W = (p, solver, TtTensor)


def _ref_task(cells):
    p, solver, TtTensor = _W
    need = set(cells)
    for c in cells:
        for fid, _ in p.mesh.cell_faces(c):
            need.add(int(p.mesh.face_left[fid]))
            r = int(p.mesh.face_right[fid])
            if r >= 0:
                need.add(r)
    f = {i: TtTensor(*p.f0.get(i)) for i in need}
    t = time.perf_counter()
    solver.step(f, p.dt, p.eps, p.cap, cells=list(cells))
    return time.perf_counter() - t


def cpu_oracle_rate(cfg, scale, ncells: int, workers: int, repeats: int = 1):
    """Cell-steps/s of the oracle on a sample of the workload's cells: each
    worker steps a strip of `ncells` consecutive cells (with the fluxes of
    every face they touch) from the workload's initial state."""
    import multiprocessing as mp
    from paper_1912_04582_b200.problems import config
    p = config(cfg, scale)
    strips = [list(range(w * ncells, (w + 1) * ncells)) for w in range(workers)]
    strips = [[c % p.mesh.ncell for c in s] for s in strips]
    ctxm = mp.get_context("spawn")
    times = []
    warm = sorted({c for st in strips for c in st})
    with ctxm.Pool(workers, initializer=_ref_worker_init, initargs=((cfg, scale, warm),)) as pool:
        pool.map(_ref_task, strips)  # warm: imports and the strips' face factors
        for _ in range(repeats):
            t = time.perf_counter()
            pool.map(_ref_task, strips)
            times.append(time.perf_counter() - t)
    return workers * ncells / min(times), times


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_1912_04582_b200.problems import config
    p = config(args.config, args.scale)
    workers = os.cpu_count() or 1
    per = 2
    import multiprocessing as mp
    from paper_1912_04582_b200.problems import config as _c  # noqa: F401
    strips = [[(w * per + k) % p.mesh.ncell for k in range(per)] for w in range(workers)]
    ctxm = mp.get_context("spawn")
    warm = sorted({c for st in strips for c in st})
    with ctxm.Pool(workers, initializer=_ref_worker_init,
                   initargs=((args.config, args.scale, warm),)) as pool:
        pool.map(_ref_task, [[0]] * workers)
        for _ in range(args.warmup):
            pool.map(_ref_task, strips)
        t = time.perf_counter()
        for _ in range(args.steps):
            pool.map(_ref_task, strips)
        el = time.perf_counter() - t
    value = workers * per * args.steps / el
    line = {"impl": "reference", "metric": "cell-steps/s", "value": value, "unit": "cell-steps/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(p, args),
            "cpu_baseline": {"value": value, "unit": "cell-steps/s", "cores": workers,
                             "kind": "port",
                             "sample": f"{workers} processes x {per} cells of the workload per "
                                       "step (faces they touch included), numpy oracle, 1 BLAS "
                                       "thread each, face factors set up before timing"},
            "e2e": {"value": value, "unit": "cell-steps/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


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
def main():
    args = parse()
    if args.e2e_steps <= 0:
        args.e2e_steps = args.steps
    if args.config == 3:
        run_config3(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
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
        ctx.set_owned(part.n_owned)
        f_local = local_state(part, pg.f0)
        ctx.upload_state(f_local)
        pack, unpack = halo.gpu_pack_unpack(ctx, torch.device("cuda", local))
        p = pg
        cells_per_rank = part.n_owned
    else:
        ctx.setup(p)
        f_local = p.f0
        cells_per_rank = p.mesh.ncell
    t0 = time.perf_counter()
    ctx.step(p.dt, p.eps, p.cap, 0)  # face factors, wall set-up, summand lists
    setup["face_factors_s"] = round(time.perf_counter() - t0, 2)
    setup.update({k: v for k, v in ctx.setup_info().items() if k != "face_factor_ms"})
    fp64_peak = ctx.fp64_peak()

    def run_steps(k):
        if part is None:
            return ctx.timed_step(p.dt, p.eps, p.cap, k)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(k):
            ctx.step(p.dt, p.eps, p.cap, 1)
            halo.exchange(part, pack, unpack, p.nv, device=torch.device("cuda", local))
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1)

    run_steps(args.warmup)
    ctx.upload_state(f_local)  # time steps 1..K from the initial state
    ctx.set_profiling(True)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        ms = run_steps(args.steps)
    torch.cuda.synchronize()
    phase_ms = ctx.phase_times()
    flops, bytes_, launches = ctx.phase_work()
    gpu_launches = ctx.launch_count()
    setup["cell_blocks"] = ctx.setup_info()["cell_blocks"]  # grown on out-of-memory
    st = ctx.download_state()
    max_rank = int(st.ranks.max())
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = ncell_total * args.steps / (ms / 1e3)

    # e2e through the public API with host buffers: upload state, one step,
    # download state -- every step
    ctx.set_profiling(False)
    # (the host state advances: steps 1..E from the initial state, as timed)
    # pinned host buffer for the state's cores (the ranks / offsets arrays
    # are small); the initial state is copied in before the timed region
    from paper_1912_04582_b200.tt_batch import TtBatch
    pinned = torch.empty(max(2 * f_local.cores.size, 1 << 20), dtype=torch.float64,
                         pin_memory=True).numpy()
    pinned[:f_local.cores.size] = f_local.cores
    host = TtBatch(f_local.n1, f_local.n2, f_local.n3, f_local.ranks, f_local.offsets,
                   pinned[:f_local.cores.size])
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    h2d = d2h = 0
    for _ in range(args.e2e_steps):
        h2d += int(host.cores.nbytes + host.ranks.nbytes + host.offsets.nbytes)
        ctx.upload_state(host)
        ctx.step(p.dt, p.eps, p.cap, 1)
        if part is not None:
            halo.exchange(part, pack, unpack, p.nv, device=torch.device("cuda", local))
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

    # roofline of the dominant kernel (the rounding phase with most time)
    names = ["moments", "shakhov_build", "round_fs", "round_collision", "round_flux",
             "round_residual", "round_update", "bookkeeping"]
    dom = int(np.argmax(phase_ms[2:7])) + 2
    dom_s = phase_ms[dom] / 1e3
    achieved = flops[dom] / dom_s / 1e12 if dom_s > 0 else 0.0
    # ncu DRAM bytes per rounded output of this phase (profiles/traffic.json),
    # times the phase's outputs per launch in this run
    per_out = traffic_from_profiles().get(names[dom] + "_bytes_per_output")
    nface_local = (part.mesh if part is not None else p.mesh).nface
    outs_per_step = {"round_flux": nface_local}.get(names[dom], cells_per_rank)
    traffic = (per_out * outs_per_step * args.steps / max(1, launches[dom]) if per_out else None)
    roofline = {"bound": "fp64", "kernel": f"round_gram_kernel ({names[dom]})",
                "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak if fp64_peak else None,
                "peak_source": "measured on this GPU by the DFMA probe in libttdvm_cuda.so",
                "flops_per_launch": flops[dom] / max(1, launches[dom]),
                "launch_ms": phase_ms[dom] / max(1, launches[dom]),
                "algorithmic_bytes_per_launch": bytes_[dom] / max(1, launches[dom]),
                "hbm_frac": (bytes_[dom] / dom_s / 1e9) / load_peaks().get("hbm_gbs", 6547.8)
                if dom_s > 0 else None,
                "traffic": traffic,
                "phase_ms": {names[i]: round(float(phase_ms[i]), 3) for i in range(8)},
                "phase_tflops": {names[i]: round(float(flops[i] / (phase_ms[i] / 1e3) / 1e12), 4)
                                 for i in range(2, 7) if phase_ms[i] > 0}}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        ncells = 2
        rate, times = cpu_oracle_rate(args.config, args.scale, ncells, 1)
        cpu = {"value": rate, "unit": "cell-steps/s", "cores": 1, "kind": "port",
               "sample": f"{ncells} cells of the workload, one step from the initial state, "
                         "numpy oracle (oracle/step.py), 1 process, 1 BLAS thread"}
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
                               cells_total=ncell_total, cells_per_gpu=cells_per_rank,
                               max_rank_after=max_rank, setup_s=setup),
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": {"value": e2e_value, "unit": "cell-steps/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "steps": args.e2e_steps},
                "gpu_launches": gpu_launches, "clocks": clk.summary()}
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
