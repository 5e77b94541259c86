"""Multi-rank path on CPU: slab partition + halo plan, and a world-size-2
gloo run of the partitioned explicit step (CPU oracle as the per-rank
compute, the product's halo.exchange as the communication) that must
reproduce the single-rank oracle step."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1912_04582_b200.mesh import (obstacle_mesh, rcb_partition, slab_partition,
                                        structured_box)
from paper_1912_04582_b200.partition import build_part


@pytest.mark.parametrize("kind,nparts", [("slab", 2), ("slab", 3), ("rcb", 2), ("rcb", 5)])
def test_halo_plan_is_consistent(kind, nparts):
    if kind == "slab":
        mesh = structured_box(6, 3, 2, periodic=(True, True, True))
        owner = slab_partition(mesh, nparts)
    else:  # config 4's shuffled obstacle mesh, recursive coordinate bisection
        mesh = obstacle_mesh((8, 6, 5), hole=2, seed=3)
        owner = rcb_partition(mesh.centroids, nparts)
        assert np.bincount(owner).max() - np.bincount(owner).min() <= 1
    parts = [build_part(mesh, owner, r) for r in range(nparts)]
    for p in parts:
        l2g = p.local_to_global
        assert np.all(owner[p.owned] == p.rank)
        assert np.all(owner[p.ghosts] != p.rank)
        for q, ids in p.send.items():
            sent = l2g[ids]
            got = parts[q].local_to_global[parts[q].recv[p.rank]]
            assert np.array_equal(sent, got)
        # owned cells see the same faces, same signs, same order as globally
        for lc in range(p.n_owned):
            gc = p.owned[lc]
            mine = [(int(p.face_global[f]), s) for f, s in p.mesh.cell_faces(lc)]
            assert mine == mesh.cell_faces(gc)
        assert sum(len(v) for v in p.recv.values()) == len(p.ghosts)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem(kind):
    from paper_1912_04582_b200.problems import obstacle_flow, periodic_box
    if kind == "slab":
        p = periodic_box((4, 2, 1), steps=2)
        return p, slab_partition(p.mesh, 2)
    p = obstacle_flow((4, 3, 3), hole=1, nv=8, seed=5)
    return p, rcb_partition(p.mesh.centroids, 2)


def _worker(rank, world, port, out, kind):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.step import OracleSolver
    from oracle.tt import TtTensor
    from paper_1912_04582_b200 import halo
    from paper_1912_04582_b200.tt_batch import TtBatch

    p, owner = _problem(kind)
    part = build_part(p.mesh, owner, rank)
    solver = OracleSolver(part.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = [TtTensor(*p.f0.get(int(g))) for g in part.local_to_global]

    def pack(ids):
        b = TtBatch.from_list([f[i] for i in ids])
        return b.ranks.ravel(), b.offsets, torch.from_numpy(b.cores.copy())

    def unpack(ids, ranks, offs, cores):
        b = TtBatch(p.nv, p.nv, p.nv, ranks.reshape(-1, 2), offs, cores.numpy())
        for k, i in enumerate(ids):
            f[int(i)] = TtTensor(*b.get(k))

    for _ in range(2):
        new, _ = solver.step(f, p.dt, p.eps, p.cap, cells=range(part.n_owned))
        f[:part.n_owned] = new
        halo.exchange(part, pack, unpack, p.nv, device="cpu")
    out[rank] = {int(part.owned[i]): f[i].to_full() for i in range(part.n_owned)}
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["slab", "rcb"])
def test_gloo_two_ranks_match_single_rank(kind):
    from oracle.step import OracleSolver
    from oracle.tt import TtTensor, rel_err

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), out, kind), nprocs=world, join=True,
                       start_method="spawn")
    p, _ = _problem(kind)
    solver = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = [TtTensor(*p.f0.get(i)) for i in range(p.mesh.ncell)]
    for _ in range(2):
        f, _ = solver.step(f, p.dt, p.eps, p.cap)
    seen = 0
    for r in range(world):
        for g, full in out[r].items():
            assert rel_err(full, f[g].to_full()) < 1e-13
            seen += 1
    assert seen == p.mesh.ncell
