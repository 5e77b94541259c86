"""The in-library NCCL halo exchange on ONE GPU.

Nothing here makes a kernel wait on another rank.  A 1-rank NCCL
communicator is created inside the library and the context exchanges its
halo WITH ITSELF: the mesh is rank 0's x-slab of a 2-slab periodic box whose
state has the period of one slab, so the ghost cells rank 1 would send are,
cell for cell, copies of rank 0's own cells one period away.  The whole
path runs for real -- dlopen of libnccl, ncclCommInitRank, the grouped
ncclSend/ncclRecv of ranks and cores on the communication stream overlapped
with the collision phases, the ghost placement, the ncclAllReduce of the
status -- and the owned cells must follow the single-rank periodic box."""
import numpy as np
import pytest

from oracle import ref
from oracle.parity import oracle_list
from oracle.step import OracleSolver
from oracle.tt import rel_err
from paper_1912_04582_b200.mesh import slab_partition
from paper_1912_04582_b200.partition import build_part, local_state
from paper_1912_04582_b200.problems import periodic_box
from paper_1912_04582_b200.tt_batch import TtBatch

pytestmark = pytest.mark.gpu


def self_halo_problem(nx=4, ny=2, nz=2):
    small = periodic_box((nx, ny, nz), steps=2)
    big = periodic_box((2 * nx, ny, nz), steps=2)
    key = {tuple(v): i for i, v in enumerate(small.mesh.cell_ijk.tolist())}
    src = np.array([key[(x % nx, y, z)] for x, y, z in big.mesh.cell_ijk.tolist()])
    f_big = small.f0.subset(src)              # period nx along x
    part = build_part(big.mesh, slab_partition(big.mesh, 2), 0)
    gkey = {tuple(v): i for i, v in enumerate(big.mesh.cell_ijk.tolist())}
    g2l = {int(g): l for l, g in enumerate(part.local_to_global)}
    recv = part.recv[1]
    send = []
    for l in recv:                             # the ghost's twin one period away, owned here
        x, y, z = big.mesh.cell_ijk[int(part.local_to_global[int(l)])]
        send.append(g2l[gkey[(int(x) - nx, int(y), int(z))]])
    return small, big, part, f_big, np.array(send, dtype=np.int32), np.asarray(recv, dtype=np.int32)


def test_self_exchange_matches_periodic_box():
    from paper_1912_04582_b200.cuda import Context
    small, big, part, f_big, send, recv = self_halo_problem()
    assert (send < part.n_owned).all() and (recv >= part.n_owned).all()
    c = Context(0)
    c.set_grid(big.nv, big.bound)
    c.set_gas(small.gas)  # (mu_ref is referred to the box length: use the one-slab box's)
    c.set_mesh(part.mesh)
    c.set_bcs(big.bcs)
    c.comm_init(1, 0, Context.nccl_unique_id())
    c.set_partition(part.n_owned, {0: send}, {0: recv})
    f_loc = local_state(part, f_big)
    # stale ghosts on purpose: the exchange at the start of the step must replace them
    stale = f_loc.subset(np.concatenate([np.arange(part.n_owned), np.zeros(len(part.ghosts), int)]))
    c.upload_state(stale)
    steps = 2
    c.step(big.dt, big.eps, big.cap, steps)
    got = c.download_state()
    stats = c.halo_stats()
    assert stats["exchanges"] == steps and stats["bytes_sent"] == stats["bytes_recv"] > 0
    # oracle: the one-slab periodic box on a single rank
    if ref.available():
        r = ref.RefSolver.for_problem(small)
        for _ in range(steps):
            r.step(small.dt, small.eps, small.cap)
        want = r.state()
    else:
        s = OracleSolver(small.mesh, small.nv, small.bound, small.gas, small.bcs)
        f = oracle_list(small.f0)
        for _ in range(steps):
            f, _ = s.step(f, small.dt, small.eps, small.cap)
        want = TtBatch.from_list(f)
    assert big.dt == small.dt
    key = {tuple(v): i for i, v in enumerate(small.mesh.cell_ijk.tolist())}
    for l in range(part.n_owned):
        x, y, z = big.mesh.cell_ijk[int(part.owned[l])]
        w = key[(int(x), int(y), int(z))]
        assert rel_err(got.full(l), want.full(w)) <= 10 * big.eps, l
    c.close()


def test_status_allreduce_reports_failure():
    """A failing step (nonpositive density) still returns through the
    ncclAllReduce of the status code with the reference's error."""
    from paper_1912_04582_b200.cuda import Context
    small, big, part, f_big, send, recv = self_halo_problem()
    c = Context(0)
    c.set_grid(big.nv, big.bound)
    c.set_gas(small.gas)  # (mu_ref is referred to the box length: use the one-slab box's)
    c.set_mesh(part.mesh)
    c.set_bcs(big.bcs)
    c.comm_init(1, 0, Context.nccl_unique_id())
    c.set_partition(part.n_owned, {0: send}, {0: recv})
    bad = local_state(part, f_big)
    bad.cores[:] = -np.abs(bad.cores)          # negative densities
    c.upload_state(bad)
    with pytest.raises(RuntimeError, match="nonpositive"):
        c.step(big.dt, big.eps, big.cap, 1)
    c.close()
