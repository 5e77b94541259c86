"""Spatial partition of the mesh across ranks and the halo plan
(SURVEY.md §8(e)): each rank owns a set of cells; its local mesh holds
every face touching an owned cell plus the neighbouring cells behind cut
faces ("ghosts").  Per step the owners send the current states of those
ghost cells; cut-face fluxes are computed on both sides, so the exchange is
the only communication.

Local numbering: owned cells first (ascending global id), then ghosts
(ascending global id); local faces in ascending global face id, so each
cell's (face, sign) list keeps the global order and a partitioned step adds
the same summands in the same order as the single-rank step.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .mesh import Mesh, _finish
from .tt_batch import TtBatch


@dataclass
class LocalPart:
    rank: int
    nparts: int
    owned: np.ndarray          # global ids of owned cells (local 0..n_owned-1)
    ghosts: np.ndarray         # global ids of ghost cells (local n_owned..)
    mesh: Mesh                 # local mesh
    face_global: np.ndarray    # local face -> global face
    send: dict = field(default_factory=dict)   # peer -> local ids to send (owned)
    recv: dict = field(default_factory=dict)   # peer -> local ids to fill (ghosts)

    @property
    def n_owned(self) -> int:
        return int(self.owned.shape[0])

    @property
    def local_to_global(self) -> np.ndarray:
        return np.concatenate([self.owned, self.ghosts])


def build_part(mesh: Mesh, owner: np.ndarray, rank: int) -> LocalPart:
    owner = np.asarray(owner, dtype=np.int32)
    nparts = int(owner.max()) + 1
    owned = np.nonzero(owner == rank)[0].astype(np.int64)
    own_mask = owner == rank
    L, R = mesh.face_left.astype(np.int64), mesh.face_right.astype(np.int64)
    touch = own_mask[L] | ((R >= 0) & own_mask[np.maximum(R, 0)])
    fids = np.nonzero(touch)[0]
    nb = np.concatenate([L[fids], R[fids][R[fids] >= 0]])
    ghosts = np.unique(nb[~own_mask[nb]])
    loc = np.concatenate([owned, ghosts])
    g2l = -np.ones(mesh.ncell, dtype=np.int64)
    g2l[loc] = np.arange(loc.shape[0])
    lf = g2l[L[fids]]
    rf = np.where(R[fids] >= 0, g2l[np.maximum(R[fids], 0)], -1)
    ijk = mesh.cell_ijk[loc] if mesh.cell_ijk is not None else None
    local = _finish(int(loc.shape[0]), lf, rf, mesh.face_group[fids], mesh.face_area[fids],
                    mesh.face_normal[fids], mesh.cell_volume[loc], mesh.group_names, mesh.shape,
                    ijk)
    if mesh.centroids is not None:
        local.centroids = mesh.centroids[loc]
    # owned cells keep the global (face, sign) order, so a partitioned step
    # adds each cell's summands in the single-rank order (bit-identical sums)
    f2l = -np.ones(mesh.nface, dtype=np.int64)
    f2l[fids] = np.arange(fids.shape[0])
    go = mesh.cell_face_off
    cnt = (go[owned + 1] - go[owned]).astype(np.int64)
    idx = np.repeat(go[owned] - np.cumsum(cnt) + cnt, cnt) + np.arange(int(cnt.sum()))
    lo_ = local.cell_face_off
    nown = owned.shape[0]
    gcnt = np.diff(lo_)[nown:]
    gidx = np.arange(int(lo_[nown]), int(lo_[-1]))
    local.cell_face_id = np.concatenate([f2l[mesh.cell_face_id[idx]],
                                         local.cell_face_id[gidx]]).astype(np.int32)
    local.cell_face_sign = np.concatenate([mesh.cell_face_sign[idx],
                                           local.cell_face_sign[gidx]]).astype(np.int8)
    off = np.zeros(loc.shape[0] + 1, dtype=np.int64)
    np.cumsum(np.concatenate([cnt, gcnt]), out=off[1:])
    local.cell_face_off = off
    part = LocalPart(rank, nparts, owned, ghosts, local, fids)
    # halo plan, both directions sorted by global id (both sides agree)
    for q in range(nparts):
        if q == rank:
            continue
        mine = ghosts[owner[ghosts] == q]                      # I receive these from q
        if mine.size:
            part.recv[q] = g2l[np.sort(mine)].astype(np.int32)
        # cells I own that are ghosts on q: owned cells adjacent to q's cells
        q_mask = owner == q
        tq = (own_mask[L] & (R >= 0) & q_mask[np.maximum(R, 0)]) | \
             ((R >= 0) & own_mask[np.maximum(R, 0)] & q_mask[L])
        cand = np.concatenate([L[tq], R[tq]])
        cand = np.unique(cand[own_mask[cand]])
        if cand.size:
            part.send[q] = g2l[cand].astype(np.int32)
    return part


def local_state(part: LocalPart, f: TtBatch) -> TtBatch:
    """The global state restricted to the local cells, in local order."""
    return f.subset(part.local_to_global)


def weak_scaling_mesh(shape_per_rank, nparts: int):
    """Global periodic box of nparts slabs along x, each shape_per_rank."""
    from .mesh import structured_box
    nx, ny, nz = shape_per_rank
    return structured_box(nx * nparts, ny, nz, periodic=(True, True, True))
