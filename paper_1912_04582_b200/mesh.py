"""Host-side mesh arrays consumed by the step.

The reference's ``UnstructuredMesh`` (proj/include/ttdvm/mesh.hpp:15-41) is
built by ``build_mesh`` (proj/src/mesh.cpp:76-196) from StarCD files; the
step only consumes its face list (area, unit normal pointing out of
``left``, left, right = -1 on boundary faces, group), cell volumes and the
per-cell (face, sign) lists, sign = +1 iff the stored normal points out of
the cell.  This module produces exactly those arrays, flattened for the C
ABI, for the synthetic structured meshes of BASELINE.json's configs, plus
periodic face pairing (absent in the reference):

* a periodic face is stored once, with ``left`` = the cell on the high side
  of the box, ``right`` = its partner on the low side, normal = +axis and
  group -1 (it is an interior face for the step);
* a periodic axis with a single cell would pair a cell with itself; its
  flux enters that cell's residual once with each sign and cancels exactly,
  so such faces are omitted (identically in the oracle and the GPU path).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


@dataclass
class Mesh:
    ncell: int
    nface: int
    face_left: np.ndarray      # int32 [nface]
    face_right: np.ndarray     # int32 [nface], -1 = boundary
    face_group: np.ndarray     # int32 [nface], -1 = interior / periodic
    face_area: np.ndarray      # f64 [nface]
    face_normal: np.ndarray    # f64 [nface, 3], unit, out of left
    cell_volume: np.ndarray    # f64 [ncell]
    cell_face_off: np.ndarray  # int64 [ncell + 1]
    cell_face_id: np.ndarray   # int32 [sum]
    cell_face_sign: np.ndarray  # int8 [sum]
    group_names: list = field(default_factory=list)
    shape: tuple = ()          # (nx, ny, nz) for structured meshes
    cell_ijk: np.ndarray | None = None  # int32 [ncell, 3]

    def cell_faces(self, c: int):
        a, b = int(self.cell_face_off[c]), int(self.cell_face_off[c + 1])
        return list(zip(self.cell_face_id[a:b].tolist(), self.cell_face_sign[a:b].tolist()))

    def min_cell_size(self) -> float:
        return float(np.min(self.cell_volume) ** (1.0 / 3.0))


def _finish(ncell, left, right, group, area, normal, volumes, group_names, shape, ijk) -> Mesh:
    nface = int(left.shape[0])
    left = np.ascontiguousarray(left, dtype=np.int32)
    right = np.ascontiguousarray(right, dtype=np.int32)
    # per-cell (face, sign) lists sorted by face id
    owners = np.concatenate([left, right[right >= 0]])
    fids = np.concatenate([np.arange(nface, dtype=np.int32),
                           np.nonzero(right >= 0)[0].astype(np.int32)])
    signs = np.concatenate([np.ones(nface, dtype=np.int8),
                            -np.ones(int((right >= 0).sum()), dtype=np.int8)])
    order = np.lexsort((fids, owners))
    owners, fids, signs = owners[order], fids[order], signs[order]
    off = np.zeros(ncell + 1, dtype=np.int64)
    np.cumsum(np.bincount(owners, minlength=ncell), out=off[1:])
    return Mesh(ncell, nface, left, right, np.ascontiguousarray(group, dtype=np.int32),
                np.ascontiguousarray(area, dtype=np.float64),
                np.ascontiguousarray(normal, dtype=np.float64).reshape(nface, 3),
                np.asarray(volumes, dtype=np.float64), off,
                np.ascontiguousarray(fids), np.ascontiguousarray(signs),
                list(group_names), tuple(shape), ijk)


def structured_box(nx: int, ny: int, nz: int, h: float = 1.0,
                   periodic=(True, True, True)) -> Mesh:
    """Box of nx*ny*nz cubes of edge h; cell id = i + nx*(j + ny*k).

    Non-periodic sides become boundary groups named ``xmin``, ``xmax``,
    ``ymin`` ... (boundary normals point out of the domain, reference
    convention proj/include/ttdvm/mesh.hpp:15-22).  Faces are ordered by
    axis, then by cell id; a low-side boundary face follows the high-side
    face of the same cell.
    """
    dims = (nx, ny, nz)
    ncell = nx * ny * nz
    ijk = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz),
                               indexing="ij"), axis=-1).transpose(2, 1, 0, 3).reshape(-1, 3)
    ijk = ijk.astype(np.int32)
    cid = np.arange(ncell, dtype=np.int64)
    stride = (1, nx, nx * ny)
    group_names = []
    gid = {}
    for ax, name in enumerate("xyz"):
        if not periodic[ax]:
            for side in ("min", "max"):
                gid[(ax, side)] = len(group_names)
                group_names.append(name + side)
    L, R, G, N = [], [], [], []
    for ax in range(3):
        nrm = np.zeros(3)
        nrm[ax] = 1.0
        pos = ijk[:, ax]
        # key orders faces: (cell, 0 = high side, 1 = low boundary side)
        keys, l_, r_, g_, n_ = [], [], [], [], []
        inner = pos + 1 < dims[ax]
        keys.append(cid[inner] * 2)
        l_.append(cid[inner]); r_.append(cid[inner] + stride[ax])
        g_.append(np.full(int(inner.sum()), -1)); n_.append(np.tile(nrm, (int(inner.sum()), 1)))
        top = pos + 1 == dims[ax]
        if periodic[ax]:
            if dims[ax] > 1:
                keys.append(cid[top] * 2)
                l_.append(cid[top]); r_.append(cid[top] - (dims[ax] - 1) * stride[ax])
                g_.append(np.full(int(top.sum()), -1)); n_.append(np.tile(nrm, (int(top.sum()), 1)))
        else:
            keys.append(cid[top] * 2)
            l_.append(cid[top]); r_.append(np.full(int(top.sum()), -1))
            g_.append(np.full(int(top.sum()), gid[(ax, "max")])); n_.append(np.tile(nrm, (int(top.sum()), 1)))
            bot = pos == 0
            keys.append(cid[bot] * 2 + 1)
            l_.append(cid[bot]); r_.append(np.full(int(bot.sum()), -1))
            g_.append(np.full(int(bot.sum()), gid[(ax, "min")])); n_.append(np.tile(-nrm, (int(bot.sum()), 1)))
        k = np.concatenate(keys)
        o = np.argsort(k, kind="stable")
        L.append(np.concatenate(l_)[o]); R.append(np.concatenate(r_)[o])
        G.append(np.concatenate(g_)[o]); N.append(np.concatenate(n_)[o])
    left = np.concatenate(L); right = np.concatenate(R)
    group = np.concatenate(G); normal = np.concatenate(N)
    area = np.full(left.shape[0], h * h)
    return _finish(ncell, left, right, group, area, normal, np.full(ncell, h ** 3),
                   group_names, dims, ijk)


def slab_partition(mesh: Mesh, nparts: int) -> np.ndarray:
    """Owner rank per cell: contiguous x-slabs (configs 2 and 5, SURVEY.md
    §8(e)).  Returns int32 [ncell]."""
    nx = mesh.shape[0]
    bounds = [(p * nx) // nparts for p in range(nparts + 1)]
    owner = np.zeros(mesh.ncell, dtype=np.int32)
    xi = mesh.cell_ijk[:, 0]
    for p in range(nparts):
        owner[(xi >= bounds[p]) & (xi < bounds[p + 1])] = p
    return owner
