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
    centroids: np.ndarray | None = None  # f64 [ncell, 3] (vertex mean, mesh.cpp:124-126)

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


# Local faces of a hexahedron in StarCD/VTK vertex order (0-3 bottom, 4-7
# top), each quad wound so its normal points out of the cell
# (proj/src/mesh.cpp:19-26).
HEX_FACES = ((0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (1, 2, 6, 5), (2, 3, 7, 6), (3, 0, 4, 7))


def _tri_vectors(p0, p1, p2, p3):
    """Vector areas of the two triangles (p0, p1, p2), (p0, p2, p3)
    (quad_geometry, proj/src/mesh.cpp:33-39)."""
    t1 = 0.5 * np.cross(p1 - p0, p2 - p0)
    t2 = 0.5 * np.cross(p2 - p0, p3 - p0)
    return t1, t2


def build_mesh(vertices: np.ndarray, cells: np.ndarray, face_group_fn=None,
               group_names=(), area: str = "reference") -> Mesh:
    """Unique-face build of ``build_mesh`` (proj/src/mesh.cpp:76-196),
    vectorised over cells.

    Cells are visited in order and their local faces in HEX_FACES order; a
    face's id is its first-discovery index, ``left`` the discovering cell
    (its winding gives the normal, pointing out of ``left``), ``right`` the
    second cell or -1.  Area and unit normal come from the two-triangle
    split; the volume from the divergence theorem over each cell's own
    outward triangulation; every cell must pass the closed-surface identity
    |sum s A n| <= 1e-10 sum A (mesh.cpp:171-181).

    ``area`` = "reference" takes the scalar sum |t1| + |t2| (mesh.cpp:38),
    "vector" the vector-area magnitude |t1 + t2|.  They agree on planar
    quads; on the non-planar quads of a jittered mesh only "vector" passes
    the reference's own closed-surface identity (DESIGN.md records this).
    ``face_group_fn(face_vertex_ids) -> int32 group per boundary face``
    tags the boundary faces (the reference matches boundary quads by their
    sorted vertex keys, mesh.cpp:183-195).
    """
    vertices = np.asarray(vertices, dtype=np.float64)
    cells = np.asarray(cells, dtype=np.int64)
    nc = cells.shape[0]
    nvtx = vertices.shape[0]
    if np.any(cells < 0) or np.any(cells >= nvtx):
        raise RuntimeError("cell references missing vertex")
    s = np.sort(cells, axis=1)
    if np.any(s[:, 1:] == s[:, :-1]):
        raise RuntimeError("cell is degenerate (repeated vertex)")
    quads = cells[:, np.array(HEX_FACES)].reshape(-1, 4)          # slot = 6 c + lf
    keys = np.sort(quads, axis=1)
    k1 = keys[:, 0] * nvtx + keys[:, 1]
    k2 = keys[:, 2] * nvtx + keys[:, 3]
    order = np.lexsort((k2, k1))                                  # stable: slots ascending
    k1s, k2s = k1[order], k2[order]
    new = np.ones(order.size, dtype=bool)
    new[1:] = (k1s[1:] != k1s[:-1]) | (k2s[1:] != k2s[:-1])
    grp = np.cumsum(new) - 1
    counts = np.bincount(grp)
    if np.any(counts > 2):
        raise RuntimeError("face shared by more than two cells")
    first_pos = np.nonzero(new)[0]
    first_slot = order[first_pos]
    fid_of_grp = np.empty(first_slot.size, dtype=np.int64)
    fid_of_grp[np.argsort(first_slot, kind="stable")] = np.arange(first_slot.size)
    face_of_slot = np.empty(order.size, dtype=np.int64)
    face_of_slot[order] = fid_of_grp[grp]
    nface = first_slot.size
    left = np.empty(nface, dtype=np.int64)
    right = np.full(nface, -1, dtype=np.int64)
    fslot = np.empty(nface, dtype=np.int64)
    fslot[fid_of_grp] = first_slot
    left[:] = fslot // 6
    two = counts == 2
    second_slot = order[first_pos[two] + 1]
    right[fid_of_grp[two]] = second_slot // 6
    fq = quads[fslot]
    p = vertices[fq]                                              # (nface, 4, 3)
    t1, t2 = _tri_vectors(p[:, 0], p[:, 1], p[:, 2], p[:, 3])
    avec = t1 + t2
    amag = np.linalg.norm(avec, axis=1)
    if area == "reference":
        ar = np.linalg.norm(t1, axis=1) + np.linalg.norm(t2, axis=1)
    elif area == "vector":
        ar = amag
    else:
        raise ValueError("area must be 'reference' or 'vector'")
    if np.any(~(ar > 0.0)) or np.any(amag <= 0.0):
        raise RuntimeError("cell has a degenerate face")
    normal = avec / amag[:, None]
    # divergence-theorem volume over each cell's outward triangulation
    pc = vertices[quads].reshape(nc, 6, 4, 3)
    c1, c2 = _tri_vectors(pc[:, :, 0], pc[:, :, 1], pc[:, :, 2], pc[:, :, 3])
    vol = (np.einsum("cfx,cfx->c", pc[:, :, 0] + pc[:, :, 1] + pc[:, :, 2], c1) / 9.0
           + np.einsum("cfx,cfx->c", pc[:, :, 0] + pc[:, :, 2] + pc[:, :, 3], c2) / 9.0)
    if np.any(~(vol > 0.0)):
        raise RuntimeError("cell has nonpositive volume (inverted ordering?)")
    # per-cell (face, sign) in HEX_FACES order (mesh.cpp:113-122)
    cf_id = face_of_slot.astype(np.int32)
    cf_sign = np.where(fslot[face_of_slot] == np.arange(order.size), 1, -1).astype(np.int8)
    off = np.arange(0, 6 * nc + 1, 6, dtype=np.int64)
    # closed-surface identity (mesh.cpp:171-181)
    contrib = (cf_sign[:, None] * ar[cf_id][:, None] * normal[cf_id]).reshape(nc, 6, 3).sum(axis=1)
    tot = ar[cf_id].reshape(nc, 6).sum(axis=1)
    bad = np.linalg.norm(contrib, axis=1) > 1e-10 * tot
    if np.any(bad):
        raise RuntimeError(f"cell {int(np.argmax(bad))} fails the closed-surface identity")
    group = np.full(nface, -1, dtype=np.int32)
    bnd = right < 0
    if np.any(bnd):
        if face_group_fn is None:
            raise RuntimeError("boundary face without a boundary tag")
        g = np.asarray(face_group_fn(fq[bnd]), dtype=np.int32)
        if np.any(g < 0):
            raise RuntimeError("boundary face without a boundary tag")
        group[bnd] = g
    return Mesh(nc, nface, left.astype(np.int32), right.astype(np.int32), group, ar, normal,
                vol, off, cf_id, cf_sign, list(group_names), (), None)


def shuffle_faces(mesh: Mesh, rng: np.random.Generator) -> Mesh:
    """Permute face ids (a face keeps its left/right/normal; cell lists are
    remapped in place)."""
    perm = rng.permutation(mesh.nface)          # new id -> old id
    inv = np.empty_like(perm)
    inv[perm] = np.arange(mesh.nface)
    return Mesh(mesh.ncell, mesh.nface, mesh.face_left[perm], mesh.face_right[perm],
                mesh.face_group[perm], mesh.face_area[perm], mesh.face_normal[perm],
                mesh.cell_volume, mesh.cell_face_off, inv[mesh.cell_face_id].astype(np.int32),
                mesh.cell_face_sign, mesh.group_names, mesh.shape, mesh.cell_ijk,
                mesh.centroids)


def rcb_partition(points: np.ndarray, nparts: int) -> np.ndarray:
    """Recursive coordinate bisection: split the
    point set at the median of its longest extent, recursively, into nparts
    (any positive count; parts differ in size by at most one point per
    level).  Returns the owner rank per point (int32)."""
    owner = np.zeros(points.shape[0], dtype=np.int32)

    def split(idx, lo, k):
        if k == 1:
            owner[idx] = lo
            return
        kl = k // 2
        pts = points[idx]
        ax = int(np.argmax(pts.max(axis=0) - pts.min(axis=0)))
        order = idx[np.argsort(pts[:, ax], kind="stable")]
        cut = (order.shape[0] * kl) // k
        split(order[:cut], lo, kl)
        split(order[cut:], lo + kl, k - kl)

    split(np.arange(points.shape[0]), 0, nparts)
    return owner


def obstacle_mesh(shape=(100, 80, 64), hole: int = 8, h: float = 1.0, jitter: float = 0.1,
                  seed: int = 4, shuffle: bool = True) -> Mesh:
    """Config 4's unstructured hex mesh: an nx x ny x nz lattice of cells of
    edge h with a centred hole^3 block of cells removed (a rigid obstacle),
    every node off the outer box jittered by U(-jitter, jitter) h per
    coordinate (seeded), cell order and face order shuffled (seeded).
    Boundary groups: 0 'inlet' (x = 0), 1 'outlet' (the five other outer
    sides), 2 'wall' (the obstacle surface)."""
    nx, ny, nz = shape
    rng = np.random.default_rng(seed)
    vi, vj, vk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1),
                             indexing="ij")
    vi, vj, vk = (a.transpose(2, 1, 0).reshape(-1) for a in (vi, vj, vk))  # id = i + (nx+1)(j + (ny+1)k)
    xyz = np.stack([vi, vj, vk], axis=1).astype(np.float64) * h
    inner = (vi > 0) & (vi < nx) & (vj > 0) & (vj < ny) & (vk > 0) & (vk < nz)
    jit = rng.uniform(-jitter, jitter, size=xyz.shape) * h
    xyz[inner] += jit[inner]
    ci, cj, ck = np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij")
    ci, cj, ck = (a.transpose(2, 1, 0).reshape(-1) for a in (ci, cj, ck))
    lo = (np.array(shape) - hole) // 2
    solid = ((ci >= lo[0]) & (ci < lo[0] + hole) & (cj >= lo[1]) & (cj < lo[1] + hole)
             & (ck >= lo[2]) & (ck < lo[2] + hole))
    ci, cj, ck = ci[~solid], cj[~solid], ck[~solid]

    def vid(i, j, k):
        return i + (nx + 1) * (j + (ny + 1) * k)

    cells = np.stack([vid(ci, cj, ck), vid(ci + 1, cj, ck), vid(ci + 1, cj + 1, ck),
                      vid(ci, cj + 1, ck), vid(ci, cj, ck + 1), vid(ci + 1, cj, ck + 1),
                      vid(ci + 1, cj + 1, ck + 1), vid(ci, cj + 1, ck + 1)], axis=1)
    ijk = np.stack([ci, cj, ck], axis=1).astype(np.int32)
    if shuffle:
        perm = rng.permutation(cells.shape[0])
        cells, ijk = cells[perm], ijk[perm]

    def groups(fv):
        fi, fj, fk = vi[fv], vj[fv], vk[fv]
        g = np.full(fv.shape[0], 2, dtype=np.int32)
        outer = (np.all(fi == 0, axis=1) | np.all(fi == nx, axis=1) | np.all(fj == 0, axis=1)
                 | np.all(fj == ny, axis=1) | np.all(fk == 0, axis=1) | np.all(fk == nz, axis=1))
        g[outer] = 1
        g[np.all(fi == 0, axis=1)] = 0
        return g

    m = build_mesh(xyz, cells, groups, ("inlet", "outlet", "wall"), area="vector")
    m.cell_ijk = ijk
    m.centroids = xyz[cells].mean(axis=1)
    m.shape = tuple(shape)
    if shuffle:
        m = shuffle_faces(m, rng)
    return m
