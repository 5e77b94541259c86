"""CPU tests of the mesh layer the step consumes (SURVEY.md §8(a) T21,
§8(f) N2): the build_mesh restatement (proj/src/mesh.cpp:76-196) on the
reference's own known answers (proj/tests/test_mesh.cpp:66-115) and on
config 4's jittered, shuffled obstacle mesh."""
import numpy as np
import pytest

from paper_1912_04582_b200.mesh import HEX_FACES, build_mesh, obstacle_mesh, structured_box

CUBE = np.array([[0, 0, 0], [1, 0, 0], [1, 1, 0], [0, 1, 0],
                 [0, 0, 1], [1, 0, 1], [1, 1, 1], [0, 1, 1]], dtype=np.float64)


def test_single_unit_cube_full_geometry():
    """test_mesh.cpp:66-88: volume 1, six unit boundary faces with axis
    normals pointing out, closed surface."""
    m = build_mesh(CUBE, np.arange(8)[None, :], lambda fv: np.zeros(fv.shape[0]), ["all"])
    assert m.ncell == 1 and m.nface == 6
    assert m.cell_volume[0] == pytest.approx(1.0, rel=1e-14)
    assert np.allclose(m.face_area, 1.0, rtol=1e-14)
    assert np.allclose(np.abs(m.face_normal).max(axis=1), 1.0, rtol=1e-14)
    assert np.all(m.face_right == -1) and np.all(m.face_group >= 0)
    closure = (m.face_area[:, None] * m.face_normal).sum(axis=0)
    assert np.linalg.norm(closure) < 1e-12
    # outward: the normal points away from the cell centre
    centre = CUBE.mean(axis=0)
    for f, q in enumerate(HEX_FACES):
        fc = CUBE[list(q)].mean(axis=0)
        assert np.dot(m.face_normal[f], fc - centre) > 0


def test_two_cells_share_one_interior_face():
    """test_mesh.cpp:90-115: left = 0, right = 1, signs +1 / -1."""
    v = np.concatenate([CUBE, CUBE[4:] + [0, 0, 1]])
    cells = np.array([[0, 1, 2, 3, 4, 5, 6, 7], [4, 5, 6, 7, 8, 9, 10, 11]])
    m = build_mesh(v, cells, lambda fv: np.zeros(fv.shape[0]), ["all"])
    interior = np.nonzero(m.face_right >= 0)[0]
    assert interior.size == 1
    f = int(interior[0])
    assert m.face_left[f] == 0 and m.face_right[f] == 1
    assert dict(m.cell_faces(0))[f] == 1 and dict(m.cell_faces(1))[f] == -1
    assert m.cell_volume.sum() == pytest.approx(2.0, rel=1e-12)


def test_build_mesh_matches_structured_box():
    """The unique-face build of a structured box gives the same geometry as
    the direct structured generator (face ids differ, the face set not)."""
    nx, ny, nz = 3, 2, 2
    m0 = structured_box(nx, ny, nz, periodic=(False, False, False))
    vid = lambda i, j, k: i + (nx + 1) * (j + (ny + 1) * k)  # noqa: E731
    ii, jj, kk = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1),
                             indexing="ij")
    xyz = np.zeros(((nx + 1) * (ny + 1) * (nz + 1), 3))
    xyz[vid(ii, jj, kk).ravel()] = np.stack([ii, jj, kk], -1).reshape(-1, 3)
    cells = []
    for k in range(nz):
        for j in range(ny):
            for i in range(nx):
                cells.append([vid(i, j, k), vid(i + 1, j, k), vid(i + 1, j + 1, k),
                              vid(i, j + 1, k), vid(i, j, k + 1), vid(i + 1, j, k + 1),
                              vid(i + 1, j + 1, k + 1), vid(i, j + 1, k + 1)])
    m = build_mesh(xyz, np.array(cells), lambda fv: np.zeros(fv.shape[0]), ["all"])
    assert m.nface == m0.nface
    assert np.allclose(m.cell_volume, 1.0)

    def key(mm):
        return sorted((int(l), int(r), tuple(np.round(n, 12))) for l, r, n in
                      zip(mm.face_left, mm.face_right, mm.face_normal))
    assert key(m) == key(m0)


def test_obstacle_mesh_config4_counts_and_geometry():
    m = obstacle_mesh((10, 8, 6), hole=2, seed=1)
    assert m.ncell == 10 * 8 * 6 - 8
    nf_expected = (11 * 8 * 6 + 10 * 9 * 6 + 10 * 8 * 7) - 3 * 2 * 2 * 1  # minus faces inside the hole
    assert m.nface == nf_expected
    g = np.bincount(m.face_group[m.face_group >= 0], minlength=3)
    assert g[0] == 8 * 6 and g[2] == 6 * 2 * 2 and g[1] == 2 * (10 * 8 + 10 * 6 + 8 * 6) - 8 * 6
    # the outer box is not jittered: its volume is exact minus the (jittered) hole
    assert 0.7 * 8 < 10 * 8 * 6 - m.cell_volume.sum() < 1.3 * 8
    assert np.allclose(np.linalg.norm(m.face_normal, axis=1), 1.0, atol=1e-14)
    # closed surface per cell with the vector area (mesh.cpp:171-181)
    s = np.zeros((m.ncell, 3))
    for c in range(m.ncell):
        for f, sg in m.cell_faces(c):
            s[c] += sg * m.face_area[f] * m.face_normal[f]
    assert np.abs(s).max() < 1e-12
    # interior faces are oblique (every node off the outer box is jittered)
    inner = m.face_right >= 0
    assert np.all((np.abs(m.face_normal[inner]) < 1.0 - 1e-9).all(axis=1))


def test_reference_area_fails_closed_surface_on_jittered_quads():
    """Recorded deviation: the reference's scalar-sum area
    |t1| + |t2| breaks its own closed-surface identity on non-planar quads,
    so the jittered config-4 mesh uses the vector-area magnitude."""
    with pytest.raises(RuntimeError, match="closed-surface"):
        from paper_1912_04582_b200 import mesh as M
        rng = np.random.default_rng(0)
        v = np.concatenate([CUBE, CUBE[4:] + [0, 0, 1]])
        v[4:8] += rng.uniform(-0.1, 0.1, size=(4, 3))
        cells = np.array([[0, 1, 2, 3, 4, 5, 6, 7], [4, 5, 6, 7, 8, 9, 10, 11]])
        M.build_mesh(v, cells, lambda fv: np.zeros(fv.shape[0]), ["all"], area="reference")


def test_obstacle_mesh_is_seeded():
    a = obstacle_mesh((6, 5, 4), hole=2, seed=7)
    b = obstacle_mesh((6, 5, 4), hole=2, seed=7)
    assert np.array_equal(a.face_normal, b.face_normal)
    assert np.array_equal(a.cell_face_id, b.cell_face_id)
