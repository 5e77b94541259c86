"""ctypes front of the COMPILED reference oracle (oracle/_ref/libttdvm_ref.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU legs (cpu_baseline / --impl reference), never by the product
package.  The library is the unmodified reference C++ (proj/src/*.cpp)
compiled by oracle/build_ref.py against the repo's Eigen/doctest subsets,
gated on the reference's own 50 unit tests, plus oracle/ref_step.cpp (the
explicit step S1 composed of reference API calls).

On the GPU box /root/reference is absent; the prebuilt .so travels with the
snapshot.  ``available()`` says whether it can be loaded.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libttdvm_ref.so")
BC_KIND = {"wall": 0, "sym-x": 1, "sym-y": 2, "sym-z": 3, "in": 4, "out": 5}

_lib = None


class _Batch(C.Structure):
    _fields_ = [("count", C.c_int32), ("n1", C.c_int32), ("n2", C.c_int32), ("n3", C.c_int32),
                ("ranks", C.c_void_p), ("offsets", C.c_void_p), ("cores", C.c_void_p)]


class _Bc(C.Structure):
    _fields_ = [("kind", C.c_int32), ("wall_temperature", C.c_double), ("free_n", C.c_double),
                ("free_t", C.c_double), ("free_u", C.c_double * 3)]


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def available() -> bool:
    try:
        lib()
        return True
    except OSError:
        return False


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) and os.path.isdir("/root/reference/proj"):
            from oracle import build_ref
            build_ref.build()
        L = C.CDLL(LIB_PATH)
        vp, i32, dbl = C.c_void_p, C.c_int32, C.c_double
        sig = {
            "ttref_create": (vp, [C.c_int, dbl, vp]),
            "ttref_destroy": (None, [vp]),
            "ttref_last_error": (C.c_char_p, [vp]),
            "ttref_set_threads": (C.c_int, [vp, C.c_int]),
            "ttref_set_mesh": (C.c_int, [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
            "ttref_set_bcs": (C.c_int, [vp, i32, vp]),
            "ttref_set_state": (C.c_int, [vp, vp]),
            "ttref_step": (C.c_int, [vp, dbl, dbl, i32, i32, vp]),
            "ttref_lusgs_step": (C.c_int, [vp, dbl, dbl, i32]),
            "ttref_times": (C.c_int, [vp, vp]),
            "ttref_layout": (C.c_int, [vp, i32, vp, vp, vp]),
            "ttref_download": (C.c_int, [vp, i32, vp]),
            "ttref_macros": (C.c_int, [vp, vp]),
            "ttref_round_sums": (C.c_int, [vp, vp, i32, vp, vp, dbl, i32]),
            "ttref_compute_macro": (C.c_int, [vp, vp, vp]),
            "ttref_collision": (C.c_int, [vp, vp, dbl]),
            "ttref_face_factors": (C.c_int, [vp, i32, vp, i32, i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _batch(b):
    s = _Batch(b.count, b.n1, b.n2, b.n3, _ptr(b.ranks), _ptr(b.offsets), _ptr(b.cores))
    return s


class RefSolver:
    """The reference's S1 step on one mesh (oracle/ref_step.cpp)."""

    STATE, PHI, J, R, RESULT = 0, 1, 2, 3, 4

    def __init__(self, nv: int, bound: float, gas, mesh=None, bcs=None, threads: int = 0):
        self.L = lib()
        self._gas = np.ascontiguousarray(gas, dtype=np.float64)
        self.h = self.L.ttref_create(int(nv), float(bound), _ptr(self._gas))
        self.nv = int(nv)
        self._check(0)
        if threads:
            self.set_threads(threads)
        if mesh is not None:
            self.set_mesh(mesh)
        if bcs is not None:
            self.set_bcs(bcs)

    @classmethod
    def for_problem(cls, p, threads: int = 0) -> "RefSolver":
        s = cls(p.nv, p.bound, p.gas, p.mesh, p.bcs, threads)
        s.set_state(p.f0)
        return s

    def _check(self, rc: int):
        if rc == 0:
            msg = self.L.ttref_last_error(self.h).decode()
            if msg:
                raise RuntimeError(msg)
            return
        msg = self.L.ttref_last_error(self.h).decode()
        raise (ValueError if rc == 1 else RuntimeError)(msg)

    def close(self):
        if self.h:
            self.L.ttref_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_threads(self, n: int):
        self._check(self.L.ttref_set_threads(self.h, int(n)))

    def set_mesh(self, m):
        self.mesh = m
        self._keep = [np.ascontiguousarray(a) for a in (
            m.face_left.astype(np.int32), m.face_right.astype(np.int32),
            m.face_group.astype(np.int32), m.face_area.astype(np.float64),
            m.face_normal.astype(np.float64), m.cell_volume.astype(np.float64),
            m.cell_face_off.astype(np.int64), m.cell_face_id.astype(np.int32),
            m.cell_face_sign.astype(np.int8))]
        self._check(self.L.ttref_set_mesh(self.h, m.ncell, m.nface, *(_ptr(a) for a in self._keep)))

    def set_bcs(self, bcs):
        arr = (_Bc * max(1, len(bcs)))()
        for g, bc in enumerate(bcs):
            arr[g].kind = BC_KIND[bc["kind"]]
            arr[g].wall_temperature = float(bc.get("t_wall", 0.0))
            arr[g].free_n = float(bc.get("n", 0.0))
            arr[g].free_t = float(bc.get("t", 0.0))
            u = bc.get("u", (0.0, 0.0, 0.0))
            for a in range(3):
                arr[g].free_u[a] = float(u[a])
        self._check(self.L.ttref_set_bcs(self.h, len(bcs), C.cast(arr, C.c_void_p)))

    def set_state(self, b):
        s = _batch(b)
        self._check(self.L.ttref_set_state(self.h, C.byref(s)))

    def step(self, dt: float, eps: float, cap: int = 0, cells=None):
        if cells is None:
            self._check(self.L.ttref_step(self.h, dt, eps, cap, 0, None))
        else:
            c = np.ascontiguousarray(cells, dtype=np.int32)
            self._check(self.L.ttref_step(self.h, dt, eps, cap, len(c), _ptr(c)))

    def lusgs_step(self, dt: float, eps: float, cap: int = 0):
        """One LU-SGS iteration over every cell (oracle/ref_step.cpp lusgs)."""
        self._check(self.L.ttref_lusgs_step(self.h, dt, eps, cap))

    def times(self):
        t = np.zeros(2)
        self._check(self.L.ttref_times(self.h, _ptr(t)))
        return float(t[0]), float(t[1])

    def fetch(self, which: int):
        from paper_1912_04582_b200.tt_batch import TtBatch
        cnt = C.c_int32(0)
        self._check(self.L.ttref_layout(self.h, which, C.byref(cnt), None, None))
        n = cnt.value
        ranks = np.zeros(2 * max(n, 1), dtype=np.int32)
        offs = np.zeros(n + 1, dtype=np.int64)
        self._check(self.L.ttref_layout(self.h, which, None, _ptr(ranks), _ptr(offs)))
        cores = np.zeros(max(1, int(offs[-1])), dtype=np.float64)
        self._check(self.L.ttref_download(self.h, which, _ptr(cores)))
        return TtBatch(self.nv, self.nv, self.nv, ranks[:2 * n].reshape(-1, 2), offs,
                       cores[:int(offs[-1])])

    def ranks_of(self, which: int) -> np.ndarray:
        """(r1, r2) of every tensor of a stage set (layout only)."""
        cnt = C.c_int32(0)
        self._check(self.L.ttref_layout(self.h, which, C.byref(cnt), None, None))
        n = cnt.value
        ranks = np.zeros(2 * max(n, 1), dtype=np.int32)
        offs = np.zeros(n + 1, dtype=np.int64)
        self._check(self.L.ttref_layout(self.h, which, None, _ptr(ranks), _ptr(offs)))
        return ranks[:2 * n].reshape(-1, 2)

    def state(self):
        return self.fetch(self.STATE)

    def macros(self, count: int):
        out = np.zeros(11 * max(count, 1))
        self._check(self.L.ttref_macros(self.h, _ptr(out)))
        return out[:11 * count].reshape(count, 11)

    # primitives (results in the RESULT set)
    def round_sums(self, b, eps: float, cap: int = 0, group_off=None, scale=None):
        nout = b.count if group_off is None else len(group_off) - 1
        go = None if group_off is None else np.ascontiguousarray(group_off, dtype=np.int64)
        sc = None if scale is None else np.ascontiguousarray(scale, dtype=np.float64)
        s = _batch(b)
        self._check(self.L.ttref_round_sums(self.h, C.byref(s), nout, _ptr(go), _ptr(sc), eps, cap))
        return self.fetch(self.RESULT)

    def compute_macro(self, b):
        out = np.zeros(11 * max(1, b.count))
        s = _batch(b)
        self._check(self.L.ttref_compute_macro(self.h, C.byref(s), _ptr(out)))
        return out[:11 * b.count].reshape(b.count, 11)

    def collision(self, b, eps: float):
        s = _batch(b)
        self._check(self.L.ttref_collision(self.h, C.byref(s), eps))
        return self.fetch(self.RESULT)

    def face_factors(self, normals, cap: int = 4, mode: int = 0):
        nrm = np.ascontiguousarray(normals, dtype=np.float64).reshape(-1, 3)
        self._check(self.L.ttref_face_factors(self.h, len(nrm), _ptr(nrm), cap, mode))
        return self.fetch(self.RESULT)
