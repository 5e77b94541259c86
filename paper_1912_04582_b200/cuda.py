"""ctypes binding of libttdvm_cuda.so -- the host-side mirror of the
reference's TT / physics / step interface over the C ABI
(include/ttdvm_cuda.h).

Names follow the reference: ``rounded`` (TtTensor::rounded,
proj/src/tt_tensor.cpp:139-193), ``compute_macro`` (physics.cpp:17-67),
``compute_collision`` (physics.cpp:112-125) and ``explicit_step`` (the step
SPEC.md:391 declares).  Errors map like the reference's exceptions:
TTDVM_EINVAL -> ValueError (std::invalid_argument), TTDVM_EDOMAIN ->
RuntimeError (std::runtime_error).  There is no CPU fallback: without the
built library or a GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .tt_batch import TtBatch

HERE = os.path.dirname(os.path.abspath(__file__))
# TTDVM_LIB overrides the library path (A/B measurements of alternative builds)
LIB_PATH = os.environ.get("TTDVM_LIB") or os.path.join(HERE, "libttdvm_cuda.so")

# every symbol declared in include/ttdvm_cuda.h
EXPORTS = (
    "ttdvm_cuda_create", "ttdvm_cuda_destroy", "ttdvm_cuda_last_error", "ttdvm_cuda_set_grid",
    "ttdvm_cuda_set_gas", "ttdvm_cuda_set_mesh", "ttdvm_cuda_set_bcs", "ttdvm_cuda_upload_state",
    "ttdvm_cuda_state_layout", "ttdvm_cuda_download_state", "ttdvm_cuda_step",
    "ttdvm_cuda_macros", "ttdvm_cuda_stage_layout", "ttdvm_cuda_stage_download",
    "ttdvm_cuda_round_batch", "ttdvm_cuda_result_layout", "ttdvm_cuda_result_download",
    "ttdvm_cuda_macro_batch", "ttdvm_cuda_collision_batch", "ttdvm_cuda_phase_times",
    "ttdvm_cuda_launch_count", "ttdvm_cuda_set_profiling", "ttdvm_cuda_phase_work",
    "ttdvm_cuda_timed_step", "ttdvm_cuda_fp64_peak", "ttdvm_cuda_round_profile",
    "ttdvm_cuda_set_owned", "ttdvm_cuda_set_blocks", "ttdvm_cuda_halo_pack", "ttdvm_cuda_halo_unpack",
    "ttdvm_cuda_face_factors", "ttdvm_cuda_wall_densities", "ttdvm_cuda_setup_info",
    "ttdvm_cuda_round_resident", "ttdvm_cuda_phase_report", "ttdvm_cuda_nccl_unique_id",
    "ttdvm_cuda_comm_init", "ttdvm_cuda_set_comm", "ttdvm_cuda_set_partition",
    "ttdvm_cuda_halo_stats", "ttdvm_cuda_lusgs_step", "ttdvm_cuda_lusgs_levels",
)

OK, EINVAL, EDOMAIN, ENOMEM, ECUDA, ENCCL = range(6)
BC_KIND = {"wall": 0, "sym-x": 1, "sym-y": 2, "sym-z": 3, "in": 4, "out": 5}
STAGE = {"phi": 0, "jr": 1, "res": 2, "fs": 3}


class TtBatchC(C.Structure):
    _fields_ = [("count", C.c_int32), ("n1", C.c_int32), ("n2", C.c_int32), ("n3", C.c_int32),
                ("ranks", C.c_void_p), ("offsets", C.c_void_p), ("cores", C.c_void_p)]


class BcC(C.Structure):
    _fields_ = [("kind", C.c_int32), ("wall_temperature", C.c_double), ("free_n", C.c_double),
                ("free_t", C.c_double), ("free_u", C.c_double * 3)]


_lib = None


def load_library(path: str = LIB_PATH):
    """Load the in-tree library (raises if it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} missing: run `python -m paper_1912_04582_b200.build` "
                          "(the product path has no CPU fallback)")
    lib = C.CDLL(path)
    vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sig = {
        "ttdvm_cuda_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
        "ttdvm_cuda_destroy": (C.c_int, [vp]),
        "ttdvm_cuda_last_error": (C.c_char_p, [vp]),
        "ttdvm_cuda_set_grid": (C.c_int, [vp, C.c_int, dbl]),
        "ttdvm_cuda_set_gas": (C.c_int, [vp, vp]),
        "ttdvm_cuda_set_mesh": (C.c_int, [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp, vp, vp]),
        "ttdvm_cuda_set_bcs": (C.c_int, [vp, i32, vp]),
        "ttdvm_cuda_upload_state": (C.c_int, [vp, vp]),
        "ttdvm_cuda_state_layout": (C.c_int, [vp, vp, vp]),
        "ttdvm_cuda_download_state": (C.c_int, [vp, vp, i64]),
        "ttdvm_cuda_step": (C.c_int, [vp, dbl, dbl, i32, i32]),
        "ttdvm_cuda_macros": (C.c_int, [vp, vp]),
        "ttdvm_cuda_stage_layout": (C.c_int, [vp, i32, vp, vp, vp]),
        "ttdvm_cuda_stage_download": (C.c_int, [vp, i32, vp, i64]),
        "ttdvm_cuda_round_batch": (C.c_int, [vp, vp, i32, vp, vp, dbl, i32, vp]),
        "ttdvm_cuda_result_layout": (C.c_int, [vp, vp, vp]),
        "ttdvm_cuda_result_download": (C.c_int, [vp, vp, i64]),
        "ttdvm_cuda_macro_batch": (C.c_int, [vp, vp, vp]),
        "ttdvm_cuda_collision_batch": (C.c_int, [vp, vp, dbl, vp]),
        "ttdvm_cuda_phase_times": (C.c_int, [vp, vp]),
        "ttdvm_cuda_launch_count": (C.c_int64, [vp]),
        "ttdvm_cuda_set_profiling": (C.c_int, [vp, C.c_int]),
        "ttdvm_cuda_phase_work": (C.c_int, [vp, vp, vp, vp]),
        "ttdvm_cuda_timed_step": (C.c_int, [vp, dbl, dbl, i32, i32, vp]),
        "ttdvm_cuda_fp64_peak": (C.c_int, [vp, vp]),
        "ttdvm_cuda_round_profile": (C.c_int, [vp, C.c_int, vp]),
        "ttdvm_cuda_set_owned": (C.c_int, [vp, i32]),
        "ttdvm_cuda_set_blocks": (C.c_int, [vp, i32]),
        "ttdvm_cuda_halo_pack": (C.c_int, [vp, i32, vp, vp, vp, vp, i64]),
        "ttdvm_cuda_halo_unpack": (C.c_int, [vp, i32, vp, vp, vp, vp]),
        "ttdvm_cuda_face_factors": (C.c_int, [vp, i32, vp, i32, i32, vp]),
        "ttdvm_cuda_wall_densities": (C.c_int, [vp, vp]),
        "ttdvm_cuda_setup_info": (C.c_int, [vp, vp]),
        "ttdvm_cuda_round_resident": (C.c_int, [vp, dbl, i32, i32, vp]),
        "ttdvm_cuda_phase_report": (C.c_int, [vp, i32, vp, vp, vp, vp]),
        "ttdvm_cuda_nccl_unique_id": (C.c_int, [vp]),
        "ttdvm_cuda_comm_init": (C.c_int, [vp, i32, i32, vp]),
        "ttdvm_cuda_set_comm": (C.c_int, [vp, vp, i32, i32]),
        "ttdvm_cuda_set_partition": (C.c_int, [vp, i32, i32, vp, vp, vp, vp, vp]),
        "ttdvm_cuda_halo_stats": (C.c_int, [vp, vp]),
        "ttdvm_cuda_lusgs_step": (C.c_int, [vp, dbl, dbl, i32, i32]),
        "ttdvm_cuda_lusgs_levels": (C.c_int, [vp, vp, vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _batch_struct(b: TtBatch):
    s = TtBatchC(b.count, b.n1, b.n2, b.n3, _ptr(b.ranks), _ptr(b.offsets), _ptr(b.cores))
    return s


class Context:
    """One CUDA context of the TT-DVM step (one per GPU / rank)."""

    def __init__(self, device: int = 0):
        self.lib = load_library()
        h = C.c_void_p()
        rc = self.lib.ttdvm_cuda_create(int(device), C.byref(h))
        if rc != OK:
            raise RuntimeError(f"ttdvm_cuda_create failed (code {rc}): no usable CUDA device")
        self.h = h
        self.n = 0
        self.mesh = None

    # -- plumbing -------------------------------------------------------------
    def _check(self, rc: int):
        if rc == OK:
            return
        msg = self.lib.ttdvm_cuda_last_error(self.h).decode()
        if rc == EINVAL:
            raise ValueError(msg)
        if rc == EDOMAIN:
            raise RuntimeError(msg)
        if rc == ENOMEM:
            raise MemoryError(msg)
        raise RuntimeError(f"CUDA error: {msg}")

    def close(self):
        if getattr(self, "h", None):
            self.lib.ttdvm_cuda_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- set-up ------------------------------------------------------------------
    def set_grid(self, n: int, bound: float):
        self._check(self.lib.ttdvm_cuda_set_grid(self.h, int(n), float(bound)))
        self.n = int(n)

    def set_gas(self, gas):
        g = np.ascontiguousarray(gas, dtype=np.float64)
        self._check(self.lib.ttdvm_cuda_set_gas(self.h, _ptr(g)))

    def set_mesh(self, m):
        self.mesh = m
        self._keep = [m.face_left, m.face_right, m.face_group, m.face_area, m.face_normal,
                      m.cell_volume, m.cell_face_off, m.cell_face_id, m.cell_face_sign]
        self._check(self.lib.ttdvm_cuda_set_mesh(
            self.h, m.ncell, m.nface, *(_ptr(np.ascontiguousarray(a)) for a in self._keep)))

    def set_bcs(self, bcs):
        arr = (BcC * max(1, len(bcs)))()
        for g, bc in enumerate(bcs):
            arr[g].kind = BC_KIND[bc["kind"]]
            arr[g].wall_temperature = float(bc.get("t_wall", 0.0))
            arr[g].free_n = float(bc.get("n", 0.0))
            arr[g].free_t = float(bc.get("t", 0.0))
            u = bc.get("u", (0.0, 0.0, 0.0))
            for a in range(3):
                arr[g].free_u[a] = float(u[a])
        self._check(self.lib.ttdvm_cuda_set_bcs(self.h, len(bcs), C.cast(arr, C.c_void_p)))

    def setup(self, problem):
        self.set_grid(problem.nv, problem.bound)
        self.set_gas(problem.gas)
        self.set_mesh(problem.mesh)
        self.set_bcs(problem.bcs)
        self.upload_state(problem.f0)

    # -- state ---------------------------------------------------------------------
    def upload_state(self, b: TtBatch):
        s = _batch_struct(b)
        self._check(self.lib.ttdvm_cuda_upload_state(self.h, C.byref(s)))

    def _fetch(self, count, layout_fn, download_fn, out=None) -> TtBatch:
        ranks = np.zeros(2 * max(count, 1), dtype=np.int32)
        offs = np.zeros(count + 1, dtype=np.int64)
        self._check(layout_fn(_ptr(ranks), _ptr(offs)))
        need = max(1, int(offs[count]))
        if out is not None and out.dtype == np.float64 and out.size >= need:
            cores = out  # caller-owned (e.g. pinned) buffer, written in place
        else:
            cores = np.empty(need, dtype=np.float64)
        self._check(download_fn(_ptr(cores), int(cores.size)))
        return TtBatch(self.n, self.n, self.n, ranks[:2 * count], offs, cores[:int(offs[count])])

    def download_state(self, out=None) -> TtBatch:
        """The state in cell order.  ``out``: optional float64 buffer (e.g.
        pinned host memory) the cores are written into when large enough."""
        count = self.mesh.ncell
        return self._fetch(count,
                           lambda r, o: self.lib.ttdvm_cuda_state_layout(self.h, r, o),
                           lambda c, cap: self.lib.ttdvm_cuda_download_state(self.h, c, cap), out)

    def stage(self, name: str) -> TtBatch:
        sid = STAGE[name]
        cnt = C.c_int32()
        self._check(self.lib.ttdvm_cuda_stage_layout(self.h, sid, C.byref(cnt), None, None))
        count = cnt.value
        return self._fetch(count,
                           lambda r, o: self.lib.ttdvm_cuda_stage_layout(self.h, sid, None, r, o),
                           lambda c, cap: self.lib.ttdvm_cuda_stage_download(self.h, sid, c, cap))

    def stage_ranks(self, name: str) -> np.ndarray:
        """(r1, r2) of every tensor of an intermediate set of the last step (no core download)."""
        sid = STAGE[name]
        cnt = C.c_int32()
        self._check(self.lib.ttdvm_cuda_stage_layout(self.h, sid, C.byref(cnt), None, None))
        ranks = np.zeros(2 * max(cnt.value, 1), dtype=np.int32)
        offs = np.zeros(cnt.value + 1, dtype=np.int64)
        self._check(self.lib.ttdvm_cuda_stage_layout(self.h, sid, None, _ptr(ranks), _ptr(offs)))
        return ranks[:2 * cnt.value].reshape(-1, 2)

    # -- the hot path ----------------------------------------------------------------
    def step(self, dt: float, eps: float, cap: int = 0, nsteps: int = 1):
        """explicit_step, nsteps times, state resident."""
        self._check(self.lib.ttdvm_cuda_step(self.h, float(dt), float(eps), int(cap), int(nsteps)))

    def lusgs_step(self, dt: float, eps: float, cap: int = 0, niter: int = 1):
        """SPEC.md:399 lusgs_step over the resident state (ttdvm_cuda_lusgs_step)."""
        self._check(self.lib.ttdvm_cuda_lusgs_step(self.h, float(dt), float(eps), int(cap),
                                                   int(niter)))

    def lusgs_levels(self):
        a, b = C.c_int32(0), C.c_int32(0)
        self._check(self.lib.ttdvm_cuda_lusgs_levels(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def set_blocks(self, nblocks: int):
        """Cell blocks of the bounded-memory step (0 = automatic)."""
        self._check(self.lib.ttdvm_cuda_set_blocks(self.h, int(nblocks)))

    def set_owned(self, nowned: int):
        """Cells [0, nowned) are stepped; the rest are halo ghosts."""
        self._check(self.lib.ttdvm_cuda_set_owned(self.h, int(nowned)))
        self.nowned = int(nowned)

    # -- in-library NCCL halo exchange (include/ttdvm_cuda.h, multi-GPU section)
    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        rc = load_library().ttdvm_cuda_nccl_unique_id(C.cast(buf, C.c_void_p))
        if rc != OK:
            raise RuntimeError("libnccl could not be loaded by libttdvm_cuda.so")
        return buf.raw

    def comm_init(self, nranks: int, rank: int, unique_id: bytes):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        self._check(self.lib.ttdvm_cuda_comm_init(self.h, int(nranks), int(rank),
                                                  C.cast(buf, C.c_void_p)))

    def set_partition(self, n_owned: int, send: dict, recv: dict):
        """send / recv: peer rank -> local cell ids (LocalPart.send / .recv)."""
        peers = sorted(set(send) | set(recv))
        s_off, r_off = np.zeros(len(peers) + 1, np.int64), np.zeros(len(peers) + 1, np.int64)
        s_ids, r_ids = [], []
        for k, q in enumerate(peers):
            a = np.asarray(send.get(q, ()), dtype=np.int32)
            b = np.asarray(recv.get(q, ()), dtype=np.int32)
            s_ids.append(a)
            r_ids.append(b)
            s_off[k + 1] = s_off[k] + a.size
            r_off[k + 1] = r_off[k] + b.size
        cat = lambda v: np.ascontiguousarray(np.concatenate(v) if v else np.zeros(0), dtype=np.int32)  # noqa: E731
        pr = np.asarray(peers, dtype=np.int32)
        si, ri = cat(s_ids), cat(r_ids)
        self._check(self.lib.ttdvm_cuda_set_partition(self.h, int(n_owned), len(peers), _ptr(pr),
                                                      _ptr(s_off), _ptr(si), _ptr(r_off), _ptr(ri)))

    def halo_stats(self) -> dict:
        out = np.zeros(4)
        self._check(self.lib.ttdvm_cuda_halo_stats(self.h, _ptr(out)))
        return {"exchanges": int(out[0]), "bytes_sent": int(out[1]), "bytes_recv": int(out[2]),
                "host_ms": float(out[3])}

    def halo_pack(self, ids: np.ndarray, dev_ptr: int, capacity: int):
        """Pack current states of local cells `ids` into the device buffer at
        dev_ptr; returns (ranks [2k] int32, offsets [k+1] int64)."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        ranks = np.zeros(2 * max(len(ids), 1), dtype=np.int32)
        offs = np.zeros(len(ids) + 1, dtype=np.int64)
        self._check(self.lib.ttdvm_cuda_halo_pack(self.h, len(ids), _ptr(ids), _ptr(ranks),
                                                  _ptr(offs), C.c_void_p(dev_ptr), int(capacity)))
        return ranks[:2 * len(ids)], offs

    def halo_size(self, ids: np.ndarray) -> int:
        """Doubles needed to pack `ids` (pack with zero capacity)."""
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        ranks = np.zeros(2 * max(len(ids), 1), dtype=np.int32)
        offs = np.zeros(len(ids) + 1, dtype=np.int64)
        rc = self.lib.ttdvm_cuda_halo_pack(self.h, len(ids), _ptr(ids), _ptr(ranks), _ptr(offs),
                                           None, 0)
        if rc not in (OK, ENOMEM):
            self._check(rc)
        return int(offs[len(ids)])

    def halo_unpack(self, ids: np.ndarray, ranks: np.ndarray, offs: np.ndarray, dev_ptr: int):
        ids = np.ascontiguousarray(ids, dtype=np.int32)
        ranks = np.ascontiguousarray(ranks, dtype=np.int32)
        offs = np.ascontiguousarray(offs, dtype=np.int64)
        self._check(self.lib.ttdvm_cuda_halo_unpack(self.h, len(ids), _ptr(ids), _ptr(ranks),
                                                    _ptr(offs), C.c_void_p(dev_ptr)))

    def macros(self) -> np.ndarray:
        nown = getattr(self, "nowned", None) or self.mesh.ncell
        out = np.zeros((nown, 11))
        self._check(self.lib.ttdvm_cuda_macros(self.h, _ptr(out)))
        return out

    def rounded(self, b: TtBatch, eps: float, cap: int = 0, group_off=None, scale=None,
                margins: bool = False, out=None):
        """Batched TtTensor::rounded of (optionally grouped, scaled) sums.
        ``out``: optional float64 (e.g. pinned) buffer for the result cores."""
        s = _batch_struct(b)
        nout = b.count if group_off is None else len(group_off) - 1
        go = None if group_off is None else np.ascontiguousarray(group_off, dtype=np.int64)
        sc = None if scale is None else np.ascontiguousarray(scale, dtype=np.float64)
        mg = np.zeros(2 * max(nout, 1)) if margins else None
        self._check(self.lib.ttdvm_cuda_round_batch(self.h, C.byref(s), nout, _ptr(go), _ptr(sc),
                                                    float(eps), int(cap), _ptr(mg)))
        self._last_nout = nout
        out = self._fetch(nout, lambda r, o: self.lib.ttdvm_cuda_result_layout(self.h, r, o),
                          lambda c, cap_: self.lib.ttdvm_cuda_result_download(self.h, c, cap_), out)
        if margins:
            return out, mg[:2 * nout].reshape(nout, 2)
        return out

    def round_resident(self, eps: float, cap: int = 0, repeats: int = 1) -> float:
        """Repeat the last rounded() on its device-resident inputs; device ms."""
        ms = np.zeros(1)
        self._check(self.lib.ttdvm_cuda_round_resident(self.h, float(eps), int(cap), int(repeats),
                                                       _ptr(ms)))
        return float(ms[0])

    def result(self) -> TtBatch:
        """The result set of the last rounding call."""
        n = self._last_nout
        return self._fetch(n, lambda r, o: self.lib.ttdvm_cuda_result_layout(self.h, r, o),
                           lambda c, cap_: self.lib.ttdvm_cuda_result_download(self.h, c, cap_))

    def compute_macro(self, b: TtBatch) -> np.ndarray:
        """Batched compute_macro: [count, 11] = n, u(3), T, rho, p, S(3), nu."""
        s = _batch_struct(b)
        out = np.zeros((max(b.count, 1), 11))
        self._check(self.lib.ttdvm_cuda_macro_batch(self.h, C.byref(s), _ptr(out)))
        return out[:b.count]

    def compute_collision(self, b: TtBatch, eps: float):
        """Batched compute_collision: returns (J_r = round(f_S - f), macros);
        J = nu * J_r with nu = macros[:, 10] (physics.cpp:118)."""
        s = _batch_struct(b)
        mac = np.zeros((max(b.count, 1), 11))
        self._check(self.lib.ttdvm_cuda_collision_batch(self.h, C.byref(s), float(eps), _ptr(mac)))
        jr = self._fetch(b.count, lambda r, o: self.lib.ttdvm_cuda_result_layout(self.h, r, o),
                         lambda c, cap: self.lib.ttdvm_cuda_result_download(self.h, c, cap))
        return jr, mac[:b.count]

    def face_factors(self, normals, cap: int = 4, mode: str = "abs", diag: bool = False):
        """VelocityGrid::abs_xi_estimate(normal, cap) ("abs"),
        xi_normal_positive / xi_normal_negative(normal, cap - 2) ("pos" /
        "neg", i.e. from_full(max/min(xi_n, 0), 1e-12, cap)) for a batch
        of unit normals (proj/src/velocity_grid.cpp:61-146)."""
        nrm = np.ascontiguousarray(np.asarray(normals, dtype=np.float64).reshape(-1, 3))
        cnt = nrm.shape[0]
        m = {"abs": 0, "pos": 1, "neg": 2}[mode]
        dg = np.zeros(4 * max(cnt, 1)) if diag else None
        self._check(self.lib.ttdvm_cuda_face_factors(self.h, cnt, _ptr(nrm), int(cap), m, _ptr(dg)))
        out = self._fetch(cnt, lambda r, o: self.lib.ttdvm_cuda_result_layout(self.h, r, o),
                          lambda c, cap_: self.lib.ttdvm_cuda_result_download(self.h, c, cap_))
        if diag:
            return out, dg[:4 * cnt].reshape(cnt, 4)
        return out

    def setup_info(self) -> dict:
        info = np.zeros(5, dtype=np.int64)
        self._check(self.lib.ttdvm_cuda_setup_info(self.h, _ptr(info)))
        return dict(oblique_normals=int(info[0]), noise_floor_normals=int(info[1]),
                    wall_faces=int(info[2]), face_factor_ms=float(info[3]) / 1000.0,
                    cell_blocks=int(info[4]))

    def wall_densities(self) -> np.ndarray:
        """n_w of the last step per wall face, in face order."""
        nw = self.setup_info()["wall_faces"]
        out = np.zeros(max(nw, 1))
        self._check(self.lib.ttdvm_cuda_wall_densities(self.h, _ptr(out)))
        return out[:nw]

    def phase_times(self) -> np.ndarray:
        out = np.zeros(8)
        self._check(self.lib.ttdvm_cuda_phase_times(self.h, _ptr(out)))
        return out

    def timed_step(self, dt: float, eps: float, cap: int = 0, nsteps: int = 1) -> float:
        """Step nsteps times; returns device ms (CUDA events on the library stream)."""
        ms = np.zeros(1)
        self._check(self.lib.ttdvm_cuda_timed_step(self.h, float(dt), float(eps), int(cap),
                                                   int(nsteps), _ptr(ms)))
        return float(ms[0])

    def phase_work(self):
        fl, by = np.zeros(8), np.zeros(8)
        la = np.zeros(8, dtype=np.int32)
        self._check(self.lib.ttdvm_cuda_phase_work(self.h, _ptr(fl), _ptr(by), _ptr(la)))
        return fl, by, la

    PHASES = ("moments", "shakhov_build", "round_fs", "round_collision", "round_flux",
              "round_residual", "round_update", "bookkeeping", "wall_densities")

    def phase_report(self) -> dict:
        """name -> (ms, flops, bytes, launches) of the last profiled call."""
        k = len(self.PHASES)
        ms, fl, by = np.zeros(k), np.zeros(k), np.zeros(k)
        la = np.zeros(k, dtype=np.int32)
        self._check(self.lib.ttdvm_cuda_phase_report(self.h, k, _ptr(ms), _ptr(fl), _ptr(by),
                                                     _ptr(la)))
        return {n: (float(ms[i]), float(fl[i]), float(by[i]), int(la[i]))
                for i, n in enumerate(self.PHASES)}

    def fp64_peak(self) -> float:
        """Measured DFMA peak in TFLOP/s."""
        t = np.zeros(1)
        self._check(self.lib.ttdvm_cuda_fp64_peak(self.h, _ptr(t)))
        return float(t[0])

    def round_profile(self, on: bool = True) -> np.ndarray:
        """Per-phase cycles of the rounding kernel since the last call."""
        out = np.zeros(16, dtype=np.uint64)
        self._check(self.lib.ttdvm_cuda_round_profile(self.h, 1 if on else 0, _ptr(out)))
        return out

    def launch_count(self) -> int:
        return int(self.lib.ttdvm_cuda_launch_count(self.h))

    def set_profiling(self, on: bool):
        self._check(self.lib.ttdvm_cuda_set_profiling(self.h, 1 if on else 0))


def explicit_step(ctx: Context, dt: float, eps: float, cap: int = 0, nsteps: int = 1):
    """SPEC.md:391's explicit_step over the resident state of ``ctx``."""
    ctx.step(dt, eps, cap, nsteps)
