"""Per-step halo exchange of TT cores between ranks.

Two phases over torch.distributed point-to-point (NCCL over NVLink on the
GPUs, gloo for the CPU tests): (1) the (r1, r2) ranks of the packed
tensors, (2) the packed cores.  Packing/unpacking is delegated to callables
so the same exchange serves the CUDA library (device buffers) and the CPU
oracle tests (host buffers).
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist


def _exchange(sends: dict, recv_like: dict, device):
    ops = []
    out = {}
    for q, t in sends.items():
        ops.append(dist.P2POp(dist.isend, t, q))
    for q, t in recv_like.items():
        out[q] = t
        ops.append(dist.P2POp(dist.irecv, t, q))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return out


def exchange(part, pack, unpack, n: int, device="cpu"):
    """pack(ids) -> (ranks int32[2k], offsets int64[k+1], cores tensor f64 on
    device); unpack(ids, ranks, offsets, cores tensor).  Peers are visited in
    the part's agreed order (cells sorted by global id)."""
    packed = {q: pack(ids) for q, ids in part.send.items()}
    # phase 1: ranks
    send_r = {q: torch.from_numpy(np.ascontiguousarray(p[0], dtype=np.int32)).to(device)
              for q, p in packed.items()}
    recv_r = {q: torch.empty(2 * len(ids), dtype=torch.int32, device=device)
              for q, ids in part.recv.items()}
    got_r = _exchange(send_r, recv_r, device)
    # phase 2: cores
    sizes = {}
    for q, t in got_r.items():
        rk = t.cpu().numpy().reshape(-1, 2)
        off = np.zeros(rk.shape[0] + 1, dtype=np.int64)
        off[1:] = np.cumsum(n * rk[:, 0] + n * rk[:, 0] * rk[:, 1] + rk[:, 1] * n)
        sizes[q] = (rk.ravel(), off)
    send_c = {q: p[2] for q, p in packed.items()}
    recv_c = {q: torch.empty(int(sizes[q][1][-1]), dtype=torch.float64, device=device)
              for q in part.recv}
    got_c = _exchange(send_c, recv_c, device)
    if device != "cpu":
        torch.cuda.synchronize()
    for q, ids in part.recv.items():
        unpack(ids, sizes[q][0], sizes[q][1], got_c[q])


def gpu_pack_unpack(ctx, device):
    """pack/unpack callables over a CUDA-library context."""

    def pack(ids):
        need = ctx.halo_size(ids)
        buf = torch.empty(max(1, need), dtype=torch.float64, device=device)
        torch.cuda.synchronize()
        ranks, offs = ctx.halo_pack(ids, buf.data_ptr(), need)
        return ranks, offs, buf[:need]

    def unpack(ids, ranks, offs, cores):
        torch.cuda.synchronize()
        ctx.halo_unpack(ids, ranks, offs, cores.data_ptr())

    return pack, unpack


class HaloExchange:
    """The per-step exchange of one rank over a CUDA-library context, with
    every buffer preallocated and reused (core buffers grow geometrically as
    the ranks rise): pack on the library's stream, one batched NCCL
    send/recv of the (r1, r2) pairs, one of the cores, unpack.  The received
    ranks cross to the host once (the library's unpack sizes the next
    state's arena from them)."""

    def __init__(self, ctx, part, device):
        self.ctx, self.part, self.device = ctx, part, device
        self.n = None
        i32, f64 = torch.int32, torch.float64
        self.send_r = {q: torch.empty(2 * len(ids), dtype=i32, device=device)
                       for q, ids in part.send.items()}
        self.recv_r = {q: torch.empty(2 * len(ids), dtype=i32, device=device)
                       for q, ids in part.recv.items()}
        self.recv_r_host = {q: torch.empty(2 * len(ids), dtype=i32, pin_memory=device.type == "cuda")
                            for q, ids in part.recv.items()}
        self.send_c = {q: torch.empty(1, dtype=f64, device=device) for q in part.send}
        self.recv_c = {q: torch.empty(1, dtype=f64, device=device) for q in part.recv}

    @staticmethod
    def _fit(bufs, q, need, device):
        if bufs[q].numel() < need:
            bufs[q] = torch.empty(int(1.5 * need) + 1, dtype=torch.float64, device=device)
        return bufs[q]

    def exchange(self):
        ctx, part, dev = self.ctx, self.part, self.device
        n = ctx.n
        sends = {}
        for q, ids in part.send.items():
            need = ctx.halo_size(ids)
            buf = self._fit(self.send_c, q, need, dev)
            ranks, _ = ctx.halo_pack(ids, buf.data_ptr(), need)  # synchronous on the library stream
            self.send_r[q].copy_(torch.from_numpy(np.ascontiguousarray(ranks, dtype=np.int32)))
            sends[q] = buf[:need]
        _exchange(self.send_r, self.recv_r, dev)
        sizes = {}
        for q in part.recv:
            self.recv_r_host[q].copy_(self.recv_r[q], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        for q in part.recv:
            rk = self.recv_r_host[q].numpy().reshape(-1, 2).astype(np.int64)
            off = np.zeros(rk.shape[0] + 1, dtype=np.int64)
            off[1:] = np.cumsum(n * rk[:, 0] + n * rk[:, 0] * rk[:, 1] + rk[:, 1] * n)
            sizes[q] = (rk.astype(np.int32).ravel(), off)
        recvs = {q: self._fit(self.recv_c, q, int(sizes[q][1][-1]), dev)[:int(sizes[q][1][-1])]
                 for q in part.recv}
        _exchange(sends, recvs, dev)
        torch.cuda.current_stream().synchronize()
        for q, ids in part.recv.items():
            ctx.halo_unpack(ids, sizes[q][0], sizes[q][1], recvs[q].data_ptr())
