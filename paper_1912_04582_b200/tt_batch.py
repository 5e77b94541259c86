"""Packed batch of order-3 TT tensors -- the host-side layout of the C ABI's
``ttdvm_tt_batch`` (include/ttdvm_cuda.h).

Per tensor, contiguous doubles, mirroring the reference's
Eigen col-major cores (proj/include/ttdvm/tt_tensor.hpp:74-76):

    [first  n1 x r1 col-major: (i, a) at i + n1*a]
    [middle n2 slices, each r1 x r2 col-major: slice j, (a, b) at j*r1*r2 + a + r1*b]
    [last   r2 x n3 col-major: (b, k) at b + r2*k]

``offsets[t]`` is the first double of tensor t; ``ranks[t] = (r1, r2)``.
"""
from __future__ import annotations

import numpy as np


def tt_size(n1: int, n2: int, n3: int, r1: int, r2: int) -> int:
    return n1 * r1 + n2 * r1 * r2 + r2 * n3


class TtBatch:
    __slots__ = ("n1", "n2", "n3", "ranks", "offsets", "cores")

    def __init__(self, n1, n2, n3, ranks, offsets, cores):
        self.n1, self.n2, self.n3 = int(n1), int(n2), int(n3)
        self.ranks = np.ascontiguousarray(ranks, dtype=np.int32).reshape(-1, 2)
        self.offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        self.cores = np.ascontiguousarray(cores, dtype=np.float64)

    @property
    def count(self) -> int:
        return int(self.ranks.shape[0])

    def __len__(self):
        return self.count

    # ------------------------------------------------------------ conversion
    @staticmethod
    def from_list(tensors, n=None) -> "TtBatch":
        """tensors: iterable of (first (n1,r1), middle (n2,r1,r2), last (r2,n3))
        or objects with .first/.middle/.last."""
        parts, ranks, offs = [], [], [0]
        n1 = n2 = n3 = None
        for t in tensors:
            first, middle, last = (t.first, t.middle, t.last) if hasattr(t, "first") else t
            n1, r1 = first.shape
            n2 = middle.shape[0]
            r2, n3 = last.shape
            parts.append(np.asarray(first, dtype=np.float64).T.ravel())
            parts.append(np.asarray(middle, dtype=np.float64).transpose(0, 2, 1).ravel())
            parts.append(np.asarray(last, dtype=np.float64).T.ravel())
            ranks.append((r1, r2))
            offs.append(offs[-1] + tt_size(n1, n2, n3, r1, r2))
        if n is not None and n1 is None:
            n1 = n2 = n3 = n
        cores = np.concatenate(parts) if parts else np.zeros(0)
        return TtBatch(n1, n2, n3, np.array(ranks, dtype=np.int32).reshape(-1, 2),
                       np.array(offs, dtype=np.int64), cores)

    def get(self, t: int):
        """(first, middle, last) numpy views (copies) of tensor t."""
        r1, r2 = (int(v) for v in self.ranks[t])
        n1, n2, n3 = self.n1, self.n2, self.n3
        o = int(self.offsets[t])
        first = self.cores[o:o + n1 * r1].reshape(r1, n1).T.copy()
        o += n1 * r1
        middle = self.cores[o:o + n2 * r1 * r2].reshape(n2, r2, r1).transpose(0, 2, 1).copy()
        o += n2 * r1 * r2
        last = self.cores[o:o + r2 * n3].reshape(n3, r2).T.copy()
        return first, middle, last

    def to_list(self):
        return [self.get(t) for t in range(self.count)]

    def full(self, t: int) -> np.ndarray:
        first, middle, last = self.get(t)
        return np.einsum("ia,jab,bk->ijk", first, middle, last, optimize=True)

    # ------------------------------------------------------- batch builders
    @staticmethod
    def uniform(count, n1, n2, n3, r1, r2, first, middle, last) -> "TtBatch":
        """All tensors at one rank: first [count,n1,r1], middle [count,n2,r1,r2],
        last [count,r2,n3]."""
        sz = tt_size(n1, n2, n3, r1, r2)
        cores = np.empty((count, sz))
        cores[:, :n1 * r1] = first.transpose(0, 2, 1).reshape(count, -1)
        cores[:, n1 * r1:n1 * r1 + n2 * r1 * r2] = middle.transpose(0, 1, 3, 2).reshape(count, -1)
        cores[:, n1 * r1 + n2 * r1 * r2:] = last.transpose(0, 2, 1).reshape(count, -1)
        ranks = np.tile(np.array([r1, r2], dtype=np.int32), (count, 1))
        offs = np.arange(count + 1, dtype=np.int64) * sz
        return TtBatch(n1, n2, n3, ranks, offs, cores.ravel())

    def uniform_cores(self):
        """Inverse of uniform() when all ranks agree."""
        r1, r2 = (int(v) for v in self.ranks[0])
        assert np.all(self.ranks[:, 0] == r1) and np.all(self.ranks[:, 1] == r2)
        n1, n2, n3 = self.n1, self.n2, self.n3
        c = self.cores.reshape(self.count, -1)
        first = c[:, :n1 * r1].reshape(-1, r1, n1).transpose(0, 2, 1)
        middle = c[:, n1 * r1:n1 * r1 + n2 * r1 * r2].reshape(-1, n2, r2, r1).transpose(0, 1, 3, 2)
        last = c[:, n1 * r1 + n2 * r1 * r2:].reshape(-1, n3, r2).transpose(0, 2, 1)
        return first, middle, last

    @staticmethod
    def from_rank_one(f1, f2, f3) -> "TtBatch":
        count, n1 = f1.shape
        n2, n3 = f2.shape[1], f3.shape[1]
        return TtBatch.uniform(count, n1, n2, n3, 1, 1, f1[:, :, None], f2[:, :, None, None],
                               f3[:, None, :])

    @staticmethod
    def random_uniform_rank(rng, count, n, r1, r2) -> "TtBatch":
        """N(0,1) cores (proj/tests/support.hpp:20-35 fixture, batched)."""
        first = rng.standard_normal((count, n, r1))
        middle = rng.standard_normal((count, n, r1, r2))
        last = rng.standard_normal((count, r2, n))
        return TtBatch.uniform(count, n, n, n, r1, r2, first, middle, last)

    def norms(self) -> np.ndarray:
        """Frobenius norms via the Gram chain (tt_tensor.cpp:282-288), batched
        over uniform ranks."""
        first, middle, last = self.uniform_cores()
        w1 = np.einsum("cia,cib->cab", first, first)
        w2 = np.einsum("cjap,cab,cjbq->cpq", middle, w1, middle, optimize=True)
        s = np.einsum("cpk,cpq,cqk->c", last, w2, last, optimize=True)
        return np.sqrt(np.maximum(s, 0.0))

    def scaled(self, s) -> "TtBatch":
        """Per-tensor scale on the first core (tt_tensor.cpp:206-210)."""
        s = np.broadcast_to(np.asarray(s, dtype=np.float64), (self.count,))
        out = TtBatch(self.n1, self.n2, self.n3, self.ranks.copy(), self.offsets.copy(),
                      self.cores.copy())
        for t in range(self.count):
            o = int(out.offsets[t])
            out.cores[o:o + self.n1 * int(self.ranks[t, 0])] *= s[t]
        return out

    @staticmethod
    def add(a: "TtBatch", b: "TtBatch") -> "TtBatch":
        """Per-tensor TT sum (tt_tensor.cpp:290-312), uniform ranks."""
        fa, ma, la = a.uniform_cores()
        fb, mb, lb = b.uniform_cores()
        count = a.count
        ra1, ra2 = fa.shape[2], la.shape[1]
        rb1, rb2 = fb.shape[2], lb.shape[1]
        first = np.concatenate([fa, fb], axis=2)
        middle = np.zeros((count, a.n2, ra1 + rb1, ra2 + rb2))
        middle[:, :, :ra1, :ra2] = ma
        middle[:, :, ra1:, ra2:] = mb
        last = np.concatenate([la, lb], axis=1)
        return TtBatch.uniform(count, a.n1, a.n2, a.n3, ra1 + rb1, ra2 + rb2, first, middle, last)

    def subset(self, idx) -> "TtBatch":
        return TtBatch.from_list([self.get(int(t)) for t in idx])
