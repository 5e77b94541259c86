"""The C++ host path (include/ttdvm_cuda.hpp -> C ABI -> CUDA): the example
driver examples/shock_tube.cpp builds and links against the in-tree library;
without a GPU it fails loudly with the reference's exception type; on a GPU
its free-running config-1 steps match the CPU oracle."""
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_bin():
    from paper_1912_04582_b200 import build
    return build.build_example()


def test_cpp_host_builds_and_fails_without_gpu():
    import torch
    exe = build_bin()
    assert os.path.exists(exe)
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    r = subprocess.run([exe, "1"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 3 and "runtime_error" in r.stderr


@pytest.mark.gpu
def test_cpp_host_shock_tube_matches_oracle(tmp_path):
    from oracle.step import OracleSolver
    from oracle.tt import TtTensor, rel_err
    from paper_1912_04582_b200.problems import config
    exe = build_bin()
    out = tmp_path / "st.bin"
    steps = 3
    r = subprocess.run([exe, str(steps), str(out)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    raw = out.read_bytes()
    nx, n, st = struct.unpack("3i", raw[:12])
    o = 12
    ranks = np.frombuffer(raw, np.int32, 2 * nx, o).reshape(nx, 2)
    o += 8 * nx
    offs = np.frombuffer(raw, np.int64, nx + 1, o)
    o += 8 * (nx + 1)
    cores = np.frombuffer(raw, np.float64, int(offs[-1]), o)
    p = config(1)
    solver = OracleSolver(p.mesh, p.nv, p.bound, p.gas, p.bcs)
    f = [TtTensor(*p.f0.get(i)) for i in range(p.mesh.ncell)]
    for _ in range(steps):
        f, _ = solver.step(f, p.dt, p.eps, p.cap)
    for c in range(nx):
        r1, r2 = ranks[c]
        a = cores[offs[c]:offs[c + 1]]
        first = a[:n * r1].reshape(r1, n).T
        mid = a[n * r1:n * r1 + n * r1 * r2].reshape(n, r2, r1).transpose(0, 2, 1)
        last = a[n * r1 + n * r1 * r2:].reshape(n, r2).T
        got = TtTensor(first, mid, last).to_full()
        assert rel_err(got, f[c].to_full()) <= 30 * p.eps, c
