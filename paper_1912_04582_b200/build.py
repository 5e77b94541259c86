"""In-tree build of libttdvm_cuda.so for sm_100a (nvcc, no JIT cache)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libttdvm_cuda.so")
SOURCES = ["round.cu", "round256.cu", "round512.cu", "round32.cu", "physics.cu", "facefactor.cu", "capi.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "--expt-relaxed-constexpr"]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "ttdvm_cuda.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    objs, procs = [], []
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    headers.append(os.path.join(os.path.dirname(HERE), "include", "ttdvm_cuda.h"))
    for s in SOURCES:  # the translation units compile in parallel
        o = os.path.join(CSRC, s.replace(".cu", ".o"))
        objs.append(o)
        deps = [os.path.join(CSRC, s), *headers]
        if s in ("round256.cu", "round512.cu", "round32.cu"):  # include round.cu
            deps.append(os.path.join(CSRC, "round.cu"))
        if not force and os.path.exists(o) and all(
                os.path.getmtime(d) <= os.path.getmtime(o) for d in deps if os.path.exists(d)):
            continue  # object newer than its source and every header
        cmd = [NVCC, *FLAGS, "-c", os.path.join(CSRC, s), "-o", o]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), cmd))
    for p, cmd in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, cmd)
    subprocess.run([NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", *objs,
                    "-o", LIB + ".tmp"], check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


EXAMPLE_SRC = os.path.join(os.path.dirname(HERE), "examples", "shock_tube.cpp")
EXAMPLE_BIN = os.path.join(os.path.dirname(HERE), "examples", "shock_tube")


def build_example(force: bool = False) -> str:
    """The C++ host driver (examples/shock_tube.cpp) over include/ttdvm_cuda.hpp,
    linked against the in-tree library."""
    lib = build()
    if (not force and os.path.exists(EXAMPLE_BIN)
            and os.path.getmtime(EXAMPLE_BIN) >= max(os.path.getmtime(EXAMPLE_SRC),
                                                     os.path.getmtime(lib))):
        return EXAMPLE_BIN
    inc = os.path.join(os.path.dirname(HERE), "include")
    subprocess.run([os.environ.get("CXX", "g++"), "-std=c++17", "-O2", "-I", inc, EXAMPLE_SRC,
                    "-L", HERE, "-lttdvm_cuda", "-Wl,-rpath,$ORIGIN/../paper_1912_04582_b200",
                    "-o", EXAMPLE_BIN], check=True)
    return EXAMPLE_BIN


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
