"""Compile the UNMODIFIED reference C++ into the CPU oracle (oracle/_ref).

TEST INFRASTRUCTURE.  Recipe only: the reference sources are compiled
where they lie under /root/reference/proj (never copied into the repo);
every output goes to oracle/_ref/ (git-ignored, shipped to the GPU box with
the snapshot like the product's own .so).  The reference's own build
(proj/CMakeLists.txt) needs Eigen and a vendored doctest, both absent here
(SURVEY.md §0 item 3, §8(c)); the repo-authored subsets in oracle/shim/
stand in for them.

Outputs:
  oracle/_ref/unit_tests     the reference's 50 doctest TEST_CASEs
                             (proj/tests/*.cpp) -- the gate of the oracle
  oracle/_ref/dropin_step    oracle/dropin_step.cpp: the product's drop-in adapter
                             (include/ttdvm_cuda_adapter.hpp) on the reference's
                             own types against the reference S1 step
  oracle/_ref/libttdvm_ref.so  proj/src/{tt_tensor,physics,velocity_grid,
                             boundary,mesh}.cpp + oracle/ref_step.cpp (the S1
                             step composed of reference API calls, C ABI for
                             ctypes), OpenMP over faces and cells.

    python oracle/build_ref.py [--force] [--test]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "_ref")
REF = os.environ.get("TTDVM_REFERENCE", "/root/reference")
PROJ = os.path.join(REF, "proj")
SRC = ["tt_tensor.cpp", "physics.cpp", "velocity_grid.cpp", "boundary.cpp", "mesh.cpp"]
TESTS = ["test_main.cpp", "test_tt_tensor.cpp", "test_velocity_grid.cpp", "test_physics.cpp",
         "test_boundary.cpp", "test_mesh.cpp"]
# the system g++ (its libgomp links OpenMP; $CXX may name a wrapper without it)
CXX = os.environ.get("TTDVM_REF_CXX", "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++")
# proj/CMakeLists.txt:3,9 -- C++20, Release -O3; -march=x86-64-v3 instead of
# -march=native because the binaries travel to the GPU box's host CPU.
# -ffp-contract=off: products and sums rounded separately, so exact
# cancellations the reference tests rely on (test_boundary.cpp:132) hold.
FLAGS = ["-std=gnu++20", "-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fPIC", "-fopenmp",
         "-I", os.path.join(HERE, "shim"), "-I", os.path.join(PROJ, "include")]
LIB = os.path.join(OUT, "libttdvm_ref.so")
UNIT = os.path.join(OUT, "unit_tests")
DROPIN = os.path.join(OUT, "dropin_step")


def _newer(target: str, deps) -> bool:
    if not os.path.exists(target):
        return False
    t = os.path.getmtime(target)
    return all(os.path.getmtime(d) <= t for d in deps if os.path.exists(d))


def _shim_headers():
    out = [os.path.join(HERE, "shim", "doctest.h")]
    d = os.path.join(HERE, "shim", "Eigen")
    out += [os.path.join(d, f) for f in os.listdir(d)]
    return out


def _compile(src: str, obj: str, extra=()):
    deps = [src, *_shim_headers()]
    inc = os.path.join(PROJ, "include", "ttdvm")
    deps += [os.path.join(inc, f) for f in os.listdir(inc)]
    if _newer(obj, deps):
        return None
    return subprocess.Popen([CXX, *FLAGS, *extra, "-c", src, "-o", obj])


def build(force: bool = False) -> tuple[str, str]:
    if not os.path.isdir(PROJ):
        raise FileNotFoundError(f"reference sources not found at {PROJ}")
    os.makedirs(os.path.join(OUT, "obj"), exist_ok=True)
    if force:
        for f in os.listdir(os.path.join(OUT, "obj")):
            os.remove(os.path.join(OUT, "obj", f))
    jobs, src_objs, test_objs = [], [], []
    for s in SRC:
        o = os.path.join(OUT, "obj", s.replace(".cpp", ".o"))
        src_objs.append(o)
        jobs.append(_compile(os.path.join(PROJ, "src", s), o))
    step_o = os.path.join(OUT, "obj", "ref_step.o")
    jobs.append(_compile(os.path.join(HERE, "ref_step.cpp"), step_o))
    for s in TESTS:
        o = os.path.join(OUT, "obj", s.replace(".cpp", ".o"))
        test_objs.append(o)
        jobs.append(_compile(os.path.join(PROJ, "tests", s), o,
                             ["-I", os.path.join(PROJ, "tests")]))
    failed = [j.args for j in jobs if j is not None and j.wait() != 0]
    if failed:
        raise RuntimeError(f"reference compile failed: {failed}")
    if force or not _newer(LIB, src_objs + [step_o]):
        subprocess.run([CXX, "-shared", "-fopenmp", *src_objs, step_o, "-o", LIB], check=True)
    if force or not _newer(UNIT, src_objs + test_objs):
        subprocess.run([CXX, "-fopenmp", *test_objs, *src_objs, "-o", UNIT], check=True)
    build_dropin(src_objs, force)
    return LIB, UNIT


def build_dropin(src_objs, force: bool = False):
    """oracle/_ref/dropin_step: include/ttdvm_cuda_adapter.hpp (the drop-in
    on the reference's own types) compiled against proj/include and linked
    with the reference objects and the product's libttdvm_cuda.so."""
    root = os.path.dirname(HERE)
    prod = os.path.join(root, "paper_1912_04582_b200")
    cuda_lib = os.path.join(prod, "libttdvm_cuda.so")
    src = os.path.join(HERE, "dropin_step.cpp")
    inc = os.path.join(root, "include")
    if not os.path.exists(cuda_lib):
        return None
    deps = [src, cuda_lib, *src_objs, *_shim_headers(),
            *(os.path.join(inc, f) for f in os.listdir(inc))]
    if not force and _newer(DROPIN, deps):
        return DROPIN
    subprocess.run([CXX, *FLAGS, "-I", inc, src, *src_objs, "-L", prod, "-lttdvm_cuda",
                    "-Wl,-rpath,$ORIGIN/../../paper_1912_04582_b200", "-o", DROPIN], check=True)
    return DROPIN


def run_unit_tests() -> subprocess.CompletedProcess:
    return subprocess.run([UNIT], capture_output=True, text=True)


if __name__ == "__main__":
    lib, unit = build(force="--force" in sys.argv)
    print(lib)
    print(unit)
    if "--test" in sys.argv:
        r = run_unit_tests()
        sys.stdout.write(r.stdout)
        sys.stderr.write(r.stderr)
        sys.exit(r.returncode)
