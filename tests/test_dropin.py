"""The drop-in boundary on the reference's own types.

include/ttdvm_cuda_adapter.hpp gives a reference maintainer
``ttdvm::cuda::explicit_step(std::vector<TtTensor>, UnstructuredMesh,
VelocityGrid, GasParameters, std::vector<BoundaryCondition>, dt, eps, cap)``
 over libttdvm_cuda.so.  oracle/build_ref.py compiles it
against the reference's headers (proj/include/ttdvm/*.hpp) and links it with
the unmodified reference into oracle/_ref/dropin_step, a C++ program that
builds the mesh, grid, boundary conditions and state with reference calls
and steps them on both sides in lock-step."""
import os
import subprocess

import pytest

from oracle import build_ref

REFERENCE_HERE = os.path.isdir(build_ref.PROJ)


@pytest.mark.skipif(not REFERENCE_HERE, reason="/root/reference absent (GPU box): prebuilt binary is used")
def test_adapter_compiles_against_reference_headers():
    build_ref.build()
    assert os.path.exists(build_ref.DROPIN)
    out = subprocess.run(["nm", "-C", "--undefined-only", build_ref.DROPIN], capture_output=True,
                         text=True).stdout
    # the program really calls the product's C ABI (not a stub)
    for sym in ("ttdvm_cuda_create", "ttdvm_cuda_set_mesh", "ttdvm_cuda_upload_state",
                "ttdvm_cuda_step", "ttdvm_cuda_download_state", "ttdvm_cuda_macros"):
        assert sym in out, sym


@pytest.mark.gpu
def test_dropin_step_matches_reference_on_its_own_types():
    if not os.path.exists(build_ref.DROPIN):
        pytest.skip("oracle/_ref/dropin_step not built")
    r = subprocess.run([build_ref.DROPIN, "3"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "dropin ok" in r.stdout, r.stdout
