"""The host-side C++ layer: the reference's C++ API implemented on the C-ABI."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_1612_00530_b200")
REF_INC = "/root/reference/proj/include"


def test_shim_is_signature_compatible_with_the_reference_headers():
    """Compile the implementation and the C++ test against the REFERENCE's own headers: every
    definition must match a reference declaration, so reference callers link unchanged.
    (Only where /root/reference is mounted; nothing is copied from it.)"""
    if not os.path.isdir(REF_INC):
        pytest.skip("reference headers not present on this machine")
    for src in (os.path.join(PKG, "cpp", "spmvcomp_host.cpp"), os.path.join(PKG, "cpp", "spmvcomp_io.cpp"),
                os.path.join(ROOT, "tests", "cpp", "test_api.cpp"), os.path.join(ROOT, "tests", "cpp", "test_io.cpp")):
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", REF_INC, "-I", os.path.join(ROOT, "include"), src],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr[-2000:]


def test_own_headers_are_self_contained():
    for h in ("spmvcomp.hpp", "grid.hpp", "stencil.hpp", "ell.hpp", "compress.hpp", "kernels.hpp", "perf_model.hpp", "errors.hpp"):
        r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-x", "c++", "-I", os.path.join(ROOT, "include"),
                            os.path.join(ROOT, "include", "spmvcomp", h)], capture_output=True, text=True)
        assert r.returncode == 0, (h, r.stderr[-1000:])


@pytest.mark.gpu
def test_cpp_api_on_gpu():
    """SPEC.md worked examples and acceptance criteria through the C++ API, on the GPU."""
    exe = os.path.join(PKG, "test_cpp_api")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", os.path.join(PKG, "cpp")], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
