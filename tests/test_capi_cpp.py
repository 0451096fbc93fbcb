"""The C++ host layer (include/epfem_gpu.hpp) and a C++ caller of the C-ABI
with no torch (tests/cpp/capi_test.cpp): compiled here with g++ against
libepfem_gpu.so (CPU test), run on the GPU against the oracle's C API."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "capi_test.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "capi_test")


def _build():
    from oracle import oracle as O
    from paper_1805_04155_b200 import build as B
    lib = B.build()
    olib = O.build()
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cuda = "/usr/local/cuda"
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", SRC, "-o", OUT, "-I", os.path.join(ROOT, "include"),
           "-I", f"{cuda}/include", lib, olib, f"-L{cuda}/lib64", "-lcudart",
           f"-Wl,-rpath,{os.path.dirname(lib)}", f"-Wl,-rpath,{os.path.dirname(olib)}", f"-Wl,-rpath,{cuda}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return OUT


def test_cpp_layer_compiles_and_links():
    assert os.access(_build(), os.X_OK)


@pytest.mark.gpu
def test_cpp_caller_matches_oracle(cuda):
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "CAPI_CPP_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
