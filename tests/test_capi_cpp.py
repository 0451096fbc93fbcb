"""The C++ host layer (include/epfem_gpu.hpp) and C++ callers of the C-ABI
with no torch: tests/cpp/capi_test.cpp (the step against the oracle's C API)
and tests/cpp/newton_test.cpp (epfem_gpu::newton_solve, solver.cpp:7-62,
against the Python newton_solve on the same problem: the same kernels in the
same order, so the same bits).  Compiled here with g++ against
libepfem_gpu.so (CPU test), run on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "cpp", "capi_test.cpp")
OUT = os.path.join(ROOT, "tests", "cpp", "_build", "capi_test")


def _build(name="capi_test"):
    src = os.path.join(ROOT, "tests", "cpp", name + ".cpp")
    out = os.path.join(ROOT, "tests", "cpp", "_build", name)
    from oracle import oracle as O
    from paper_1805_04155_b200 import build as B
    lib = B.build()
    olib = O.build()
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cuda = "/usr/local/cuda"
    cmd = ["g++", "-std=c++17", "-O2", "-Wall", src, "-o", out, "-I", os.path.join(ROOT, "include"),
           "-I", f"{cuda}/include", lib, olib, f"-L{cuda}/lib64", "-lcudart",
           f"-Wl,-rpath,{os.path.dirname(lib)}", f"-Wl,-rpath,{os.path.dirname(olib)}", f"-Wl,-rpath,{cuda}/lib64"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
    return out


def test_cpp_layer_compiles_and_links():
    assert os.access(_build(), os.X_OK)
    assert os.access(_build("newton_test"), os.X_OK)


@pytest.mark.gpu
def test_cpp_caller_matches_oracle(cuda):
    exe = _build()
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "CAPI_CPP_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.gpu
def test_cpp_newton_solve_equals_python(cuda, tmp_path):
    """The cantilever step of tests/test_solver.py (cfg2's material, 6 x 6
    Q2-8, left edge clamped, right edge pulled by 0.004: yielding) through
    epfem_gpu::newton_solve (C++, no torch) and through the Python
    newton_solve: the same Newton iteration count, plastic count and u bit for
    bit (the Python one is checked against the reference loop restated on the
    oracle in tests/test_solver.py)."""
    import numpy as np
    import torch

    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.solver import NewtonSettings, SolveSettings, newton_solve
    from paper_1805_04155_b200.synthetic import CONFIGS
    cfg = CONFIGS["cfg2"]
    mesh = cfg.mesh(6)
    mat = cfg.material(mesh.n_int)
    x = mesh.coord.reshape(-1, 2)
    n_dofs = x.shape[0] * 2
    dirichlet = np.zeros(n_dofs)
    free = np.ones(n_dofs, bool)
    left, right = np.isclose(x[:, 0], 0.0), np.isclose(x[:, 0], x[:, 0].max())
    free[2 * np.nonzero(left)[0]] = False
    free[2 * np.nonzero(left)[0] + 1] = False
    free[2 * np.nonzero(right)[0]] = False
    dirichlet[2 * np.nonzero(right)[0]] = 0.004 * x[:, 0].max()
    f_ext = np.zeros(n_dofs)
    eps, max_iters, rel_tol = 1e-9, 25, 1e-12
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, cuda), mat)
    res = newton_solve(gc, mat, P.IntegrationState.zero(mesh.n_int, device=cuda),
                       torch.from_numpy(dirichlet), torch.from_numpy(free), torch.from_numpy(f_ext),
                       NewtonSettings(eps_newton=eps, max_iters=max_iters, linear=SolveSettings(rel_tol=rel_tol)))
    d = str(tmp_path)
    fam = {"P1": 0, "P2": 1, "Q1": 2, "Q2": 3}[cfg.family]
    np.array([fam, 2, 1, cfg.young, cfg.poisson, cfg.p1, cfg.p2, eps, max_iters, rel_tol, mesh.n_int],
             dtype=np.float64).tofile(d + "/meta.bin")
    np.ascontiguousarray(mesh.coord, dtype=np.float64).tofile(d + "/coord.bin")
    np.ascontiguousarray(mesh.elem, dtype=np.int32).tofile(d + "/elem.bin")
    dirichlet.tofile(d + "/dirichlet.bin")
    free.astype(np.uint8).tofile(d + "/free.bin")
    f_ext.tofile(d + "/fext.bin")
    r = subprocess.run([_build("newton_test"), d], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "NEWTON_CPP_OK" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]
    iters, npl = (int(v) for v in open(d + "/stats.txt").read().split())
    u_cpp = np.fromfile(d + "/u.bin", dtype=np.float64)
    assert iters == res.record.newton_iters and npl == res.record.n_plastic
    assert 0 < npl < mesh.n_int
    assert np.array_equal(u_cpp.view(np.uint64), res.u.cpu().numpy().view(np.uint64))
