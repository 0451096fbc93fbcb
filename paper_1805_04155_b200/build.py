"""Build libepfem_gpu.so in-tree with nvcc for sm_100a (no JIT, no torch
extension machinery: the product is a plain C-ABI shared library).

    python -m paper_1805_04155_b200.build            # incremental
    python -m paper_1805_04155_b200.build --force
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OBJ = os.path.join(PKG, "_obj")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libepfem_gpu.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                      "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
                      "-I", os.path.join(ROOT, "include")]

# per-source extra flags: the constitutive kernel reproduces the reference's
# (FMA-free) operation order bit for bit.
SOURCES = {
    "constitutive.cu": ["--fmad=false"],
    "assembly.cu": [],
    "tangent.cu": [],
    "capi.cu": [],
    "solve.cu": [],
    "exchange.cu": [],
    "tables.cpp": [],
}
HEADERS = ["common.cuh", "kernels.cuh", "delta.cuh", "tma.cuh"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


LIB_DEBUG = os.path.join(LIBDIR, "debug", "libepfem_gpu.so")


def build(force: bool = False, verbose: bool = False, debug_checks: bool = False) -> str:
    """debug_checks: the test build with device-side bounds / single-writer
    assertions (EPFEM_DEBUG_CHECKS=1) into lib/debug/ (own object dir)."""
    OBJ = os.path.join(PKG, "_obj_debug") if debug_checks else globals()["OBJ"]
    LIB = LIB_DEBUG if debug_checks else globals()["LIB"]
    os.makedirs(OBJ, exist_ok=True)
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "epfem_gpu.h")]
    objs, jobs = [], []
    for src, extra in SOURCES.items():
        path = os.path.join(CSRC, src)
        obj = os.path.join(OBJ, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + hdrs + [__file__]):
            if src.endswith(".cpp"):
                cmd = ["g++", "-O2", "-fPIC", "-std=c++17", "-ffp-contract=off",
                       "-I", "/usr/local/cuda/include", "-I", os.path.join(ROOT, "include"),
                       "-c", path, "-o", obj]
            else:
                cmd = [nvcc()] + NVCC_COMMON + extra + (["-DEPFEM_DEBUG_CHECKS=1"] if debug_checks else []) + \
                    ["-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            jobs.append((cmd, subprocess.Popen(cmd)))
    # the translation units compile in parallel
    failed = [cmd for cmd, p in jobs if p.wait() != 0]
    if failed:
        raise subprocess.CalledProcessError(1, failed[0])
    if force or _stale(LIB, objs):
        cmd = [nvcc()] + ARCH + ["-shared", "-o", LIB] + objs + ["-lcudart_static", "-ldl"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--debug-checks", action="store_true")
    args = ap.parse_args(argv)
    print(build(force=args.force, verbose=args.verbose, debug_checks=args.debug_checks))


if __name__ == "__main__":
    sys.exit(main())
