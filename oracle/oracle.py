"""TEST INFRASTRUCTURE ONLY — ctypes wrapper around the CPU restatement.

Only tests/, ``__graft_entry__.smoke()`` (as the checker) and bench.py's
``cpu_baseline`` / ``--impl reference`` leg may import this module.  The
product package never does.  See oracle/epfem_oracle.cpp for what is restated
(reference file:line citations there) and how it is pinned.

Array conventions mirror the reference's column-major Eigen storage: a numpy
array of shape (n_int, 6) in C order has the same bytes as the reference's
6 x n_int ``Mat``; DS is (n_int, 36) with each row a column-major 6x6 block.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "epfem_oracle.cpp")
LIB = os.path.join(HERE, "_build", "libepfem_oracle.so")

FAMILIES = {"P1": 0, "P2": 1, "Q1": 2, "Q2": 3}

_lib = None


def build(force: bool = False) -> str:
    """Compile the restatement with the reference's FP contract (no FMA)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        subprocess.check_call(
            ["g++", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-std=c++17",
             "-o", LIB, SRC])
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build()
        _lib = C.CDLL(LIB)
        _declare(_lib)
    return _lib


_P = C.c_void_p
_D = C.POINTER(C.c_double)
_I64 = C.POINTER(C.c_int64)
_I32 = C.POINTER(C.c_int32)
_U8 = C.POINTER(C.c_uint8)


def _declare(L):
    L.or_last_error.restype = C.c_char_p
    L.or_quadrature.restype = C.c_int
    L.or_quadrature.argtypes = [C.c_int, C.c_int, _P, _P]
    L.or_basis.argtypes = [C.c_int, C.c_int, _P, C.c_int, _P, _P]
    L.or_structured_mesh.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_double, C.c_double, C.c_double, _P,
                                     _I64, _I64, _P, _P, _P]
    L.or_elastic_moduli.argtypes = [C.c_double, C.c_double, _D, _D]
    L.or_dp_parameters.argtypes = [C.c_double, C.c_double, C.c_int, _D, _D]
    L.or_constitutive_elastic.argtypes = [C.c_int64] + [_P] * 5
    L.or_constitutive_vm.argtypes = [C.c_int64] + [_P] * 13
    L.or_constitutive_dp.argtypes = [C.c_int64] + [_P] * 11
    L.or_constitutive_dp.restype = C.c_int64
    L.or_cache_build.restype = _P
    L.or_cache_build.argtypes = [C.c_int, C.c_int, C.c_int64, _P, C.c_int64, _P, _P, _P]
    L.or_cache_free.argtypes = [_P]
    L.or_cache_info.argtypes = [_P, _P, _P]
    L.or_cache_arrays.argtypes = [_P, _P, _P, _P]
    L.or_cache_K_elast.argtypes = [_P, _P, _P, _P]
    L.or_cache_B.argtypes = [_P, _P, _P, _P]
    L.or_cache_strains.argtypes = [_P, _P, _P]
    L.or_cache_internal_forces.argtypes = [_P, _P, _P]
    for f in ("or_cache_tangent",):
        getattr(L, f).restype = _P
    L.or_cache_tangent.argtypes = [_P, C.c_int64, _P, _P]
    L.or_cache_direct.restype = _P
    L.or_cache_direct.argtypes = [_P, _P]
    L.or_cache_elastic.restype = _P
    L.or_cache_elastic.argtypes = [_P]
    L.or_k_info.argtypes = [_P, _I64, _I64]
    L.or_k_copy.argtypes = [_P, _P, _P, _P]
    L.or_k_free.argtypes = [_P]
    L.or_time_iteration.restype = C.c_double
    L.or_time_iteration.argtypes = [_P, C.c_int, _P, _P, _P, _P, _P, _I64]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    pass


def _err():
    return OracleError(lib().or_last_error().decode())


def node_count(family: str, dim: int) -> int:
    return lib().or_node_count(FAMILIES[family], dim)


def quadrature(family: str, dim: int):
    L = lib()
    nq = L.or_quadrature(FAMILIES[family], dim, None, None)
    pts = np.zeros((nq, dim))
    w = np.zeros(nq)
    L.or_quadrature(FAMILIES[family], dim, _ptr(pts), _ptr(w))
    return pts, w


def basis(family: str, dim: int, pts: np.ndarray):
    pts = _f64(pts)
    m = pts.shape[0]
    npn = node_count(family, dim)
    vals = np.zeros((npn, m))
    grads = np.zeros((dim, npn, m))
    lib().or_basis(FAMILIES[family], dim, _ptr(pts), m, _ptr(vals), _ptr(grads))
    return vals, grads


def structured_mesh(family, dim, nx, ny, nz=0, hx=None, hy=None, hz=None, active=None):
    """mesh.cpp:136-210 restated. Returns coord (n_n, dim), elem (n_e, n_p), fine (n_n, 3)."""
    hx = 1.0 / nx if hx is None else hx
    hy = 1.0 / ny if hy is None else hy
    hz = (1.0 / nz if nz else 0.0) if hz is None else hz
    L = lib()
    act = None if active is None else np.ascontiguousarray(active, dtype=np.uint8)
    nn, ne = C.c_int64(), C.c_int64()
    fam = FAMILIES[family]
    L.or_structured_mesh(fam, dim, nx, ny, nz, hx, hy, hz, _ptr(act), C.byref(nn), C.byref(ne),
                         None, None, None)
    npn = node_count(family, dim)
    coord = np.zeros((nn.value, dim))
    elem = np.zeros((ne.value, npn), dtype=np.int32)
    fine = np.zeros((nn.value, 3), dtype=np.int32)
    L.or_structured_mesh(fam, dim, nx, ny, nz, hx, hy, hz, _ptr(act), C.byref(nn), C.byref(ne),
                         _ptr(coord), _ptr(elem), _ptr(fine))
    return coord, elem, fine


def elastic_moduli(young, poisson):
    k, g = C.c_double(), C.c_double()
    lib().or_elastic_moduli(young, poisson, C.byref(k), C.byref(g))
    return k.value, g.value


def dp_parameters(c0, phi, three_d=True):
    e, c = C.c_double(), C.c_double()
    lib().or_dp_parameters(c0, phi, 1 if three_d else 0, C.byref(e), C.byref(c))
    return e.value, c.value


def _bcast(x, n):
    return _f64(np.broadcast_to(np.asarray(x, dtype=np.float64), (n,)).copy())


def constitutive_elastic(E, G, K):
    E = _f64(E)
    n = E.shape[0]
    S = np.zeros((n, 6))
    DS = np.zeros((n, 36))
    lib().or_constitutive_elastic(n, _ptr(E), _ptr(_bcast(G, n)), _ptr(_bcast(K, n)),
                                  _ptr(S), _ptr(DS))
    return dict(S=S, DS=DS)


def constitutive_vm(E, Ep, Hard, G, K, a, Y):
    E = _f64(E)
    n = E.shape[0]
    out = dict(S=np.zeros((n, 6)), DS=np.zeros((n, 36)), Ep=np.zeros((n, 6)),
               Hard=np.zeros((n, 6)), plastic=np.zeros(n, np.uint8), crit=np.zeros(n))
    lib().or_constitutive_vm(n, _ptr(E), _ptr(_f64(Ep)), _ptr(_f64(Hard)),
                             _ptr(_bcast(G, n)), _ptr(_bcast(K, n)), _ptr(_bcast(a, n)),
                             _ptr(_bcast(Y, n)), _ptr(out["S"]), _ptr(out["DS"]),
                             _ptr(out["Ep"]), _ptr(out["Hard"]), _ptr(out["plastic"]),
                             _ptr(out["crit"]))
    return out


def constitutive_dp(E, Ep, G, K, eta, c):
    E = _f64(E)
    n = E.shape[0]
    out = dict(S=np.zeros((n, 6)), DS=np.zeros((n, 36)), Ep=np.zeros((n, 6)),
               smooth=np.zeros(n, np.uint8), apex=np.zeros(n, np.uint8))
    rc = lib().or_constitutive_dp(n, _ptr(E), _ptr(_f64(Ep)), _ptr(_bcast(G, n)),
                                  _ptr(_bcast(K, n)), _ptr(_bcast(eta, n)), _ptr(_bcast(c, n)),
                                  _ptr(out["S"]), _ptr(out["DS"]), _ptr(out["Ep"]),
                                  _ptr(out["smooth"]), _ptr(out["apex"]))
    if rc != 0:
        raise _err()
    out["plastic"] = out["smooth"] | out["apex"]
    return out


class Csr:
    """Square sparse matrix from the oracle (CSC of a structurally symmetric
    pattern == CSR arrays)."""

    def __init__(self, indptr, indices, data):
        self.indptr, self.indices, self.data = indptr, indices, data

    @property
    def n(self):
        return self.indptr.shape[0] - 1

    @property
    def nnz(self):
        return self.indices.shape[0]

    def to_scipy_csc(self):
        import scipy.sparse as sp
        return sp.csc_matrix((self.data, self.indices, self.indptr), shape=(self.n, self.n))

    def dense(self):
        return self.to_scipy_csc().toarray()


def _take_k(handle):
    L = lib()
    if not handle:
        raise _err()
    rows, nnz = C.c_int64(), C.c_int64()
    L.or_k_info(handle, C.byref(rows), C.byref(nnz))
    indptr = np.zeros(rows.value + 1, np.int64)
    indices = np.zeros(nnz.value, np.int32)
    data = np.zeros(nnz.value)
    L.or_k_copy(handle, _ptr(indptr), _ptr(indices), _ptr(data))
    L.or_k_free(handle)
    return Csr(indptr, indices, data)


class Cache:
    """build_assembly_cache restated (assembly.cpp:148-180)."""

    def __init__(self, family, dim, coord, elem, shear, bulk):
        L = lib()
        self.family, self.dim = family, dim
        coord = _f64(coord)
        elem = np.ascontiguousarray(elem, dtype=np.int32)
        n_q = quadrature(family, dim)[0].shape[0]
        n_int = elem.shape[0] * n_q
        self._h = L.or_cache_build(FAMILIES[family], dim, coord.shape[0], _ptr(coord),
                                   elem.shape[0], _ptr(elem), _ptr(_bcast(shear, n_int)),
                                   _ptr(_bcast(bulk, n_int)))
        if not self._h:
            raise _err()
        info = np.zeros(8, np.int64)
        secs = C.c_double()
        L.or_cache_info(self._h, _ptr(info), C.byref(secs))
        (self.n_int, self.n_dofs, self.nnz, self.nnz_B, self.n_q, self.n_p,
         self.n_strain, self.n_e) = (int(v) for v in info)
        self.elastic_assembly_seconds = secs.value

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            lib().or_cache_free(h)
            self._h = None

    def arrays(self):
        det = np.zeros(self.n_int)
        w = np.zeros(self.n_int)
        inv = np.zeros((self.n_int, self.dim * self.dim))
        lib().or_cache_arrays(self._h, _ptr(det), _ptr(w), _ptr(inv))
        return det, w, inv

    def K_elast(self) -> Csr:
        indptr = np.zeros(self.n_dofs + 1, np.int64)
        indices = np.zeros(self.nnz, np.int32)
        data = np.zeros(self.nnz)
        lib().or_cache_K_elast(self._h, _ptr(indptr), _ptr(indices), _ptr(data))
        return Csr(indptr, indices, data)

    def B(self):
        import scipy.sparse as sp
        indptr = np.zeros(self.n_dofs + 1, np.int64)
        indices = np.zeros(self.nnz_B, np.int32)
        data = np.zeros(self.nnz_B)
        lib().or_cache_B(self._h, _ptr(indptr), _ptr(indices), _ptr(data))
        return sp.csc_matrix((data, indices, indptr), shape=(self.n_strain * self.n_int, self.n_dofs))

    def strains(self, u):
        u = _f64(u)
        E = np.zeros((self.n_int, 6))
        lib().or_cache_strains(self._h, _ptr(u), _ptr(E))
        return E

    def internal_forces(self, S):
        F = np.zeros(self.n_dofs)
        lib().or_cache_internal_forces(self._h, _ptr(_f64(S)), _ptr(F))
        return F

    def tangent(self, DS, plastic) -> Csr:
        DS = _f64(DS)
        pl = np.ascontiguousarray(plastic, dtype=np.uint8)
        return _take_k(lib().or_cache_tangent(self._h, pl.shape[0], _ptr(DS), _ptr(pl)))

    def direct(self, DS) -> Csr:
        return _take_k(lib().or_cache_direct(self._h, _ptr(_f64(DS))))

    def elastic(self) -> Csr:
        return _take_k(lib().or_cache_elastic(self._h))

    def time_iteration(self, model, E, Ep=None, Hard=None, p1=None, p2=None):
        """Reference timed region (solver.cpp:24,28-29); returns (seconds, n_plastic)."""
        n = self.n_int
        npl = C.c_int64()
        secs = lib().or_time_iteration(self._h, model, _ptr(_f64(E)), _ptr(_f64(Ep)),
                                       _ptr(_f64(Hard)),
                                       _ptr(None if p1 is None else _bcast(p1, n)),
                                       _ptr(None if p2 is None else _bcast(p2, n)),
                                       C.byref(npl))
        if secs < 0:
            raise _err()
        return secs, npl.value


class CscMatrix:
    """General (possibly non-square) CSC result of the linalg entry points."""

    def __init__(self, rows, cols, indptr, indices, data):
        self.rows, self.cols = rows, cols
        self.indptr, self.indices, self.data = indptr, indices, data

    @property
    def nnz(self):
        return self.indices.shape[0]

    def dense(self):
        import scipy.sparse as sp
        return sp.csc_matrix((self.data, self.indices, self.indptr),
                             shape=(self.rows, self.cols)).toarray()


def _take_csc(handle):
    L = lib()
    if not handle:
        raise _err()
    rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
    L.or_k_shape(handle, C.byref(rows), C.byref(cols))
    L.or_k_info(handle, C.byref(rows), C.byref(nnz))
    indptr = np.zeros(cols.value + 1, np.int64)
    indices = np.zeros(nnz.value, np.int32)
    data = np.zeros(nnz.value)
    L.or_k_copy(handle, _ptr(indptr), _ptr(indices), _ptr(data))
    L.or_k_free(handle)
    return CscMatrix(rows.value, cols.value, indptr, indices, data)


def from_triplets(rows, cols, values, n_rows, n_cols) -> CscMatrix:
    """linalg.cpp:10-26: duplicates summed, explicit zeros kept."""
    L = lib()
    L.or_from_triplets.restype = _P
    L.or_from_triplets.argtypes = [C.c_int64, _P, _P, _P, C.c_int64, C.c_int64]
    L.or_k_shape.argtypes = [_P, _I64, _I64]
    r = np.ascontiguousarray(rows, np.int64)
    c = np.ascontiguousarray(cols, np.int64)
    v = _f64(values)
    return _take_csc(L.or_from_triplets(r.shape[0], _ptr(r), _ptr(c), _ptr(v), n_rows, n_cols))


def sandwich(B_dense, D_dense) -> CscMatrix:
    """linalg.cpp:28-35 on matrices given densely (stored entries = nonzeros)."""
    L = lib()
    L.or_sandwich.restype = _P
    L.or_sandwich.argtypes = [C.c_int64, _P, _P, _P, C.c_int64, C.c_int64,
                              C.c_int64, _P, _P, _P, C.c_int64]
    L.or_k_shape.argtypes = [_P, _I64, _I64]
    B = np.asarray(B_dense, np.float64)
    D = np.asarray(D_dense, np.float64)
    br, bc = np.nonzero(B)
    dr, dc = np.nonzero(D)
    bv, dv = _f64(B[br, bc]), _f64(D[dr, dc])
    br, bc, dr, dc = (np.ascontiguousarray(x, np.int64) for x in (br, bc, dr, dc))
    return _take_csc(L.or_sandwich(br.shape[0], _ptr(br), _ptr(bc), _ptr(bv), B.shape[0],
                                   B.shape[1], dr.shape[0], _ptr(dr), _ptr(dc), _ptr(dv),
                                   D.shape[0]))
