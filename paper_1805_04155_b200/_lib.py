"""ctypes binding of libepfem_gpu.so (include/epfem_gpu.h).

The shared library is built in-tree by ``paper_1805_04155_b200.build`` (nvcc,
sm_100a).  Loading fails loudly when it is missing: the package has no CPU
compute path to fall back to.
"""
from __future__ import annotations

import ctypes as C
import os

from .build import LIB

_P = C.c_void_p
_I64 = C.c_int64
_D = C.c_double


class Material(C.Structure):
    _fields_ = [("model", C.c_int), ("n_int", _I64), ("shear", _P), ("bulk", _P),
                ("p1", _P), ("p2", _P), ("shear_u", _D), ("bulk_u", _D),
                ("p1_u", _D), ("p2_u", _D)]


class MeshView(C.Structure):
    _fields_ = [("dim", C.c_int), ("family", C.c_int), ("n_nodes", _I64),
                ("n_elements", _I64), ("coord", _P), ("elem", _P)]


class ConstitutiveOut(C.Structure):
    _fields_ = [("S", _P), ("flags", _P), ("D", _P), ("DS", _P), ("Ep", _P), ("Hard", _P),
                ("plastic_mask", _P), ("smooth_mask", _P), ("apex_mask", _P), ("crit", _P)]


class CacheInfo(C.Structure):
    _fields_ = [("dim", C.c_int), ("family", C.c_int), ("n_p", C.c_int), ("n_q", C.c_int),
                ("n_strain", C.c_int), ("max_row_nodes", C.c_int), ("n_nodes", _I64),
                ("n_elements", _I64), ("n_int", _I64), ("n_dofs", _I64), ("nnz", _I64),
                ("build_seconds", _D), ("pattern_seconds", _D), ("elastic_seconds", _D)]


D_STRIDE = 24  # EPFEM_D_STRIDE
FLAG_PLASTIC, FLAG_SMOOTH, FLAG_APEX = 1, 2, 4
MODEL_ELASTIC, MODEL_VON_MISES, MODEL_DRUCKER_PRAGER = 0, 1, 2
FAMILIES = {"P1": 0, "P2": 1, "Q1": 2, "Q2": 3}
# packed D entry k holds D(D_ROW[k], D_COL[k]) (epfem_gpu.h)
D_ROW = [0, 0, 0, 1, 1, 3, 0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 3, 4, 4, 5]
D_COL = [0, 1, 3, 1, 3, 3, 2, 4, 5, 2, 4, 5, 2, 3, 4, 5, 4, 5, 4, 5, 5]

EXPORTS = [
    "epfem_last_error", "epfem_abi_version", "epfem_ctx_create", "epfem_ctx_set_stream",
    "epfem_ctx_set_sync", "epfem_ctx_sync", "epfem_ctx_destroy", "epfem_elastic_moduli",
    "epfem_dp_parameters", "epfem_constitutive", "epfem_cache_build", "epfem_cache_destroy",
    "epfem_cache_get_info", "epfem_cache_pattern", "epfem_cache_K_elast", "epfem_cache_geometry",
    "epfem_cache_workspace",
    "epfem_assemble_elastic", "epfem_assemble_tangent", "epfem_assemble_tangent_ds",
    "epfem_newton_step", "epfem_newton_step_u", "epfem_newton_step_f", "epfem_constitutive_delta", "epfem_assemble_rows", "epfem_assemble_rows_range", "epfem_newton_range",
    "epfem_delta_range", "epfem_strains", "epfem_internal_forces", "epfem_restricted_solve",
    "epfem_restricted_solve_blocked", "epfem_energy_norm",
    "epfem_restricted_solve_direct", "epfem_nccl_unique_id", "epfem_ctx_attach_nccl", "epfem_ctx_set_nccl_comm", "epfem_exchange_interface",
]

_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("EPFEM_GPU_LIB", LIB)  # tuning experiments: an in-tree variant build
    if not os.path.exists(path):
        raise ImportError(
            f"libepfem_gpu.so not found at {path}; build it with "
            "`python -m paper_1805_04155_b200.build` (there is no CPU fallback)")
    L = C.CDLL(path)
    L.epfem_last_error.restype = C.c_char_p
    L.epfem_abi_version.restype = C.c_int
    L.epfem_ctx_create.argtypes = [C.c_int, _P, C.POINTER(_P)]
    L.epfem_ctx_set_stream.argtypes = [_P, _P]
    L.epfem_ctx_set_sync.argtypes = [_P, C.c_int]
    L.epfem_ctx_sync.argtypes = [_P]
    L.epfem_ctx_destroy.argtypes = [_P]
    L.epfem_elastic_moduli.argtypes = [_D, _D, C.POINTER(_D), C.POINTER(_D)]
    L.epfem_dp_parameters.argtypes = [_D, _D, C.c_int, C.POINTER(_D), C.POINTER(_D)]
    L.epfem_constitutive.argtypes = [_P, C.POINTER(Material), _P, _P, _P,
                                     C.POINTER(ConstitutiveOut)]
    L.epfem_cache_build.argtypes = [_P, C.POINTER(MeshView), C.POINTER(Material), C.POINTER(_P)]
    L.epfem_cache_destroy.argtypes = [_P]
    L.epfem_cache_get_info.argtypes = [_P, C.POINTER(CacheInfo)]
    L.epfem_cache_pattern.argtypes = [_P, C.POINTER(_P), C.POINTER(_P)]
    L.epfem_cache_K_elast.argtypes = [_P, C.POINTER(_P)]
    L.epfem_cache_geometry.argtypes = [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]
    L.epfem_cache_workspace.argtypes = [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_I64)]
    L.epfem_assemble_elastic.argtypes = [_P, _P, _P]
    L.epfem_assemble_tangent.argtypes = [_P, _P, _I64, _P, _P, _P]
    L.epfem_assemble_tangent_ds.argtypes = [_P, _P, _I64, _P, _P, _P]
    L.epfem_newton_step.argtypes = [_P, _P, C.POINTER(Material), _P, _P, _P,
                                    C.POINTER(ConstitutiveOut), _P]
    L.epfem_newton_step_u.argtypes = [_P, _P, C.POINTER(Material), _P, _P, _P,
                                      C.POINTER(ConstitutiveOut), _P, _P]
    L.epfem_newton_step_f.argtypes = [_P, _P, C.POINTER(Material), _P, _P, _P,
                                      C.POINTER(ConstitutiveOut), _P, _P]
    L.epfem_constitutive_delta.argtypes = [_P, _P, C.POINTER(Material), _P, _P, _P,
                                           C.POINTER(ConstitutiveOut)]
    L.epfem_assemble_rows.argtypes = [_P, _P, _P]
    L.epfem_assemble_rows_range.argtypes = [_P, _P, _P, C.c_int64, C.c_int64]
    L.epfem_newton_range.argtypes = [_P, _P, C.POINTER(Material), _P, _P, _P,
                                     C.POINTER(ConstitutiveOut), C.c_int64, C.c_int64]
    L.epfem_delta_range.argtypes = [_P, _P, C.c_int64, _P, _P, C.c_int64, C.c_int64]
    L.epfem_strains.argtypes = [_P, _P, _P, _P]
    L.epfem_internal_forces.argtypes = [_P, _P, _P, _P]
    L.epfem_restricted_solve.argtypes = [_P, _I64, _P, _P, _P, _P, _P, _D, _I64, _P, C.POINTER(_I64),
                                         C.POINTER(_D)]
    L.epfem_restricted_solve_blocked.argtypes = [_P, _I64, _P, _P, _P, _P, _P, _D, _I64, C.c_int, _P,
                                                 C.POINTER(_I64), C.POINTER(_D)]
    L.epfem_energy_norm.argtypes = [_P, _I64, _P, _P, _P, _P, C.POINTER(_D)]
    L.epfem_restricted_solve_direct.argtypes = [_P, _I64, _P, _P, _P, _P, _P, _D, _P, C.POINTER(C.c_int),
                                                C.POINTER(_D)]
    L.epfem_nccl_unique_id.argtypes = [_P]
    L.epfem_ctx_attach_nccl.argtypes = [_P, _P, C.c_int, C.c_int]
    L.epfem_ctx_set_nccl_comm.argtypes = [_P, _P, C.c_int, C.c_int]
    L.epfem_exchange_interface.argtypes = [_P, _P, _P, C.c_int64, C.c_int64, C.c_int64, C.c_int64]
    _lib = L
    return L


def last_error() -> str:
    return lib().epfem_last_error().decode()
