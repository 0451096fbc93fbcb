"""Reference-mirror host API over the C-ABI (include/epfem_gpu.h).

Same names, argument meaning and error behaviour as the reference's
constitutive / assembly entry points (/root/reference/proj/include/epfem):

    elastic_moduli, dp_parameters              constitutive.hpp:11-16
    MaterialField, uniform_*                   constitutive.hpp:18-44
    IntegrationState (+ zero)                  constitutive.hpp:48-59
    constitutive_elastic / _vm / _dp           constitutive.hpp:67-93
    evaluate_constitutive                      constitutive.hpp:96-98
    build_assembly_cache, AssemblyCache        assembly.hpp:35-53
    assemble_elastic_stiffness                 assembly.hpp:55
    assemble_tangent_stiffness                 assembly.hpp:59-60
    internal_forces                            assembly.hpp:63
    Error                                      types.hpp:20-22

Arrays are torch tensors on a CUDA device.  A tensor of shape (n_int, 6) has
the bytes of the reference's 6 x n_int column-major ``Mat``; DS is
(n_int, 36), one column-major 6x6 block per row.  Sparse results are
``CsrMatrix`` (int64 row_ptr, int32 col_idx, float64 values) whose arrays
equal the reference's Eigen CSC arrays (K is structurally symmetric).

These calls are synchronous and raise ``Error`` with the reference's message,
like the reference.  The stream-ordered hot path used by the benchmark is
``TangentEngine``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Union

import torch

from . import _lib as L
from .mesh import ElementType, StructuredMesh, node_count, quad_count


class Error(RuntimeError):
    """epfem::Error (types.hpp:20-22)."""


def _check(rc: int):
    if rc != 0:
        raise Error(L.last_error())


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


def _stream_handle(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class Context:
    """One epfem_ctx per (device, stream)."""

    def __init__(self, device: Union[int, torch.device] = 0, stream: Optional[torch.cuda.Stream] = None,
                 synchronous: bool = True):
        dev = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.device = dev
        h = C.c_void_p()
        st = (stream.cuda_stream if stream is not None else _stream_handle(dev))
        _check(L.lib().epfem_ctx_create(dev.index or 0, C.c_void_p(st), C.byref(h)))
        self._h = h
        _check(L.lib().epfem_ctx_set_sync(self._h, 1 if synchronous else 0))

    @property
    def handle(self):
        return self._h

    def set_stream(self, stream: torch.cuda.Stream):
        _check(L.lib().epfem_ctx_set_stream(self._h, C.c_void_p(stream.cuda_stream)))

    def use_current_stream(self):
        _check(L.lib().epfem_ctx_set_stream(self._h, C.c_void_p(_stream_handle(self.device))))

    def sync(self):
        _check(L.lib().epfem_ctx_sync(self._h))

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and L._lib is not None:
            L._lib.epfem_ctx_destroy(h)
            self._h = None


_default_ctx: dict = {}


def default_context(device=None) -> Context:
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    key = dev.index or 0
    ctx = _default_ctx.get(key)
    if ctx is None:
        ctx = Context(key, synchronous=True)
        _default_ctx[key] = ctx
    ctx.use_current_stream()
    return ctx


# ---------------------------------------------------------------------------
# constitutive.hpp

def elastic_moduli(young: float, poisson: float) -> tuple[float, float]:
    """(bulk K, shear G) = (E/(3(1-2nu)), E/(2(1+nu))) (constitutive.cpp:11-18)."""
    k, g = C.c_double(), C.c_double()
    _check(L.lib().epfem_elastic_moduli(young, poisson, C.byref(k), C.byref(g)))
    return k.value, g.value


class DPMode:
    plane_strain = 0
    three_d = 1


def dp_parameters(c0: float, phi: float, mode: int = DPMode.three_d) -> tuple[float, float]:
    """(eta, c) of the Drucker-Prager cone (constitutive.cpp:20-30)."""
    e, c = C.c_double(), C.c_double()
    _check(L.lib().epfem_dp_parameters(c0, phi, mode, C.byref(e), C.byref(c)))
    return e.value, c.value


Scalar = Union[float, torch.Tensor]


@dataclass
class VonMisesParams:
    a: Scalar   # kinematic hardening modulus
    Y: Scalar   # yield stress


@dataclass
class DruckerPragerParams:
    eta: Scalar
    c: Scalar


@dataclass
class MaterialField:
    """Per-integration-point moduli and plastic model (constitutive.hpp:18-38).

    Each field is either a python float (uniform) or a CUDA float64 tensor of
    length n_int.
    """

    n_int: int
    shear: Scalar
    bulk: Scalar
    plastic: Union[None, VonMisesParams, DruckerPragerParams] = None

    def is_elastic(self) -> bool:
        return self.plastic is None

    @property
    def model(self) -> int:
        if self.plastic is None:
            return L.MODEL_ELASTIC
        return L.MODEL_VON_MISES if isinstance(self.plastic, VonMisesParams) else L.MODEL_DRUCKER_PRAGER

    def slice(self, p0: int, p1: int) -> "MaterialField":
        """The field of points [p0, p1): per-point arrays sliced, uniform values kept."""
        cut = (lambda v: v[p0:p1] if isinstance(v, torch.Tensor) else v)
        plastic = self.plastic
        if isinstance(plastic, VonMisesParams):
            plastic = VonMisesParams(cut(plastic.a), cut(plastic.Y))
        elif isinstance(plastic, DruckerPragerParams):
            plastic = DruckerPragerParams(cut(plastic.eta), cut(plastic.c))
        return MaterialField(p1 - p0, cut(self.shear), cut(self.bulk), plastic)

    def view(self) -> L.Material:
        m = L.Material()
        m.model = self.model
        m.n_int = self.n_int

        def put(val, arr_name, u_name):
            if isinstance(val, torch.Tensor):
                if val.numel() != self.n_int or val.dtype != torch.float64 or not val.is_cuda:
                    raise Error("material field: arrays must be float64 CUDA tensors of length n_int")
                setattr(m, arr_name, C.c_void_p(val.contiguous().data_ptr()))
                setattr(m, u_name, 0.0)
            else:
                setattr(m, arr_name, None)
                setattr(m, u_name, float(val))

        put(self.shear, "shear", "shear_u")
        put(self.bulk, "bulk", "bulk_u")
        p1 = p2 = 0.0
        if isinstance(self.plastic, VonMisesParams):
            p1, p2 = self.plastic.a, self.plastic.Y
        elif isinstance(self.plastic, DruckerPragerParams):
            p1, p2 = self.plastic.eta, self.plastic.c
        put(p1, "p1", "p1_u")
        put(p2, "p2", "p2_u")
        return m


def uniform_elastic(n_int: int, bulk: float, shear: float) -> MaterialField:
    return MaterialField(n_int, shear, bulk, None)


def uniform_von_mises(n_int: int, bulk: float, shear: float, a: float, Y: float) -> MaterialField:
    return MaterialField(n_int, shear, bulk, VonMisesParams(a, Y))


def uniform_drucker_prager(n_int: int, bulk: float, shear: float, eta: float, c: float) -> MaterialField:
    return MaterialField(n_int, shear, bulk, DruckerPragerParams(eta, c))


def _f64(n, cols, device):
    return torch.empty((n, cols), dtype=torch.float64, device=device) if cols else \
        torch.empty((n,), dtype=torch.float64, device=device)


def _u8(n, device):
    return torch.empty((n,), dtype=torch.uint8, device=device)


@dataclass
class IntegrationState:
    """constitutive.hpp:48-59 (masks are bool tensors).  ``D``/``flags`` carry
    the compact hot-path form: packed tangent at plastic points and the flag
    byte (include/epfem_gpu.h)."""

    E: torch.Tensor
    Ep: torch.Tensor
    Hard: torch.Tensor
    S: torch.Tensor
    DS: Optional[torch.Tensor]
    plastic_mask: torch.Tensor
    smooth_mask: torch.Tensor
    apex_mask: torch.Tensor
    D: Optional[torch.Tensor] = None
    flags: Optional[torch.Tensor] = None

    @staticmethod
    def zero(n_int: int, device="cuda") -> "IntegrationState":
        z6 = lambda: torch.zeros((n_int, 6), dtype=torch.float64, device=device)
        zb = lambda: torch.zeros((n_int,), dtype=torch.bool, device=device)
        return IntegrationState(z6(), z6(), z6(), z6(),
                                torch.zeros((n_int, 36), dtype=torch.float64, device=device),
                                zb(), zb(), zb())


def _check_strain(E: torch.Tensor, name: str):
    if E.dim() != 2 or E.shape[1] != 6 or E.dtype != torch.float64 or not E.is_cuda:
        raise Error(f"{name}: strains must be a CUDA float64 tensor of shape (n_int, 6)")


def _run_constitutive(E, Ep_prev, Hard_prev, mat: MaterialField, *, want_ds=True, want_D=True,
                      want_hist=True, want_crit=False, ctx=None):
    n = E.shape[0]
    dev = E.device
    ctx = ctx or default_context(dev)
    out = dict(S=_f64(n, 6, dev), flags=_u8(n, dev),
               plastic=_u8(n, dev), smooth=_u8(n, dev), apex=_u8(n, dev))
    if want_D:
        out["D"] = _f64(n, L.D_STRIDE, dev)
    if want_ds:
        out["DS"] = _f64(n, 36, dev)
    if want_hist:
        out["Ep"] = _f64(n, 6, dev)
        out["Hard"] = _f64(n, 6, dev)
    if want_crit:
        out["crit"] = _f64(n, 0, dev)
    o = L.ConstitutiveOut()
    o.S, o.flags = _ptr(out["S"]), _ptr(out["flags"])
    o.D, o.DS = _ptr(out.get("D")), _ptr(out.get("DS"))
    o.Ep, o.Hard = _ptr(out.get("Ep")), _ptr(out.get("Hard"))
    o.plastic_mask, o.smooth_mask, o.apex_mask = _ptr(out["plastic"]), _ptr(out["smooth"]), _ptr(out["apex"])
    o.crit = _ptr(out.get("crit"))
    mv = mat.view()
    E = E.contiguous()
    Ep_prev = None if Ep_prev is None else Ep_prev.contiguous()
    Hard_prev = None if Hard_prev is None else Hard_prev.contiguous()
    _check(L.lib().epfem_constitutive(ctx.handle, C.byref(mv), _ptr(E), _ptr(Ep_prev),
                                      _ptr(Hard_prev), C.byref(o)))
    for k in ("plastic", "smooth", "apex"):
        out[k] = out[k].bool()
    return out


@dataclass
class ElasticEval:
    S: torch.Tensor
    DS: torch.Tensor


@dataclass
class VonMisesEval:
    S: torch.Tensor
    DS: torch.Tensor
    Ep: torch.Tensor
    Hard: torch.Tensor
    plastic_mask: torch.Tensor
    crit: torch.Tensor


@dataclass
class DruckerPragerEval:
    S: torch.Tensor
    DS: torch.Tensor
    Ep: torch.Tensor
    smooth_mask: torch.Tensor
    apex_mask: torch.Tensor


def constitutive_elastic(E: torch.Tensor, mat: MaterialField) -> ElasticEval:
    """S = C E, DS = C at every point (constitutive.cpp:76-88)."""
    _check_strain(E, "constitutive_elastic")
    if mat.n_int != E.shape[0]:
        raise Error("constitutive_elastic: size mismatch")
    el = MaterialField(mat.n_int, mat.shear, mat.bulk, None)
    o = _run_constitutive(E, None, None, el, want_D=False, want_hist=False)
    return ElasticEval(o["S"], o["DS"])


def constitutive_vm(E, Ep_prev, Hard_prev, mat: MaterialField) -> VonMisesEval:
    """Radial return with linear kinematic hardening (constitutive.cpp:90-135)."""
    if not isinstance(mat.plastic, VonMisesParams):
        raise Error("bad_variant_access: material is not von Mises")
    _check_strain(E, "constitutive_vm")
    n = E.shape[0]
    if Ep_prev.shape[0] != n or Hard_prev.shape[0] != n or mat.n_int != n:
        raise Error("constitutive_vm: size mismatch")
    o = _run_constitutive(E, Ep_prev, Hard_prev, mat, want_D=False, want_crit=True)
    return VonMisesEval(o["S"], o["DS"], o["Ep"], o["Hard"], o["plastic"], o["crit"])


def constitutive_dp(E, Ep_prev, mat: MaterialField) -> DruckerPragerEval:
    """Drucker-Prager smooth-portion / apex return (constitutive.cpp:137-196)."""
    if not isinstance(mat.plastic, DruckerPragerParams):
        raise Error("bad_variant_access: material is not Drucker-Prager")
    _check_strain(E, "constitutive_dp")
    n = E.shape[0]
    if Ep_prev.shape[0] != n or mat.n_int != n:
        raise Error("constitutive_dp: size mismatch")
    o = _run_constitutive(E, Ep_prev, None, mat, want_D=False)
    return DruckerPragerEval(o["S"], o["DS"], o["Ep"], o["smooth"], o["apex"])


def evaluate_constitutive(E: torch.Tensor, prev: IntegrationState, mat: MaterialField,
                          *, full_ds: bool = True) -> IntegrationState:
    """Model dispatch used by the Newton loop (constitutive.cpp:198-225).

    Returns E, updated Ep/Hard, S, the reference's full DS (unless
    ``full_ds=False``), the masks and the compact ``D``/``flags``."""
    _check_strain(E, "evaluate_constitutive")
    n = E.shape[0]
    if mat.n_int != n:
        raise Error("evaluate_constitutive: size mismatch")
    if mat.model == L.MODEL_VON_MISES and (prev.Ep.shape[0] != n or prev.Hard.shape[0] != n):
        raise Error("constitutive_vm: size mismatch")
    if mat.model == L.MODEL_DRUCKER_PRAGER and prev.Ep.shape[0] != n:
        raise Error("constitutive_dp: size mismatch")
    ep = prev.Ep if mat.model != L.MODEL_ELASTIC else None
    hd = prev.Hard if mat.model == L.MODEL_VON_MISES else None
    o = _run_constitutive(E, ep, hd, mat, want_ds=full_ds)
    return IntegrationState(E=E, Ep=o["Ep"], Hard=o["Hard"], S=o["S"], DS=o.get("DS"),
                            plastic_mask=o["plastic"], smooth_mask=o["smooth"],
                            apex_mask=o["apex"], D=o["D"], flags=o["flags"])


# ---------------------------------------------------------------------------
# assembly.hpp

@dataclass
class CsrMatrix:
    """Square sparse matrix on the device: CSR == the reference's CSC arrays."""

    row_ptr: torch.Tensor   # int64, n + 1
    col_idx: torch.Tensor   # int32, nnz
    values: torch.Tensor    # float64, nnz

    @property
    def n(self) -> int:
        return self.row_ptr.numel() - 1

    @property
    def shape(self):
        return (self.n, self.n)

    def nonZeros(self) -> int:
        return self.values.numel()

    nnz = property(nonZeros)

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.csr_matrix((self.values.cpu().numpy(), self.col_idx.cpu().numpy(),
                              self.row_ptr.cpu().numpy()), shape=self.shape)

    def matvec(self, x: torch.Tensor, rows_per_chunk: int = 1 << 20) -> torch.Tensor:
        """y = K x with int64 offsets (valid past 2^31 nonzeros), chunked by rows."""
        y = torch.empty((self.n,), dtype=self.values.dtype, device=self.values.device)
        for r0 in range(0, self.n, rows_per_chunk):
            r1 = min(self.n, r0 + rows_per_chunk)
            off = self.row_ptr[r0:r1 + 1]
            a, b = int(off[0]), int(off[-1])
            prod = self.values[a:b] * x[self.col_idx[a:b].long()]
            y[r0:r1] = torch.segment_reduce(prod, "sum", offsets=off - a, unsafe=True)
        return y


@dataclass
class Mesh:
    """Device mesh (mesh.hpp:15-35, geometry only)."""

    elem_type: ElementType
    coord: torch.Tensor   # (n_nodes, dim) float64
    elem: torch.Tensor    # (n_elements, n_p) int32

    @property
    def dim(self):
        return self.elem_type.dim

    @property
    def n_nodes(self):
        return self.coord.shape[0]

    @property
    def n_elements(self):
        return self.elem.shape[0]

    def n_dofs(self):
        return self.dim * self.n_nodes

    @staticmethod
    def from_structured(m: StructuredMesh, device="cuda") -> "Mesh":
        return Mesh(m.elem_type, torch.from_numpy(m.coord).to(device),
                    torch.from_numpy(m.elem).to(device))


class _DeviceArray:
    """__cuda_array_interface__ wrapper around memory owned by the C library."""

    _TYPESTR = {torch.float64: "<f8", torch.int64: "<i8", torch.int32: "<i4", torch.uint8: "|u1"}

    def __init__(self, ptr: int, n: int, dtype):
        self.__cuda_array_interface__ = {
            "shape": (n,), "typestr": self._TYPESTR[dtype], "data": (ptr, False),
            "version": 3, "strides": None}


def _tensor_view(ptr: int, n: int, dtype, device) -> torch.Tensor:
    """Copy a device array owned by the C library into a fresh torch tensor."""
    if n == 0:
        return torch.empty((0,), dtype=dtype, device=device)
    with torch.cuda.device(device):
        return torch.as_tensor(_DeviceArray(ptr, n, dtype), device=device).clone()


class AssemblyCache:
    """build_assembly_cache result (assembly.hpp:35-53), device-resident.

    Holds geometry (det, inv, weight), the CSR pattern, the element->slot map
    and K_elast inside the C library; B itself is never materialised."""

    def __init__(self, mesh: Mesh, mat: MaterialField, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context(mesh.coord.device)
        self.device = mesh.coord.device
        self.mesh = mesh
        self.dim = mesh.dim
        self.n_strain = 6 if mesh.dim == 3 else 3
        coord = mesh.coord.contiguous()
        elem = mesh.elem.contiguous()
        if coord.dtype != torch.float64 or elem.dtype != torch.int32:
            raise Error("build_assembly_cache: coord must be float64 and elem int32")
        if elem.shape[1] != node_count(mesh.elem_type):
            raise Error("build_assembly_cache: element node count mismatch")
        mv = L.MeshView(mesh.dim, mesh.elem_type.code, mesh.n_nodes, mesh.n_elements,
                        C.c_void_p(coord.data_ptr()), C.c_void_p(elem.data_ptr()))
        matv = mat.view()
        self._mat = mat  # keep tensors alive
        h = C.c_void_p()
        _check(L.lib().epfem_cache_build(self.ctx.handle, C.byref(mv), C.byref(matv), C.byref(h)))
        self._h = h
        info = L.CacheInfo()
        _check(L.lib().epfem_cache_get_info(self._h, C.byref(info)))
        self.info = info
        self.n_int = info.n_int
        self.n_q = info.n_q
        self.n_p = info.n_p
        self.nnz = info.nnz
        self.elastic_assembly_seconds = info.build_seconds
        self.shear, self.bulk = mat.shear, mat.bulk
        rp, ci = C.c_void_p(), C.c_void_p()
        _check(L.lib().epfem_cache_pattern(self._h, C.byref(rp), C.byref(ci)))
        self._row_ptr_ptr, self._col_idx_ptr = rp.value, ci.value
        kv = C.c_void_p()
        _check(L.lib().epfem_cache_K_elast(self._h, C.byref(kv)))
        self._kel_ptr = kv.value
        # pattern tensors (copied once; shared by every returned CsrMatrix)
        self.row_ptr = _tensor_view(rp.value, info.n_dofs + 1, torch.int64, self.device)
        self.col_idx = _tensor_view(ci.value, info.nnz, torch.int32, self.device)

    @property
    def handle(self):
        return self._h

    @property
    def K_elast(self) -> CsrMatrix:
        return CsrMatrix(self.row_ptr, self.col_idx,
                         _tensor_view(self._kel_ptr, self.nnz, torch.float64, self.device))

    def K_elast_ptr(self) -> int:
        return self._kel_ptr

    @property
    def jac(self):
        det, w, inv = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(L.lib().epfem_cache_geometry(self._h, C.byref(det), C.byref(w), C.byref(inv)))
        n = self.n_int
        return (_tensor_view(det.value, n, torch.float64, self.device),
                _tensor_view(inv.value, n * self.dim * self.dim, torch.float64, self.device)
                .view(n, self.dim * self.dim))

    @property
    def weight(self) -> torch.Tensor:
        det, w, inv = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(L.lib().epfem_cache_geometry(self._h, C.byref(det), C.byref(w), C.byref(inv)))
        return _tensor_view(w.value, self.n_int, torch.float64, self.device)

    def workspace(self) -> tuple[torch.Tensor, torch.Tensor]:
        """(records, emask) of the last tangent step: symmetric element deltas
        (n_elements x record doubles) and the plastic-point bitmask per
        element (records of elements with mask 0 are stale).  Copies."""
        rec, em, nd = C.c_void_p(), C.c_void_p(), C.c_int64()
        _check(L.lib().epfem_cache_workspace(self._h, C.byref(rec), C.byref(em), C.byref(nd)))
        ne = self.info.n_elements
        r = _tensor_view(rec.value, ne * nd.value, torch.float64, self.device).view(ne, nd.value)
        m = _tensor_view(em.value, ne, torch.int32, self.device)
        return r, m

    def strains(self, u: torch.Tensor) -> torch.Tensor:
        """E = B u, 6 x n_int with 2D rows {0,1,3} (assembly.cpp:135-146)."""
        if u.numel() != self.info.n_dofs or u.dtype != torch.float64:
            raise Error("strains: size mismatch")
        E = torch.empty((self.n_int, 6), dtype=torch.float64, device=self.device)
        self.ctx.use_current_stream()
        _check(L.lib().epfem_strains(self.ctx.handle, self._h, _ptr(u.contiguous()), _ptr(E)))
        return E

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and L._lib is not None:
            L._lib.epfem_cache_destroy(h)
            self._h = None


def build_assembly_cache(mesh: Union[Mesh, StructuredMesh], mat: MaterialField) -> AssemblyCache:
    if isinstance(mesh, StructuredMesh):
        mesh = Mesh.from_structured(mesh)
    return AssemblyCache(mesh, mat)


def assemble_elastic_stiffness(cache: AssemblyCache) -> CsrMatrix:
    """sandwich(B, D_elast) recomputed (assembly.cpp:182-184)."""
    vals = torch.empty((cache.nnz,), dtype=torch.float64, device=cache.device)
    cache.ctx.use_current_stream()
    _check(L.lib().epfem_assemble_elastic(cache.ctx.handle, cache.handle, _ptr(vals)))
    return CsrMatrix(cache.row_ptr, cache.col_idx, vals)


def assemble_tangent_stiffness(cache: AssemblyCache, DS: torch.Tensor,
                               plastic_cols: torch.Tensor) -> CsrMatrix:
    """K_elast + B^T (D_tangent - D_elast) B (assembly.cpp:186-213).

    DS is (n_int, 36) in the reference layout; plastic_cols a bool mask."""
    if DS.dim() != 2 or DS.shape[0] != cache.n_int or DS.shape[1] != 36 or \
            plastic_cols.numel() != cache.n_int:
        raise Error("assemble_tangent_stiffness: size mismatch")
    vals = torch.empty((cache.nnz,), dtype=torch.float64, device=cache.device)
    pm = plastic_cols.to(torch.uint8).contiguous()
    cache.ctx.use_current_stream()
    _check(L.lib().epfem_assemble_tangent_ds(cache.ctx.handle, cache.handle, cache.n_int,
                                             _ptr(DS.contiguous()), _ptr(pm), _ptr(vals)))
    return CsrMatrix(cache.row_ptr, cache.col_idx, vals)


def assemble_tangent_packed(cache: AssemblyCache, D: torch.Tensor, flags: torch.Tensor,
                            out: Optional[torch.Tensor] = None) -> CsrMatrix:
    """Hot-path form: packed D (n_int, 24) at plastic points + flag bytes."""
    if D.shape[0] != cache.n_int or flags.numel() != cache.n_int:
        raise Error("assemble_tangent_stiffness: size mismatch")
    vals = out if out is not None else torch.empty((cache.nnz,), dtype=torch.float64, device=cache.device)
    cache.ctx.use_current_stream()
    _check(L.lib().epfem_assemble_tangent(cache.ctx.handle, cache.handle, cache.n_int,
                                          _ptr(D), _ptr(flags), _ptr(vals)))
    return CsrMatrix(cache.row_ptr, cache.col_idx, vals)


def internal_forces(cache: AssemblyCache, S: torch.Tensor) -> torch.Tensor:
    """F = B^T (weight * S) (assembly.cpp:215-225)."""
    if S.shape[0] != cache.n_int:
        raise Error("internal_forces: size mismatch")
    F = torch.empty((cache.info.n_dofs,), dtype=torch.float64, device=cache.device)
    cache.ctx.use_current_stream()
    _check(L.lib().epfem_internal_forces(cache.ctx.handle, cache.handle, _ptr(S.contiguous()), _ptr(F)))
    return F


def unpack_D(D: torch.Tensor) -> torch.Tensor:
    """Packed (n, 24) tangent -> (n, 36) column-major 6x6 blocks."""
    n = D.shape[0]
    full = torch.zeros((n, 6, 6), dtype=D.dtype, device=D.device)
    for k, (i, j) in enumerate(zip(L.D_ROW, L.D_COL)):
        full[:, j, i] = D[:, k]
        full[:, i, j] = D[:, k]
    return full.reshape(n, 36)


# ---------------------------------------------------------------------------
# Hot path: stream-ordered engine with preallocated buffers

class TangentEngine:
    """One Newton iteration's hot path on device-resident data:

        K1  constitutive  (E, Ep, Hard) -> S, flags, packed D at plastic points
        K2+K6 tangent     K = K_elast + sum_plastic B^T w (D - C) B

    Asynchronous on the current (or given) stream; ``capture()`` records both
    launches in a CUDA graph so a step is one graph launch.
    """

    def __init__(self, cache: AssemblyCache, mat: MaterialField, stream: Optional[torch.cuda.Stream] = None,
                 fused: bool = True):
        self.fused = fused
        self.cache = cache
        self.mat = mat
        self.device = cache.device
        self.stream = stream or torch.cuda.current_stream(self.device)
        self.ctx = Context(self.device.index or 0, stream=self.stream, synchronous=False)
        n = cache.n_int
        self.S = torch.empty((n, 6), dtype=torch.float64, device=self.device)
        self.flags = torch.empty((n,), dtype=torch.uint8, device=self.device)
        self.D = torch.empty((n, L.D_STRIDE), dtype=torch.float64, device=self.device)
        self.K = torch.empty((cache.nnz,), dtype=torch.float64, device=self.device)
        self._mv = mat.view()
        self._out = L.ConstitutiveOut()
        self._out.S, self._out.flags, self._out.D = _ptr(self.S), _ptr(self.flags), _ptr(self.D)
        self.graph = None
        self._graph_inputs = None

    def step(self, E: torch.Tensor, Ep: Optional[torch.Tensor] = None,
             Hard: Optional[torch.Tensor] = None):
        lib = L.lib()
        if self.fused:
            _check(lib.epfem_newton_step(self.ctx.handle, self.cache.handle, C.byref(self._mv),
                                         _ptr(E), _ptr(Ep), _ptr(Hard), C.byref(self._out),
                                         _ptr(self.K)))
            return self.S, self.flags, self.D, self.K
        _check(lib.epfem_constitutive(self.ctx.handle, C.byref(self._mv), _ptr(E), _ptr(Ep),
                                      _ptr(Hard), C.byref(self._out)))
        _check(lib.epfem_assemble_tangent(self.ctx.handle, self.cache.handle, self.cache.n_int,
                                          _ptr(self.D), _ptr(self.flags), _ptr(self.K)))
        return self.S, self.flags, self.D, self.K

    def step_u(self, u: torch.Tensor, Ep: Optional[torch.Tensor] = None,
               Hard: Optional[torch.Tensor] = None, E_out: Optional[torch.Tensor] = None):
        """The step from nodal displacements: E = B u is formed inside
        the constitutive kernel (epfem_newton_step_u); same bits as
        cache.strains(u) followed by step()."""
        _check(L.lib().epfem_newton_step_u(self.ctx.handle, self.cache.handle, C.byref(self._mv),
                                           _ptr(u), _ptr(Ep), _ptr(Hard), C.byref(self._out),
                                           _ptr(E_out), _ptr(self.K)))
        return self.S, self.flags, self.D, self.K

    def step_f(self, E: torch.Tensor, Ep: Optional[torch.Tensor] = None,
               Hard: Optional[torch.Tensor] = None, F: Optional[torch.Tensor] = None):
        """step() plus the internal forces F = B^T (w S) of its stresses
        (internal_forces, assembly.cpp:215-225; the reference forms them every
        Newton iteration, solver.cpp:25) in one call (epfem_newton_step_f),
        bitwise cache.internal_forces(S).  Returns (S, flags, D, K, F)."""
        if F is None:
            F = torch.empty((self.cache.info.n_dofs,), dtype=torch.float64, device=self.device)
        _check(L.lib().epfem_newton_step_f(self.ctx.handle, self.cache.handle, C.byref(self._mv),
                                           _ptr(E), _ptr(Ep), _ptr(Hard), C.byref(self._out),
                                           _ptr(self.K), _ptr(F)))
        return self.S, self.flags, self.D, self.K, F

    def capture(self, E, Ep=None, Hard=None):
        """Record step() on fixed input buffers into a CUDA graph."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.ctx.set_stream(s)
            self.step(E, Ep, Hard)  # warm-up outside capture
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.ctx.set_stream(torch.cuda.current_stream(self.device))
                self.step(E, Ep, Hard)
        torch.cuda.current_stream(self.device).wait_stream(s)
        self.ctx.set_stream(self.stream)
        self.graph = g
        self._graph_inputs = (E, Ep, Hard)
        return g

    def capture_u(self, u, Ep=None, Hard=None, E_out=None):
        """Record step_u() on fixed buffers into a CUDA graph (replay())."""
        s = torch.cuda.Stream(self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.ctx.set_stream(s)
            self.step_u(u, Ep, Hard, E_out)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                self.ctx.set_stream(torch.cuda.current_stream(self.device))
                self.step_u(u, Ep, Hard, E_out)
        torch.cuda.current_stream(self.device).wait_stream(s)
        self.ctx.set_stream(self.stream)
        self.graph = g
        self._graph_inputs = (u, Ep, Hard, E_out)
        return g

    def replay(self):
        with torch.cuda.stream(self.stream):
            self.graph.replay()
        return self.S, self.flags, self.D, self.K

    def sync(self):
        self.ctx.sync()
