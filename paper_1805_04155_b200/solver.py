"""The semismooth-Newton time step on the GPU:
``newton_solve`` mirrors proj/src/solver.cpp:7-62 and proj/include/epfem/solver.hpp,
``restricted_solve`` / ``energy_norm`` mirror proj/src/linalg.cpp:69-121.

Every iteration stays on the device: strains E = B u (K8), the step with its
internal forces (constitutive update, tangent K, F = B^T (w S);
epfem_newton_step_f), the restricted solve of K[free, free] du = (f_ext -
F)[free] (the reference's default LinearSolver::direct: device sparse
Cholesky + refinement, epfem_restricted_solve_direct; or its
LinearSolver::conjugate_gradient: Jacobi-preconditioned device CG,
epfem_restricted_solve), and the energy-norm stopping test with K_elast.  The host reads
back only the scalars of the stopping test.
"""
from __future__ import annotations

import ctypes as C
import enum
import warnings
from dataclasses import dataclass, field
from typing import List, Optional

import torch

from . import _lib as L
from .api import (AssemblyCache, CsrMatrix, Error, IntegrationState, MaterialField, TangentEngine, _ptr,
                  evaluate_constitutive)


class SolverError(Error):
    """epfem::SolverError (types.hpp): a linear solve above tolerance."""

    def __init__(self, msg: str, residual: float = float("inf")):
        super().__init__(msg)
        self.residual = residual


class NonConvergenceError(Error):
    """epfem::NonConvergenceError: the Newton iteration did not converge."""


class LinearSolver(enum.Enum):
    direct = 0
    conjugate_gradient = 1


@dataclass
class SolveSettings:
    """linalg.hpp:19-22.  ``direct`` (the default, the reference's
    SimplicialLDLT + up to three refinement sweeps, linalg.cpp:84-96) runs
    epfem_restricted_solve_direct: K[free, free] formed on the device, sparse
    Cholesky (QR when not positive definite) from cuSOLVER, refinement on the
    true residual.  Only when cuSOLVER cannot be loaded does the Jacobi CG
    stand in, with a warning (once per process) and ``SolveInfo.substituted``
    / the time-step record's ``direct_substituted`` saying so."""
    method: LinearSolver = LinearSolver.direct
    rel_tol: float = 1e-10


@dataclass
class NewtonSettings:
    """solver.hpp:9-15.  ``on_failure`` ("halve_step" or "error") is read by
    the load drivers (benchmarks.py), as in the reference."""
    eps_newton: float = 1e-10
    max_iters: int = 25
    linear: SolveSettings = field(default_factory=SolveSettings)
    on_failure: str = "halve_step"


@dataclass
class IterationSample:
    n_plastic: int = 0
    tangent_seconds: float = 0.0


@dataclass
class TimeStepRecord:
    """solver.hpp:22-30 (+ the per-iteration CG counts and stopping ratios)."""
    step: int = 0
    load: float = 0.0            # zeta (traction scale) or u_D
    derived_scalar: float = 0.0  # work (VM) or normalised pressure (DP)
    newton_iters: int = 0
    n_plastic: int = 0
    tangent_seconds: float = 0.0
    iterations: List[IterationSample] = field(default_factory=list)
    linear_iters: List[int] = field(default_factory=list)
    ratios: List[float] = field(default_factory=list)  # |du|_e / (|u_prev|_e + |u|_e) per iteration
    direct_substituted: bool = False  # LinearSolver.direct requested: Jacobi CG stood in


@dataclass
class NewtonResult:
    u: torch.Tensor
    state: IntegrationState
    record: TimeStepRecord


def _mask_u8(free_mask: Optional[torch.Tensor], n: int, device) -> Optional[torch.Tensor]:
    if free_mask is None:
        return None
    if free_mask.numel() != n:
        raise Error("restricted_solve: dimension mismatch")
    return free_mask.to(device=device, dtype=torch.uint8).contiguous()


@dataclass
class SolveInfo:
    """What a restricted_solve did: CG iterations and the true relative residual."""
    iterations: int = 0
    residual: float = 0.0
    substituted: bool = False  # LinearSolver.direct requested, CG ran


_warned_direct = False


def restricted_solve(K: CsrMatrix, rhs: torch.Tensor, free_mask: Optional[torch.Tensor] = None,
                     settings: SolveSettings = SolveSettings(), ctx=None,
                     info: Optional[SolveInfo] = None, block: int = 1) -> torch.Tensor:
    """Solve K[free, free] x = rhs[free]; x is zero on fixed dofs (linalg.cpp:69-115).
    Raises SolverError with the reference's message above tolerance; `info`
    (optional) receives the iteration count and the residual.  ``block`` > 1
    (the mesh dimension) uses the node-block Jacobi preconditioner
    (epfem_restricted_solve_blocked) instead of the scalar one."""
    global _warned_direct
    from .api import default_context
    n = K.n
    if rhs.numel() != n:
        raise Error("restricted_solve: dimension mismatch")
    dev = K.values.device
    ctx = ctx or default_context(dev)
    ctx.use_current_stream()
    x = torch.empty((n,), dtype=torch.float64, device=dev)
    substituted = False
    if settings.method == LinearSolver.direct and block == 1:
        sweeps, res = C.c_int(), C.c_double()
        rc = L.lib().epfem_restricted_solve_direct(ctx.handle, n, _ptr(K.row_ptr), _ptr(K.col_idx),
                                                   _ptr(K.values), _ptr(rhs.contiguous()),
                                                   _ptr(_mask_u8(free_mask, n, dev)), settings.rel_tol, _ptr(x),
                                                   C.byref(sweeps), C.byref(res))
        if rc != 6:  # EPFEM_ERR_UNSUPPORTED: no cuSOLVER (or past int32 sizes) -> CG below
            if info is not None:
                info.iterations, info.residual, info.substituted = sweeps.value, res.value, False
            if rc == 7:  # EPFEM_ERR_SOLVER
                raise SolverError(L.last_error(), res.value)
            if rc != 0:
                raise Error(L.last_error())
            return x
        substituted = True
        if not _warned_direct:
            _warned_direct = True
            warnings.warn("restricted_solve: LinearSolver.direct is unavailable on this device ("
                          + L.last_error() + "); Jacobi-preconditioned CG runs under the same tolerance",
                          RuntimeWarning, stacklevel=2)
    it, res = C.c_int64(), C.c_double()
    rc = L.lib().epfem_restricted_solve_blocked(ctx.handle, n, _ptr(K.row_ptr), _ptr(K.col_idx),
                                                _ptr(K.values), _ptr(rhs.contiguous()),
                                                _ptr(_mask_u8(free_mask, n, dev)), settings.rel_tol, 0, int(block),
                                                _ptr(x), C.byref(it), C.byref(res))
    if info is not None:
        info.iterations, info.residual, info.substituted = it.value, res.value, substituted
    if rc == 7:  # EPFEM_ERR_SOLVER
        raise SolverError(L.last_error(), res.value)
    if rc != 0:
        raise Error(L.last_error())
    return x


def energy_norm(K: CsrMatrix, v: torch.Tensor, ctx=None) -> float:
    """sqrt(max(v . K v, 0)) (linalg.cpp:117-121)."""
    from .api import default_context
    if v.numel() != K.n:
        raise Error("energy_norm: dimension mismatch")
    ctx = ctx or default_context(K.values.device)
    ctx.use_current_stream()
    out = C.c_double()
    rc = L.lib().epfem_energy_norm(ctx.handle, K.n, _ptr(K.row_ptr), _ptr(K.col_idx), _ptr(K.values),
                                   _ptr(v.contiguous()), C.byref(out))
    if rc != 0:
        raise Error(L.last_error())
    return out.value


def newton_solve(cache: AssemblyCache, mat: MaterialField, state_prev: IntegrationState,
                 dirichlet: torch.Tensor, free_mask: torch.Tensor, f_ext: torch.Tensor,
                 settings: NewtonSettings = NewtonSettings(),
                 u_start: Optional[torch.Tensor] = None) -> NewtonResult:
    """One time step of the semismooth Newton iteration (solver.cpp:7-62):
    starts from the Dirichlet lift (free dofs from u_start when given), stops
    on |du|_e <= eps (|u_prev|_e + |u|_e) in the K_elast energy norm
    (converged at once when both vanish), commits Ep / Hard from a final
    constitutive evaluation at the converged displacement."""
    if settings.eps_newton <= 0.0 or settings.max_iters < 1:
        raise Error("newton_solve: invalid settings")
    dev = cache.device
    n = cache.info.n_dofs
    free = free_mask.to(device=dev, dtype=torch.bool)
    u = dirichlet.to(device=dev, dtype=torch.float64).clone()
    if u_start is not None:
        u = torch.where(free, u_start.to(dev, torch.float64), u)
    fext = f_ext.to(device=dev, dtype=torch.float64)
    Ke = cache.K_elast
    eng = TangentEngine(cache, mat)
    ep = state_prev.Ep if mat.model != L.MODEL_ELASTIC else None
    hd = state_prev.Hard if mat.model == L.MODEL_VON_MISES else None
    F = torch.empty((n,), dtype=torch.float64, device=dev)
    rec = TimeStepRecord()
    converged = False
    for it in range(1, settings.max_iters + 1):
        E = cache.strains(u)
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        S, flags, D, Kv, F = eng.step_f(E, ep, hd, F)
        t1.record()
        Kt = CsrMatrix(cache.row_ptr, cache.col_idx, Kv)
        lin = SolveInfo()
        # scalar Jacobi CG (Eigen's iterates) for both methods: the node-block
        # preconditioner (block = dim) saved only 5-28 % of the CG iterations
        # on the footing (tools/footing_bench.py)
        du = restricted_solve(Kt, fext - F, free, settings.linear, ctx=eng.ctx, info=lin)
        torch.cuda.synchronize(dev)
        n_pl = int((flags & 1).sum().item())
        rec.iterations.append(IterationSample(n_pl, t0.elapsed_time(t1) * 1e-3))
        rec.linear_iters.append(lin.iterations)
        rec.direct_substituted = rec.direct_substituted or lin.substituted
        rec.tangent_seconds += rec.iterations[-1].tangent_seconds
        rec.newton_iters = it
        norm_prev = energy_norm(Ke, u, ctx=eng.ctx)
        u = u + du
        norm_curr = energy_norm(Ke, u, ctx=eng.ctx)
        denom = norm_prev + norm_curr
        ndu = energy_norm(Ke, du, ctx=eng.ctx)
        rec.ratios.append(ndu / denom if denom > 0.0 else 0.0)
        if denom == 0.0 or ndu <= settings.eps_newton * denom:
            converged = True
            break
    if not converged:
        err = NonConvergenceError(f"newton_solve: no convergence within {settings.max_iters} iterations")
        err.record = rec
        raise err
    state = evaluate_constitutive(cache.strains(u), state_prev, mat)
    rec.n_plastic = int(state.plastic_mask.sum().item())
    return NewtonResult(u=u, state=state, record=rec)
