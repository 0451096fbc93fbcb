"""Seeded synthetic inputs for the BASELINE configurations.

There is no public dataset for this path: inputs are smooth random
displacement fields on the structured meshes, turned into strains E = B u by
the GPU strain kernel, and scaled so a target fraction of integration points
is plastic.  Plastic history is zero (Ep = Hard = 0).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import api
from .mesh import StructuredMesh, structured_mesh

SEED_BASE = 180504155


@dataclass(frozen=True)
class Config:
    """One BASELINE.json configuration."""

    name: str
    family: str
    dim: int
    n: int                    # cells per axis
    model: str                # "elastic" | "vm" | "dp"
    young: float
    poisson: float
    p1: float = 0.0           # VM: a        DP: c0
    p2: float = 0.0           # VM: Y        DP: phi
    target: float = 0.0       # plastic fraction

    @property
    def seed(self) -> int:
        return SEED_BASE + int(self.name[-1])

    def material(self, n_int: int) -> api.MaterialField:
        K, G = api.elastic_moduli(self.young, self.poisson)
        if self.model == "elastic":
            return api.uniform_elastic(n_int, K, G)
        if self.model == "vm":
            return api.uniform_von_mises(n_int, K, G, self.p1, self.p2)
        eta, c = api.dp_parameters(self.p1, self.p2, api.DPMode.three_d)
        return api.uniform_drucker_prager(n_int, K, G, eta, c)

    def mesh(self, n: int | None = None, z_range=None) -> StructuredMesh:
        n = self.n if n is None else n
        return structured_mesh(self.family, self.dim, n, n, n if self.dim == 3 else 0,
                               z_range=z_range)

    def with_(self, **kw) -> "Config":
        d = dict(self.__dict__)
        d.update(kw)
        return Config(**d)


# BASELINE.json "configs" (unit square / cube)
CONFIGS = {
    "cfg1": Config("cfg1", "P1", 2, 256, "elastic", 206900.0, 0.29),
    "cfg2": Config("cfg2", "Q2", 2, 512, "vm", 206900.0, 0.29, 1.0e4, 450.0, 0.30),
    "cfg3": Config("cfg3", "P2", 3, 64, "dp", 1.0e7, 0.48, 450.0, math.pi / 9.0, 0.40),
    "cfg4": Config("cfg4", "Q1", 3, 160, "vm", 206900.0, 0.29, 1.0e4, 450.0, 0.25),
    "cfg5": Config("cfg5", "Q2", 3, 100, "dp", 1.0e7, 0.48, 450.0, math.pi / 9.0, 0.50),
}


def displacement(coord: np.ndarray, seed: int, shear: float = 0.0) -> np.ndarray:
    """u_i(x) = sum_{m<8} a_mi sin(2 pi k_m.x + phi_mi) / |k_m|  (+ shear x_2 on u_1).

    k_m in {1,2,3}^dim, phi ~ U[0, 2 pi), a ~ U[0.5, 1]; rng = default_rng(seed).
    Returns the dof vector (node-major, direction-minor)."""
    rng = np.random.default_rng(seed)
    dim = coord.shape[1]
    k = rng.integers(1, 4, size=(8, dim)).astype(np.float64)
    phi = rng.uniform(0.0, 2.0 * math.pi, size=(8, dim))
    amp = rng.uniform(0.5, 1.0, size=(8, dim))
    u = np.zeros_like(coord)
    for m in range(8):
        arg = 2.0 * math.pi * (coord @ k[m])
        inv = 1.0 / np.linalg.norm(k[m])
        for i in range(dim):
            u[:, i] += amp[m, i] * np.sin(arg + phi[m, i]) * inv
    if shear:
        u[:, 0] += shear * coord[:, 1]
    return u.reshape(-1)


def plastic_fraction(E: torch.Tensor, mat: api.MaterialField, ctx=None) -> float:
    o = api._run_constitutive(E, None, None, mat, want_ds=False, want_D=False, want_hist=False,
                              ctx=ctx)
    return float(o["plastic"].double().mean().item())


def calibrate(E1: torch.Tensor, mat: api.MaterialField, target: float,
              E0: torch.Tensor | None = None, iters: int = 48) -> tuple[float, float]:
    """Scale s so that E = E0 + s E1 has the target plastic fraction.

    target 0 -> half of the first-yield scale; otherwise bisection (the
    fraction is monotone in s at zero history).  Returns (s, fraction)."""
    base = E0 if E0 is not None else torch.zeros_like(E1)

    def frac(s):
        return plastic_fraction(base + s * E1, mat)

    lo, hi = 0.0, 1.0
    while frac(hi) <= max(target, 1e-12) and hi < 1e12:
        lo, hi = hi, hi * 4.0
    if target <= 0.0:
        for _ in range(iters):
            mid = 0.5 * (lo + hi)
            if frac(mid) > 0.0:
                hi = mid
            else:
                lo = mid
        s = 0.5 * lo
        return s, frac(s)
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        if frac(mid) < target:
            lo = mid
        else:
            hi = mid
    return hi, frac(hi)


@dataclass
class Workload:
    cfg: Config
    mesh: StructuredMesh
    cache: api.AssemblyCache
    mat: api.MaterialField
    E: torch.Tensor
    scale: float
    shear: float
    fraction: float


def make_workload(cfg: Config, n: int | None = None, target: float | None = None,
                  device="cuda", z_range=None) -> Workload:
    """Mesh + cache + calibrated strains for one configuration."""
    target = cfg.target if target is None else target
    mesh = cfg.mesh(n, z_range=z_range)
    mat = cfg.material(mesh.n_int)
    cache = api.build_assembly_cache(api.Mesh.from_structured(mesh, device), mat)
    u1 = torch.from_numpy(displacement(mesh.coord, cfg.seed)).to(device)
    E1 = cache.strains(u1)
    if cfg.model == "elastic":
        return Workload(cfg, mesh, cache, mat, E1, 1.0, 0.0, 0.0)
    shear = 0.0
    E0 = None
    if target >= 1.0:
        K, G = api.elastic_moduli(cfg.young, cfg.poisson)
        if cfg.model == "vm":
            gamma = 2.0 * cfg.p2 / (math.sqrt(2.0) * G)
        else:
            eta, c = api.dp_parameters(cfg.p1, cfg.p2)
            gamma = 4.0 * c / G
        shear = gamma
        u0 = torch.from_numpy(displacement(mesh.coord, cfg.seed, 0.0) * 0.0).to(device)
        coord = torch.from_numpy(mesh.coord).to(device)
        u0 = u0.view(-1, cfg.dim)
        u0[:, 0] = gamma * coord[:, 1]
        E0 = cache.strains(u0.reshape(-1))
        # largest perturbation that keeps every point plastic
        lo, hi = 0.0, 1.0
        while plastic_fraction(E0 + hi * E1, mat) >= 1.0 and hi < 1e12:
            lo, hi = hi, hi * 4.0
        for _ in range(40):
            mid = 0.5 * (lo + hi)
            if plastic_fraction(E0 + mid * E1, mat) >= 1.0:
                lo = mid
            else:
                hi = mid
        s = 0.5 * lo
        E = E0 + s * E1
        return Workload(cfg, mesh, cache, mat, E, s, shear, plastic_fraction(E, mat))
    s, f = calibrate(E1, mat, target)
    return Workload(cfg, mesh, cache, mat, (s * E1).contiguous(), s, shear, f)
