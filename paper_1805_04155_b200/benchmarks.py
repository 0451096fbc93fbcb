"""The paper's displacement-driven strip-footing benchmark over the GPU path
(SURVEY §8(f) rank 4): the mesh with its Dirichlet data
(``build_mesh_footing``, proj/src/mesh.cpp:260-291, with ``Mesh::free_mask`` /
``dirichlet_values`` / ``constrain``, mesh.cpp:12-25,212-216) and the load
driver ``run_dp_footing`` (proj/src/benchmarks.cpp:120-205): Drucker-Prager
(E = 1e7, nu = 0.48, c0 = 450, phi = pi/9), adaptive footing displacement
increments (halved on a Newton failure, doubled when the pressure settles),
the normalised footing pressure per step.

Every Newton time step runs on the device (``solver.newton_solve``); the
reaction on the footing comes from ``internal_forces`` (K9).  The host holds
only the mesh numbering and the Dirichlet tables, as the reference does.

The L-shaped elastic body (``build_mesh_elastic_body``, mesh.cpp:222-258)
carries the two traction drivers: ``run_elastic`` (one elastic step under a
volume force and a top traction, benchmarks.cpp:36-66) and ``run_vm_cyclic``
(von Mises, traction cycled 0 -> 1 -> -1 -> 0, benchmarks.cpp:68-118).  Their
external forces come from ``forces.external_forces`` (2D and 3D).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np
import torch

from . import api as A
from .forces import boundary_faces, constant_force, external_forces
from .mesh import StructuredMesh, structured_mesh
from .solver import NewtonSettings, TimeStepRecord, newton_solve


def default_layers(h: float) -> int:
    """mesh.cpp:218-220: 3D extrusion layers tracking the in-plane density."""
    return max(1, int(_lround(1.0 / h)))


def _lround(x: float) -> int:
    """std::lround: halves away from zero (Python's round() is to even)."""
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


@dataclass
class BoundaryMesh:
    """A structured mesh with the reference Mesh's Dirichlet data
    (mesh.hpp:18-34): per node and direction, free or constrained, the fixed
    value and the load pattern scaled by the load factor.  Arrays are
    (n_nodes, dim), so ``reshape(-1)`` is the reference's dof order dim * j + i."""
    mesh: StructuredMesh
    free_dof: np.ndarray
    dirichlet_fixed: np.ndarray
    dirichlet_load: np.ndarray
    neumann_faces: list = field(default_factory=list)  # (element, local face), sorted

    @property
    def dim(self) -> int:
        return self.mesh.dim

    @property
    def n_nodes(self) -> int:
        return self.mesh.n_nodes

    @property
    def n_dofs(self) -> int:
        return self.mesh.n_dofs

    def free_mask(self) -> np.ndarray:
        """Mesh::free_mask (mesh.cpp:12-17)."""
        return self.free_dof.reshape(-1).copy()

    def dirichlet_values(self, load_scale: float) -> np.ndarray:
        """Mesh::dirichlet_values (mesh.cpp:19-27): fixed + scale * load at
        constrained dofs, zero at free ones."""
        v = self.dirichlet_fixed + load_scale * self.dirichlet_load
        return np.where(self.free_dof, 0.0, v).reshape(-1)

    def constrain(self, direction: int, nodes: np.ndarray, fixed: float, load: float) -> None:
        """constrain (mesh.cpp:212-216) on a node set; a later call overrides
        an earlier one on the same (direction, node), as in the reference's
        per-node sequence."""
        self.free_dof[nodes, direction] = False
        self.dirichlet_fixed[nodes, direction] = fixed
        self.dirichlet_load[nodes, direction] = load


def build_mesh_footing(level: int, family: str, dim: int, layers: int = -1) -> BoundaryMesh:
    """build_mesh_footing (mesh.cpp:260-291): the 10 x 10 (x 1) half-domain
    under a rigid rough strip footing of unit width at the top left.  Sides
    slide (u1 = 0), the base slides (u2 = 0), the footing nodes carry
    u2 = -u_D (load pattern -1) and u1 = 0; 3D fronts have u3 = 0."""
    if level < 0:
        raise A.Error("build_mesh_footing: level must be >= 0")
    quadratic = family in ("P2", "Q2")
    cells = (5 if quadratic else 10) << level
    h = 10.0 / cells
    nz, hz = 0, None
    if dim == 3:
        nz = layers if layers > 0 else default_layers(h)
        hz = 1.0 / nz
    m = structured_mesh(family, dim, cells, cells, nz, hx=h, hy=h, hz=hz)
    n = m.n_nodes
    bm = BoundaryMesh(m, np.ones((n, dim), bool), np.zeros((n, dim)), np.zeros((n, dim)))
    amax, bmax, cmax = 2 * cells, 2 * cells, 2 * nz
    a, b, c = m.fine[:, 0], m.fine[:, 1], m.fine[:, 2]
    a_foot = _lround(2.0 / h)  # footing over x1 in [0, 1]: fine coordinate a <= 2 / hx
    bm.constrain(0, np.nonzero((a == 0) | (a == amax))[0], 0.0, 0.0)
    bm.constrain(1, np.nonzero(b == 0)[0], 0.0, 0.0)
    foot = np.nonzero((b == bmax) & (a <= a_foot))[0]
    bm.constrain(1, foot, 0.0, -1.0)  # u2 = -u_D under the footing
    bm.constrain(0, foot, 0.0, 0.0)   # rough footing
    if dim == 3:
        bm.constrain(2, np.nonzero((c == 0) | (c == cmax))[0], 0.0, 0.0)
    return bm


def build_mesh_elastic_body(level: int, family: str, dim: int, layers: int = -1) -> BoundaryMesh:
    """build_mesh_elastic_body (mesh.cpp:222-258): the 10 x 10 (x 1) square
    without its bottom-left 5 x 5 block.  Left side: u1 = 0 (symmetry); bottom:
    u2 = 0 and u1 = u_D (load pattern 1); 3D fronts u3 = 0; Neumann faces on
    the top edge."""
    if level < 0:
        raise A.Error("build_mesh_elastic_body: level must be >= 0")
    block = 5 << level
    cells = 2 * block
    h = 5.0 / block
    nz, hz = 0, None
    if dim == 3:
        nz = layers if layers > 0 else default_layers(h)
        hz = 1.0 / nz
    active = np.ones((cells, cells), bool)
    active[:block, :block] = False  # (j, i): remove the bottom-left block
    m = structured_mesh(family, dim, cells, cells, nz, hx=h, hy=h, hz=hz, active=active)
    n = m.n_nodes
    bm = BoundaryMesh(m, np.ones((n, dim), bool), np.zeros((n, dim)), np.zeros((n, dim)))
    a, b, c = m.fine[:, 0], m.fine[:, 1], m.fine[:, 2]
    bmax, cmax = 2 * cells, 2 * nz
    bm.constrain(0, np.nonzero(a == 0)[0], 0.0, 0.0)  # symmetry on the left
    bottom = np.nonzero(b == 0)[0]
    bm.constrain(1, bottom, 0.0, 0.0)                  # bottom: u.n = 0, u1 = u_D
    bm.constrain(0, bottom, 0.0, 1.0)
    if dim == 3:
        bm.constrain(2, np.nonzero((c == 0) | (c == cmax))[0], 0.0, 0.0)
    from .forces import face_nodes
    faces = face_nodes(family, dim)
    bm.neumann_faces = [(e, f) for e, f in boundary_faces(m)
                        if all(m.fine[m.elem[e, p], 1] == bmax for p in faces[f])]
    return bm


@dataclass
class BenchmarkConfig:
    """benchmarks.hpp:7-19 (the footing's fields)."""
    dim: int = 2
    elem: str = "P1"
    level: int = 1
    layers: int = -1
    newton: NewtonSettings = field(default_factory=NewtonSettings)
    n_steps: int = 40
    du0: float = 1e-3
    u_max: float = 1.0
    theta: float = 1e-3


@dataclass
class RunResults:
    """benchmarks.hpp:26-37 (the footing's fields)."""
    mesh: BoundaryMesh
    records: List[TimeStepRecord] = field(default_factory=list)
    u: Optional[torch.Tensor] = None
    displacement_snapshots: list = field(default_factory=list)
    hardening_snapshots: list = field(default_factory=list)  # (step, mean |Hard| per element)
    n_int: int = 0
    limit_pressure: float = 0.0
    completed: bool = True


def vm_load_scale(t: float) -> float:
    """benchmarks.cpp:31-35: 0 -> 1 on [0, 1], 1 -> -1 on [1, 3], -1 -> 0 on [3, 4]."""
    if t <= 1.0:
        return t
    if t <= 3.0:
        return 2.0 - t
    return t - 4.0


def _cell_mean_hardening(n_elements: int, Hard: torch.Tensor) -> np.ndarray:
    """benchmarks.cpp:15-26: per element, the mean over its points of
    stress_norm(Hard) (voigt.hpp:39-41), summed in point order."""
    h = Hard.cpu().numpy().reshape(n_elements, -1, 6)
    nrm = np.sqrt((h[..., 0] ** 2 + h[..., 1] ** 2 + h[..., 2] ** 2)
                  + 2.0 * (h[..., 3] ** 2 + h[..., 4] ** 2 + h[..., 5] ** 2))
    acc = np.zeros(n_elements)
    for q in range(nrm.shape[1]):
        acc = acc + nrm[:, q]
    return acc / nrm.shape[1]


def _traction_setup(config: BenchmarkConfig, mat_fn, device):
    bm = build_mesh_elastic_body(config.level, config.elem, config.dim, config.layers)
    m = bm.mesh
    bulk, shear = A.elastic_moduli(206900.0, 0.29)
    mat = mat_fn(m.n_int, bulk, shear)
    cache = A.build_assembly_cache(A.Mesh.from_structured(m, device), mat)
    return bm, m, mat, cache, cache.weight.cpu().numpy()


def run_elastic(config: BenchmarkConfig, device="cuda") -> RunResults:
    """run_elastic (benchmarks.cpp:36-66): one elastic step, unit volume force
    and traction 200 in x2, u_D = 0.5 on the bottom segment."""
    bm, m, mat, cache, w = _traction_setup(config, A.uniform_elastic, device)
    out = RunResults(mesh=bm, n_int=cache.n_int)
    dev = cache.device
    e2 = [0.0] * m.dim
    e2[1] = 1.0
    t2 = [0.0] * m.dim
    t2[1] = 200.0
    f = external_forces(m, w, constant_force(e2), constant_force(t2), bm.neumann_faces)
    ft = torch.from_numpy(f).to(dev)
    res = newton_solve(cache, mat, A.IntegrationState.zero(cache.n_int, device=dev),
                       torch.from_numpy(bm.dirichlet_values(0.5)), torch.from_numpy(bm.free_mask()), ft,
                       config.newton)
    rec = res.record
    rec.step, rec.load, rec.derived_scalar = 1, 1.0, float(torch.dot(ft, res.u).item())
    out.u = res.u
    out.records.append(rec)
    out.displacement_snapshots.append((1, res.u))
    return out


def run_vm_cyclic(config: BenchmarkConfig, device="cuda") -> RunResults:
    """run_vm_cyclic (benchmarks.cpp:68-118): von Mises (a = 1e4,
    Y = 450 sqrt(2/3)), traction scale zeta(t_k), t_k = 4k / n_steps, each
    step a newton_solve from the committed state with a warm start; Newton
    failure is an error; snapshots nearest t = 1, 2, 3, 4."""
    bm, m, mat, cache, w = _traction_setup(
        config, lambda n, k, g: A.uniform_von_mises(n, k, g, 1e4, 450.0 * math.sqrt(2.0 / 3.0)), device)
    out = RunResults(mesh=bm, n_int=cache.n_int)
    dev = cache.device
    t2 = [0.0] * m.dim
    t2[1] = 200.0
    f_max = torch.from_numpy(external_forces(m, w, None, constant_force(t2), bm.neumann_faces)).to(dev)
    dirichlet = torch.from_numpy(bm.dirichlet_values(0.0))
    free = torch.from_numpy(bm.free_mask())
    settings = NewtonSettings(eps_newton=config.newton.eps_newton, max_iters=config.newton.max_iters,
                              linear=config.newton.linear, on_failure="error")
    state = A.IntegrationState.zero(cache.n_int, device=dev)
    u_prev = torch.zeros(bm.n_dofs, dtype=torch.float64, device=dev)
    for k in range(1, config.n_steps + 1):
        t = 4.0 * k / config.n_steps
        zeta = vm_load_scale(t)
        res = newton_solve(cache, mat, state, dirichlet, free, zeta * f_max, settings, u_prev)
        state = res.state
        out.u = res.u
        u_prev = res.u
        rec = res.record
        rec.step, rec.load, rec.derived_scalar = k, zeta, float(torch.dot(f_max, res.u).item())
        out.records.append(rec)
        for j in range(1, 5):
            if k == (j * config.n_steps + 2) // 4:
                out.hardening_snapshots.append((k, _cell_mean_hardening(m.n_elements, state.Hard)))
                out.displacement_snapshots.append((k, out.u))
    return out


def run_dp_footing(config: BenchmarkConfig, device="cuda") -> RunResults:
    """run_dp_footing (benchmarks.cpp:120-205) with every Newton step on the GPU."""
    bm = build_mesh_footing(config.level, config.elem, config.dim, config.layers)
    res_all = RunResults(mesh=bm)
    m = bm.mesh
    bulk, shear = A.elastic_moduli(1e7, 0.48)
    eta, cohesion = A.dp_parameters(450.0, math.pi / 9.0,
                                    A.DPMode.three_d if m.dim == 3 else A.DPMode.plane_strain)
    mat = A.uniform_drucker_prager(m.n_int, bulk, shear, eta, cohesion)
    cache = A.build_assembly_cache(A.Mesh.from_structured(m, device), mat)
    res_all.n_int = cache.n_int
    dev = cache.device
    n = bm.n_dofs
    f_ext = torch.zeros(n, dtype=torch.float64, device=dev)
    free = torch.from_numpy(bm.free_mask()).to(dev)
    # footing dofs (x2) carry the load pattern; their reactions give the mean
    # pressure over the unit footing area
    footing = torch.from_numpy(m.dim * np.nonzero(bm.dirichlet_load[:, 1] != 0.0)[0] + 1).to(dev)
    state = A.IntegrationState.zero(cache.n_int, device=dev)
    u_prev = torch.zeros(n, dtype=torch.float64, device=dev)
    u_d, du, p_prev, step, c0 = 0.0, config.du0, 0.0, 0, 450.0
    halve_on_failure = config.newton.on_failure != "error"
    while u_d < config.u_max - 1e-14:
        increment = min(du, config.u_max - u_d)
        solved = False
        while True:
            try:
                dirichlet = torch.from_numpy(bm.dirichlet_values(u_d + increment))
                res = newton_solve(cache, mat, state, dirichlet, free, f_ext, config.newton, u_prev)
                solved = True
                break
            except A.Error:
                if not halve_on_failure:
                    raise
                increment *= 0.5
                if increment < 1e-9 * config.u_max:  # limit load reached
                    break
        if not solved:
            res_all.completed = False
            break
        u_d += increment
        du = increment
        state = res.state
        res_all.u = res.u
        u_prev = res.u
        F = A.internal_forces(cache, state.S)
        reaction = 0.0
        for f in F[footing].cpu().tolist():  # node order, one rounding per add (benchmarks.cpp:177-178)
            reaction += f
        pressure = -reaction  # footing area 1 x 1
        step += 1
        rec = res.record
        rec.step, rec.load, rec.derived_scalar = step, u_d, pressure / c0
        res_all.records.append(rec)
        res_all.limit_pressure = pressure
        if abs(pressure - p_prev) < config.theta * max(abs(pressure), 1e-300):
            du *= 2.0
        p_prev = pressure
    if res_all.records:
        res_all.displacement_snapshots.append((res_all.records[-1].step, res_all.u))
    return res_all


# ------------------------------------------------------------- mesh text I/O
def _g17(x: float) -> str:
    """operator<< on a double at precision(17) (printf %.17g)."""
    return "%.17g" % x


def write_mesh_text(bm: BoundaryMesh, path: str) -> None:
    """write_mesh_text (mesh.cpp:323-354): header, nodes, elements, the
    constrained dofs in (node, direction) order, the Neumann faces."""
    m = bm.mesh
    try:
        out = open(path, "w")
    except OSError:
        raise A.Error("write_mesh_text: cannot open " + path) from None
    with out:
        w = out.write
        w("epfem-mesh 1\n")
        w(f"dim {m.dim}\n")
        w(f"elem {m.elem_type.family}\n")
        w(f"nodes {m.n_nodes}\n")
        for n in range(m.n_nodes):
            w(str(n) + "".join(" " + _g17(float(v)) for v in m.coord[n]) + "\n")
        w(f"elements {m.n_elements} {m.elem.shape[1]}\n")
        for e in range(m.n_elements):
            w(str(e) + "".join(f" {int(v)}" for v in m.elem[e]) + "\n")
        con = np.argwhere(~bm.free_dof)  # row-major: node, then direction
        w(f"dirichlet {con.shape[0]}\n")
        for n, i in con:
            w(f"{n} {i} {_g17(float(bm.dirichlet_fixed[n, i]))} {_g17(float(bm.dirichlet_load[n, i]))}\n")
        w(f"neumann {len(bm.neumann_faces)}\n")
        for e, f in bm.neumann_faces:
            w(f"{e} {f}\n")


def read_mesh_text(path: str) -> BoundaryMesh:
    """read_mesh_text (mesh.cpp:356-410), with its error messages.  The mesh
    carries no fine-grid indices (``fine`` is None)."""
    from .mesh import ElementType, node_count
    try:
        toks = open(path).read().split()
    except OSError:
        raise A.Error("read_mesh_text: cannot open " + path) from None
    pos = 0

    def nxt(conv=str):
        nonlocal pos
        if pos >= len(toks):
            raise A.Error("read_mesh_text: truncated file " + path)
        pos += 1
        try:
            return conv(toks[pos - 1])
        except ValueError:
            raise A.Error("read_mesh_text: truncated file " + path) from None
    if len(toks) < 2 or toks[0] != "epfem-mesh" or toks[1] != "1":
        raise A.Error("read_mesh_text: unrecognized header in " + path)
    pos = 2
    nxt()
    dim = nxt(int)
    nxt()
    family = nxt()
    if family not in ("P1", "P2", "Q1", "Q2"):
        raise A.Error("unknown element family: " + family)
    t = ElementType(family, dim)
    nxt()
    n_nodes = nxt(int)
    coord = np.zeros((n_nodes, dim))
    for _ in range(n_nodes):
        nid = nxt(int)
        for i in range(dim):
            coord[nid, i] = nxt(float)
    nxt()
    n_elems, n_p = nxt(int), nxt(int)
    if n_p != node_count(t):
        raise A.Error("read_mesh_text: node count mismatch for element type")
    elem = np.zeros((n_elems, n_p), np.int32)
    for _ in range(n_elems):
        eid = nxt(int)
        for p in range(n_p):
            v = nxt(int)
            if v < 0 or v >= n_nodes:
                raise A.Error("read_mesh_text: node index out of range")
            elem[eid, p] = v
    m = StructuredMesh(t, coord, elem, None, (0, 0, 0))
    bm = BoundaryMesh(m, np.ones((n_nodes, dim), bool), np.zeros((n_nodes, dim)), np.zeros((n_nodes, dim)))
    nxt()
    for _ in range(nxt(int)):
        n, d, fx, ld = nxt(int), nxt(int), nxt(float), nxt(float)
        bm.constrain(d, np.array([n]), fx, ld)
    nxt()
    for _ in range(nxt(int)):
        bm.neumann_faces.append((nxt(int), nxt(int)))
    return bm
