"""External forces for the paper's load drivers (host side, one-time per
driver, like the reference): ``external_forces`` (proj/src/assembly.cpp:231-296)
with a volume force at the volume quadrature points (weights |det J| w_q from
the device cache) and a traction on the mesh's Neumann faces with the face
rule and the face restriction of the basis (reference_elements.cpp:87-115,
117-135,196-244,392-412,466-498); ``boundary_faces`` (mesh.cpp:293-310).

2D faces are segments (Gauss rules, segment basis); 3D faces use the 2D
volume rule and basis of the same family (triangles for tetrahedra,
quadrilaterals for hexahedra) with the area element |t1 x t2|.
"""
from __future__ import annotations

import math
from typing import Callable, Optional

import numpy as np

from . import api as A
from .mesh import StructuredMesh

ForceField = Callable[[np.ndarray], np.ndarray]  # x (n, dim) -> value (n, dim)

# face_nodes (reference_elements.cpp:466-494), 2D
FACE_NODES_2D = {
    "P1": [[0, 1], [1, 2], [2, 0]],
    "P2": [[0, 1, 3], [1, 2, 4], [2, 0, 5]],
    "Q1": [[0, 1], [1, 2], [2, 3], [3, 0]],
    "Q2": [[0, 1, 4], [1, 2, 5], [2, 3, 6], [3, 0, 7]],
}
FACE_NODES_3D = {
    "P1": [[0, 2, 1], [0, 1, 3], [1, 2, 3], [0, 3, 2]],
    "P2": [[0, 2, 1, 6, 5, 4], [0, 1, 3, 4, 7, 9], [1, 2, 3, 5, 8, 7], [0, 3, 2, 9, 8, 6]],
    "Q1": [[0, 1, 2, 3], [4, 5, 6, 7], [0, 1, 5, 4], [1, 2, 6, 5], [2, 3, 7, 6], [3, 0, 4, 7]],
    "Q2": [[0, 1, 2, 3, 8, 9, 10, 11], [4, 5, 6, 7, 12, 13, 14, 15], [0, 1, 5, 4, 8, 17, 12, 16],
           [1, 2, 6, 5, 9, 18, 13, 17], [2, 3, 7, 6, 10, 19, 14, 18], [3, 0, 4, 7, 11, 16, 15, 19]],
}


def face_nodes(family: str, dim: int) -> list:
    """face_nodes (reference_elements.cpp:466-494)."""
    return (FACE_NODES_2D if dim == 2 else FACE_NODES_3D)[family]


_QUAD_CORNERS = [(-1, -1), (1, -1), (1, 1), (-1, 1)]
_HEX_CORNERS = [(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1),
                (-1, -1, 1), (1, -1, 1), (1, 1, 1), (-1, 1, 1)]
_HEX_EDGES = [(0, -1, -1), (1, 0, -1), (0, 1, -1), (-1, 0, -1), (0, -1, 1), (1, 0, 1),
              (0, 1, 1), (-1, 0, 1), (-1, -1, 0), (1, -1, 0), (1, 1, 0), (-1, 1, 0)]
_QUAD_EDGES = [(0, -1), (1, 0), (0, 1), (-1, 0)]


def constant_force(value) -> ForceField:
    """constant_force (assembly.cpp:227-229)."""
    v = np.asarray(value, dtype=np.float64)
    return lambda x: np.broadcast_to(v, (x.shape[0], v.size))


def gauss_segment(n: int):
    """gauss_segment (reference_elements.cpp:20-44)."""
    if n == 1:
        return np.array([0.0]), np.array([2.0])
    if n == 2:
        g = 1.0 / math.sqrt(3.0)
        return np.array([-g, g]), np.array([1.0, 1.0])
    if n == 3:
        g = math.sqrt(3.0 / 5.0)
        return np.array([-g, 0.0, g]), np.array([5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0])
    raise A.Error("unsupported segment rule")


def _segment_basis(order: int, x: np.ndarray):
    """segment_basis (reference_elements.cpp:87-115): values, d/dx (n_fp, m)."""
    if order == 1:
        return np.stack([0.5 * (1.0 - x), 0.5 * (1.0 + x)]), np.stack([np.full_like(x, -0.5), np.full_like(x, 0.5)])
    return (np.stack([0.5 * x * (x - 1.0), 0.5 * x * (x + 1.0), 1.0 - x * x]),
            np.stack([x - 0.5, x + 0.5, -2.0 * x]))


def volume_rule_2d(family: str):
    """quadrature_volume (reference_elements.cpp:345-374) in 2D: points (2, n_q), weights."""
    if family == "P1":
        return np.full((2, 1), 1.0 / 3.0), np.array([0.5])
    if family == "P2":
        return np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5]]), np.full(3, 1.0 / 6.0)
    x1, w1 = gauss_segment(2 if family == "Q1" else 3)
    n1 = x1.size
    pts = np.zeros((2, n1 * n1))
    w = np.zeros(n1 * n1)
    for q in range(n1 * n1):  # tensor_rule: axis 0 fastest, weight = running product
        idx, acc = q, 1.0
        for i in range(2):
            k = idx % n1
            idx //= n1
            pts[i, q] = x1[k]
            acc *= w1[k]
        w[q] = acc
    return pts, w


def volume_basis_values_2d(family: str, pts: np.ndarray) -> np.ndarray:
    """Shape-function values (n_p, m) of the 2D bases (reference_elements.cpp:117-135,196-244)."""
    x, y = pts[0], pts[1]
    if family == "P1":
        return np.stack([1.0 - x - y, x, y])
    if family == "P2":
        z = 1.0 - x - y
        return np.stack([z * (2 * z - 1), x * (2 * x - 1), y * (2 * y - 1), 4 * z * x, 4 * x * y, 4 * z * y])
    if family == "Q1":
        return np.stack([0.25 * (1 + sx * x) * (1 + sy * y) for sx, sy in _QUAD_CORNERS])
    vals = []
    for sx, sy in _QUAD_CORNERS:
        ax, ay = 1 + sx * x, 1 + sy * y
        vals.append(0.25 * ax * ay * (sx * x + sy * y - 1))
    for sx, sy in _QUAD_EDGES:
        vals.append(0.5 * (1 - x * x) * (1 + sy * y) if sx == 0 else 0.5 * (1 + sx * x) * (1 - y * y))
    return np.stack(vals)


def volume_basis_grads_2d(family: str, pts: np.ndarray) -> np.ndarray:
    """Reference gradients (2, n_p, m) of the 2D bases (reference_elements.cpp:117-135,196-244)."""
    x, y = pts[0], pts[1]
    one, zero = np.ones_like(x), np.zeros_like(x)
    if family == "P1":
        return np.stack([np.stack([-one, one, zero]), np.stack([-one, zero, one])])
    if family == "P2":
        z = 1.0 - x - y
        return np.stack([np.stack([1 - 4 * z, 4 * x - 1, zero, 4 * (z - x), 4 * y, -4 * y]),
                         np.stack([1 - 4 * z, zero, 4 * y - 1, -4 * x, 4 * x, 4 * (z - y)])])
    if family == "Q1":
        return np.stack([np.stack([0.25 * sx * (1 + sy * y) for sx, sy in _QUAD_CORNERS]),
                         np.stack([0.25 * sy * (1 + sx * x) for sx, sy in _QUAD_CORNERS])])
    gx, gy = [], []
    for sx, sy in _QUAD_CORNERS:
        ax, ay = 1 + sx * x, 1 + sy * y
        r = sx * x + sy * y - 1
        gx.append(0.25 * sx * (ay * r + ax * ay))
        gy.append(0.25 * sy * (ax * r + ax * ay))
    for sx, sy in _QUAD_EDGES:
        if sx == 0:
            gx.append(-x * (1 + sy * y))
            gy.append(0.5 * sy * (1 - x * x))
        else:
            gx.append(0.5 * sx * (1 - y * y))
            gy.append(-y * (1 + sx * x))
    return np.stack([np.stack(gx), np.stack(gy)])


def volume_rule_3d(family: str):
    """quadrature_volume (reference_elements.cpp:20-84,345-372) in 3D: points (3, n_q), weights."""
    if family == "P1":
        return np.full((3, 1), 0.25), np.array([1.0 / 6.0])
    if family == "P2":  # the reference's 11-point tetrahedron rule (Keast), its literals
        a, b, f, g = 0.399403576166799, 0.100596423833201, 0.071428571428571, 0.785714285714286
        w1, w2, w3 = -0.013155555555555, 0.007622222222222, 0.024888888888888
        pts = np.array([[0.25, f, g, f, f, a, b, b, a, a, b],
                        [0.25, f, f, g, f, b, a, b, a, b, a],
                        [0.25, f, f, f, g, b, b, a, b, a, a]])
        return pts, np.array([w1, w2, w2, w2, w2, w3, w3, w3, w3, w3, w3])
    x1, w1 = gauss_segment(2 if family == "Q1" else 3)
    n1 = x1.size
    pts = np.zeros((3, n1 ** 3))
    w = np.zeros(n1 ** 3)
    for q in range(n1 ** 3):
        idx, acc = q, 1.0
        for i in range(3):
            k = idx % n1
            idx //= n1
            pts[i, q] = x1[k]
            acc *= w1[k]
        w[q] = acc
    return pts, w


def volume_basis_values_3d(family: str, pts: np.ndarray) -> np.ndarray:
    """Shape-function values (n_p, m) of the 3D bases (reference_elements.cpp:137-194,246-304)."""
    x, y, z = pts[0], pts[1], pts[2]
    if family == "P1":
        return np.stack([1.0 - x - y - z, x, y, z])
    if family == "P2":
        x0 = 1.0 - x - y - z
        return np.stack([x0 * (2 * x0 - 1), x * (2 * x - 1), y * (2 * y - 1), z * (2 * z - 1), 4 * x0 * x,
                         4 * x * y, 4 * x0 * y, 4 * x * z, 4 * y * z, 4 * x0 * z])
    if family == "Q1":
        return np.stack([0.125 * (1 + sx * x) * (1 + sy * y) * (1 + sz * z) for sx, sy, sz in _HEX_CORNERS])
    vals = []
    for sx, sy, sz in _HEX_CORNERS:
        ax, ay, az = 1 + sx * x, 1 + sy * y, 1 + sz * z
        vals.append(0.125 * ax * ay * az * (sx * x + sy * y + sz * z - 2))
    c = (x, y, z)
    for e in _HEX_EDGES:
        v = [1 - c[i] * c[i] if e[i] == 0 else 1 + e[i] * c[i] for i in range(3)]
        vals.append(0.25 * v[0] * v[1] * v[2])
    return np.stack(vals)


def boundary_faces(mesh: StructuredMesh) -> list:
    """boundary_faces (mesh.cpp:293-310): the (element, face) pairs whose node
    set occurs once, sorted."""
    faces = face_nodes(mesh.elem_type.family, mesh.dim)
    table = {}
    for e in range(mesh.n_elements):
        for f, loc in enumerate(faces):
            key = tuple(sorted(int(mesh.elem[e, p]) for p in loc))
            ent = table.setdefault(key, [0, (e, f)])
            ent[0] += 1
    return sorted(v[1] for v in table.values() if v[0] == 1)


def boundary_nodes(mesh: StructuredMesh) -> list:
    """boundary_nodes (mesh.cpp:312-321): the nodes of the boundary faces, ascending."""
    faces = face_nodes(mesh.elem_type.family, mesh.dim)
    on = np.zeros(mesh.n_nodes, bool)
    for e, f in boundary_faces(mesh):
        on[mesh.elem[e, faces[f]]] = True
    return np.nonzero(on)[0].tolist()


def external_forces(mesh: StructuredMesh, weight: np.ndarray, volume_force: Optional[ForceField] = None,
                    traction: Optional[ForceField] = None, neumann_faces: Optional[list] = None) -> np.ndarray:
    """external_forces (assembly.cpp:231-296): f += w * value at every
    (element, point, node, direction) in the reference's loop order (one
    rounding per add, np.add.at is sequential in index order)."""
    dim = mesh.dim
    fam = mesh.elem_type.family
    f = np.zeros(mesh.n_dofs)
    coord, elem = mesh.coord, mesh.elem
    if volume_force is not None:
        if dim == 2:
            pts, _ = volume_rule_2d(fam)
            vals = volume_basis_values_2d(fam, pts)  # (n_p, n_q)
        else:
            pts, _ = volume_rule_3d(fam)
            vals = volume_basis_values_3d(fam, pts)
        n_p, n_q = vals.shape
        # x_q = sum_p N_p(q) x_p, accumulated over p in order
        x = np.zeros((mesh.n_elements, n_q, dim))
        for p in range(n_p):
            x += vals[p][None, :, None] * coord[elem[:, p]][:, None, :]
        value = np.asarray(volume_force(x.reshape(-1, dim)), dtype=np.float64).reshape(mesh.n_elements, n_q, dim)
        w = weight.reshape(mesh.n_elements, n_q)[:, :, None] * vals.T[None, :, :]  # (e, q, p)
        contrib = w[:, :, :, None] * value[:, :, None, :]                        # (e, q, p, i)
        dofs = dim * elem[:, None, :, None] + np.arange(dim)[None, None, None, :]
        dofs = np.broadcast_to(dofs, contrib.shape)
        np.add.at(f, dofs.reshape(-1), contrib.reshape(-1))
    if traction is not None:
        if not neumann_faces:
            raise A.Error("external_forces: traction given but mesh has no Neumann faces")
        if dim == 2:
            quadratic = fam in ("P2", "Q2")
            fx, fw = gauss_segment({"P1": 1, "P2": 2, "Q1": 2, "Q2": 3}[fam])
            vals, g1 = _segment_basis(2 if quadratic else 1, fx)  # (n_fp, n_fq)
            grads = g1[None]                                      # (dim - 1, n_fp, n_fq)
        else:
            fpts, fw = volume_rule_2d(fam)
            vals = volume_basis_values_2d(fam, fpts)
            grads = volume_basis_grads_2d(fam, fpts)
        faces = face_nodes(fam, dim)
        for e, fi in neumann_faces:
            nodes = [int(elem[e, p]) for p in faces[fi]]
            for q in range(fw.size):
                x = np.zeros(dim)
                t = np.zeros((dim - 1, dim))
                for p, node in enumerate(nodes):
                    x += vals[p, q] * coord[node]
                    for k in range(dim - 1):
                        t[k] += grads[k, p, q] * coord[node]
                if dim == 3:
                    a, b = t[0], t[1]
                    cr = (a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0])
                    area = math.sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2])
                else:
                    area = math.sqrt(t[0, 0] * t[0, 0] + t[0, 1] * t[0, 1])
                value = np.asarray(traction(x[None, :]), dtype=np.float64).reshape(dim)
                for p, node in enumerate(nodes):
                    w = fw[q] * area * vals[p, q]
                    for i in range(dim):
                        f[dim * node + i] += w * value[i]
    return f
