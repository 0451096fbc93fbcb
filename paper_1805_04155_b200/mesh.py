"""Structured meshes with the reference's numbering (mesh.cpp:36-210).

The numbering fixes the CSR pattern bit for bit, so the generator follows the
reference exactly: a fine grid at half the cell spacing; nodes are the used
fine points numbered in (z, y, x) lexicographic order; elements are listed in
cell order (k, j, i) and, inside a cell, in the cell-pattern order (Kuhn
tetrahedra with the odd-permutation vertex swap, reference corner/mid-edge
orders).  Coordinates are ``0.5 * h * fine_index`` like the reference.

Vectorised numpy; a 160^3 hex mesh takes a few seconds.  Arrays use the
reference's byte layout: ``coord`` is (n_nodes, dim) C-order == dim x n_nodes
column-major, ``elem`` is (n_elements, n_p) int32 == n_p x n_elements.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import FAMILIES

_NODE_COUNT = {("P1", 2): 3, ("P2", 2): 6, ("Q1", 2): 4, ("Q2", 2): 8,
               ("P1", 3): 4, ("P2", 3): 10, ("Q1", 3): 8, ("Q2", 3): 20}
_QUAD_COUNT = {("P1", 2): 1, ("P2", 2): 3, ("Q1", 2): 4, ("Q2", 2): 9,
               ("P1", 3): 1, ("P2", 3): 11, ("Q1", 3): 8, ("Q2", 3): 27}

_HEX_CORNERS = [(-1, -1, -1), (1, -1, -1), (1, 1, -1), (-1, 1, -1),
                (-1, -1, 1), (1, -1, 1), (1, 1, 1), (-1, 1, 1)]
_HEX_EDGES = [(0, -1, -1), (1, 0, -1), (0, 1, -1), (-1, 0, -1),
              (0, -1, 1), (1, 0, 1), (0, 1, 1), (-1, 0, 1),
              (-1, -1, 0), (1, -1, 0), (1, 1, 0), (-1, 1, 0)]


@dataclass(frozen=True)
class ElementType:
    """epfem::ElementType (reference_elements.hpp:12-17)."""

    family: str
    dim: int

    @property
    def code(self) -> int:
        return FAMILIES[self.family]


def node_count(t: ElementType) -> int:
    return _NODE_COUNT[(t.family, t.dim)]


def quad_count(t: ElementType) -> int:
    return _QUAD_COUNT[(t.family, t.dim)]


def cell_patterns(t: ElementType) -> list[list[tuple[int, int, int]]]:
    """Fine-grid offsets of every element inside one cell (mesh.cpp:36-119)."""
    quadratic = t.family in ("P2", "Q2")
    out = []
    if t.dim == 2:
        if t.family in ("P1", "P2"):
            for tri in (((0, 0), (2, 0), (2, 2)), ((0, 0), (2, 2), (0, 2))):
                nodes = [(x, y, 0) for x, y in tri]
                if quadratic:
                    for a, b in ((0, 1), (1, 2), (0, 2)):
                        nodes.append(((nodes[a][0] + nodes[b][0]) // 2,
                                      (nodes[a][1] + nodes[b][1]) // 2, 0))
                out.append(nodes)
        else:
            nodes = [(0, 0, 0), (2, 0, 0), (2, 2, 0), (0, 2, 0)]
            if quadratic:
                nodes += [(1, 0, 0), (2, 1, 0), (1, 2, 0), (0, 1, 0)]
            out.append(nodes)
        return out
    if t.family in ("P1", "P2"):
        perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
        odd = [False, True, True, False, False, True]
        for perm, is_odd in zip(perms, odd):
            v = [[0, 0, 0]]
            for k in range(3):
                nxt = list(v[-1])
                nxt[perm[k]] += 2
                v.append(nxt)
            if is_odd:
                v[2], v[3] = v[3], v[2]
            nodes = [tuple(x) for x in v]
            if quadratic:
                for a, b in ((0, 1), (1, 2), (0, 2), (1, 3), (2, 3), (0, 3)):
                    nodes.append(tuple((v[a][d] + v[b][d]) // 2 for d in range(3)))
            out.append(nodes)
        return out
    nodes = [tuple(c + 1 for c in p) for p in _HEX_CORNERS]
    if quadratic:
        nodes += [tuple(c + 1 for c in p) for p in _HEX_EDGES]
    out.append(nodes)
    return out


@dataclass
class StructuredMesh:
    """Host-side mesh (numpy)."""

    elem_type: ElementType
    coord: np.ndarray   # (n_nodes, dim) float64
    elem: np.ndarray    # (n_elements, n_p) int32
    fine: np.ndarray    # (n_nodes, 3) int32 fine-grid index per node
    shape: tuple        # (nx, ny, nz)

    @property
    def dim(self) -> int:
        return self.elem_type.dim

    @property
    def n_nodes(self) -> int:
        return self.coord.shape[0]

    @property
    def n_elements(self) -> int:
        return self.elem.shape[0]

    @property
    def n_dofs(self) -> int:
        return self.dim * self.n_nodes

    @property
    def n_int(self) -> int:
        return self.n_elements * quad_count(self.elem_type)


def structured_mesh(family: str, dim: int, nx: int, ny: int, nz: int = 0,
                    hx: float | None = None, hy: float | None = None,
                    hz: float | None = None, active: np.ndarray | None = None,
                    z_range: tuple[int, int] | None = None,
                    slab: tuple[int, int] | None = None) -> StructuredMesh:
    """build_structured (mesh.cpp:136-210) on an nx x ny (x nz) cell grid.

    ``active`` is an (ny, nx) in-plane cell mask (all active by default).
    ``slab=(k0, k1)`` (alias ``z_range`` in 3D) restricts the cells along the
    LAST axis (z in 3D, y in 2D) to k0 <= k < k1: a slab of the full grid,
    numbered as its own mesh.  Because the numbering is last-axis-major, the
    slab's nodes are a contiguous range of the full mesh's nodes, in the same
    order; fine indices and coordinates stay global.
    """
    t = ElementType(family, dim)
    hx = 1.0 / nx if hx is None else hx
    hy = 1.0 / ny if hy is None else hy
    if dim == 3:
        hz = 1.0 / nz if hz is None else hz
    pats = np.array(cell_patterns(t), dtype=np.int64)  # (n_pat, n_p, 3)
    slab = slab if slab is not None else z_range
    k0, k1 = (0, nz) if dim == 3 else (0, 1)
    jlo, jhi = 0, ny
    if slab is not None:
        if dim == 3:
            k0, k1 = slab
        else:
            jlo, jhi = slab
    fx = 2 * nx + 1
    fy = 2 * (jhi - jlo) + 1
    fz = 2 * (k1 - k0) + 1 if dim == 3 else 1
    act = np.ones((ny, nx), dtype=bool) if active is None else np.asarray(active, bool).reshape(ny, nx)
    act = act[jlo:jhi]
    jj, ii = np.nonzero(act)                      # row-major: j slow, i fast (local j)
    kk = np.arange(k1 - k0, dtype=np.int64)
    # cells in (k, j, i) order
    ck = np.repeat(kk, jj.size)
    cj = np.tile(jj.astype(np.int64), kk.size)
    ci = np.tile(ii.astype(np.int64), kk.size)
    # fine ids (local z) of every (cell, pattern, node)
    a = 2 * ci[:, None, None] + pats[None, :, :, 0]
    b = 2 * cj[:, None, None] + pats[None, :, :, 1]
    c = (2 * ck[:, None, None] + pats[None, :, :, 2]) if dim == 3 else np.zeros_like(a)
    fid = (c * fy + b) * fx + a                   # (n_cells, n_pat, n_p)
    used = np.zeros(fx * fy * fz, dtype=bool)
    used[fid.ravel()] = True
    node_of = np.cumsum(used, dtype=np.int64) - 1
    n_nodes = int(used.sum())
    elem = node_of[fid].reshape(-1, pats.shape[1]).astype(np.int32)
    ids = np.flatnonzero(used)
    fa = ids % fx
    fb = (ids // fx) % fy + 2 * jlo
    fc = ids // (fx * fy) + (2 * k0 if dim == 3 else 0)
    coord = np.empty((n_nodes, dim))
    coord[:, 0] = 0.5 * hx * fa
    coord[:, 1] = 0.5 * hy * fb
    if dim == 3:
        coord[:, 2] = 0.5 * hz * fc
    fine = np.stack([fa, fb, fc], axis=1).astype(np.int32)
    return StructuredMesh(t, coord, elem, fine, (nx, ny, nz))
