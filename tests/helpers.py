"""Shared test helpers: the reference tests' small meshes, a dense
element-loop stiffness oracle (restating tests/test_assembly.cpp:38-98),
and row-scaled comparisons."""
from __future__ import annotations

import math

import numpy as np

FAMILIES = ["P1", "P2", "Q1", "Q2"]
GOLDEN = __import__("os").path.join(__import__("os").path.dirname(__file__), "golden")


def lround(x: float) -> int:
    return int(math.floor(x + 0.5)) if x >= 0 else -int(math.floor(-x + 0.5))


def elastic_body_grid(level: int, family: str, dim: int):
    """build_mesh_elastic_body grid (mesh.cpp:224-238): L-shaped 10x10 minus
    the bottom-left 5x5 block, thickness 1 in 3D."""
    block = 5 << level
    nx = ny = 2 * block
    h = 5.0 / block
    active = np.ones((ny, nx), np.uint8)
    active[:block, :block] = 0
    nz = max(1, lround(1.0 / h)) if dim == 3 else 0
    hz = 1.0 / nz if dim == 3 else 0.0
    return dict(nx=nx, ny=ny, nz=nz, hx=h, hy=h, hz=hz, active=active)


def footing_grid(level: int, family: str, dim: int):
    """build_mesh_footing grid (mesh.cpp:260-275): 10x10 (x 1) domain."""
    quadratic = family in ("P2", "Q2")
    cells = (5 if quadratic else 10) << level
    h = 10.0 / cells
    nz = max(1, lround(1.0 / h)) if dim == 3 else 0
    hz = 1.0 / nz if dim == 3 else 0.0
    return dict(nx=cells, ny=cells, nz=nz, hx=h, hy=h, hz=hz, active=None)


def small_mesh(oracle, family: str, dim: int):
    """tests/test_assembly.cpp:17-21: elastic body (2D) / footing (3D), level 0."""
    g = elastic_body_grid(0, family, dim) if dim == 2 else footing_grid(0, family, dim)
    coord, elem, fine = oracle.structured_mesh(family, dim, g["nx"], g["ny"], g["nz"], g["hx"],
                                               g["hy"], g["hz"], g["active"])
    return coord, elem


def dense_elastic_oracle(oracle, family, dim, coord, elem, bulk, shear):
    """Element loop with its own Jacobian and B block, dense scatter."""
    pts, wq = oracle.quadrature(family, dim)
    _, grads = oracle.basis(family, dim, pts)          # (dim, n_p, n_q)
    n_p, n_q = grads.shape[1], grads.shape[2]
    ns = 6 if dim == 3 else 3
    C6 = np.zeros((6, 6))
    iota = np.array([1, 1, 1, 0, 0, 0.0])
    dev = np.diag([1, 1, 1, 0.5, 0.5, 0.5]) - np.outer(iota, iota) / 3.0
    C6 = bulk * np.outer(iota, iota) + 2.0 * shear * dev
    rows = [0, 1, 2, 3, 4, 5] if dim == 3 else [0, 1, 3]
    Cr = C6[np.ix_(rows, rows)]
    ndof = dim * coord.shape[0]
    K = np.zeros((ndof, ndof))
    for e in range(elem.shape[0]):
        X = coord[elem[e]]                              # (n_p, dim)
        ke = np.zeros((dim * n_p, dim * n_p))
        for q in range(n_q):
            J = grads[:, :, q] @ X                      # J(i,j) = sum_p g_i(p) x_j(p)
            Ji = np.linalg.inv(J)
            dphi = Ji @ grads[:, :, q]                  # (dim, n_p)
            B = np.zeros((ns, dim * n_p))
            for p in range(n_p):
                d = dphi[:, p]
                if dim == 3:
                    B[0, 3 * p] = d[0]; B[1, 3 * p + 1] = d[1]; B[2, 3 * p + 2] = d[2]
                    B[3, 3 * p] = d[1]; B[3, 3 * p + 1] = d[0]
                    B[4, 3 * p + 1] = d[2]; B[4, 3 * p + 2] = d[1]
                    B[5, 3 * p] = d[2]; B[5, 3 * p + 2] = d[0]
                else:
                    B[0, 2 * p] = d[0]; B[1, 2 * p + 1] = d[1]
                    B[2, 2 * p] = d[1]; B[2, 2 * p + 1] = d[0]
            ke += wq[q] * abs(np.linalg.det(J)) * B.T @ Cr @ B
        dofs = (dim * elem[e][:, None] + np.arange(dim)[None, :]).reshape(-1)
        K[np.ix_(dofs, dofs)] += ke
    return K


def row_scaled_error(got_vals, want_vals, row_ptr, base_vals=None):
    """max_ij |dK_ij| / max_k |K_ref(i,k)| (SURVEY.md §8(a) parity definition).

    ``base_vals`` (K_elast) widens the row scale to max_k(|K_ref|, |K_elast|):
    Drucker-Prager apex points have D = 0, so K_elast + dK cancels to round-off
    in rows surrounded by apex points and |K_ref| alone is no scale for the
    rounding of either implementation there."""
    got = np.asarray(got_vals)
    want = np.asarray(want_vals)
    rp = np.asarray(row_ptr)
    diff = np.abs(got - want)
    rows = np.repeat(np.arange(rp.shape[0] - 1), np.diff(rp))
    rowmax = np.zeros(rp.shape[0] - 1)
    np.maximum.at(rowmax, rows, np.abs(want))
    if base_vals is not None:
        np.maximum.at(rowmax, rows, np.abs(np.asarray(base_vals)))
    scale = np.where(rowmax > 0, rowmax, 1.0)
    return float((diff / scale[rows]).max()) if diff.size else 0.0


def sym_block(rng, scale=1.0):
    A = rng.uniform(-scale, scale, size=(6, 6))
    return 0.5 * (A + A.T)


def elastic_C(bulk, shear):
    iota = np.array([1, 1, 1, 0, 0, 0.0])
    dev = np.diag([1, 1, 1, 0.5, 0.5, 0.5]) - np.outer(iota, iota) / 3.0
    return bulk * np.outer(iota, iota) + 2.0 * shear * dev
