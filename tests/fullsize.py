"""Test infrastructure: full-size parity of the BASELINE configurations.

The oracle (oracle/epfem_oracle.cpp, the reference algorithm restated with
int32 Eigen-style indices) cannot hold configs 3-5 whole
(nnz(D B) > 2^31, SURVEY §8 size table), so their K is checked on slabs:

  * a slab = the elements of cell layers [k0, k1) along the last axis (z in
    3D).  Elements are numbered in cell order (k, j, i) (mesh.cpp:192-204),
    so a slab is a contiguous element range, and its points a contiguous
    point range;
  * the oracle assembles the slab as a mesh of its own (its nodes renumbered
    by a monotone map, so sorted columns stay sorted) from the SAME strains
    as the full-size GPU run;
  * a node whose every element lies in the slab has its complete K rows in
    the slab's K: those global rows of the full-size GPU K must have the
    oracle's pattern bit for bit (global column ids) and values within
    1e-12 row-scaled.

tests/test_fullsize_method.py checks this comparison itself on the CPU
(slab oracle rows == whole-mesh oracle rows at small sizes).
"""
from __future__ import annotations

import numpy as np



def row_scaled_error(got, want, rp, base=None):
    """helpers.row_scaled_error for large row sets (every row non-empty):
    max |got - want| / max_k max(|want|, |base|) over each row."""
    a = np.abs(want)
    if base is not None:
        a = np.maximum(a, np.abs(base))
    rowmax = np.maximum.reduceat(a, rp[:-1]) if a.size else a
    scale = np.where(rowmax > 0, rowmax, 1.0)
    lens = np.diff(rp)
    return float((np.abs(got - want) / np.repeat(scale, lens)).max()) if a.size else 0.0


def layer_elements(elem: np.ndarray, n_layers: int) -> int:
    """Elements per cell layer of a structured mesh with n_layers layers."""
    assert elem.shape[0] % n_layers == 0
    return elem.shape[0] // n_layers


def slab_submesh(coord: np.ndarray, elem: np.ndarray, e0: int, e1: int):
    """The elements [e0, e1) as a mesh of their own: (nodes, coord_l, elem_l)
    with nodes = sorted global ids of the used nodes (local id = position)."""
    es = elem[e0:e1]
    nodes = np.unique(es)
    elem_l = np.searchsorted(nodes, es).astype(np.int32)
    return nodes, np.ascontiguousarray(coord[nodes]), np.ascontiguousarray(elem_l)


def complete_nodes(elem: np.ndarray, n_nodes: int, e0: int, e1: int, nodes: np.ndarray) -> np.ndarray:
    """Boolean mask over `nodes`: True where every element of the node lies
    in [e0, e1) (element counts in the slab == in the whole mesh)."""
    glob = np.bincount(elem.ravel(), minlength=n_nodes)
    loc = np.bincount(elem[e0:e1].ravel(), minlength=n_nodes)
    return glob[nodes] == loc[nodes]


def global_rows(dim: int, indptr: np.ndarray, indices: np.ndarray, nodes: np.ndarray, local_nodes: np.ndarray):
    """Rows of the local nodes `local_nodes` (ascending) of a slab matrix,
    with columns mapped to global dof ids: (row_ptr relative, global cols,
    value positions into the slab matrix's data)."""
    rows = (dim * local_nodes[:, None] + np.arange(dim)[None, :]).ravel()
    starts, ends = indptr[rows], indptr[rows + 1]
    lens = ends - starts
    rp = np.zeros(rows.size + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    pos = np.repeat(starts - rp[:-1], lens) + np.arange(rp[-1])
    lc = indices[pos].astype(np.int64)
    gc = dim * nodes[lc // dim] + lc % dim
    return rp, gc, pos


def compare_slab_rows(dim, nodes, complete, slab_K, slab_Kel, got_row_ptr, got_col, got_val, tol=1e-12):
    """Compare the complete rows of a slab-oracle matrix with the rows of the
    full-size matrix.  slab_K / slab_Kel: oracle Csr (tangent, K_elast) of
    the slab; got_row_ptr: the full matrix's row_ptr (numpy int64, all rows);
    got_col / got_val: callables (v0, v1) -> numpy arrays of that value range
    of the full matrix (fetched lazily: the full arrays can be tens of GB).
    Returns (rows compared, max row-scaled error)."""
    loc = np.flatnonzero(complete)
    assert loc.size > 0, "slab has no complete node"
    # complete nodes are contiguous in global numbering for a full-width slab
    g = nodes[loc]
    assert np.array_equal(g, np.arange(g[0], g[0] + g.size)), "complete nodes not contiguous"
    r0, r1 = dim * int(g[0]), dim * (int(g[-1]) + 1)
    v0, v1 = int(got_row_ptr[r0]), int(got_row_ptr[r1])
    rp, gcol, pos = global_rows(dim, slab_K.indptr, slab_K.indices, nodes, loc)
    # pattern: bit for bit
    want_rp = got_row_ptr[r0:r1 + 1] - v0
    assert np.array_equal(rp, want_rp), "row lengths differ"
    col = got_col(v0, v1)
    assert np.array_equal(gcol.astype(np.int32), col), "column ids differ"
    # values: row-scaled (rows scaled by max(|K_ref|, |K_elast|) as in test_gpu_parity)
    val = got_val(v0, v1)
    err = row_scaled_error(val, slab_K.data[pos], rp, slab_Kel.data[pos])
    assert err <= tol, err
    return r1 - r0, err
