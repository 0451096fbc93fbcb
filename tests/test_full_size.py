"""Full-size parity: every BASELINE configuration at its BASELINE size, GPU
hot path against the oracle (north_star: "oracle-matching K/stress/D on all
five configs"; the reference path is evaluate_constitutive +
assemble_tangent_stiffness, constitutive.cpp:198-225, assembly.cpp:186-213).

Per configuration, on the workload bench.py times (make_workload: seeded
smooth displacement, calibrated plastic fraction, zero history):
  * numbering: the product's mesh (paper_1805_04155_b200/mesh.py) equals the
    oracle's restatement of mesh.cpp:36-210 at full size, coordinates bit
    for bit (the pattern follows from it);
  * constitutive, EVERY integration point: plastic / smooth / apex flags and
    S bit for bit, the packed D bit for bit at every plastic point (the
    oracle's D blocks are checked bitwise symmetric, so the 21 packed
    entries are the whole block), oracle run chunk-wise from the same E
    bytes;
  * K: cfg1 and cfg2 whole (pattern bit for bit, values <= 1e-12 row-scaled);
    cfg3-5 (too large for the oracle's int32 indices) on three 2-layer slabs
    -- bottom, middle, top -- assembled by the oracle as meshes of their own
    (tests/fullsize.py; the method is checked on the CPU by
    tests/test_fullsize_method.py): the complete rows of every slab against
    the same global rows of the full-size GPU K, pattern bit for bit with
    global column ids, values <= 1e-12 row-scaled.
"""
import gc as _gc
import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest
import torch

from fullsize import compare_slab_rows, complete_nodes, layer_elements, row_scaled_error, slab_submesh

pytestmark = pytest.mark.gpu

D_ROW = [0, 0, 0, 1, 1, 3, 0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 3, 4, 4, 5]
D_COL = [0, 1, 3, 1, 3, 3, 2, 4, 5, 2, 4, 5, 2, 3, 4, 5, 4, 5, 4, 5, 5]
CHUNK = 1 << 20
FULL_NNZ = {"cfg1": 1_841_156, "cfg2": 49_315_844, "cfg3": 547_739_145,
            "cfg4": 1_001_561_769, "cfg5": 2_118_711_609}  # SURVEY §8 size table


def _oracle_eval(oracle, cfg, E):
    K, G = oracle.elastic_moduli(cfg.young, cfg.poisson)
    if cfg.model == "vm":
        return oracle.constitutive_vm(E, None, None, G, K, cfg.p1, cfg.p2)
    if cfg.model == "dp":
        eta, c = oracle.dp_parameters(cfg.p1, cfg.p2)
        return oracle.constitutive_dp(E, None, G, K, eta, c)
    return None


def _check_points(oracle, cfg, E, S, flags, Dp, pl_index):
    """Every point: flags, S bitwise; D bitwise at plastic points.  Returns
    (n_plastic, n_smooth, n_apex) from the oracle."""
    n = E.shape[0]
    starts = list(range(0, n, CHUNK))
    cols = np.array(D_COL) * 6 + np.array(D_ROW)   # packed k -> column-major 6x6 position
    colsT = np.array(D_ROW) * 6 + np.array(D_COL)

    def one(a):
        b = min(n, a + CHUNK)
        ref = _oracle_eval(oracle, cfg, E[a:b])
        fl = flags[a:b]
        pl = ref["plastic"].astype(bool)
        assert np.array_equal(fl & 1, ref["plastic"]), f"plastic flags differ in [{a}, {b})"
        if cfg.model == "dp":
            assert np.array_equal((fl >> 1) & 1, ref["smooth"]), f"smooth flags differ in [{a}, {b})"
            assert np.array_equal((fl >> 2) & 1, ref["apex"]), f"apex flags differ in [{a}, {b})"
        assert np.array_equal(S[a:b].view(np.uint64), ref["S"].view(np.uint64)), f"S differs in [{a}, {b})"
        # packed rows of this chunk's plastic points
        i0, i1 = np.searchsorted(pl_index, [a, b])
        DS = ref["DS"][pl]
        assert np.array_equal(DS[:, cols].view(np.uint64), DS[:, colsT].view(np.uint64)), "oracle D not symmetric"
        assert np.array_equal(Dp[i0:i1, :21].view(np.uint64), DS[:, cols].view(np.uint64)), \
            f"D differs in [{a}, {b})"
        sm = int(ref["smooth"].sum()) if cfg.model == "dp" else 0
        ap = int(ref["apex"].sum()) if cfg.model == "dp" else 0
        return int(pl.sum()), sm, ap

    with ThreadPoolExecutor(8) as ex:
        res = list(ex.map(one, starts))
    return tuple(int(sum(r[k] for r in res)) for k in range(3))


def _slab_K(oracle, cfg, coord, elem, E, nq, e0, e1):
    K, G = oracle.elastic_moduli(cfg.young, cfg.poisson)
    nodes, cl, el = slab_submesh(coord, elem, e0, e1)
    comp = complete_nodes(elem, coord.shape[0], e0, e1, nodes)
    sc = oracle.Cache(cfg.family, cfg.dim, cl, el, G, K)
    ref = _oracle_eval(oracle, cfg, E[e0 * nq:e1 * nq])
    Ks = sc.tangent(ref["DS"], ref["plastic"])
    return nodes, comp, Ks, sc.K_elast()


def _log(rec):
    """EPFEM_PARITY_LOG=<file>: append one JSON record per configuration
    (the evidence copied into profiles/)."""
    path = os.environ.get("EPFEM_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


@pytest.mark.parametrize("name,variant", [("cfg1", ""), ("cfg2", ""), ("cfg3", ""), ("cfg4", ""), ("cfg5", ""),
                                          ("cfg3", "apex"), ("cfg4", "0.0"), ("cfg4", "0.5"), ("cfg4", "1.0"),
                                          ("cfg5", "0.0"), ("cfg5", "1.0")])
def test_full_size_parity(cuda, oracle, name, variant):
    """variant "apex" (Drucker-Prager): the workload's strains plus the
    hydrostatic tension c / (3 K eta) on every point, the apex threshold of
    a zero deviator, so the apex branch (constitutive.cpp:188-193) is taken
    at a large fraction of the points, as the reference's forced-apex test
    does at its scale (tests/test_constitutive.cpp:432-435).  A numeric
    variant is the plastic fraction of BASELINE's sweeps (configs 4 and 5:
    0 / 25 / 50 / 100 % and 0 / 50 / 100 %; 100 % through a simple shear
    above first yield plus the perturbation, synthetic.make_workload)."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, make_workload
    cfg = CONFIGS[name]
    n = cfg.n
    nz = n if cfg.dim == 3 else 0
    target = float(variant) if variant not in ("", "apex") else None
    wl = make_workload(cfg, device=cuda, target=target)
    coord, elem, _ = oracle.structured_mesh(cfg.family, cfg.dim, n, n, nz)
    assert np.array_equal(wl.mesh.coord.view(np.uint64), coord.view(np.uint64))
    assert np.array_equal(wl.mesh.elem, elem)
    gcache = wl.cache
    nq = gcache.info.n_q
    rp = gcache.row_ptr.cpu().numpy()
    K, G = oracle.elastic_moduli(cfg.young, cfg.poisson)
    # size-independent properties of the whole pattern: SURVEY's nonzero
    # count, columns strictly ascending in every row; K_elast symmetric with
    # the rigid translations in its nullspace
    assert gcache.nnz == FULL_NNZ[name] and rp[0] == 0 and rp[-1] == gcache.nnz
    ci = gcache.col_idx
    starts = torch.zeros(gcache.nnz, dtype=torch.bool, device=cuda)
    starts[gcache.row_ptr[:-1].clamp(max=gcache.nnz - 1)] = True
    assert bool(((ci[1:] > ci[:-1]) | starts[1:]).all())
    Kel_g = gcache.K_elast
    ones = torch.ones(gcache.info.n_dofs, dtype=torch.float64, device=cuda)
    assert float(Kel_g.matvec(ones).abs().max()) <= 1e-9 * float(Kel_g.values.abs().max())
    x = torch.randn(gcache.info.n_dofs, dtype=torch.float64, device=cuda)
    y = torch.randn(gcache.info.n_dofs, dtype=torch.float64, device=cuda)
    lhs, rhs = float(y @ Kel_g.matvec(x)), float(x @ Kel_g.matvec(y))
    assert abs(lhs - rhs) <= 1e-9 * max(abs(lhs), 1.0)
    del ci, starts, ones, x, y

    def fetch(t):
        return lambda v0, v1: t[v0:v1].cpu().numpy()

    if cfg.model == "elastic":
        oc = oracle.Cache(cfg.family, cfg.dim, coord, elem, G, K)
        Kel = oc.K_elast()
        assert np.array_equal(rp, Kel.indptr) and np.array_equal(gcache.col_idx.cpu().numpy(), Kel.indices)
        err = row_scaled_error(gcache.K_elast.values.cpu().numpy(), Kel.data, Kel.indptr)
        assert err <= 1e-12, err
        _log({"config": name, "n_int": int(gcache.n_int), "K": "whole matrix (K_elast)", "rows": int(rp.size - 1),
              "nnz": int(rp[-1]), "pattern": "bitwise", "K_err": err})
        return

    E_run = wl.E
    if variant == "apex":
        eta, c = oracle.dp_parameters(cfg.p1, cfg.p2)
        E_run = wl.E.clone()
        E_run[:, :3] += c / (3.0 * K * eta)
    eng = P.TangentEngine(gcache, wl.mat)
    S, flags, D, Kv = eng.step(E_run)
    eng.sync()
    E_h = E_run.cpu().numpy()
    fl_h = flags.cpu().numpy()
    pl_index = np.flatnonzero(fl_h & 1)
    Dp = D[torch.from_numpy(pl_index).to(cuda)].cpu().numpy()
    npl, nsm, nap = _check_points(oracle, cfg, E_h, S.cpu().numpy(), fl_h, Dp, pl_index)
    assert npl == pl_index.size
    if target == 0.0:
        # an all-elastic iteration returns K bitwise equal to K_elast (assembly.cpp:190)
        assert npl == 0 and torch.equal(Kv, gcache.K_elast.values)
    elif target == 1.0:
        assert npl == fl_h.size
    else:
        assert 0 < npl < fl_h.size
    if variant == "apex":
        assert nap > 0.1 * fl_h.size and nsm > 0.1 * fl_h.size, (nsm, nap)
    rec = {"config": name + (f"+{variant}" if variant else ""), "n_int": int(fl_h.size), "plastic": npl,
           "smooth": nsm, "apex": nap, "flags_S_D": "bitwise, every point"}
    del Dp
    if cfg.dim == 2:
        # whole mesh: the oracle holds cfg2 (49.3 M nonzeros)
        oc = oracle.Cache(cfg.family, cfg.dim, coord, elem, G, K)
        ref = _oracle_eval(oracle, cfg, E_h)
        Kref = oc.tangent(ref["DS"], ref["plastic"])
        assert np.array_equal(rp, Kref.indptr)
        assert np.array_equal(gcache.col_idx.cpu().numpy(), Kref.indices)
        err = row_scaled_error(Kv.cpu().numpy(), Kref.data, Kref.indptr, oc.K_elast().data)
        assert err <= 1e-12, err
        rec.update(K="whole matrix", rows=int(rp.size - 1), nnz=int(rp[-1]), pattern="bitwise", K_err=err)
        _log(rec)
        return
    per = layer_elements(elem, n)
    slabs = [(0, 2), (n // 2 - 1, n // 2 + 1), (n - 2, n)]
    with ThreadPoolExecutor(3) as ex:
        outs = list(ex.map(lambda s: _slab_K(oracle, cfg, coord, elem, E_h, nq, s[0] * per, s[1] * per), slabs))
    total, errs = 0, []
    for nodes, comp, Ks, Kel in outs:
        rows, err = compare_slab_rows(cfg.dim, nodes, comp, Ks, Kel, rp, fetch(gcache.col_idx), fetch(Kv))
        total += rows
        errs.append(err)
    assert total > 0
    rec.update(K=f"complete rows of 2-layer slabs {slabs}", rows=int(total), pattern="bitwise",
               K_err=max(errs), nnz=int(rp[-1]))
    _log(rec)
    del outs, eng, S, flags, D, Kv, wl, gcache
    _gc.collect()
    torch.cuda.empty_cache()
