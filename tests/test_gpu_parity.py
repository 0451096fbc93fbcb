"""GPU parity: the C-ABI kernels against the pinned CPU oracle.

Bar (BASELINE.json north_star):
  * CSR pattern (row_ptr, col_idx) and plastic / smooth / apex flags bit-exact;
  * K row-scaled |dK_ij| <= 1e-12 max_k |K_ref(i,k)|;
  * S within 1e-12 of max(|sigma|_inf, yield); D within 1e-12 ||C||_max —
    the constitutive kernel reproduces the oracle's operation order without
    FMA, so S/D/Ep/Hard are in fact compared bit for bit;
  * an all-elastic iteration returns K bitwise equal to K_elast.
"""
import math
import os

import numpy as np
import pytest
import torch

from helpers import FAMILIES, GOLDEN, elastic_C, row_scaled_error, small_mesh, sym_block

pytestmark = pytest.mark.gpu


def _g(name):
    return np.load(os.path.join(GOLDEN, name + ".npy"))


def _t(a, dev, dtype=torch.float64):
    return torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dtype)


def _np(t):
    return t.detach().cpu().numpy()


def _blocks(DS):
    return DS.reshape(-1, 6, 6).transpose(0, 2, 1)


# ---------------------------------------------------------------------------
# K1 constitutive

def test_vm_batch_bitwise_vs_oracle(cuda, oracle):
    import paper_1805_04155_b200 as P
    E, Ep, H = _g("vm_E"), _g("vm_Ep"), _g("vm_Hard")
    G, K, a, Y = _g("vm_G"), _g("vm_K"), _g("vm_a"), _g("vm_Y")
    ref = oracle.constitutive_vm(E, Ep, H, G, K, a, Y)
    n = E.shape[0]
    mat = P.MaterialField(n, _t(G, cuda), _t(K, cuda), P.VonMisesParams(_t(a, cuda), _t(Y, cuda)))
    ev = P.constitutive_vm(_t(E, cuda), _t(Ep, cuda), _t(H, cuda), mat)
    assert np.array_equal(_np(ev.plastic_mask).astype(np.uint8), ref["plastic"])
    for k, got in (("S", ev.S), ("DS", ev.DS), ("Ep", ev.Ep), ("Hard", ev.Hard), ("crit", ev.crit)):
        assert np.array_equal(_np(got), ref[k]), k
    st = P.evaluate_constitutive(_t(E, cuda), P.IntegrationState(_t(E, cuda), _t(Ep, cuda), _t(H, cuda),
                                 None, None, None, None, None), mat)
    pl = ref["plastic"].astype(bool)
    assert np.array_equal(_np(st.flags) & 1, ref["plastic"])
    D = _np(P.unpack_D(st.D))[pl]
    assert np.array_equal(D, ref["DS"][pl])


def test_dp_batch_bitwise_vs_oracle(cuda, oracle):
    import paper_1805_04155_b200 as P
    E, Ep = _g("dp_E"), _g("dp_Ep")
    G, K, eta, c = _g("dp_G"), _g("dp_K"), _g("dp_eta"), _g("dp_c")
    ref = oracle.constitutive_dp(E, Ep, G, K, eta, c)
    n = E.shape[0]
    mat = P.MaterialField(n, _t(G, cuda), _t(K, cuda), P.DruckerPragerParams(_t(eta, cuda), _t(c, cuda)))
    ev = P.constitutive_dp(_t(E, cuda), _t(Ep, cuda), mat)
    assert np.array_equal(_np(ev.smooth_mask).astype(np.uint8), ref["smooth"])
    assert np.array_equal(_np(ev.apex_mask).astype(np.uint8), ref["apex"])
    for k, got in (("S", ev.S), ("DS", ev.DS), ("Ep", ev.Ep)):
        assert np.array_equal(_np(got), ref[k]), k
    prev = P.IntegrationState(_t(E, cuda), _t(Ep, cuda), torch.zeros((n, 6), dtype=torch.float64, device=cuda),
                              None, None, None, None, None)
    st = P.evaluate_constitutive(_t(E, cuda), prev, mat)
    fl = _np(st.flags)
    assert np.array_equal((fl >> 1) & 1, ref["smooth"]) and np.array_equal((fl >> 2) & 1, ref["apex"])
    assert np.abs(_np(st.Hard)).max() == 0.0  # evaluate_constitutive keeps Hard = 0 for DP
    pl = ref["plastic"].astype(bool)
    assert np.array_equal(_np(P.unpack_D(st.D))[pl], ref["DS"][pl])


def test_elastic_model_and_uniform_material(cuda, oracle):
    import paper_1805_04155_b200 as P
    E = np.random.default_rng(3).uniform(-1, 1, (777, 6))
    K, G = 2.0, 1.5
    ref = oracle.constitutive_elastic(E, G, K)
    ev = P.constitutive_elastic(_t(E, cuda), P.uniform_elastic(777, K, G))
    assert np.array_equal(_np(ev.S), ref["S"]) and np.array_equal(_np(ev.DS), ref["DS"])


def test_constitutive_known_answers(cuda):
    import paper_1805_04155_b200 as P
    G, K, eta, c = 1.2, 2.1, 0.4, 0.6
    E = torch.zeros((2, 6), dtype=torch.float64, device=cuda)
    E[1, :3] = 10.0
    ev = P.constitutive_dp(E, torch.zeros_like(E), P.uniform_drucker_prager(2, K, G, eta, c))
    assert not bool(ev.apex_mask[0]) and bool(ev.apex_mask[1])
    assert torch.allclose(ev.S[1, :3], torch.full((3,), c / eta, dtype=torch.float64, device=cuda), rtol=1e-13)
    assert float(ev.DS[1].abs().max()) == 0.0
    E = torch.zeros((1, 6), dtype=torch.float64, device=cuda)
    E[0, 3] = 2.0
    ev = P.constitutive_vm(E, torch.zeros_like(E), torch.zeros_like(E), P.uniform_von_mises(1, 1.7, 1.1, 0.0, 0.8))
    assert bool(ev.plastic_mask[0]) and float(ev.Hard.abs().max()) == 0.0


def test_constitutive_size_mismatch_raises(cuda):
    import paper_1805_04155_b200 as P
    E = torch.zeros((4, 6), dtype=torch.float64, device=cuda)
    with pytest.raises(P.Error, match="constitutive_vm: size mismatch"):
        P.constitutive_vm(E, E[:3], E, P.uniform_von_mises(4, 1, 1, 0, 1))


# ---------------------------------------------------------------------------
# assembly, all eight element types

def _caches(cuda, oracle, family, dim, young=10.0, nu=0.3):
    import paper_1805_04155_b200 as P
    coord, elem = small_mesh(oracle, family, dim)
    K, G = oracle.elastic_moduli(young, nu)
    ocache = oracle.Cache(family, dim, coord, elem, G, K)
    mesh = P.Mesh(P.ElementType(family, dim), _t(coord, cuda), _t(elem, cuda, torch.int32))
    gcache = P.build_assembly_cache(mesh, P.uniform_elastic(ocache.n_int, K, G))
    return ocache, gcache, K, G


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("family", FAMILIES)
def test_pattern_and_elastic_stiffness(cuda, oracle, family, dim):
    import paper_1805_04155_b200 as P
    oc, gc, K, G = _caches(cuda, oracle, family, dim)
    ref = oc.K_elast()
    assert gc.nnz == ref.nnz
    assert np.array_equal(_np(gc.row_ptr), ref.indptr)
    assert np.array_equal(_np(gc.col_idx), ref.indices)
    kel = _np(gc.K_elast.values)
    assert row_scaled_error(kel, ref.data, ref.indptr) <= 1e-12
    # recomputed elastic assembly is deterministic
    again = _np(P.assemble_elastic_stiffness(gc).values)
    assert np.array_equal(again.view(np.uint64), kel.view(np.uint64))
    # geometry (jacobians, assembly.cpp:20-61) bit for bit: the kernel rounds
    # every product and sum in the reference's order (delta.cuh point_geometry)
    det, w, inv = oc.arrays()
    gdet, ginv = gc.jac
    assert np.array_equal(_np(gdet).view(np.uint64), det.view(np.uint64))
    assert np.array_equal(_np(gc.weight).view(np.uint64), w.view(np.uint64))
    assert np.array_equal(_np(ginv).reshape(inv.shape).view(np.uint64), inv.view(np.uint64))


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("family", FAMILIES)
def test_tangent_matches_oracle(cuda, oracle, family, dim):
    import paper_1805_04155_b200 as P
    oc, gc, K, G = _caches(cuda, oracle, family, dim, 5.0, 0.2)
    rng = np.random.default_rng(41)
    C = elastic_C(K, G)
    n = oc.n_int
    kel = _np(gc.K_elast.values)
    for frac in (0.0, 0.5, 1.0):
        pl = (rng.uniform(size=n) < frac).astype(np.uint8)
        D = np.stack([C + 0.3 * sym_block(rng) if p else C for p in pl])
        DS = D.transpose(0, 2, 1).reshape(n, 36).copy()
        ref = oc.tangent(DS, pl)
        got = P.assemble_tangent_stiffness(gc, _t(DS, cuda), _t(pl, cuda, torch.uint8).bool())
        gv = _np(got.values)
        assert row_scaled_error(gv, ref.data, ref.indptr, kel) <= 1e-12, frac
        # packed hot-path layout
        Dp = np.zeros((n, 24))
        from paper_1805_04155_b200._lib import D_COL, D_ROW
        Dp[:, :21] = D[:, D_ROW, D_COL]
        gp = _np(P.assemble_tangent_packed(gc, _t(Dp, cuda), _t(pl, cuda, torch.uint8)).values)
        assert np.array_equal(gp.view(np.uint64), gv.view(np.uint64))
        if frac == 0.0:
            assert np.array_equal(gv.view(np.uint64), kel.view(np.uint64))


@pytest.mark.parametrize("model", ["vm", "dp"])
@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("family", FAMILIES)
def test_fused_step_all_element_types(cuda, oracle, family, dim, model):
    """The fused Newton step (each element type's default kernel: 2D warp,
    3D tetrahedra warp / row pairs, 3D hexahedra CTA) vs the oracle's
    evaluate_constitutive + assemble_tangent_stiffness on random strains,
    and bitwise vs the separate constitutive + tangent calls."""
    import paper_1805_04155_b200 as P
    oc, gc, K, G = _caches(cuda, oracle, family, dim, 5.0, 0.2)
    n = oc.n_int
    E = np.random.default_rng(47).uniform(-1e-3, 1e-3, (n, 6))
    if dim == 2:
        E[:, [2, 4, 5]] = 0.0  # plane strain
    if model == "vm":
        a = 0.05
        Y = float(np.median(oracle.constitutive_vm(E, None, None, G, K, a, 0.0)["crit"]))
        mat = P.uniform_von_mises(n, K, G, a, Y)
        ref = oracle.constitutive_vm(E, None, None, G, K, a, Y)
    else:
        eta, _ = P.dp_parameters(1.0, np.pi / 9)
        # c at the median of rho / sqrt2 + eta p (constitutive.cpp:157-166): about half yields
        tr = E[:, 0] + E[:, 1] + E[:, 2]
        dev = E.copy()
        dev[:, :3] -= tr[:, None] / 3.0
        dev[:, 3:] *= 0.5
        rho = 2.0 * G * np.sqrt(np.maximum(0.0, (E * dev).sum(1)))
        c = float(np.median(rho / np.sqrt(2.0) + eta * K * tr))
        mat = P.uniform_drucker_prager(n, K, G, eta, c)
        ref = oracle.constitutive_dp(E, None, G, K, eta, c)
    pl = ref["plastic"]
    assert 0 < pl.sum() < n
    Kref = oc.tangent(ref["DS"], pl)
    Et = _t(E, cuda)
    eng = P.TangentEngine(gc, mat)
    S, flags, D, Kv = eng.step(Et)
    eng.sync()
    assert np.array_equal(_np(flags) & 1, pl)
    assert np.array_equal(_np(S), ref["S"])
    assert row_scaled_error(_np(Kv), Kref.data, Kref.indptr, oc.K_elast().data) <= 1e-12
    sep = P.TangentEngine(gc, mat, fused=False)
    S2, f2, D2, K2 = sep.step(Et)
    sep.sync()
    assert np.array_equal(_np(K2).view(np.uint64), _np(Kv).view(np.uint64))


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("family", FAMILIES)
def test_strains_and_internal_forces(cuda, oracle, family, dim):
    import paper_1805_04155_b200 as P
    oc, gc, K, G = _caches(cuda, oracle, family, dim, 3.0, 0.3)
    u = np.random.default_rng(43).uniform(-1, 1, oc.n_dofs)
    E_ref = oc.strains(u)
    E = _np(gc.strains(_t(u, cuda)))
    assert np.abs(E - E_ref).max() <= 1e-12 * np.abs(E_ref).max()
    S = oracle.constitutive_elastic(E_ref, G, K)["S"]
    F_ref = oc.internal_forces(S)
    F = _np(P.internal_forces(gc, _t(S, cuda)))
    assert np.abs(F - F_ref).max() <= 1e-12 * np.abs(F_ref).max()


def test_degenerate_element_reported(cuda):
    import paper_1805_04155_b200 as P
    coord = torch.tensor([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0.0]], dtype=torch.float64, device=cuda)
    elem = torch.tensor([[0, 1, 2, 3]], dtype=torch.int32, device=cuda)
    with pytest.raises(P.Error, match="jacobians: nonpositive det J in element 0"):
        P.build_assembly_cache(P.Mesh(P.ElementType("P1", 3), coord, elem), P.uniform_elastic(1, 1.0, 1.0))


def test_tangent_size_mismatch(cuda, oracle):
    import paper_1805_04155_b200 as P
    oc, gc, K, G = _caches(cuda, oracle, "Q1", 2)
    DS = torch.zeros((gc.n_int - 1, 36), dtype=torch.float64, device=cuda)
    with pytest.raises(P.Error, match="assemble_tangent_stiffness: size mismatch"):
        P.assemble_tangent_stiffness(gc, DS, torch.zeros(gc.n_int - 1, dtype=torch.bool, device=cuda))


# ---------------------------------------------------------------------------
# BASELINE configurations: full hot path on reduced meshes vs the oracle's
# reference-algorithm pipeline (evaluate_constitutive + assemble_tangent_stiffness)

REDUCED = {"cfg1": 16, "cfg2": 24, "cfg3": 5, "cfg4": 8, "cfg5": 5}


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_config_pipeline_vs_oracle(cuda, oracle, name):
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, displacement
    cfg = CONFIGS[name]
    n = REDUCED[name]
    mesh = cfg.mesh(n)
    mat = cfg.material(mesh.n_int)
    K, G = P.elastic_moduli(cfg.young, cfg.poisson)
    oc = oracle.Cache(cfg.family, cfg.dim, mesh.coord, mesh.elem, G, K)
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, cuda), mat)
    assert np.array_equal(_np(gc.row_ptr), oc.K_elast().indptr)
    assert np.array_equal(_np(gc.col_idx), oc.K_elast().indices)
    u = displacement(mesh.coord, cfg.seed)
    E1 = oc.strains(u)
    if cfg.model == "elastic":
        assert row_scaled_error(_np(gc.K_elast.values), oc.K_elast().data, oc.K_elast().indptr) <= 1e-12
        return
    # scale so that a fraction of points yields (oracle decides, same E bytes to both)
    if cfg.model == "vm":
        crit = oracle.constitutive_vm(E1, None, None, G, K, cfg.p1, 0.0)["crit"]  # |s_tr| at Y=0
        s = cfg.p2 / np.quantile(crit, 1.0 - cfg.target)
    else:
        eta, c = P.dp_parameters(cfg.p1, cfg.p2)
        s = 1.0
        for _ in range(60):
            f = oracle.constitutive_dp(s * E1, None, G, K, eta, c)["plastic"].mean()
            s *= 1.3 if f < cfg.target else 0.8
            if abs(f - cfg.target) < 0.05:
                break
    E = s * E1
    if cfg.model == "vm":
        ref = oracle.constitutive_vm(E, None, None, G, K, cfg.p1, cfg.p2)
    else:
        eta, c = P.dp_parameters(cfg.p1, cfg.p2)
        ref = oracle.constitutive_dp(E, None, G, K, eta, c)
    pl = ref["plastic"]
    assert 0 < pl.sum() < pl.size
    Kref = oc.tangent(ref["DS"], pl)
    eng = P.TangentEngine(gc, mat)
    Et = _t(E, cuda)
    S, flags, D, Kv = eng.step(Et)
    eng.sync()
    assert np.array_equal(_np(flags) & 1, pl)
    if cfg.model == "dp":
        assert np.array_equal((_np(flags) >> 1) & 1, ref["smooth"])
        assert np.array_equal((_np(flags) >> 2) & 1, ref["apex"])
    assert np.array_equal(_np(S), ref["S"])
    m = pl.astype(bool)
    assert np.array_equal(_np(P.unpack_D(D))[m], ref["DS"][m])
    assert row_scaled_error(_np(Kv), Kref.data, Kref.indptr, oc.K_elast().data) <= 1e-12
    # CUDA-graph replay gives the same bits
    eng.capture(Et)
    eng.replay()
    torch.cuda.synchronize()
    assert np.array_equal(_np(eng.K).view(np.uint64), _np(Kv).view(np.uint64))
    # the fused Newton step and the separate constitutive + tangent calls agree bitwise
    sep = P.TangentEngine(gc, mat, fused=False)
    S2, f2, D2, K2 = sep.step(Et)
    sep.sync()
    assert np.array_equal(_np(f2), _np(eng.flags)) and np.array_equal(_np(S2), _np(eng.S))
    assert np.array_equal(_np(K2).view(np.uint64), _np(eng.K).view(np.uint64))


@pytest.mark.parametrize("name", ["cfg2", "cfg4"])
def test_slab_data_path_on_one_rank(cuda, name):
    """dist.DistributedTangent (K1 on own points, exchange, tangent on the
    extended slab) run as a single rank equals the fused single-GPU step."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.dist import DistributedTangent, make_plan
    from paper_1805_04155_b200.synthetic import CONFIGS, displacement
    cfg = CONFIGS[name]
    n = REDUCED[name]
    plan = make_plan(cfg.family, cfg.dim, n, 1, 0)
    dt = DistributedTangent(plan, cfg.material, cuda)
    from paper_1805_04155_b200.synthetic import calibrate
    E1 = dt.cache.strains(torch.from_numpy(displacement(plan.mesh.coord, cfg.seed)).to(cuda))
    s, frac = calibrate(E1, dt.mat_ext, 0.3)
    assert 0.2 < frac < 0.4
    E = (s * E1).contiguous()
    S, flags, K = dt.step(E)
    dt.ctx.sync()
    eng = P.TangentEngine(dt.cache, dt.mat_ext)
    S2, f2, D2, K2 = eng.step(E)
    eng.sync()
    assert np.array_equal(_np(flags), _np(f2)) and np.array_equal(_np(S), _np(S2))
    assert np.array_equal(_np(K).view(np.uint64), _np(K2).view(np.uint64))


@pytest.mark.parametrize("name", ["cfg2", "cfg4", "cfg3"])
def test_assemble_rows_by_node_ranges(cuda, name):
    """epfem_assemble_rows_range over three uneven node ranges writes the same K bits as the whole
    row stream, and a range leaves the other rows untouched; a range outside the mesh is rejected."""
    import ctypes as C

    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.dist import DistributedTangent, make_plan
    from paper_1805_04155_b200.synthetic import CONFIGS, calibrate, displacement
    api = P.api
    cfg = CONFIGS[name]
    plan = make_plan(cfg.family, cfg.dim, REDUCED[name], 1, 0)
    dt = DistributedTangent(plan, cfg.material, cuda)
    E1 = dt.cache.strains(torch.from_numpy(displacement(plan.mesh.coord, cfg.seed)).to(cuda))
    s, _ = calibrate(E1, dt.mat_ext, 0.4)
    eng = P.TangentEngine(dt.cache, dt.mat_ext)
    S, f, D, K = eng.step((s * E1).contiguous())
    eng.sync()
    Kref = K.clone()
    n_nodes = dt.cache.info.n_nodes
    lib = api.L.lib()
    eng.K.fill_(float("nan"))
    eng.ctx.use_current_stream()
    cuts = [0, n_nodes // 3 + 1, n_nodes // 3 + 2, n_nodes]
    api._check(lib.epfem_assemble_rows_range(eng.ctx.handle, dt.cache.handle, api._ptr(eng.K), cuts[1], cuts[2]))
    eng.sync()
    written = int((~torch.isnan(eng.K)).sum())
    assert 0 < written < eng.K.numel() // 2
    for a, b in zip(cuts[:-1], cuts[1:]):
        api._check(lib.epfem_assemble_rows_range(eng.ctx.handle, dt.cache.handle, api._ptr(eng.K), a, b))
    eng.sync()
    assert np.array_equal(_np(eng.K).view(np.uint64), _np(Kref).view(np.uint64))
    rc = lib.epfem_assemble_rows_range(eng.ctx.handle, dt.cache.handle, api._ptr(eng.K), 0, n_nodes + 1)
    assert rc != 0 and b"node range" in lib.epfem_last_error()


@pytest.mark.parametrize("name,world", [("cfg2", 2), ("cfg2", 3), ("cfg4", 2), ("cfg3", 3), ("cfg5", 2)])
def test_slab_ranks_emulated_in_one_process(cuda, name, world):
    """The N-rank data path (dist.py) with the NCCL exchange replaced by the
    equivalent device copy, all ranks in one process one after another (no
    rank waits on another): the owned K rows of all ranks, concatenated, are
    bitwise the single-GPU fused step's K, and flags / S match per point."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.dist import DistributedTangent, make_plan
    from paper_1805_04155_b200.synthetic import CONFIGS, calibrate, displacement
    cfg = CONFIGS[name]
    n = {"cfg2": 24, "cfg4": 6, "cfg3": 6, "cfg5": 4}[name]
    mesh = cfg.mesh(n)
    mat = cfg.material(mesh.n_int)
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, cuda), mat)
    E1 = gc.strains(torch.from_numpy(displacement(mesh.coord, cfg.seed)).to(cuda))
    s, frac = calibrate(E1, mat, 0.35)
    E = (s * E1).contiguous()
    eng = P.TangentEngine(gc, mat)
    Sg, fg, Dg, Kg = eng.step(E)
    eng.sync()
    plans = [make_plan(cfg.family, cfg.dim, n, world, r) for r in range(world)]
    dts = [DistributedTangent(p, cfg.material, cuda) for p in plans]
    per_layer = plans[0].layer_elems
    nq = plans[0].n_q
    for p, dt in zip(plans, dts):
        k0, k1 = p.own_layers
        Eo = E[k0 * per_layer * nq:k1 * per_layer * nq].contiguous()
        n_e = p.mesh.n_elements
        top = max(p.halo_elems, n_e - p.layer_elems)
        if p.rank + 1 < p.world and top > p.halo_elems:  # the order of dt.step(): top layer first
            dt.update_own(Eo, elems=(top, n_e))
            dt.update_own(Eo, elems=(p.halo_elems, top))
        else:
            dt.update_own(Eo)
    for r in range(1, world):  # the exchange: top layer of r-1 -> halo of r
        s0, s1 = plans[r - 1].send_points
        h0, h1 = plans[r].halo_points
        dts[r].flags[h0:h1] = dts[r - 1].flags[s0:s1]
        dts[r].D[h0:h1] = dts[r - 1].D[s0:s1]
    rp = _np(gc.row_ptr)
    Kg_np = _np(Kg)
    for p, dt in zip(plans, dts):
        S, f, Kown = dt.assemble()
        dt.ctx.sync()
        k0, k1 = p.own_layers
        q0, q1 = k0 * per_layer * nq, k1 * per_layer * nq
        assert np.array_equal(_np(f), _np(fg[q0:q1])) and np.array_equal(_np(S), _np(Sg[q0:q1]))
        g0, g1 = p.global_rows
        want = Kg_np[rp[g0]:rp[g1]]
        assert np.array_equal(_np(Kown).view(np.uint64), want.view(np.uint64)), (p.rank, g0, g1)
    assert sum(p.global_rows[1] - p.global_rows[0] for p in plans) == gc.info.n_dofs


# ---------------------------------------------------------------------------
# the opt-in FP64 tensor-pipe phase 2 (EPFEM_FUSED=mma, read once per
# process): in a fresh interpreter, same bar as the default path
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4", "cfg5"])
def test_mma_phase2(cuda, oracle, name):
    import subprocess
    import sys
    env = dict(os.environ, EPFEM_FUSED="mma")
    n = {"cfg2": 24, "cfg3": 4, "cfg4": 6, "cfg5": 3}[name]
    r = subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "variant_check.py"), name,
                        str(n)], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


@pytest.mark.parametrize("name", ["cfg2", "cfg1", "cfg3", "cfg4", "cfg5"])
def test_newton_step_from_displacements(cuda, name):
    """epfem_newton_step_u (strains fused into the constitutive kernel,
    SURVEY §8(f) rank 1) gives the bits of epfem_strains + epfem_newton_step,
    and E_out the bits of epfem_strains."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, calibrate, displacement
    cfg = CONFIGS[name]
    mesh = cfg.mesh(REDUCED[name] * (2 if cfg.dim == 2 else 1))
    mat = cfg.material(mesh.n_int)
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, cuda), mat)
    u1 = torch.from_numpy(displacement(mesh.coord, cfg.seed)).to(cuda)
    E1 = gc.strains(u1)
    s = calibrate(E1, mat, 0.3)[0] if cfg.model != "elastic" else 1.0
    u = (s * u1).contiguous()
    E = gc.strains(u)
    e1, e2 = P.TangentEngine(gc, mat), P.TangentEngine(gc, mat)
    S1, f1, D1, K1 = e1.step(E)
    Eo = torch.empty_like(E)
    S2, f2, D2, K2 = e2.step_u(u, E_out=Eo)
    torch.cuda.synchronize()
    assert np.array_equal(_np(Eo).view(np.uint64), _np(E).view(np.uint64))
    assert np.array_equal(_np(f1), _np(f2)) and np.array_equal(_np(S1), _np(S2))
    m = (_np(f1) & 1).astype(bool)
    assert np.array_equal(_np(D1)[m], _np(D2)[m])
    assert np.array_equal(_np(K1).view(np.uint64), _np(K2).view(np.uint64))
    if cfg.model != "elastic":
        assert 0.2 < m.mean() < 0.4


@pytest.mark.parametrize("k5", ["gather", "rows"])
def test_elastic_assembly_both_paths(cuda, oracle, k5):
    """K5 through either implementation (EPFEM_K5, read once per process):
    the pattern / K_elast / tangent tests of all 8 element types in a fresh
    interpreter."""
    import subprocess
    import sys
    env = dict(os.environ, EPFEM_K5=k5)
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        os.path.join(os.path.dirname(__file__), "test_gpu_parity.py"),
                        "-k", "pattern_and_elastic or tangent_matches_oracle or all_element_types"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


@pytest.mark.parametrize("name", ["cfg2", "cfg1", "cfg3", "cfg4", "cfg5"])
def test_newton_step_with_internal_forces(cuda, oracle, name):
    """epfem_newton_step_f (fused in 2D): S, flags, D
    and K are the bits of epfem_newton_step, F the bits of K9
    (epfem_internal_forces on the step's S), and F matches the oracle's
    internal_forces (assembly.cpp:215-225) within 1e-12 of max |F|."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, calibrate, displacement
    cfg = CONFIGS[name]
    mesh = cfg.mesh(REDUCED[name])
    mat = cfg.material(mesh.n_int)
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, cuda), mat)
    u = torch.from_numpy(displacement(mesh.coord, cfg.seed)).to(cuda)
    E1 = gc.strains(u)
    s = calibrate(E1, mat, 0.3)[0] if cfg.model != "elastic" else 1.0
    E = (s * E1).contiguous()
    e1, e2 = P.TangentEngine(gc, mat), P.TangentEngine(gc, mat)
    S1, f1, D1, K1 = e1.step(E)
    S2, f2, D2, K2, F = e2.step_f(E)
    torch.cuda.synchronize()
    assert np.array_equal(_np(f1), _np(f2)) and np.array_equal(_np(S1), _np(S2))
    m = (_np(f1) & 1).astype(bool)
    assert np.array_equal(_np(D1)[m], _np(D2)[m])
    assert np.array_equal(_np(K1).view(np.uint64), _np(K2).view(np.uint64))
    F9 = P.internal_forces(gc, S2)
    torch.cuda.synchronize()
    assert np.array_equal(_np(F).view(np.uint64), _np(F9).view(np.uint64))
    K, G = P.elastic_moduli(cfg.young, cfg.poisson)
    oc = oracle.Cache(cfg.family, cfg.dim, mesh.coord, mesh.elem, G, K)
    Fref = oc.internal_forces(_np(S2))
    assert np.abs(_np(F) - Fref).max() <= 1e-12 * np.abs(Fref).max()


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("family", FAMILIES)
def test_single_cell_mesh_all_plastic(cuda, oracle, family, dim):
    """Edge case: a one-cell mesh (one element, or the cell's 2 / 6 simplices;
    a CTA or warp group far from full) with every point plastic: flags and S
    bitwise, K within 1e-12 row-scaled of the oracle."""
    import paper_1805_04155_b200 as P
    coord, elem, _ = oracle.structured_mesh(family, dim, 1, 1, 1 if dim == 3 else 0)
    K, G = oracle.elastic_moduli(206900.0, 0.29)
    oc = oracle.Cache(family, dim, coord, elem, G, K)
    mesh = P.Mesh(P.ElementType(family, dim), _t(coord, cuda), _t(elem, cuda, torch.int32))
    n = oc.n_int
    E = np.random.default_rng(5).uniform(-1e-3, 1e-3, (n, 6))
    if dim == 2:
        E[:, [2, 4, 5]] = 0.0
    a = 1.0e4
    Y = 0.5 * float(oracle.constitutive_vm(E, None, None, G, K, a, 0.0)["crit"].min())
    ref = oracle.constitutive_vm(E, None, None, G, K, a, Y)
    assert ref["plastic"].all()
    mat = P.uniform_von_mises(n, K, G, a, Y)
    gc = P.build_assembly_cache(mesh, mat)
    eng = P.TangentEngine(gc, mat)
    S, flags, D, Kv = eng.step(_t(E, cuda))
    eng.sync()
    assert np.array_equal(_np(flags) & 1, ref["plastic"])
    assert np.array_equal(_np(S), ref["S"])
    Kref = oc.tangent(ref["DS"], ref["plastic"])
    assert row_scaled_error(_np(Kv), Kref.data, Kref.indptr, oc.K_elast().data) <= 1e-12


def test_empty_constitutive_batch(cuda):
    """Edge case: zero integration points (the reference's 6 x 0 Mat) returns
    empty outputs without a launch error."""
    import paper_1805_04155_b200 as P
    K, G = P.elastic_moduli(206900.0, 0.29)
    mat = P.uniform_von_mises(0, K, G, 1.0e4, 450.0)
    st = P.evaluate_constitutive(torch.zeros((0, 6), dtype=torch.float64, device=cuda),
                                 P.IntegrationState.zero(0, device=cuda), mat)
    assert st.S.shape[0] == 0 and st.plastic_mask.numel() == 0
