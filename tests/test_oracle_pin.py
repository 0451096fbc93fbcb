"""Pin the CPU restatement (oracle/) against the reference's own tests.

The reference cannot be built here (no Eigen), so the oracle is pinned
against every known answer and independent in-test oracle the reference's
test-suite holds for this path:
  * tests/test_constitutive.cpp — moduli / DP parameters (:205-245), tensor-space
    oracles on the seeded 1000-point batches (:307-375, :415-466; fixtures from
    tests/golden/gen_golden.cpp), apex / a=0 / huge-Y / yield-surface known
    answers (:267-305, :377-413), finite-difference tangents (:468-561);
  * tests/test_assembly.cpp — dense element-loop K oracle for all 8 element
    types (:299-327), tangent split identity incl. bitwise 0% (:329-365),
    B reproduces fields and weights integrate the domain (:192-260),
    internal forces (:367-392), degenerate element (:478-488);
  * tests/test_linalg.cpp — from_triplets duplicates / empty / range (:15-50),
    sandwich special cases and dense triple product (:52-88).
"""
import math
import os

import numpy as np
import pytest

from helpers import (FAMILIES, GOLDEN, dense_elastic_oracle, elastic_C, small_mesh, sym_block)


def _g(name):
    return np.load(os.path.join(GOLDEN, name + ".npy"))


def _blocks(DS):
    return DS.reshape(-1, 6, 6).transpose(0, 2, 1)  # column-major blocks -> D[q][i][j]


IOTA = np.array([1, 1, 1, 0, 0, 0.0])
DEV = np.diag([1, 1, 1, 0.5, 0.5, 0.5]) - np.outer(IOTA, IOTA) / 3.0


def stress_norm(s):
    return np.sqrt((s[..., :3] ** 2).sum(-1) + 2.0 * (s[..., 3:] ** 2).sum(-1))


def to_strain(s):
    e = s.copy()
    e[..., 3:] *= 2.0
    return e


# ---------------------------------------------------------------------------
# constitutive known answers

def test_elastic_moduli_known_answers(oracle):
    K, G = oracle.elastic_moduli(206900.0, 0.29)
    assert K == pytest.approx(206900.0 / 1.26, rel=1e-12)
    assert G == pytest.approx(206900.0 / 2.58, rel=1e-12)
    K, G = oracle.elastic_moduli(1e7, 0.48)
    assert K == pytest.approx(8.3333e7, rel=1e-4)
    assert G == pytest.approx(3.3784e6, rel=1e-4)


def test_dp_parameters_known_answers(oracle):
    eta, c = oracle.dp_parameters(450.0, math.pi / 9.0, True)
    assert eta == pytest.approx(0.354515, rel=1e-5)
    assert c == pytest.approx(438.31, rel=1e-4)
    eta3, c3 = oracle.dp_parameters(450.0, 1e-9, True)
    assert abs(eta3) < 1e-6
    assert c3 == pytest.approx(450.0 * 6.0 / (3.0 * math.sqrt(3.0)), rel=1e-6)
    eta2, c2 = oracle.dp_parameters(450.0, 1e-9, False)
    assert abs(eta2) < 1e-6 and c2 == pytest.approx(450.0, rel=1e-6)


def test_voigt_identities():
    assert np.abs(DEV @ IOTA).max() <= 1e-15
    vol = np.outer(IOTA, IOTA)
    assert np.abs(vol @ vol - 3 * vol).max() <= 1e-15


def test_elastic_model(oracle):
    E = np.zeros((3, 6))
    E[1, :3] = 0.3
    E[2] = np.random.default_rng(5).uniform(-1, 1, 6)
    o = oracle.constitutive_elastic(E, 1.5, 2.0)
    assert np.abs(o["S"][0]).max() <= 1e-15
    assert np.allclose(o["S"][1, :3], 3 * 2.0 * 0.3, rtol=1e-13)
    C = elastic_C(2.0, 1.5)
    assert np.abs(o["S"][2] - C @ E[2]).max() <= 1e-13
    assert np.abs(_blocks(o["DS"]) - C).max() <= 1e-15


def test_vm_basics(oracle):
    G, K, Y = 1.1, 1.7, 0.8
    z = np.zeros((1, 6))
    o = oracle.constitutive_vm(z, z, z, G, K, 0.5, Y)
    assert np.abs(o["S"]).max() == 0.0 and o["plastic"][0] == 0
    E = np.zeros((1, 6))
    E[0, 3] = 2.0
    o = oracle.constitutive_vm(E, z, z, G, K, 0.0, Y)
    assert o["plastic"][0] == 1
    dev_s = DEV @ to_strain(o["S"][0])
    assert stress_norm(dev_s) == pytest.approx(Y, rel=1e-12)
    assert np.abs(o["Hard"]).max() == 0.0
    E = np.random.default_rng(7).uniform(-1, 1, (1, 6))
    o = oracle.constitutive_vm(E, z, z, G, K, 0.5, 1e9)
    el = oracle.constitutive_elastic(E, G, K)
    assert np.abs(o["S"] - el["S"]).max() <= 1e-14
    assert np.abs(o["DS"] - el["DS"]).max() <= 1e-14
    assert o["plastic"][0] == 0


def test_dp_basics(oracle):
    G, K, eta, c = 1.2, 2.1, 0.4, 0.6
    z = np.zeros((1, 6))
    o = oracle.constitutive_dp(z, z, G, K, eta, c)
    assert np.abs(o["S"]).max() == 0.0 and not o["smooth"][0] and not o["apex"][0]
    E = np.zeros((1, 6))
    E[0, :3] = 10.0
    o = oracle.constitutive_dp(E, z, G, K, eta, c)
    assert o["apex"][0] == 1
    assert np.allclose(o["S"][0, :3], c / eta, rtol=1e-13)
    assert np.abs(o["S"][0, 3:]).max() <= 1e-15
    assert np.abs(o["DS"]).max() == 0.0
    E = np.zeros((1, 6))
    E[0, 0], E[0, 1], E[0, 3] = 1.5, -0.2, 0.7
    o = oracle.constitutive_dp(E, z, G, K, eta, c)
    assert o["smooth"][0] == 1
    S = o["S"][0]
    dev_s = DEV @ to_strain(S)
    yld = stress_norm(dev_s) / math.sqrt(2.0) + (eta / 3.0) * S[:3].sum() - c
    assert abs(yld) <= 1e-9 * c


def test_dp_zero_deviator_goes_to_apex(oracle):
    # With a zero deviator rho = 0, so crit2 == crit1: a point past the cone
    # returns to the apex and the "zero deviator in smooth return" guard
    # (constitutive.cpp:173-174) cannot fire for finite input.
    E = np.zeros((2, 6))
    E[:, :3] = [[1.0] * 3, [-1.0] * 3]
    o = oracle.constitutive_dp(E, np.zeros((2, 6)), 1.0, 1.0, 0.5, 0.1)
    assert o["apex"].tolist() == [1, 0] and o["smooth"].tolist() == [0, 0]


# ---------------------------------------------------------------------------
# seeded batches vs the reference's tensor-space oracles (golden fixtures)

def test_vm_batch_matches_tensor_oracle(oracle):
    E, Ep, H = _g("vm_E"), _g("vm_Ep"), _g("vm_Hard")
    G, K, a, Y = _g("vm_G"), _g("vm_K"), _g("vm_a"), _g("vm_Y")
    o = oracle.constitutive_vm(E, Ep, H, G, K, a, Y)
    assert np.abs(o["S"] - _g("vm_S_tensor")).max() <= 1e-12
    assert np.abs(o["Ep"] - _g("vm_Ep_tensor")).max() <= 1e-12
    assert np.abs(o["Hard"] - _g("vm_Hard_tensor")).max() <= 1e-12
    pl = _g("vm_plastic_tensor").astype(np.uint8)
    assert np.array_equal(o["plastic"], pl)
    assert pl.sum() > 100 and (1 - pl).sum() > 100
    C = np.stack([elastic_C(k, g) for k, g in zip(K, G)])
    el = np.einsum("qij,qj->qi", C, E - o["Ep"])
    assert (np.abs(o["S"] - el).max(1) <= 1e-10 * (1 + np.abs(el).max(1))).all()
    m = pl.astype(bool)
    shifted = (DEV @ to_strain(o["S"][m]).T).T - o["Hard"][m]
    assert np.allclose(stress_norm(shifted), Y[m], rtol=1e-9)
    D = _blocks(o["DS"])
    assert (np.abs(D - D.transpose(0, 2, 1)).max((1, 2)) <= 1e-10 * np.abs(D).max((1, 2))).all()


def test_dp_batch_matches_tensor_oracle(oracle):
    E, Ep = _g("dp_E"), _g("dp_Ep")
    G, K, eta, c = _g("dp_G"), _g("dp_K"), _g("dp_eta"), _g("dp_c")
    o = oracle.constitutive_dp(E, Ep, G, K, eta, c)
    assert np.abs(o["S"] - _g("dp_S_tensor")).max() <= 1e-12
    assert np.abs(o["Ep"] - _g("dp_Ep_tensor")).max() <= 1e-12
    sm, ap = _g("dp_smooth_tensor").astype(np.uint8), _g("dp_apex_tensor").astype(np.uint8)
    assert np.array_equal(o["smooth"], sm) and np.array_equal(o["apex"], ap)
    assert sm.sum() > 50 and ap.sum() > 50 and (1 - sm - ap).sum() > 50
    C = np.stack([elastic_C(k, g) for k, g in zip(K, G)])
    el = np.einsum("qij,qj->qi", C, E - o["Ep"])
    assert (np.abs(o["S"] - el).max(1) <= 1e-10 * (1 + np.abs(el).max(1))).all()


def _fd(fn, E, h):
    fd = np.zeros((6, 6))
    for j in range(6):
        Ep_, Em_ = E.copy(), E.copy()
        Ep_[j] += h
        Em_[j] -= h
        fd[:, j] = (fn(Ep_) - fn(Em_)) / (2 * h)
    return fd


def test_consistent_tangents_match_finite_differences(oracle):
    rng = np.random.default_rng(17)
    G, K = 1.3, 2.2
    tol = 1e-5
    cn = np.linalg.norm(elastic_C(K, G))
    for a in (0.7, 0.0):
        Y = 0.6
        done = {True: 0, False: 0}
        while min(done.values()) < 20:
            E = rng.uniform(-1, 1, 6)
            Ep = 0.2 * rng.uniform(-1, 1, (1, 6))
            H = (DEV @ rng.uniform(-0.1, 0.1, 6))[None]
            o = oracle.constitutive_vm(E[None], Ep, H, G, K, a, Y)
            if abs(o["crit"][0]) < 1e-3 * Y:
                continue
            pl = bool(o["crit"][0] > 0)
            if done[pl] >= 20:
                continue
            h = 1e-6 * (1 + np.linalg.norm(E))
            fd = _fd(lambda x: oracle.constitutive_vm(x[None], Ep, H, G, K, a, Y)["S"][0], E, h)
            D = _blocks(o["DS"])[0]
            assert np.linalg.norm(fd - D) / max(np.linalg.norm(D), 1e-8 * cn) <= tol
            done[pl] += 1
    eta, c = 0.35, 0.5
    done = [0, 0, 0]
    while min(done) < 20:
        E = rng.uniform(-1, 1, 6)
        if rng.uniform() < 0.4:
            E[:3] += 2.0 + 2.0 * rng.uniform()
            E[3:] *= 0.1
        de = DEV @ E
        rho = 2 * G * math.sqrt(max(0.0, E @ de))
        p = K * E[:3].sum()
        c1 = rho / math.sqrt(2) + eta * p - c
        c2 = eta * p - K * eta * eta * rho / (G * math.sqrt(2)) - c
        m = 1e-3 * c
        reg = 0 if c1 < -m else (1 if (c1 > m and c2 < -m) else (2 if (c1 > m and c2 > m) else -1))
        if reg < 0 or done[reg] >= 20:
            continue
        z = np.zeros((1, 6))
        o = oracle.constitutive_dp(E[None], z, G, K, eta, c)
        h = 1e-6 * (1 + np.linalg.norm(E))
        fd = _fd(lambda x: oracle.constitutive_dp(x[None], z, G, K, eta, c)["S"][0], E, h)
        D = _blocks(o["DS"])[0]
        assert np.linalg.norm(fd - D) / max(np.linalg.norm(D), 1e-8 * cn) <= tol
        done[reg] += 1


# ---------------------------------------------------------------------------
# assembly

@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("family", FAMILIES)
def test_elastic_stiffness_equals_dense_element_loop(oracle, family, dim):
    coord, elem = small_mesh(oracle, family, dim)
    assert dim * coord.shape[0] <= 2000
    K, G = oracle.elastic_moduli(10.0, 0.3)
    cache = oracle.Cache(family, dim, coord, elem, G, K)
    dense = dense_elastic_oracle(oracle, family, dim, coord, elem, K, G)
    Kel = cache.K_elast().dense()
    scale = np.abs(dense).max()
    assert np.abs(Kel - dense).max() <= 1e-10 * scale
    t = np.ones(dim * coord.shape[0])
    assert np.abs(Kel @ t).max() <= 1e-9 * scale
    assert np.abs(Kel - Kel.T).max() <= 1e-10 * scale
    # structural pattern: every dof pair of nodes sharing an element
    adj = set()
    for e in elem:
        for a in e:
            for b in e:
                adj.add((int(a), int(b)))
    assert cache.nnz == dim * dim * len(adj)


@pytest.mark.parametrize("dim", [2, 3])
def test_tangent_split_identity(oracle, dim):
    rng = np.random.default_rng(41)
    coord, elem = small_mesh(oracle, "Q1", dim)
    K, G = oracle.elastic_moduli(5.0, 0.2)
    cache = oracle.Cache("Q1", dim, coord, elem, G, K)
    C = elastic_C(K, G)
    n = cache.n_int
    Kel = cache.K_elast()
    for frac in (0.0, 0.5, 1.0):
        pl = (np.arange(n) < frac * n).astype(np.uint8)
        D = np.stack([C + 0.3 * sym_block(rng) if p else C for p in pl])
        DS = D.transpose(0, 2, 1).reshape(n, 36)
        split = cache.tangent(DS, pl)
        direct = cache.direct(DS)
        assert np.array_equal(split.indptr, Kel.indptr) and np.array_equal(split.indices, Kel.indices)
        scale = np.abs(direct.data).max()
        assert np.abs(split.dense() - direct.dense()).max() <= 1e-10 * scale
        if frac == 0.0:
            assert split.nnz == Kel.nnz
            assert np.array_equal(split.data.view(np.uint64), Kel.data.view(np.uint64))


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("family", FAMILIES)
def test_B_reproduces_fields_and_weights_integrate_domain(oracle, family, dim):
    coord, elem = small_mesh(oracle, family, dim)
    K, G = oracle.elastic_moduli(1.0, 0.25)
    cache = oracle.Cache(family, dim, coord, elem, G, K)
    nn = coord.shape[0]
    trans = np.tile(0.3 + 0.1 * np.arange(dim), nn)
    assert np.abs(cache.strains(trans)).max() <= 1e-12
    u = np.zeros((nn, dim))
    u[:, 0] = coord[:, 1]
    E = cache.strains(u.reshape(-1))
    assert np.allclose(E[:, 3], 1.0, rtol=1e-10)
    assert np.abs(E[:, :2]).max() <= 1e-10
    A = np.zeros((dim, dim))
    A[0, 0], A[0, 1], A[1, 0], A[1, 1] = 0.02, 0.01, -0.015, 0.03
    if dim == 3:
        A[2, 2], A[0, 2], A[2, 1] = -0.01, 0.007, 0.004
    Ea = cache.strains((coord @ A.T).reshape(-1))
    sym = 0.5 * (A + A.T)
    exp = np.zeros(6)
    exp[0], exp[1], exp[3] = sym[0, 0], sym[1, 1], 2 * sym[0, 1]
    if dim == 3:
        exp[2], exp[4], exp[5] = sym[2, 2], 2 * sym[1, 2], 2 * sym[2, 0]
    assert np.abs(Ea - exp).max() <= 1e-10
    det, w, _ = cache.arrays()
    assert w.sum() == pytest.approx(75.0 if dim == 2 else 100.0, rel=1e-10)
    if not (family == "P2" and dim == 3):
        assert w.min() > 0


def test_internal_forces(oracle):
    coord, elem = small_mesh(oracle, "P2", 2)
    K, G = oracle.elastic_moduli(3.0, 0.3)
    cache = oracle.Cache("P2", 2, coord, elem, G, K)
    assert np.abs(cache.internal_forces(np.zeros((cache.n_int, 6)))).max() == 0.0
    u = np.random.default_rng(43).uniform(-1, 1, cache.n_dofs)
    S = oracle.constitutive_elastic(cache.strains(u), G, K)["S"]
    F = cache.internal_forces(S)
    Ku = cache.K_elast().to_scipy_csc() @ u
    assert np.abs(F - Ku).max() <= 1e-10 * np.abs(Ku).max()


def test_degenerate_element_is_reported(oracle):
    coord = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [1, 1, 0.0]])
    elem = np.array([[0, 1, 2, 3]], np.int32)
    with pytest.raises(oracle.OracleError, match="element 0"):
        oracle.Cache("P1", 3, coord, elem, 1.0, 1.0)


# ---------------------------------------------------------------------------
# linalg semantics (the Eigen boundary)

def test_from_triplets_semantics(oracle):
    A = oracle.from_triplets([0, 0], [0, 0], [2.0, 3.0], 2, 2)
    assert A.nnz == 1 and A.dense()[0, 0] == pytest.approx(5.0)
    E = oracle.from_triplets([], [], [], 3, 4)
    assert E.nnz == 0 and (E.rows, E.cols) == (3, 4)
    rng = np.random.default_rng(11)
    r, c, v = rng.integers(0, 8, 200), rng.integers(0, 8, 200), rng.uniform(-1, 1, 200)
    want = np.zeros((8, 8))
    np.add.at(want, (r, c), v)
    assert np.abs(oracle.from_triplets(r, c, v, 8, 8).dense() - want).max() <= 1e-14
    with pytest.raises(oracle.OracleError):
        oracle.from_triplets([5], [0], [1.0], 3, 3)
    # explicit zeros are kept (structural semantics)
    assert oracle.from_triplets([1], [1], [0.0], 2, 2).nnz == 1


def test_sandwich_semantics(oracle):
    rng = np.random.default_rng(13)
    Bd = np.where(rng.uniform(-1, 1, (6, 4)) > 0, rng.uniform(-1, 1, (6, 4)), 0.0)
    BtB = oracle.sandwich(Bd, np.eye(6))
    assert np.abs(BtB.dense() - Bd.T @ Bd).max() <= 1e-13
    assert np.linalg.eigvalsh(BtB.dense()).min() >= -1e-12
    assert oracle.sandwich(Bd, np.zeros((6, 6))).nnz == 0
    with pytest.raises(oracle.OracleError):
        oracle.sandwich(Bd, np.eye(5))
    rng = np.random.default_rng(17)
    Bd = np.where(rng.uniform(-1, 1, (9, 6)) > -0.2, rng.uniform(-1, 1, (9, 6)), 0.0)
    Dd = np.where(rng.uniform(-1, 1, (9, 9)) > 0.3, rng.uniform(-1, 1, (9, 9)), 0.0)
    want = Bd.T @ Dd @ Bd
    got = oracle.sandwich(Bd, Dd).dense()
    assert np.abs(got - want).max() <= 1e-10 * np.abs(want).max()


def test_cfg1_pattern_size_matches_survey(oracle):
    coord, elem, _ = oracle.structured_mesh("P1", 2, 256, 256)
    K, G = oracle.elastic_moduli(206900.0, 0.29)
    cache = oracle.Cache("P1", 2, coord, elem, G, K)
    assert (coord.shape[0], elem.shape[0], cache.n_dofs, cache.nnz) == (66049, 131072, 132098, 1841156)
