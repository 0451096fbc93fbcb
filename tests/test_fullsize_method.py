"""CPU check of the full-size parity method (tests/fullsize.py): the complete
rows of a slab assembled by the oracle as a mesh of its own equal the same
rows of the whole mesh's oracle K (pattern bit for bit with global column
ids, values within 1e-12 row-scaled), for slabs at the bottom, inside and at
the top of meshes of the BASELINE element types."""
import numpy as np
import pytest

from fullsize import compare_slab_rows, complete_nodes, layer_elements, slab_submesh


def _strains_and_state(oracle, cfg, oc, coord, target):
    from paper_1805_04155_b200.synthetic import displacement
    K, G = oracle.elastic_moduli(cfg.young, cfg.poisson)
    E1 = oc.strains(displacement(coord, cfg.seed))
    if cfg.model == "vm":
        crit = oracle.constitutive_vm(E1, None, None, G, K, cfg.p1, 0.0)["crit"]
        return (cfg.p2 / np.quantile(crit, 1.0 - target)) * E1
    eta, c = oracle.dp_parameters(cfg.p1, cfg.p2)
    s = 1.0
    for _ in range(60):
        f = oracle.constitutive_dp(s * E1, None, G, K, eta, c)["plastic"].mean()
        s *= 1.3 if f < target else 0.8
        if abs(f - target) < 0.05:
            break
    return s * E1


def _evaluate(oracle, cfg, E):
    K, G = oracle.elastic_moduli(cfg.young, cfg.poisson)
    if cfg.model == "vm":
        return oracle.constitutive_vm(E, None, None, G, K, cfg.p1, cfg.p2)
    eta, c = oracle.dp_parameters(cfg.p1, cfg.p2)
    return oracle.constitutive_dp(E, None, G, K, eta, c)


@pytest.mark.parametrize("name,n", [("cfg2", 8), ("cfg3", 4), ("cfg4", 6), ("cfg5", 3)])
def test_slab_rows_equal_whole_mesh_rows(oracle, name, n):
    from paper_1805_04155_b200.synthetic import CONFIGS
    cfg = CONFIGS[name]
    nz = n if cfg.dim == 3 else 0
    coord, elem, _ = oracle.structured_mesh(cfg.family, cfg.dim, n, n, nz)
    K, G = oracle.elastic_moduli(cfg.young, cfg.poisson)
    oc = oracle.Cache(cfg.family, cfg.dim, coord, elem, G, K)
    E = _strains_and_state(oracle, cfg, oc, coord, 0.4)
    ref = _evaluate(oracle, cfg, E)
    Kfull = oc.tangent(ref["DS"], ref["plastic"])
    nq = oc.n_q
    per = layer_elements(elem, n)
    for k0, k1 in ((0, 2), (n // 2 - 1, n // 2 + 1), (n - 2, n)):
        e0, e1 = k0 * per, k1 * per
        nodes, cl, el = slab_submesh(coord, elem, e0, e1)
        comp = complete_nodes(elem, coord.shape[0], e0, e1, nodes)
        sc = oracle.Cache(cfg.family, cfg.dim, cl, el, G, K)
        sref = _evaluate(oracle, cfg, E[e0 * nq:e1 * nq])
        assert np.array_equal(sref["plastic"], ref["plastic"][e0 * nq:e1 * nq])
        Ks = sc.tangent(sref["DS"], sref["plastic"])
        rows, err = compare_slab_rows(cfg.dim, nodes, comp, Ks, sc.K_elast(), Kfull.indptr,
                                      lambda v0, v1: Kfull.indices[v0:v1], lambda v0, v1: Kfull.data[v0:v1])
        assert rows > 0 and err <= 1e-12


def test_slab_comparison_detects_a_wrong_value_and_a_wrong_column(oracle):
    """The comparison has teeth: one perturbed value (1e-10 relative) or one
    shifted column id in the full matrix fails it."""
    from paper_1805_04155_b200.synthetic import CONFIGS
    cfg = CONFIGS["cfg4"]
    n = 4
    coord, elem, _ = oracle.structured_mesh(cfg.family, 3, n, n, n)
    K, G = oracle.elastic_moduli(cfg.young, cfg.poisson)
    oc = oracle.Cache(cfg.family, 3, coord, elem, G, K)
    Kel = oc.K_elast()
    per = layer_elements(elem, n)
    e0, e1 = per, 3 * per
    nodes, cl, el = slab_submesh(coord, elem, e0, e1)
    comp = complete_nodes(elem, coord.shape[0], e0, e1, nodes)
    sc = oracle.Cache(cfg.family, 3, cl, el, G, K)
    Ks = sc.K_elast()
    g0 = 3 * int(nodes[np.flatnonzero(comp)[0]])
    k = int(Kel.indptr[g0]) + 1
    data = Kel.data.copy()
    data[k] *= 1.0 + 1e-10
    with pytest.raises(AssertionError):
        compare_slab_rows(3, nodes, comp, Ks, Ks, Kel.indptr, lambda a, b: Kel.indices[a:b], lambda a, b: data[a:b])
    cols = Kel.indices.copy()
    cols[k] += 1
    with pytest.raises(AssertionError):
        compare_slab_rows(3, nodes, comp, Ks, Ks, Kel.indptr, lambda a, b: cols[a:b], lambda a, b: Kel.data[a:b])
    compare_slab_rows(3, nodes, comp, Ks, Ks, Kel.indptr, lambda a, b: Kel.indices[a:b], lambda a, b: Kel.data[a:b])
