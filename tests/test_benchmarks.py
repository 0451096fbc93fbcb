"""The strip-footing benchmark: the mesh and its
Dirichlet data against the reference's per-node constraint loop
(mesh.cpp:260-291) restated over the oracle's mesh numbering (CPU), and the
load driver run_dp_footing (benchmarks.cpp:120-205) on the GPU against the
same driver restated on the oracle with the reference's direct solves."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")


def _footing_ref(O, level, family, dim, layers=-1):
    """mesh.cpp:260-291 restated per node, in the reference's call order
    (a later constrain on the same dof overrides an earlier one)."""
    cells = (5 if family in ("P2", "Q2") else 10) << level
    h = 10.0 / cells
    nz = 0
    if dim == 3:
        nz = layers if layers > 0 else max(1, int(math.floor(1.0 / h + 0.5)))
    coord, elem, fine = O.structured_mesh(family, dim, cells, cells, nz, h, h, (1.0 / nz if nz else None))
    n = coord.shape[0]
    free = np.ones((n, dim), bool)
    fixed = np.zeros((n, dim))
    load = np.zeros((n, dim))

    def constrain(d, node, f, l):
        free[node, d] = False
        fixed[node, d] = f
        load[node, d] = l
    a_foot = int(math.floor(2.0 / h + 0.5))
    amax, bmax, cmax = 2 * cells, 2 * cells, 2 * nz
    for node in range(n):
        a, b, c = (int(x) for x in fine[node])
        if a == 0 or a == amax:
            constrain(0, node, 0.0, 0.0)
        if b == 0:
            constrain(1, node, 0.0, 0.0)
        if b == bmax and a <= a_foot:
            constrain(1, node, 0.0, -1.0)
            constrain(0, node, 0.0, 0.0)
        if dim == 3 and (c == 0 or c == cmax):
            constrain(2, node, 0.0, 0.0)
    return coord, elem, free, fixed, load


@pytest.mark.parametrize("family,dim,level", [("P1", 2, 0), ("P2", 2, 1), ("Q1", 2, 0), ("Q2", 2, 0),
                                              ("P1", 3, 0), ("Q2", 3, 0)])
def test_footing_mesh_matches_reference_loop(oracle, family, dim, level):
    from paper_1805_04155_b200.benchmarks import build_mesh_footing
    bm = build_mesh_footing(level, family, dim)
    coord, elem, free, fixed, load = _footing_ref(oracle, level, family, dim)
    assert np.array_equal(bm.mesh.coord, coord)
    assert np.array_equal(bm.mesh.elem, elem)
    assert np.array_equal(bm.free_dof, free)
    assert np.array_equal(bm.dirichlet_fixed, fixed)
    assert np.array_equal(bm.dirichlet_load, load)
    # the footing is the unit segment x1 in [0, 1] of the top edge
    foot = np.nonzero(load[:, 1] != 0.0)[0]
    assert np.all(coord[foot, 1] == 10.0) and coord[foot, 0].max() == 1.0 and coord[foot, 0].min() == 0.0
    # Mesh::free_mask / dirichlet_values: dof order dim * node + direction
    v = bm.dirichlet_values(0.25)
    assert np.array_equal(bm.free_mask(), free.reshape(-1))
    assert np.all(v[dim * foot + 1] == -0.25)
    assert np.all(v[free.reshape(-1)] == 0.0)
    assert np.count_nonzero(v) == foot.size


def test_footing_mesh_rejects_negative_level():
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.benchmarks import build_mesh_footing
    with pytest.raises(P.Error, match="build_mesh_footing: level must be >= 0"):
        build_mesh_footing(-1, "P1", 2)


def _footing_driver_ref(O, bm, du0, u_max, theta, eps, max_iters):
    """benchmarks.cpp:120-205 and solver.cpp:7-62 restated on the oracle, with
    the reference's default direct restricted solve (no step failures
    expected at these increments)."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    m = bm.mesh
    K, G = O.elastic_moduli(1e7, 0.48)
    eta, c = O.dp_parameters(450.0, math.pi / 9.0, three_d=(m.dim == 3))
    oc = O.Cache(m.elem_type.family, m.dim, m.coord, m.elem, G, K)
    Ke = oc.K_elast()
    Kes = sp.csr_matrix((Ke.data, Ke.indices, Ke.indptr))

    def en(v):
        return np.sqrt(max(v @ (Kes @ v), 0.0))
    free = bm.free_mask()
    fi = np.nonzero(free)[0]
    foot = m.dim * np.nonzero(bm.dirichlet_load[:, 1] != 0.0)[0] + 1
    Ep = np.zeros((m.n_int, 6))
    u_prev = np.zeros(bm.n_dofs)
    u_d, du, p_prev, out = 0.0, du0, 0.0, []
    while u_d < u_max - 1e-14:
        inc = min(du, u_max - u_d)
        u = bm.dirichlet_values(u_d + inc)
        u[fi] = u_prev[fi]
        for it in range(1, max_iters + 1):
            st = O.constitutive_dp(oc.strains(u), Ep, G, K, eta, c)
            F = oc.internal_forces(st["S"])
            Kt = oc.tangent(st["DS"], st["plastic"])
            Ks = sp.csr_matrix((Kt.data, Kt.indices, Kt.indptr))
            d = np.zeros_like(u)
            d[fi] = spl.spsolve(Ks[fi][:, fi].tocsc(), -F[fi])
            npv = en(u)
            u = u + d
            ncu = en(u)
            if npv + ncu == 0.0 or en(d) <= eps * (npv + ncu):
                break
        else:
            raise AssertionError("reference Newton did not converge")
        st = O.constitutive_dp(oc.strains(u), Ep, G, K, eta, c)
        Ep = st["Ep"]
        u_d += inc
        du = inc
        u_prev = u
        F = oc.internal_forces(st["S"])
        reaction = 0.0
        for f in F[foot]:
            reaction += f
        p = -reaction
        out.append((u_d, it, int(st["plastic"].sum()), p / 450.0))
        if abs(p - p_prev) < theta * max(abs(p), 1e-300):
            du *= 2.0
        p_prev = p
    return out, u_prev


@pytest.mark.gpu
def test_run_dp_footing_matches_reference_driver(cuda, oracle):
    """Level-0 P1 footing, 6 footing increments of 1e-3 into plasticity: the
    GPU driver (the reference's default direct restricted solve on the device)
    and the restated reference driver (direct solves) take the same load path
    with the same plastic counts and normalised pressures within 1e-7, and
    Newton iteration counts within one: a converged plastic point sits on the
    yield surface, so the next step's first iterate can flip it on a 1e-14
    difference between two exact solves (the cyclic test allows the same)."""
    from paper_1805_04155_b200.benchmarks import BenchmarkConfig, run_dp_footing
    from paper_1805_04155_b200.solver import NewtonSettings, SolveSettings
    cfg = BenchmarkConfig(dim=2, elem="P1", level=0, du0=1e-3, u_max=6e-3, theta=1e-3,
                          newton=NewtonSettings(eps_newton=1e-10, max_iters=25,
                                                linear=SolveSettings(rel_tol=1e-12), on_failure="error"))
    res = run_dp_footing(cfg, device=cuda)
    ref, u_ref = _footing_driver_ref(oracle, res.mesh, cfg.du0, cfg.u_max, cfg.theta, 1e-10, 25)
    assert res.completed and len(res.records) == len(ref)
    assert ref[-1][2] > 0, "the footing must yield within the load path"
    for rec, (load, iters, n_pl, p) in zip(res.records, ref):
        assert rec.load == load
        assert abs(rec.newton_iters - iters) <= 1
        assert rec.n_plastic == n_pl
        assert abs(rec.derived_scalar - p) <= 1e-7 * abs(p)
        assert not rec.direct_substituted
    u = res.u.cpu().numpy()
    assert np.abs(u - u_ref).max() <= 1e-8 * np.abs(u_ref).max()
    assert abs(res.limit_pressure - res.records[-1].derived_scalar * 450.0) <= 1e-12 * abs(res.limit_pressure)


@pytest.mark.gpu
def test_run_dp_footing_through_the_limit_load(cuda, oracle):
    """ADVICE (round 1): the footing through its limit load at the default
    restricted-solve tolerance (rel_tol 1e-10, LinearSolver::direct): level-0
    P1 to u_D = 0.02, where the pressure plateaus (the increment doubles once
    the pressure stops changing, benchmarks.cpp:177-178).  The GPU driver and
    the restated reference driver (direct solves) take the same load path, and
    the pressure at every step and the limit pressure agree within 1e-6."""
    from paper_1805_04155_b200.benchmarks import BenchmarkConfig, run_dp_footing
    from paper_1805_04155_b200.solver import NewtonSettings
    cfg = BenchmarkConfig(dim=2, elem="P1", level=0, du0=1e-3, u_max=2e-2, theta=1e-3,
                          newton=NewtonSettings(eps_newton=1e-10, max_iters=25, on_failure="error"))
    res = run_dp_footing(cfg, device=cuda)
    ref, _ = _footing_driver_ref(oracle, res.mesh, cfg.du0, cfg.u_max, cfg.theta, 1e-10, 25)
    assert res.completed and len(res.records) == len(ref)
    loads = [r.load for r in res.records]
    assert loads == [x[0] for x in ref]
    assert loads[-1] == pytest.approx(2e-2)
    for rec, (load, iters, n_pl, p) in zip(res.records, ref):
        assert abs(rec.derived_scalar - p) <= 1e-6 * abs(p)
        assert not rec.direct_substituted
    # at the limit the last increments change the pressure by well under 1 %
    assert abs(ref[-1][3] - ref[-2][3]) <= 1e-2 * abs(ref[-1][3])


# ---------------------------------------------------------------- elastic body
def _elastic_body_ref(O, level, family, dim=2):
    """mesh.cpp:222-258 restated per node over the oracle's numbering."""
    block = 5 << level
    cells, h = 2 * block, 5.0 / block
    nz = max(1, int(math.floor(1.0 / h + 0.5))) if dim == 3 else 0
    active = np.ones((cells, cells), np.uint8)
    active[:block, :block] = 0
    coord, elem, fine = O.structured_mesh(family, dim, cells, cells, nz, h, h, (1.0 / nz if nz else None), active)
    n = coord.shape[0]
    free = np.ones((n, dim), bool)
    fixed = np.zeros((n, dim))
    load = np.zeros((n, dim))

    def constrain(d, node, f, l):
        free[node, d] = False
        fixed[node, d] = f
        load[node, d] = l
    for node in range(n):
        a, b = int(fine[node, 0]), int(fine[node, 1])
        if a == 0:
            constrain(0, node, 0.0, 0.0)
        if b == 0:
            constrain(1, node, 0.0, 0.0)
            constrain(0, node, 0.0, 1.0)
        if dim == 3 and fine[node, 2] in (0, 2 * nz):
            constrain(2, node, 0.0, 0.0)
    return coord, elem, free, fixed, load


@pytest.mark.parametrize("family", ["P1", "P2", "Q1", "Q2"])
def test_elastic_body_3d_mesh_and_forces(oracle, family):
    """3D body (one layer): mesh and Dirichlet data equal the reference's
    loop; Neumann faces lie on the top face; a unit volume force sums to the
    volume (75) and the traction 200 to 200 x 10 x 1 (face rule = the 2D
    volume rule, area element |t1 x t2|)."""
    from paper_1805_04155_b200.benchmarks import build_mesh_elastic_body
    from paper_1805_04155_b200.forces import constant_force, external_forces, face_nodes
    bm = build_mesh_elastic_body(0, family, 3)
    coord, elem, free, fixed, load = _elastic_body_ref(oracle, 0, family, 3)
    m = bm.mesh
    assert np.array_equal(m.coord, coord) and np.array_equal(m.elem, elem)
    assert np.array_equal(bm.free_dof, free)
    assert np.array_equal(bm.dirichlet_fixed, fixed) and np.array_equal(bm.dirichlet_load, load)
    assert len(bm.neumann_faces) == (20 if family in ("P1", "P2") else 10)
    for e, f in bm.neumann_faces:
        assert np.all(coord[elem[e, face_nodes(family, 3)[f]], 1] == 10.0)
    K, G = oracle.elastic_moduli(206900.0, 0.29)
    w = oracle.Cache(family, 3, coord, elem, G, K).arrays()[1]
    fv = external_forces(m, np.asarray(w), constant_force([0.0, 1.0, 0.0]))
    assert abs(fv[1::3].sum() - 75.0) <= 1e-11 * 75.0 and np.all(fv[0::3] == 0.0) and np.all(fv[2::3] == 0.0)
    ft = external_forces(m, np.asarray(w), None, constant_force([0.0, 200.0, 0.0]), bm.neumann_faces)
    assert abs(ft[1::3].sum() - 2000.0) <= 1e-11 * 2000.0
    assert np.all(ft[1::3][coord[:, 1] != 10.0] == 0.0)


@pytest.mark.parametrize("family,level", [("P1", 0), ("P2", 0), ("Q1", 1), ("Q2", 0)])
def test_elastic_body_mesh_and_forces(oracle, family, level):
    """The L-shaped body's mesh and Dirichlet data equal the reference's loop;
    Neumann faces are the top edge; the consistent loads of a unit volume
    force sum to the area (75) and those of the traction 200 to 200 x 10, with
    the known nodal split along the top edge (linear: h/2 at the ends, h
    inside; quadratic: h/6 at corners, 2h/3 at midsides)."""
    from paper_1805_04155_b200.benchmarks import build_mesh_elastic_body
    from paper_1805_04155_b200.forces import FACE_NODES_2D, constant_force, external_forces
    bm = build_mesh_elastic_body(level, family, 2)
    coord, elem, free, fixed, load = _elastic_body_ref(oracle, level, family)
    m = bm.mesh
    assert np.array_equal(m.coord, coord) and np.array_equal(m.elem, elem)
    assert np.array_equal(bm.free_dof, free)
    assert np.array_equal(bm.dirichlet_fixed, fixed) and np.array_equal(bm.dirichlet_load, load)
    cells = 10 << level
    assert len(bm.neumann_faces) == cells
    for e, f in bm.neumann_faces:
        assert np.all(coord[elem[e, FACE_NODES_2D[family][f]], 1] == 10.0)
    # weights |det J| w_q of an affine structured mesh: the oracle's cache
    K, G = oracle.elastic_moduli(206900.0, 0.29)
    oc = oracle.Cache(family, 2, coord, elem, G, K)
    w = oc.arrays()[1]
    fv = external_forces(m, np.asarray(w), constant_force([0.0, 1.0]))
    assert abs(fv[1::2].sum() - 75.0) <= 1e-12 * 75.0 and np.all(fv[0::2] == 0.0)
    ft = external_forces(m, np.asarray(w), None, constant_force([0.0, 200.0]), bm.neumann_faces)
    assert abs(ft[1::2].sum() - 2000.0) <= 1e-11 * 2000.0 and np.all(ft[0::2] == 0.0)
    top = np.nonzero(coord[:, 1] == 10.0)[0]
    top = top[np.argsort(coord[top, 0])]
    hh = 10.0 / cells
    expect = np.zeros(top.size)
    if family in ("P1", "Q1"):
        expect[:] = 200.0 * hh
        expect[[0, -1]] = 100.0 * hh
    else:
        expect[0::2] = 200.0 * hh / 3.0
        expect[[0, -1]] = 200.0 * hh / 6.0
        expect[1::2] = 200.0 * hh * 2.0 / 3.0
    assert np.allclose(ft[2 * top + 1], expect, rtol=1e-12, atol=0.0)
    assert np.count_nonzero(ft) == top.size


def _traction_driver_ref(O, bm, model, f_steps, dirichlet, eps, max_iters):
    """solver.cpp:7-62 restated on the oracle over a sequence of load steps
    (external force per step), committing Ep / Hard, direct restricted solves."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    m = bm.mesh
    K, G = O.elastic_moduli(206900.0, 0.29)
    oc = O.Cache(m.elem_type.family, m.dim, m.coord, m.elem, G, K)
    Ke = oc.K_elast()
    Kes = sp.csr_matrix((Ke.data, Ke.indices, Ke.indptr))

    def en(v):
        return np.sqrt(max(v @ (Kes @ v), 0.0))

    def const(E, Ep, Hard):
        if model == "elastic":
            return O.constitutive_vm(E, Ep, Hard, G, K, 0.0, 1e300)
        return O.constitutive_vm(E, Ep, Hard, G, K, 1e4, 450.0 * math.sqrt(2.0 / 3.0))
    fi = np.nonzero(bm.free_mask())[0]
    Ep = np.zeros((m.n_int, 6))
    Hard = np.zeros((m.n_int, 6))
    u_prev = np.zeros(bm.n_dofs)
    out = []
    for f_ext in f_steps:
        u = dirichlet.copy()
        u[fi] = u_prev[fi]
        for it in range(1, max_iters + 1):
            st = const(oc.strains(u), Ep, Hard)
            F = oc.internal_forces(st["S"])
            Kt = oc.tangent(st["DS"], st["plastic"])
            Ks = sp.csr_matrix((Kt.data, Kt.indices, Kt.indptr))
            d = np.zeros_like(u)
            d[fi] = spl.spsolve(Ks[fi][:, fi].tocsc(), (f_ext - F)[fi])
            npv = en(u)
            u = u + d
            ncu = en(u)
            if npv + ncu == 0.0 or en(d) <= eps * (npv + ncu):
                break
        else:
            raise AssertionError("reference Newton did not converge")
        st = const(oc.strains(u), Ep, Hard)
        Ep, Hard = st["Ep"], st["Hard"]
        u_prev = u
        out.append((it, int(st["plastic"].sum()), u))
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("family,dim", [("Q2", 2), ("Q1", 3)])
def test_run_elastic_and_vm_cyclic_match_reference_drivers(cuda, oracle, family, dim):
    """run_elastic and run_vm_cyclic (8 steps, traction to +-1 and back) on the
    level-0 Q2-8 (2D) and Q1 (3D, one layer) bodies vs the same drivers restated on the oracle with direct
    solves: plastic counts per step equal, Newton iterations within one (see
    below), u within 1e-8, the traction work f.u within 1e-9."""
    from paper_1805_04155_b200.benchmarks import (BenchmarkConfig, run_elastic, run_vm_cyclic,
                                                  vm_load_scale)
    from paper_1805_04155_b200.solver import NewtonSettings, SolveSettings
    ns = NewtonSettings(eps_newton=1e-10, max_iters=25, linear=SolveSettings(rel_tol=1e-12))
    cfg = BenchmarkConfig(dim=dim, elem=family, level=0, n_steps=8, newton=ns)
    el = run_elastic(cfg, device=cuda)
    bm = el.mesh
    from paper_1805_04155_b200.forces import constant_force, external_forces
    K, G = oracle.elastic_moduli(206900.0, 0.29)
    w = oracle.Cache(family, dim, bm.mesh.coord, bm.mesh.elem, G, K).arrays()[1]
    e2 = [0.0, 1.0, 0.0][:dim]
    t2 = [0.0, 200.0, 0.0][:dim]
    f = external_forces(bm.mesh, np.asarray(w), constant_force(e2), constant_force(t2), bm.neumann_faces)
    (it, npl, u_ref), = _traction_driver_ref(oracle, bm, "elastic", [f], bm.dirichlet_values(0.5), 1e-10, 25)
    u = el.u.cpu().numpy()
    assert el.records[0].newton_iters == it and npl == 0
    assert np.abs(u - u_ref).max() <= 1e-8 * np.abs(u_ref).max()
    assert abs(el.records[0].derived_scalar - f @ u_ref) <= 1e-9 * abs(f @ u_ref)

    cy = run_vm_cyclic(cfg, device=cuda)
    fmax = external_forces(bm.mesh, np.asarray(w), None, constant_force(t2), bm.neumann_faces)
    zetas = [vm_load_scale(4.0 * k / 8) for k in range(1, 9)]
    ref = _traction_driver_ref(oracle, bm, "vm", [z * fmax for z in zetas], bm.dirichlet_values(0.0), 1e-10, 25)
    assert len(cy.records) == 8 and [r.load for r in cy.records] == zetas
    assert max(r[1] for r in ref) > 0, "the cyclic traction must yield"
    for rec, (it, npl, u_r) in zip(cy.records, ref):
        # a warm start from the previous step's converged u puts the points
        # that were plastic there exactly on the yield surface (crit = 0 up to
        # rounding), so the first iterations' active sets follow the 1e-12
        # differences between the device CG and the direct solve: the count
        # may differ by one; the converged state may not
        assert abs(rec.newton_iters - it) <= 1
        assert rec.n_plastic == npl
        assert abs(rec.derived_scalar - fmax @ u_r) <= 1e-9 * max(abs(fmax @ u_r), 1e-30)
    assert np.abs(cy.u.cpu().numpy() - ref[-1][2]).max() <= 1e-8 * np.abs(ref[-1][2]).max()
    assert [k for k, _ in cy.hardening_snapshots] == [2, 4, 6, 8]


# ------------------------------------------------------------- mesh text I/O
@pytest.mark.parametrize("builder,family,dim", [("footing", "P2", 2), ("body", "Q2", 2), ("footing", "Q1", 3)])
def test_mesh_text_round_trip(tmp_path, builder, family, dim):
    """write_mesh_text / read_mesh_text (mesh.cpp:323-410): every array comes
    back bit for bit (%.17g round-trips doubles)."""
    from paper_1805_04155_b200.benchmarks import (build_mesh_elastic_body, build_mesh_footing, read_mesh_text,
                                                  write_mesh_text)
    bm = (build_mesh_footing if builder == "footing" else build_mesh_elastic_body)(0, family, dim)
    p = str(tmp_path / "m.txt")
    write_mesh_text(bm, p)
    rb = read_mesh_text(p)
    assert rb.mesh.elem_type == bm.mesh.elem_type
    assert np.array_equal(rb.mesh.coord, bm.mesh.coord) and np.array_equal(rb.mesh.elem, bm.mesh.elem)
    assert np.array_equal(rb.free_dof, bm.free_dof)
    assert np.array_equal(rb.dirichlet_fixed, bm.dirichlet_fixed)
    assert np.array_equal(rb.dirichlet_load, bm.dirichlet_load)
    assert rb.neumann_faces == bm.neumann_faces


def test_mesh_text_format_and_errors(tmp_path):
    """The reference's text layout on a 1-cell P1 mesh (h = 0.1), and its
    error messages for a bad header, a wrong node count, an out-of-range node
    and a truncated file."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.benchmarks import BoundaryMesh, read_mesh_text, write_mesh_text
    m = P.structured_mesh("P1", 2, 1, 1, hx=0.1, hy=0.1)
    bm = BoundaryMesh(m, np.ones((4, 2), bool), np.zeros((4, 2)), np.zeros((4, 2)))
    bm.constrain(1, np.array([0, 1]), 0.0, 0.0)
    bm.constrain(0, np.array([3]), 0.25, -1.0)
    bm.neumann_faces = [(1, 0)]
    p = tmp_path / "m.txt"
    write_mesh_text(bm, str(p))
    lines = p.read_text().splitlines()
    assert lines[:4] == ["epfem-mesh 1", "dim 2", "elem P1", "nodes 4"]
    assert lines[4:8] == ["0 0 0", "1 0.10000000000000001 0", "2 0 0.10000000000000001",
                          "3 0.10000000000000001 0.10000000000000001"]
    assert lines[8] == "elements 2 3"
    assert lines[9:11] == ["0 " + " ".join(map(str, m.elem[0])), "1 " + " ".join(map(str, m.elem[1]))]
    assert lines[11:] == ["dirichlet 3", "0 1 0 0", "1 1 0 0", "3 0 0.25 -1", "neumann 1", "1 0"]
    bad = tmp_path / "bad.txt"
    for text, msg in [("epfem-mesh 2\n", "unrecognized header"),
                      (p.read_text().replace("elements 2 3", "elements 2 4"), "node count mismatch"),
                      (p.read_text().replace("\n1 " + " ".join(map(str, m.elem[1])), "\n1 0 1 7"),
                       "node index out of range"),
                      ("\n".join(lines[:12]) + "\n", "truncated file")]:
        bad.write_text(text)
        with pytest.raises(P.Error, match=msg):
            read_mesh_text(str(bad))


@pytest.mark.parametrize("family,dim", [("P1", 2), ("Q2", 2), ("P2", 3), ("Q2", 3)])
def test_boundary_nodes_of_a_box(family, dim):
    """boundary_faces / boundary_nodes (mesh.cpp:293-321) on a structured box:
    the boundary nodes are exactly those on the box's faces, and every
    boundary face lies in one of them."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.forces import boundary_faces, boundary_nodes, face_nodes
    m = P.structured_mesh(family, dim, 3, 2, 2 if dim == 3 else 0)
    x = m.coord
    on = np.zeros(m.n_nodes, bool)
    for d in range(dim):
        on |= (x[:, d] == 0.0) | (x[:, d] == x[:, d].max())
    assert boundary_nodes(m) == np.nonzero(on)[0].tolist()
    for e, f in boundary_faces(m):
        fx = x[m.elem[e, face_nodes(family, dim)[f]]]
        assert any(np.all(fx[:, d] == v) for d in range(dim) for v in (0.0, x[:, d].max()))
