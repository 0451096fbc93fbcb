"""Newton-loop linear algebra and the Newton time step on the GPU (SURVEY
§8(f) rank 3) against the reference's own tests (tests/test_linalg.cpp:90-162)
and a restatement of newton_solve (solver.cpp:7-62) on the oracle with the
reference's default direct solve."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


def _csr(A, dev):
    import scipy.sparse as sp
    import paper_1805_04155_b200 as P
    M = sp.csr_matrix(A)
    M.sort_indices()
    return P.CsrMatrix(torch.from_numpy(M.indptr.astype(np.int64)).to(dev),
                       torch.from_numpy(M.indices.astype(np.int32)).to(dev),
                       torch.from_numpy(M.data.astype(np.float64)).to(dev))


def test_restricted_solve_trivial_cases(cuda):
    """test_linalg.cpp:90-110: identity, and a decoupled 2x2 with one fixed dof."""
    from paper_1805_04155_b200.solver import restricted_solve
    x = restricted_solve(_csr(np.eye(3), cuda), torch.tensor([1.0, 0.0, 0.0], dtype=torch.float64, device=cuda),
                         torch.ones(3, dtype=torch.bool, device=cuda)).cpu().numpy()
    assert abs(x[0] - 1.0) < 1e-12 and np.abs(x[1:]).max() <= 1e-15
    x2 = restricted_solve(_csr(np.diag([2.0, 2.0]), cuda), torch.tensor([2.0, 4.0], dtype=torch.float64, device=cuda),
                          torch.tensor([True, False], device=cuda)).cpu().numpy()
    assert abs(x2[0] - 1.0) < 1e-12 and x2[1] == 0.0


def test_restricted_solve_random_spd(cuda):
    """test_linalg.cpp:112-151: K = A^T A + 0.5 I, random free set, vs a dense solve."""
    from paper_1805_04155_b200.solver import SolveSettings, LinearSolver, restricted_solve
    rng = np.random.default_rng(23)
    n = 20
    A = rng.uniform(-1, 1, (n, n))
    Kd = A.T @ A + 0.5 * np.eye(n)
    rhs = rng.uniform(-1, 1, n)
    mask = rng.uniform(size=n) < 0.7
    mask[0] = True
    x = restricted_solve(_csr(Kd, cuda), torch.from_numpy(rhs).to(cuda), torch.from_numpy(mask).to(cuda),
                         SolveSettings(LinearSolver.conjugate_gradient, 1e-12)).cpu().numpy()
    f = np.nonzero(mask)[0]
    xf = np.linalg.solve(Kd[np.ix_(f, f)], rhs[f])
    assert np.abs(x[f] - xf).max() <= 1e-9 * np.abs(xf).max()
    assert np.all(x[~mask] == 0.0)
    # deterministic: the same bits on a second solve
    x2 = restricted_solve(_csr(Kd, cuda), torch.from_numpy(rhs).to(cuda), torch.from_numpy(mask).to(cuda),
                          SolveSettings(LinearSolver.conjugate_gradient, 1e-12)).cpu().numpy()
    assert np.array_equal(x.view(np.uint64), x2.view(np.uint64))


def test_restricted_solve_reports_singular_systems(cuda):
    """test_linalg.cpp:153-162: rank-deficient K, incompatible rhs -> SolverError:
    with the default direct method the factorisation fails (the reference's
    SimplicialLDLT meets a zero pivot: "factorization failed", linalg.cpp:86-88);
    with conjugate gradients the residual stays above the tolerance."""
    from paper_1805_04155_b200.solver import LinearSolver, SolveSettings, SolverError, restricted_solve
    rhs = torch.tensor([1.0, -1.0], dtype=torch.float64, device=cuda)
    with pytest.raises(SolverError, match="restricted_solve: factorization failed"):
        restricted_solve(_csr(np.ones((2, 2)), cuda), rhs)
    with pytest.raises(SolverError, match="restricted_solve: residual .* above tolerance"):
        restricted_solve(_csr(np.ones((2, 2)), cuda), rhs, None, SolveSettings(LinearSolver.conjugate_gradient))


def test_energy_norm(cuda):
    from paper_1805_04155_b200.solver import energy_norm
    rng = np.random.default_rng(5)
    A = rng.uniform(-1, 1, (12, 12))
    Kd = A.T @ A
    v = rng.uniform(-1, 1, 12)
    e = energy_norm(_csr(Kd, cuda), torch.from_numpy(v).to(cuda))
    assert abs(e - np.sqrt(v @ Kd @ v)) <= 1e-12 * np.sqrt(v @ Kd @ v)


def _newton_ref(O, oc, mat_args, dirichlet, free, f_ext, eps, max_iters):
    """solver.cpp:7-62 restated on the oracle (test infrastructure), with the
    reference's default direct restricted solve (scipy spsolve on K[free, free])."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    G, K, a, Y = mat_args
    Ke = oc.K_elast()
    Kes = sp.csr_matrix((Ke.data, Ke.indices, Ke.indptr))

    def en(v):
        return np.sqrt(max(v @ (Kes @ v), 0.0))
    u = dirichlet.copy()
    fi = np.nonzero(free)[0]
    for it in range(1, max_iters + 1):
        E = oc.strains(u)
        st = O.constitutive_vm(E, None, None, G, K, a, Y)
        F = oc.internal_forces(st["S"])
        Kt = oc.tangent(st["DS"], st["plastic"])
        Ks = sp.csr_matrix((Kt.data, Kt.indices, Kt.indptr))
        du = np.zeros_like(u)
        du[fi] = spl.spsolve(Ks[fi][:, fi].tocsc(), (f_ext - F)[fi])
        npv = en(u)
        u = u + du
        ncu = en(u)
        if npv + ncu == 0.0 or en(du) <= eps * (npv + ncu):
            st = O.constitutive_vm(oc.strains(u), None, None, G, K, a, Y)
            return u, it, int(st["plastic"].sum())
    raise AssertionError("reference Newton did not converge")


def test_newton_solve_matches_reference(cuda, oracle):
    """A 2D Q2-8 von Mises time step (cfg2's material): left edge clamped, the
    right edge pulled by u_x = delta (yielding), GPU newton_solve (device CG,
    rel_tol 1e-12) vs the restated reference with a direct solve: the same
    number of Newton iterations and plastic points, u within 1e-8."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.solver import NewtonSettings, SolveSettings, newton_solve
    from paper_1805_04155_b200.synthetic import CONFIGS
    cfg = CONFIGS["cfg2"]
    mesh = cfg.mesh(6)
    mat = cfg.material(mesh.n_int)
    K, G = P.elastic_moduli(cfg.young, cfg.poisson)
    x = mesh.coord.reshape(-1, 2)
    n_dofs = x.shape[0] * 2
    dirichlet = np.zeros(n_dofs)
    free = np.ones(n_dofs, bool)
    left, right = np.isclose(x[:, 0], 0.0), np.isclose(x[:, 0], x[:, 0].max())
    free[2 * np.nonzero(left)[0]] = False
    free[2 * np.nonzero(left)[0] + 1] = False
    free[2 * np.nonzero(right)[0]] = False
    dirichlet[2 * np.nonzero(right)[0]] = 0.004 * x[:, 0].max()
    f_ext = np.zeros(n_dofs)
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, cuda), mat)
    res = newton_solve(gc, mat, P.IntegrationState.zero(mesh.n_int, device=cuda),
                       torch.from_numpy(dirichlet), torch.from_numpy(free), torch.from_numpy(f_ext),
                       NewtonSettings(eps_newton=1e-9, max_iters=25, linear=SolveSettings(rel_tol=1e-12)))
    oc = oracle.Cache(cfg.family, cfg.dim, mesh.coord, mesh.elem, G, K)
    u_ref, iters_ref, npl_ref = _newton_ref(oracle, oc, (G, K, cfg.p1, cfg.p2), dirichlet, free, f_ext, 1e-9, 25)
    u = res.u.cpu().numpy()
    assert 0 < npl_ref < mesh.n_int, npl_ref
    assert res.record.newton_iters == iters_ref
    assert res.record.n_plastic == npl_ref
    assert np.abs(u - u_ref).max() <= 1e-8 * np.abs(u_ref).max()
    assert np.all(u[~free] == dirichlet[~free])


def test_newton_iterates_follow_the_reference_when_diverging(cuda, oracle):
    """A single too-large load step (16 x 16, the right edge pulled to 0.004
    from the bare Dirichlet lift) is outside the semismooth Newton's basin for
    the reference too: the GPU loop's stopping ratios |du|_e / (|u_prev|_e +
    |u|_e) follow the restated reference's over the first iterations, and both
    raise NonConvergenceError."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as spl
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS
    cfg = CONFIGS["cfg2"]
    mesh = cfg.mesh(16)
    mat = cfg.material(mesh.n_int)
    K, G = P.elastic_moduli(cfg.young, cfg.poisson)
    x = mesh.coord
    nd = x.shape[0] * 2
    dirichlet, free = np.zeros(nd), np.ones(nd, bool)
    left, right = np.isclose(x[:, 0], 0.0), np.isclose(x[:, 0], x[:, 0].max())
    free[2 * np.nonzero(left)[0]] = free[2 * np.nonzero(left)[0] + 1] = False
    free[2 * np.nonzero(right)[0]] = False
    dirichlet[2 * np.nonzero(right)[0]] = 0.004
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, cuda), mat)
    with pytest.raises(P.NonConvergenceError) as ex:
        P.newton_solve(gc, mat, P.IntegrationState.zero(mesh.n_int, device=cuda), torch.from_numpy(dirichlet),
                       torch.from_numpy(free), torch.zeros(nd, dtype=torch.float64),
                       P.NewtonSettings(eps_newton=1e-9, max_iters=4, linear=P.SolveSettings(rel_tol=1e-12)))
    gpu = ex.value.record.ratios
    oc = oracle.Cache(cfg.family, cfg.dim, mesh.coord, mesh.elem, G, K)
    Ke = oc.K_elast()
    Kes = sp.csr_matrix((Ke.data, Ke.indices, Ke.indptr))
    en = lambda v: np.sqrt(max(v @ (Kes @ v), 0.0))  # noqa: E731
    u, fi, ref = dirichlet.copy(), np.nonzero(free)[0], []
    for _ in range(4):
        st = oracle.constitutive_vm(oc.strains(u), None, None, G, K, cfg.p1, cfg.p2)
        F = oc.internal_forces(st["S"])
        Kt = oc.tangent(st["DS"], st["plastic"])
        Ks = sp.csr_matrix((Kt.data, Kt.indices, Kt.indptr))
        du = np.zeros_like(u)
        du[fi] = spl.spsolve(Ks[fi][:, fi].tocsc(), (-F)[fi])
        a = en(u)
        u = u + du
        ref.append(en(du) / (a + en(u)))
    assert len(gpu) == 4
    assert np.allclose(gpu, ref, rtol=1e-6, atol=0), (gpu, ref)


@pytest.mark.parametrize("block", [2, 3])
def test_restricted_solve_block_jacobi(cuda, block):
    """The node-block Jacobi CG (epfem_restricted_solve_blocked) solves the
    same restricted SPD system as the scalar one, to the same tolerance, with
    fixed dofs zero; a dimension not divisible by the block is rejected."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.solver import LinearSolver, SolveInfo, SolveSettings, restricted_solve
    rng = np.random.default_rng(7 + block)
    n = 60 * block
    A = rng.standard_normal((n, n))
    A = A @ A.T + n * np.eye(n)
    A[np.abs(A) < 0.5] = 0.0
    A = 0.5 * (A + A.T) + n * np.eye(n)
    b = rng.standard_normal(n)
    free = rng.random(n) > 0.2
    K = _csr(A, cuda)
    s = SolveSettings(LinearSolver.conjugate_gradient, rel_tol=1e-12)
    i1, ib = SolveInfo(), SolveInfo()
    x1 = restricted_solve(K, torch.from_numpy(b).to(cuda), torch.from_numpy(free).to(cuda), s, info=i1).cpu().numpy()
    xb = restricted_solve(K, torch.from_numpy(b).to(cuda), torch.from_numpy(free).to(cuda), s, info=ib,
                          block=block).cpu().numpy()
    fi = np.nonzero(free)[0]
    ref = np.zeros(n)
    ref[fi] = np.linalg.solve(A[np.ix_(fi, fi)], b[fi])
    assert np.all(xb[~free] == 0.0)
    assert np.abs(xb - ref).max() <= 1e-9 * np.abs(ref).max()
    assert np.abs(x1 - ref).max() <= 1e-9 * np.abs(ref).max()
    assert ib.residual <= 1e-12
    with pytest.raises(P.Error, match="dimension mismatch"):
        restricted_solve(_csr(A[:n - 1, :n - 1], cuda), torch.from_numpy(b[:n - 1]).to(cuda), None, s, block=block)


def test_restricted_solve_direct(cuda):
    """LinearSolver::direct (linalg.cpp:84-96) on the device: a random SPD
    system with a random free set vs a dense solve, zero on fixed dofs,
    deterministic; an indefinite (not positive definite) restricted system
    through the QR fallback; the reference's singular case raises SolverError
    (tests/test_linalg.cpp:153-162)."""
    from paper_1805_04155_b200.solver import SolveInfo, SolveSettings, SolverError, restricted_solve
    rng = np.random.default_rng(31)
    n = 80
    A = rng.uniform(-1, 1, (n, n))
    Kd = A.T @ A + 0.5 * np.eye(n)
    rhs = rng.uniform(-1, 1, n)
    mask = rng.uniform(size=n) < 0.7
    info = SolveInfo()
    x = restricted_solve(_csr(Kd, cuda), torch.from_numpy(rhs).to(cuda), torch.from_numpy(mask).to(cuda),
                         SolveSettings(rel_tol=1e-12), info=info).cpu().numpy()
    f = np.nonzero(mask)[0]
    xf = np.linalg.solve(Kd[np.ix_(f, f)], rhs[f])
    assert np.abs(x[f] - xf).max() <= 1e-10 * np.abs(xf).max()
    assert np.all(x[~mask] == 0.0) and not info.substituted and info.residual <= 1e-12 and info.iterations >= 1
    x2 = restricted_solve(_csr(Kd, cuda), torch.from_numpy(rhs).to(cuda), torch.from_numpy(mask).to(cuda),
                          SolveSettings(rel_tol=1e-12)).cpu().numpy()
    assert np.array_equal(x.view(np.uint64), x2.view(np.uint64))
    # symmetric indefinite: Cholesky declines, QR solves
    S = rng.uniform(-1, 1, (n, n))
    S = 0.5 * (S + S.T) + np.diag(np.where(np.arange(n) % 2 == 0, 3.0, -3.0))
    xs = restricted_solve(_csr(S, cuda), torch.from_numpy(rhs).to(cuda), None, SolveSettings(rel_tol=1e-10)).cpu().numpy()
    assert np.abs(xs - np.linalg.solve(S, rhs)).max() <= 1e-8 * np.abs(np.linalg.solve(S, rhs)).max()


def test_restricted_solve_direct_sparse_path(cuda, monkeypatch):
    """The sparse cuSOLVER path (restricted systems above the dense limit;
    forced here with EPFEM_DIRECT_DENSE_MAX=0): Cholesky with the cached
    symbolic analysis on an SPD system, repeated with new values on the same
    pattern, and the QR fallback on an indefinite one."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.solver import SolveInfo, SolveSettings, restricted_solve
    monkeypatch.setenv("EPFEM_DIRECT_DENSE_MAX", "0")
    ctx = P.Context(cuda)
    rng = np.random.default_rng(37)
    n = 120
    # banded SPD (a 1D chain with a few couplings), like a mesh numbering
    A = np.zeros((n, n))
    for i in range(n):
        for j in range(max(0, i - 4), min(n, i + 5)):
            A[i, j] = rng.uniform(-1, 1)
    Kd = A @ A.T + n * np.eye(n)
    mask = rng.uniform(size=n) < 0.8
    f = np.nonzero(mask)[0]
    M = _csr(Kd, cuda)
    for scale in (1.0, 3.0):  # second call: same pattern and mask, new values (numeric factorisation only)
        M.values.mul_(scale)
        Ks = Kd * (3.0 if scale == 3.0 else 1.0)
        rhs = rng.uniform(-1, 1, n)
        info = SolveInfo()
        x = restricted_solve(M, torch.from_numpy(rhs).to(cuda), torch.from_numpy(mask).to(cuda),
                             SolveSettings(rel_tol=1e-12), ctx=ctx, info=info).cpu().numpy()
        xf = np.linalg.solve(Ks[np.ix_(f, f)], rhs[f])
        assert np.abs(x[f] - xf).max() <= 1e-10 * np.abs(xf).max()
        assert np.all(x[~mask] == 0.0) and not info.substituted and info.residual <= 1e-12
    S = rng.uniform(-1, 1, (n, n))
    S = 0.5 * (S + S.T) + np.diag(np.where(np.arange(n) % 2 == 0, 3.0, -3.0))
    rhs = rng.uniform(-1, 1, n)
    xs = restricted_solve(_csr(S, cuda), torch.from_numpy(rhs).to(cuda), None, SolveSettings(rel_tol=1e-10),
                          ctx=ctx).cpu().numpy()
    ref = np.linalg.solve(S, rhs)
    assert np.abs(xs - ref).max() <= 1e-8 * np.abs(ref).max()


@pytest.mark.parametrize("dense_max", ["16384", "0"])
def test_restricted_solve_direct_pattern_rewritten_in_place(cuda, monkeypatch, dense_max):
    """The direct solve caches the restricted pattern and its analysis; the
    key is the pattern's content, so a caller that rewrites row_ptr / col_idx
    in place (same addresses, same n, same free mask, same nnz) gets a solve
    of the new matrix, not of the cached pattern."""
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.solver import SolveSettings, restricted_solve
    monkeypatch.setenv("EPFEM_DIRECT_DENSE_MAX", dense_max)
    ctx = P.Context(cuda)
    rng = np.random.default_rng(41)
    n = 60

    def spd(offsets):
        A = np.eye(n) * 8.0
        for d in offsets:
            for i in range(n - d):
                A[i, i + d] = A[i + d, i] = rng.uniform(-1, 1)
        return A

    # offsets (1, 4) and (2, 3): the same nnz (2 (59 + 56) = 2 (58 + 57)), different columns
    import scipy.sparse as sp
    c1, c2 = sp.csr_matrix(spd((1, 4))), sp.csr_matrix(spd((2, 3)))
    c1.sort_indices()
    c2.sort_indices()
    assert c1.nnz == c2.nnz and not np.array_equal(c1.indices, c2.indices)
    M = P.CsrMatrix(torch.from_numpy(c1.indptr.astype(np.int64)).to(cuda),
                    torch.from_numpy(c1.indices.astype(np.int32)).to(cuda),
                    torch.from_numpy(c1.data.astype(np.float64)).to(cuda))
    rhs = rng.uniform(-1, 1, n)
    b = torch.from_numpy(rhs).to(cuda)
    x1 = restricted_solve(M, b, None, SolveSettings(rel_tol=1e-12), ctx=ctx).cpu().numpy()
    assert np.abs(x1 - np.linalg.solve(c1.toarray(), rhs)).max() <= 1e-10
    M.row_ptr.copy_(torch.from_numpy(c2.indptr.astype(np.int64)))
    M.col_idx.copy_(torch.from_numpy(c2.indices.astype(np.int32)))
    M.values.copy_(torch.from_numpy(c2.data.astype(np.float64)))
    x2 = restricted_solve(M, b, None, SolveSettings(rel_tol=1e-12), ctx=ctx).cpu().numpy()
    assert np.abs(x2 - np.linalg.solve(c2.toarray(), rhs)).max() <= 1e-10
