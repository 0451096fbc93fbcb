import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1805_04155_b200 as P
import paper_1805_04155_b200.solver as S
from paper_1805_04155_b200.benchmarks import BenchmarkConfig, run_dp_footing
from paper_1805_04155_b200.solver import NewtonSettings, SolveSettings, LinearSolver, SolveInfo
import scipy.sparse as sp, scipy.sparse.linalg as spl
dev = torch.device('cuda', 0)
orig = S.restricted_solve
log = []
def wrapped(K, rhs, free_mask=None, settings=SolveSettings(), ctx=None, info=None, block=1):
    x = orig(K, rhs, free_mask, settings, ctx=ctx, info=info, block=block)
    A = sp.csr_matrix((K.values.cpu().numpy(), K.col_idx.cpu().numpy(), K.row_ptr.cpu().numpy()))
    f = free_mask.cpu().numpy().astype(bool)
    fi = np.nonzero(f)[0]
    b = rhs.cpu().numpy()
    xs = np.zeros_like(b); xs[fi] = spl.spsolve(A[fi][:, fi].tocsc(), b[fi])
    xx = x.cpu().numpy()
    log.append((settings.method.name, info.iterations if info else None, info.residual if info else None,
                float(np.abs(xx - xs).max() / max(np.abs(xs).max(), 1e-300))))
    return x
S.restricted_solve = wrapped
cfg = BenchmarkConfig(dim=2, elem="P1", level=0, du0=1e-3, u_max=2e-3, theta=1e-3,
                      newton=NewtonSettings(eps_newton=1e-10, max_iters=25, linear=SolveSettings(LinearSolver.direct, rel_tol=1e-12), on_failure="error"))
res = run_dp_footing(cfg, device=dev)
for l in log: print(l)
