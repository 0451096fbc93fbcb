import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1805_04155_b200 as P
from paper_1805_04155_b200.benchmarks import build_mesh_footing
from paper_1805_04155_b200.solver import SolveSettings, LinearSolver, restricted_solve, SolveInfo
dev = torch.device('cuda', 0)
for fam, lvl in (("P1", 2), ("Q2", 3)):
    bm = build_mesh_footing(lvl, fam, 2)
    m = bm.mesh
    K_, G_ = P.elastic_moduli(1e7, 0.48)
    cache = P.build_assembly_cache(P.Mesh.from_structured(m, dev), P.uniform_elastic(m.n_int, K_, G_))
    Ke = cache.K_elast
    free = torch.from_numpy(bm.free_mask()).to(dev)
    b = torch.randn(cache.info.n_dofs, dtype=torch.float64, device=dev)
    ctx = P.Context(0, synchronous=True)
    for meth in (LinearSolver.direct, LinearSolver.conjugate_gradient):
        info = SolveInfo()
        restricted_solve(Ke, b, free, SolveSettings(meth, 1e-10), ctx=ctx, info=info)
        torch.cuda.synchronize(); t = time.perf_counter()
        for _ in range(10): restricted_solve(Ke, b, free, SolveSettings(meth, 1e-10), ctx=ctx, info=info)
        torch.cuda.synchronize(); print(fam, lvl, meth.name, cache.info.n_dofs, 'ms/solve', round((time.perf_counter() - t) * 100, 2), info)
