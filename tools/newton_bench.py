"""Time one Newton time step on the GPU: the cfg2
material on an n x n Q2-8 mesh, left edge clamped, right edge pulled into
yield; per-iteration step (constitutive + K + F) time, CG iterations and
the whole solve.  Not a product path.

    python tools/newton_bench.py [n]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(n=64):
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS
    dev = torch.device("cuda", 0)
    cfg = CONFIGS["cfg2"]
    mesh = cfg.mesh(int(n))
    mat = cfg.material(mesh.n_int)
    x = mesh.coord
    nd = x.shape[0] * 2
    dirichlet, free = np.zeros(nd), np.ones(nd, bool)
    left, right = np.isclose(x[:, 0], 0.0), np.isclose(x[:, 0], x[:, 0].max())
    free[2 * np.nonzero(left)[0]] = free[2 * np.nonzero(left)[0] + 1] = False
    free[2 * np.nonzero(right)[0]] = False
    dirichlet[2 * np.nonzero(right)[0]] = 0.004
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, dev), mat)
    args = (gc, mat, P.IntegrationState.zero(mesh.n_int, device=dev), torch.from_numpy(dirichlet),
            torch.from_numpy(free), torch.zeros(nd, dtype=torch.float64),
            P.NewtonSettings(eps_newton=1e-9, linear=P.SolveSettings(rel_tol=1e-10)))
    P.newton_solve(*args)  # warm-up
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = P.newton_solve(*args)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    print(json.dumps({"mesh": f"Q2-8 {n}x{n}", "dofs": nd, "n_int": mesh.n_int, "newton_iters": r.record.newton_iters,
                      "n_plastic": r.record.n_plastic, "cg_iters": r.record.linear_iters,
                      "step_ms": [round(s.tangent_seconds * 1e3, 4) for s in r.record.iterations],
                      "solve_wall_s": round(wall, 4)}))


if __name__ == "__main__":
    main(*sys.argv[1:])
