"""Time Newton time steps on the GPU: the cfg2
material on an n x n Q2-8 mesh, left edge clamped, the right edge pulled to
u_x = delta in `steps` load increments (each a newton_solve from the previous
step's committed state and a warm start, as the reference's drivers load); per-iteration step
(constitutive + K + F) time, CG iterations, wall time.  Not a product path.

    python tools/newton_bench.py [n] [delta] [steps]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(n=64, delta=0.004, steps=8):
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS
    dev = torch.device("cuda", 0)
    cfg = CONFIGS["cfg2"]
    mesh = cfg.mesh(int(n))
    mat = cfg.material(mesh.n_int)
    x = mesh.coord
    nd = x.shape[0] * 2
    free = np.ones(nd, bool)
    left, right = np.isclose(x[:, 0], 0.0), np.isclose(x[:, 0], x[:, 0].max())
    free[2 * np.nonzero(left)[0]] = free[2 * np.nonzero(left)[0] + 1] = False
    free[2 * np.nonzero(right)[0]] = False
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, dev), mat)
    settings = P.NewtonSettings(eps_newton=1e-9, linear=P.SolveSettings(rel_tol=1e-10))
    state, u, out = P.IntegrationState.zero(mesh.n_int, device=dev), None, []
    torch.cuda.synchronize()
    t = time.perf_counter()
    for k in range(1, int(steps) + 1):
        dirichlet = np.zeros(nd)
        dirichlet[2 * np.nonzero(right)[0]] = float(delta) * k / int(steps)
        # warm start: the affine field of the load on the first step (the bare Dirichlet lift
        # concentrates the whole pull in the last element column), then the previous step's u
        # scaled to the new load
        if u is None:
            u0 = np.zeros(nd)
            u0[0::2] = float(delta) * k / int(steps) * x[:, 0] / x[:, 0].max()
            u_start = torch.from_numpy(u0)
        else:
            u_start = u * (k / (k - 1))
        try:
            r = P.newton_solve(gc, mat, state, torch.from_numpy(dirichlet), torch.from_numpy(free),
                               torch.zeros(nd, dtype=torch.float64), settings, u_start=u_start)
        except P.NonConvergenceError as e:
            out.append({"step": k, "nonconvergence": e.record.ratios[:8]})
            break
        state, u = r.state, r.u
        out.append({"step": k, "newton_iters": r.record.newton_iters, "n_plastic": r.record.n_plastic,
                    "cg_iters": r.record.linear_iters, "step_ms": [round(s.tangent_seconds * 1e3, 4)
                                                                   for s in r.record.iterations]})
    torch.cuda.synchronize()
    print(json.dumps({"mesh": f"Q2-8 {n}x{n}", "dofs": nd, "n_int": mesh.n_int, "delta": float(delta),
                      "load_steps": out, "wall_s": round(time.perf_counter() - t, 3)}))


if __name__ == "__main__":
    main(*sys.argv[1:])
