"""Time the paper's strip-footing benchmark (run_dp_footing, benchmarks.cpp:120-205)
with every Newton step on the GPU: load steps, Newton and CG iterations, the
normalised pressure path, wall time.  Not a product path.

    python tools/footing_bench.py [level] [family] [dim] [u_max] [du0] [direct|conjugate_gradient]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def main(level=2, family="P1", dim=2, u_max=0.02, du0=1e-3, method="direct"):
    from paper_1805_04155_b200.benchmarks import BenchmarkConfig, run_dp_footing
    from paper_1805_04155_b200.solver import LinearSolver, NewtonSettings, SolveSettings
    cfg = BenchmarkConfig(dim=int(dim), elem=family, level=int(level), du0=float(du0), u_max=float(u_max),
                          newton=NewtonSettings(eps_newton=1e-10,
                                                linear=SolveSettings(LinearSolver[method], rel_tol=1e-10)))
    torch.cuda.synchronize()
    t = time.perf_counter()
    res = run_dp_footing(cfg)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t
    recs = res.records
    print(json.dumps({
        "benchmark": "dp_footing", "family": family, "dim": int(dim), "level": int(level),
        "n_int": res.n_int, "n_dofs": res.mesh.n_dofs, "completed": res.completed,
        "steps": len(recs), "newton_iters": sum(r.newton_iters for r in recs),
        "linear_solver": method, "linear_iters": sum(sum(r.linear_iters) for r in recs),
        "tangent_seconds": sum(r.tangent_seconds for r in recs),
        "wall_s": wall, "u_D": [r.load for r in recs], "p_over_c0": [r.derived_scalar for r in recs],
        "n_plastic": [r.n_plastic for r in recs]}))


if __name__ == "__main__":
    main(*sys.argv[1:])
