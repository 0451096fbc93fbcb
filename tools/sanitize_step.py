"""One Newton step of a reduced BASELINE configuration through every hot
kernel (the fused update + element deltas, the row stream, the separate
constitutive + tangent path, the step from displacements and with internal
forces) for compute-sanitizer (tools/sanitize.sh).

    python tools/sanitize_step.py cfg4 6
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main(name, n):
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, calibrate, displacement
    dev = torch.device("cuda", 0)
    cfg = CONFIGS[name]
    mesh = cfg.mesh(n)
    mat = cfg.material(mesh.n_int)
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, dev), mat)
    u1 = torch.from_numpy(displacement(mesh.coord, cfg.seed)).to(dev)
    E1 = gc.strains(u1)
    s, frac = calibrate(E1, mat, 0.4)
    E = (s * E1).contiguous()
    eng = P.TangentEngine(gc, mat)
    eng.step(E)
    sep = P.TangentEngine(gc, mat, fused=False)
    sep.step(E)
    eng.step_u((s * u1).contiguous())
    eng.step_f(E)
    torch.cuda.synchronize()
    same = torch.equal(eng.K, sep.K)
    print(f"sanitize_step {name} n={n} plastic={frac:.2f} fused==separate {same}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
