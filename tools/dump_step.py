"""Debug helper: run one Newton step on a reduced BASELINE config and save
K, S, flags to gpurun_out/<tag>.npz (compare kernel paths across processes).

    EPFEM_MEGA=0 python tools/dump_step.py cfg2 24 twolaunch
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(name, n, tag, reps=1):
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, calibrate, displacement
    dev = torch.device("cuda", 0)
    cfg = CONFIGS[name]
    mesh = cfg.mesh(int(n))
    mat = cfg.material(mesh.n_int)
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, dev), mat)
    u = torch.from_numpy(displacement(mesh.coord, cfg.seed)).to(dev)
    E1 = gc.strains(u)
    s, _ = calibrate(E1, mat, cfg.target)
    E = (s * E1).contiguous()
    eng = P.TangentEngine(gc, mat)
    outs = []
    for _ in range(int(reps)):
        S, flags, D, Kv = eng.step(E)
        eng.sync()
        outs.append(Kv.cpu().numpy().copy())
    np.savez(f"gpurun_out/{tag}.npz", K=outs[-1], K0=outs[0], S=S.cpu().numpy(), flags=flags.cpu().numpy(),
             row_ptr=gc.row_ptr.cpu().numpy(), col_idx=gc.col_idx.cpu().numpy(), elem=mesh.elem)
    print(tag, "plastic", float((flags & 1).float().mean()), "reps", reps,
          "first==last", bool(np.array_equal(outs[0].view(np.uint64), outs[-1].view(np.uint64))))


if __name__ == "__main__":
    main(*sys.argv[1:])
