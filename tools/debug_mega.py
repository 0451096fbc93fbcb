"""Debug (not a product path): one-launch step vs the two launches in one
process; saves K (both), K_elast and the differing entries' context."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main(name, n, reps):
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
    Ep0 = torch.zeros_like(E)
    Hard0 = torch.zeros_like(E)
    eng = P.TangentEngine(gc, mat)
    lib, C_ = P.api.L.lib(), P.api.C
    P.api._check(lib.epfem_constitutive_delta(eng.ctx.handle, gc.handle, C_.byref(eng._mv), P.api._ptr(E),
                                              P.api._ptr(Ep0), P.api._ptr(Hard0), C_.byref(eng._out)))
    K2 = torch.empty_like(eng.K)
    P.api._check(lib.epfem_assemble_rows(eng.ctx.handle, gc.handle, P.api._ptr(K2)))
    torch.cuda.synchronize()
    R2, M2 = [x.cpu().numpy() for x in gc.workspace()]
    D2 = eng.D.cpu().numpy().copy()
    K2 = K2.cpu().numpy()
    Ke = gc.K_elast.values.cpu().numpy()
    rp = gc.row_ptr.cpu().numpy()
    rows = np.repeat(np.arange(rp.size - 1), np.diff(rp))
    for r in range(int(reps)):
        S, flags, D, Kv = eng.step(E, Ep0, Hard0)
        eng.sync()
        K = Kv.cpu().numpy()
        R, M = [x.cpu().numpy() for x in gc.workspace()]
        pl = M != 0
        rd = np.nonzero((R.view(np.uint64) != R2.view(np.uint64)).any(axis=1) & pl)[0]
        Dm = (flags.cpu().numpy() & 1).astype(bool)
        dd = np.nonzero((D.cpu().numpy().view(np.uint64) != D2.view(np.uint64)).any(axis=1) & Dm)[0]
        print(f"rep {r}: masks equal {np.array_equal(M, M2)}, records differing {rd.size} of {pl.sum()} "
              f"(elements {rd[:12]}), D differing {dd.size}")
        for e in rd[:3]:
            c = np.nonzero(R[e].view(np.uint64) != R2[e].view(np.uint64))[0]
            print(f"   element {e} mask {M[e]:09b} entries {c[:16]} mega {R[e][c[:3]]} two {R2[e][c[:3]]}")
        d = np.nonzero(K.view(np.uint64) != K2.view(np.uint64))[0]
        if r == 0:
            np.savez("gpurun_out/debug_mega.npz", K=K, K2=K2, Ke=Ke, R=R, M=M, row_ptr=rp,
                     col_idx=gc.col_idx.cpu().numpy(), elem=mesh.elem, d=d)
        print(f"rep {r}: {d.size} differing entries")
        for i in d[:6]:
            print(f"   idx {i} row {rows[i]} col {gc.col_idx[i].item()} two {K2[i]!r} mega {K[i]!r} "
                  f"Kelast {Ke[i]!r} two-Ke {K2[i]-Ke[i]!r} mega-Ke {K[i]-Ke[i]!r}")


if __name__ == "__main__":
    main(*sys.argv[1:])
