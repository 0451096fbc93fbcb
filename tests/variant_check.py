"""Subprocess body of test_gpu_parity.test_kernel_variants: the library reads
its kernel-variant switch (EPFEM_FUSED) once per process, so each variant is
checked in a fresh interpreter.  For one BASELINE configuration on a reduced
mesh: fused Newton step vs the oracle (flags and S bit-exact, K row-scaled
<= 1e-12) and the separate constitutive + tangent calls bitwise equal to the
fused step.  Prints OK on success, raises otherwise.

    EPFEM_FUSED=mma python tests/variant_check.py cfg2 24
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from helpers import row_scaled_error  # noqa: E402


def main(name, n):
    import paper_1805_04155_b200 as P
    from oracle import oracle as O
    from paper_1805_04155_b200.synthetic import CONFIGS, displacement
    O.build()
    dev = torch.device("cuda", 0)
    cfg = CONFIGS[name]
    mesh = cfg.mesh(n)
    mat = cfg.material(mesh.n_int)
    K, G = P.elastic_moduli(cfg.young, cfg.poisson)
    oc = O.Cache(cfg.family, cfg.dim, mesh.coord, mesh.elem, G, K)
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, dev), mat)
    E1 = oc.strains(displacement(mesh.coord, cfg.seed))
    if cfg.model == "vm":
        crit = O.constitutive_vm(E1, None, None, G, K, cfg.p1, 0.0)["crit"]
        E = (cfg.p2 / np.quantile(crit, 1.0 - cfg.target)) * E1
        ref = O.constitutive_vm(E, None, None, G, K, cfg.p1, cfg.p2)
    else:
        eta, c = P.dp_parameters(cfg.p1, cfg.p2)
        s = 1.0
        for _ in range(60):
            f = O.constitutive_dp(s * E1, None, G, K, eta, c)["plastic"].mean()
            s *= 1.3 if f < cfg.target else 0.8
            if abs(f - cfg.target) < 0.05:
                break
        E = s * E1
        ref = O.constitutive_dp(E, None, G, K, eta, c)
    pl = ref["plastic"]
    assert 0 < pl.sum() < pl.size
    Kref = oc.tangent(ref["DS"], pl)
    Et = torch.from_numpy(np.ascontiguousarray(E)).to(dev)
    eng = P.TangentEngine(gc, mat)
    S, flags, D, Kv = eng.step(Et)
    eng.sync()
    assert np.array_equal(flags.cpu().numpy() & 1, pl)
    assert np.array_equal(S.cpu().numpy(), ref["S"])
    err = row_scaled_error(Kv.cpu().numpy(), Kref.data, Kref.indptr, oc.K_elast().data)
    assert err <= 1e-12, err
    sep = P.TangentEngine(gc, mat, fused=False)
    S2, f2, D2, K2 = sep.step(Et)
    sep.sync()
    assert np.array_equal(K2.cpu().numpy().view(np.uint64), Kv.cpu().numpy().view(np.uint64))
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("EPFEM_")) or "default"
    print(f"OK {tag} {name} n={n} plastic={pl.mean():.2f} err={err:.2e}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]))
