"""Timing experiment (not a product path): K8 strains, K9 internal forces and
the strain-fused / force-fused steps on one BASELINE configuration.

    python tools/time_k8k9.py cfg4 [cfg3 ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main(names):
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, make_workload
    dev = torch.device("cuda", 0)
    for name in names:
        cfg = CONFIGS[name]
        wl = make_workload(cfg, device=dev)
        cache = wl.cache
        E = wl.E.contiguous()
        Ep = torch.zeros_like(E)
        Hd = torch.zeros_like(E) if cfg.model == "vm" else None
        u = torch.randn(cache.info.n_dofs, dtype=torch.float64, device=dev) * 1e-4
        eng = P.TangentEngine(cache, wl.mat)
        eng.step(E, Ep, Hd)
        S = eng.S

        fns = {
            "strains": lambda: cache.strains(u),
            "forces": lambda: P.api.internal_forces(cache, S),
            "step": lambda: eng.step(E, Ep, Hd),
            "step_f": lambda: eng.step_f(E, Ep, Hd),
        }
        out = {"config": name}
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for nm, fn in fns.items():
            for _ in range(3):
                fn()
            torch.cuda.synchronize(dev)
            ev[0].record()
            for _ in range(10):
                fn()
            ev[1].record()
            torch.cuda.synchronize(dev)
            out[nm + "_ms"] = round(ev[0].elapsed_time(ev[1]) / 10, 4)
        print(json.dumps(out), flush=True)
        del eng, wl, cache
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main(sys.argv[1:] or ["cfg4"])
