"""Timing experiment (not a product path): the halves of the Newton step on
one BASELINE configuration, each launched alone on one stream with CUDA
events (after warm-up):

  fused      epfem_constitutive_delta (update + element deltas, one kernel)
  rows       epfem_assemble_rows (row stream)
  lean       epfem_constitutive, hot-path outputs only (S, flags, packed D)
  delta      epfem_delta_range over all elements (element deltas from D)
  step       epfem_newton_step (fused + rows)
  separate   lean + delta + rows

    python tools/time_paths.py cfg4 [cfg5 ...]     (prints one JSON line per config)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main(names, target=None):
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, make_workload
    dev = torch.device("cuda", 0)
    lib = P.api.L.lib()
    C = P.api.C
    for name in names:
        cfg = CONFIGS[name]
        wl = make_workload(cfg, device=dev, target=target)
        cache, mat = wl.cache, wl.mat
        E = wl.E.contiguous()
        Ep = torch.zeros_like(E)
        Hd = torch.zeros_like(E) if cfg.model == "vm" else None
        st = torch.cuda.Stream(dev)
        eng = P.TangentEngine(cache, mat, stream=st)
        h = eng.ctx.handle

        def fused():
            P.api._check(lib.epfem_constitutive_delta(h, cache.handle, C.byref(eng._mv), P.api._ptr(E),
                                                      P.api._ptr(Ep), P.api._ptr(Hd), C.byref(eng._out)))

        def rows():
            P.api._check(lib.epfem_assemble_rows(h, cache.handle, P.api._ptr(eng.K)))

        def lean():
            P.api._check(lib.epfem_constitutive(h, C.byref(eng._mv), P.api._ptr(E), P.api._ptr(Ep),
                                                P.api._ptr(Hd), C.byref(eng._out)))

        def delta():
            P.api._check(lib.epfem_delta_range(h, cache.handle, cache.n_int, P.api._ptr(eng.D),
                                               P.api._ptr(eng.flags), 0, cache.info.n_elements))

        def step():
            fused()
            rows()

        def separate():
            lean()
            delta()
            rows()

        out = {"config": name, "plastic_fraction": wl.fraction}
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(st):
            for nm, fn in (("fused", fused), ("rows", rows), ("lean", lean), ("delta", delta), ("step", step),
                           ("separate", separate)):
                for _ in range(3):
                    fn()
                torch.cuda.synchronize(dev)
                reps = 10
                ev[0].record(st)
                for _ in range(reps):
                    fn()
                ev[1].record(st)
                torch.cuda.synchronize(dev)
                out[nm + "_ms"] = ev[0].elapsed_time(ev[1]) / reps
        out["EPFEM_FUSED"] = os.environ.get("EPFEM_FUSED", "")
        print(json.dumps(out), flush=True)
        del eng, wl, cache, E, Ep, Hd
        torch.cuda.empty_cache()


if __name__ == "__main__":
    args = sys.argv[1:] or ["cfg4"]
    tgt = None
    if args and args[0].startswith("--target="):
        tgt = float(args[0].split("=")[1])
        args = args[1:]
    main(args, tgt)
