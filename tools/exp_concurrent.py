"""Timing experiment (not a product path): does the row stream overlap the
fused constitutive+delta kernel if both run concurrently on two streams?
The concurrent case assembles from the PREVIOUS step's workspace, so only its
timing is meaningful.

    python tools/exp_concurrent.py [--config cfg2] [--reps 30]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--prio", action="store_true", help="row stream on a high-priority stream")
    args = ap.parse_args()
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, make_workload
    dev = torch.device("cuda", 0)
    cfg = CONFIGS[args.config]
    wl = make_workload(cfg, device=dev)
    cache, mat = wl.cache, wl.mat
    sa, sb = torch.cuda.Stream(dev), torch.cuda.Stream(dev, priority=-1 if args.prio else 0)
    eng = P.TangentEngine(cache, mat, stream=sa)
    ctx_b = P.Context(0, stream=sb, synchronous=False)
    E = wl.E.contiguous()
    Ep0 = torch.zeros_like(E)
    Hard0 = torch.zeros_like(E) if cfg.model == "vm" else None
    lib, C_ = P.api.L.lib(), P.api.C

    def fused():
        P.api._check(lib.epfem_constitutive_delta(eng.ctx.handle, cache.handle, C_.byref(eng._mv),
                                                  P.api._ptr(E), P.api._ptr(Ep0), P.api._ptr(Hard0),
                                                  C_.byref(eng._out)))

    def rows(ctx):
        P.api._check(lib.epfem_assemble_rows(ctx.handle, cache.handle, P.api._ptr(eng.K)))

    main_s = torch.cuda.current_stream(dev)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev[0].record(main_s)
        for _ in range(args.reps):
            fn()
        ev[1].record(main_s)
        torch.cuda.synchronize()
        return ev[0].elapsed_time(ev[1]) / args.reps

    def seq():
        sa.wait_stream(main_s)
        fused()
        rows(eng.ctx)
        main_s.wait_stream(sa)

    def conc():
        sa.wait_stream(main_s)
        sb.wait_stream(main_s)
        fused()
        rows(ctx_b)
        main_s.wait_stream(sa)
        main_s.wait_stream(sb)

    def only_f():
        sa.wait_stream(main_s)
        fused()
        main_s.wait_stream(sa)

    def only_r():
        sb.wait_stream(main_s)
        rows(ctx_b)
        main_s.wait_stream(sb)

    eng2 = P.TangentEngine(cache, mat, stream=sa, fused=False)

    def cons():
        sa.wait_stream(main_s)
        P.api._check(lib.epfem_constitutive(eng2.ctx.handle, C_.byref(eng2._mv), P.api._ptr(E),
                                            P.api._ptr(Ep0), P.api._ptr(Hard0), C_.byref(eng2._out)))
        main_s.wait_stream(sa)

    def tang():
        sa.wait_stream(main_s)
        P.api._check(lib.epfem_assemble_tangent(eng2.ctx.handle, cache.handle, cache.n_int,
                                                P.api._ptr(eng2.D), P.api._ptr(eng2.flags),
                                                P.api._ptr(eng2.K)))
        main_s.wait_stream(sa)

    print(f"separate path: constitutive {timeit(cons):.4f} ms, assemble_tangent (delta + rows) "
          f"{timeit(tang):.4f} ms")
    print(f"{args.config} prio={args.prio}: fused alone {timeit(only_f):.4f} ms, rows alone {timeit(only_r):.4f} ms, "
          f"sequential {timeit(seq):.4f} ms, concurrent {timeit(conc):.4f} ms")


if __name__ == "__main__":
    main()
