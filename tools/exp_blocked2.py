"""Timing experiment (not a product path): the cfg4 step in blocks of cell layers on TWO streams.
Stream A (low priority) runs the fused kernel of block 0, 1, 2, ... back to back (epfem_newton_range);
stream B (high priority) runs, after block k's event, the row stream of the node planes that block
completes (epfem_assemble_rows_range), so a block's element records are read back while L2-resident
and the drain of one kernel is filled by the other stream's CTAs.  Compared with the plain step.

    python tools/exp_blocked2.py [layers per block ...]
"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def main(blocks):
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, make_workload
    api = P.api
    dev = torch.device("cuda", 0)
    lib = api.L.lib()
    cfg = CONFIGS["cfg4"]
    wl = make_workload(cfg, device=dev)
    cache, mat = wl.cache, wl.mat
    E = wl.E.contiguous()
    Ep = torch.zeros_like(E)
    Hd = torch.zeros_like(E)
    lo, hi = torch.cuda.Stream.priority_range()
    sA = torch.cuda.Stream(dev, priority=lo)
    sA1 = torch.cuda.Stream(dev, priority=lo)
    sB = torch.cuda.Stream(dev, priority=hi)
    eng = P.TangentEngine(cache, mat, stream=sA)
    h = eng.ctx.handle
    n = cfg.n
    nq = 8
    layer_e, plane_n = n * n, (n + 1) * (n + 1)
    n_layers = n

    def set_stream(st):
        api._check(lib.epfem_ctx_set_stream(h, C.c_void_p(st.cuda_stream)))

    def plain():
        set_stream(sA)
        api._check(lib.epfem_constitutive_delta(h, cache.handle, C.byref(eng._mv), api._ptr(E), api._ptr(Ep),
                                                api._ptr(Hd), C.byref(eng._out)))
        api._check(lib.epfem_assemble_rows(h, cache.handle, api._ptr(eng.K)))

    mats = {}

    def fused_range(e0, e1):
        q0, q1 = e0 * nq, e1 * nq
        out = api.L.ConstitutiveOut()
        out.S, out.flags, out.D = api._ptr(eng.S[q0:q1]), api._ptr(eng.flags[q0:q1]), api._ptr(eng.D[q0:q1])
        if (q0, q1) not in mats:
            mats[(q0, q1)] = mat.slice(q0, q1)
        mv = mats[(q0, q1)].view()
        api._check(lib.epfem_newton_range(h, cache.handle, C.byref(mv), api._ptr(E[q0:q1]), api._ptr(Ep[q0:q1]),
                                          api._ptr(Hd[q0:q1]), C.byref(out), e0, e1))

    def blocked(L, two_streams=True, alt=False):
        nb = (n_layers + L - 1) // L
        evs = [torch.cuda.Event() for _ in range(nb)]
        if alt:
            sA1.wait_stream(sA)
        for k in range(nb):
            z0, z1 = k * L, min((k + 1) * L, n_layers)
            sF = sA1 if (alt and k % 2) else sA
            set_stream(sF)
            fused_range(z0 * layer_e, z1 * layer_e)
            evs[k].record(sF)
            # node planes complete after layers < z1: planes [z0, z1) (plus the top plane at the end)
            p0, p1 = z0, (z1 if z1 < n_layers else n_layers + 1)
            if two_streams:
                sB.wait_event(evs[k])
                set_stream(sB)
            api._check(lib.epfem_assemble_rows_range(h, cache.handle, api._ptr(eng.K), p0 * plane_n, p1 * plane_n))
        if two_streams:
            sA.wait_stream(sB)
        if alt:
            sA.wait_stream(sA1)

    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record(sA)
        for _ in range(reps):
            fn()
        ev[1].record(sA)
        torch.cuda.synchronize(dev)
        return ev[0].elapsed_time(ev[1]) / reps

    out = {"plain_ms": timeit(plain)}
    plain()
    torch.cuda.synchronize(dev)
    Kref = eng.K.clone()
    for L in blocks:
        eng.K.zero_()
        t2 = timeit(lambda: blocked(L, True))
        torch.cuda.synchronize(dev)
        same = bool(torch.equal(eng.K, Kref))
        t1 = timeit(lambda: blocked(L, False))
        eng.K.zero_()
        t3 = timeit(lambda: blocked(L, True, True))
        torch.cuda.synchronize(dev)
        same3 = bool(torch.equal(eng.K, Kref))
        out[f"L{L}"] = {"two_streams_ms": t2, "one_stream_ms": t1, "three_streams_ms": t3, "K_bitwise": same and same3}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [4, 8, 16, 32])
