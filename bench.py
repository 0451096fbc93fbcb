#!/usr/bin/env python
"""Benchmark: one semismooth-Newton iteration of the hot path.

A step = K1 constitutive update (E, Ep, Hard -> S, flags, packed D at plastic
points) + K2/K6 tangent assembly (K = K_elast + sum_plastic B^T w (D - C) B
into the cached CSR pattern) over the whole configuration, inputs resident in
HBM.  Default workload: the largest single-GPU BASELINE configuration,
configs[3] = "cfg4" (3D Q1 hexahedra 160^3, von Mises a = 1e4, Y = 450, 25 %
plastic, 32.8 M integration points, 1.0 G nonzeros); the same run adds lean
lines for cfg5 (Q2-20 hexahedra 100^3, Drucker-Prager, 50 % plastic; the
largest by bytes) and cfg3 (P2 tetrahedra, DP, 40 %) under "extra_configs".

    python bench.py [--gpus N --steps K --warmup W] [--config cfgX] [--impl reference]

Prints ONE JSON line on rank 0 (driver contract): value = integration
points / s over all ranks; e2e = the same through the public API with host
buffers (H2D E, D2H S + flags + K every step); roofline = the dominant kernel
against MEASURED_PEAKS.json; cpu_baseline = the oracle port of the reference
algorithm on one cell-layer slab of the configuration, pinned to one core.
--impl reference: the same port on every host core over a partition of the
whole configuration into cell-layer slabs (the reference arm).
"""
from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tangent-stiffness assembly: integration points/s and achieved HBM GB/s vs peak"


# optimal FMA per plastic point of the element delta:
# n_p n_s g + n_p (n_p + 1) / 2 g dim, g = 9 (3D) / 4 (2D)
FMA_PER_PLASTIC_POINT = {("P1", 2): 84, ("Q2", 2): 384, ("P2", 3): 2025, ("Q1", 3): 1404, ("Q2", 3): 6750}


def load_fp64_peak():
    p = os.path.join(ROOT, "profiles", "fp64_peak.json")
    try:
        d = json.load(open(p))
        return float(d["fp64_tflops"]), d["source"]
    except (OSError, ValueError, KeyError):
        return 36.6, "fallback (tools/fp64_peak.cu measurement, DESIGN.md)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# ---------------------------------------------------------------------------
# algorithmic bytes

def algorithmic_bytes(cfg, n_int, n_plastic, nnz, n_nodes, n_e, n_p):
    """constitutive 8 (E + Ep [+ Hard for VM] + S) + 1 flag
    byte per point + 288 B of D per plastic point; assembly one write of
    every K value + coordinates + connectivity."""
    hist = 6 if cfg.model == "vm" else 0  # Hard read only for VM
    epr = 6 if cfg.model != "elastic" else 0
    constitutive = 8 * (6 + epr + hist + 6) * n_int + n_int + 288 * n_plastic
    assembly = 8 * nnz + 8 * cfg.dim * n_nodes + 4 * n_p * n_e
    return constitutive, assembly


# ---------------------------------------------------------------------------
# clocks sampling during the timed region

class ClockSampler:
    """SM clock + throttle reasons polled through NVML in a thread for the
    duration of the timed region (the same counters `nvidia-smi
    --query-gpu=clocks.sm,clocks_event_reasons.*` reads; NVML polls fast
    enough for sub-100-ms regions).  Falls back to no samples without NVML."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index=0):
        self.index = index
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self._N = N
            self._h = N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        except Exception:
            self._N = None
        return self

    def _poll(self):
        N = self._N
        self.samples.append(float(N.nvmlDeviceGetClockInfo(self._h, N.NVML_CLOCK_SM)))
        mask = N.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        for nm, bit in self.REASONS.items():
            if mask & bit:
                self.reasons.add(nm)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._poll()
            except Exception:
                return
            time.sleep(0.0005)

    def __exit__(self, *a):
        self._stop.set()
        if self._N is not None:
            self._t.join(timeout=2)
            try:
                self._poll()  # at least one sample at the end of the region
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "source": "NVML polled during the timed region"}


# ---------------------------------------------------------------------------
# CPU baseline: the oracle port of the reference algorithm
#
# The configuration is partitioned into cell-layer slabs along the last axis
# (z in 3D, y in 2D).  A slab's elements are a contiguous range
# of the full mesh (cell order (k, j, i), mesh.cpp:192-204), so the slab is
# cut out of the full oracle mesh with bitwise the same coordinates, and its
# points are the full workload's points.  A worker process, pinned to one
# core (the reference is single-threaded), builds the oracle cache of each of
# its slabs (untimed, like the reference's one-time build_assembly_cache) and
# times `reps` iterations of evaluate_constitutive + assemble_tangent_stiffness
# on it with the reference's own steady_clock timer (oracle mode A,
# solver.cpp:24,27-32).

SLAB_LAYERS = {"cfg1": 256, "cfg2": 64, "cfg3": 8, "cfg4": 5, "cfg5": 4}  # layers per slab


def _cpu_worker(name, slabs, core, scale, reps, warmup, conn):
    """Run in a spawned process: for each slab (k0, k1) build the oracle cache
    and time `warmup` + `reps` iterations.  Sends back, per slab, (n_int,
    [t per rep], n_plastic).  scale None: calibrate this slab's strains to
    the configuration's plastic fraction by the unit-scale yield quantile."""
    try:
        if core is not None:
            os.sched_setaffinity(0, {core})
        sys.path.insert(0, ROOT)
        import numpy as np
        from oracle import oracle as O
        from paper_1805_04155_b200.synthetic import CONFIGS, displacement
        cfg = CONFIGS[name]
        n = cfg.n
        coord, elem, _ = O.structured_mesh(cfg.family, cfg.dim, n, n, n if cfg.dim == 3 else 0)
        per = elem.shape[0] // n
        K, G = O.elastic_moduli(cfg.young, cfg.poisson)
        out = []
        for k0, k1 in slabs:
            es = elem[k0 * per:k1 * per]
            nodes = np.unique(es)
            el = np.searchsorted(nodes, es).astype(np.int32)
            cl = np.ascontiguousarray(coord[nodes])
            cache = O.Cache(cfg.family, cfg.dim, cl, el, G, K)
            if cfg.model == "elastic":
                # the timed region is assemble_elastic_stiffness inside the cache build: one build per
                # iteration (the first `warmup` builds untimed)
                times = []
                for it in range(warmup + reps):
                    if it:
                        del cache
                        cache = O.Cache(cfg.family, cfg.dim, cl, el, G, K)
                    if it >= warmup:
                        times.append(cache.elastic_assembly_seconds)
                out.append((cache.n_int, times, 0))
                del cache
                continue
            E1 = cache.strains(displacement(cl, cfg.seed))
            if cfg.model == "vm":
                p1, p2, model = cfg.p1, cfg.p2, 1
                g = O.constitutive_vm(E1, None, None, G, K, cfg.p1, 0.0)["crit"]  # |s_tr| at unit scale
            else:
                eta, c = O.dp_parameters(cfg.p1, cfg.p2)
                p1, p2, model = eta, c, 2
                # crit1 at unit scale and c = 0 (crit1 is linear in the scale at zero history)
                e = E1
                tr = (e[:, 0] + e[:, 1]) + e[:, 2]
                dev = e.copy()
                dev[:, :3] -= tr[:, None] / 3.0
                dev[:, 3:] *= 0.5
                ne = np.sqrt(np.maximum(0.0, (e * dev).sum(axis=1)))
                g = 2.0 * G * ne / np.sqrt(2.0) + eta * K * tr
            s = scale if scale is not None else p2 / np.quantile(g, 1.0 - cfg.target)
            E = s * E1
            z = np.zeros_like(E)
            for _ in range(warmup):
                cache.time_iteration(model, E, z, z if model == 1 else None, p1, p2)
            times, npl = [], 0
            for _ in range(reps):
                t, npl = cache.time_iteration(model, E, z, z if model == 1 else None, p1, p2)
                times.append(t)
            out.append((cache.n_int, times, npl))
            del cache, E1, E, z
        conn.send(("ok", out))
    except Exception as exc:  # reported by the parent
        import traceback
        conn.send(("error", traceback.format_exc()))
    finally:
        conn.close()


def cpu_run(name, assignments, scale, reps, warmup, pin=True):
    """assignments: one list of slabs per worker process (worker w pinned to
    core w).  Returns per-worker results (see _cpu_worker)."""
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    procs, pipes = [], []
    for w, slabs in enumerate(assignments):
        r, s_ = ctx.Pipe(duplex=False)
        p = ctx.Process(target=_cpu_worker, args=(name, slabs, w if pin else None, scale, reps, warmup, s_))
        p.start()
        procs.append(p)
        pipes.append(r)
    res = []
    for p, r in zip(procs, pipes):
        status, payload = r.recv()
        p.join()
        if status != "ok":
            raise RuntimeError("CPU baseline worker failed:\n" + payload)
        res.append(payload)
    return res


def cpu_baseline(name, scale):
    """ours-arm cpu_baseline: one slab of the reference arm's
    partition (the bottom SLAB_LAYERS[name] cell layers) on core 0, 1 warm-up
    + median of 3 iterations."""
    from paper_1805_04155_b200.synthetic import CONFIGS
    cfg = CONFIGS[name]
    L = min(SLAB_LAYERS[name], cfg.n)
    t0 = time.perf_counter()
    (res,) = cpu_run(name, [[(0, L)]], scale, reps=3, warmup=1)
    n_int, times, npl = res[0]
    t = statistics.median(times)
    return {"value": n_int / t, "unit": "ip/s", "cores": 1, "kind": "port",
            "host_nproc": os.cpu_count(), "pinned": "core 0 (sched_setaffinity)",
            "sample": (f"one {cfg.n}^{cfg.dim - 1} x {L} cell-layer slab of {name} (layers 0..{L - 1}, {n_int} "
                       f"integration points, the same strains as the GPU workload), oracle mode A = "
                       f"evaluate_constitutive + assemble_tangent_stiffness restated with Eigen's sparse "
                       f"semantics, 1 warm-up + median of 3 iterations ({t:.3f} s/iter)"),
            "n_plastic": npl, "wall_s": time.perf_counter() - t0}


# ---------------------------------------------------------------------------

def run_reference(args, rank, world):
    """--impl reference: the reference algorithm (oracle mode A; the
    reference itself cannot be built here) over a partition of
    the WHOLE configuration into cell-layer slabs, on every host core: worker
    w (pinned to core w) owns a contiguous run of slabs; per slab the cache
    is built once (untimed), then warm-up + `steps` iterations are timed.
    Step k of the whole configuration takes max over workers of the sum of
    their slabs' k-th iteration times (the workers run concurrently); value =
    the configuration's points / the median step time."""
    from paper_1805_04155_b200.synthetic import CONFIGS
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    cores = os.cpu_count() or 1
    L = min(SLAB_LAYERS[args.config], cfg.n)
    slabs = [(k, min(cfg.n, k + L)) for k in range(0, cfg.n, L)]
    W = max(1, min(cores, len(slabs)))
    assign = [slabs[w * len(slabs) // W:(w + 1) * len(slabs) // W] for w in range(W)]
    t0 = time.perf_counter()
    if args.ref_reps is not None:
        reps = max(1, min(args.steps, args.ref_reps))
    else:
        # --steps K timed whole-configuration steps, bounded so the arm ends within a few minutes:
        # one iteration of the first slab on core 0 estimates a step (the busiest worker's slabs)
        budget = float(os.environ.get("EPFEM_REF_BUDGET_S", "180"))
        (cal,) = cpu_run(args.config, [[slabs[0]]], None, 1, 0)
        est = cal[0][1][0] * max(len(a) for a in assign)
        reps = max(1, min(args.steps, int(budget / max(est, 1e-9))))
    warm = 1 if args.warmup > 0 else 0
    res = cpu_run(args.config, assign, None, reps, warm)
    wall = time.perf_counter() - t0
    n_int = sum(r[0] for wr in res for r in wr)
    step_t = [max(sum(r[1][k] for r in wr) for wr in res) for k in range(reps)]
    t = statistics.median(step_t)
    npl = sum(r[2] for wr in res for r in wr)
    value = n_int / t
    sample = (f"the whole {args.config} ({n_int} integration points) partitioned into {len(slabs)} "
              f"{cfg.n}^{cfg.dim - 1} x {L} cell-layer slabs on {W} worker processes pinned one per core; "
              f"oracle mode A = evaluate_constitutive + assemble_tangent_stiffness restated (Eigen "
              f"sparse semantics), caches built once untimed, {warm} warm-up + {reps} timed iterations "
              f"per slab; a step = max over workers of its slabs' summed iteration times")
    line = {
        "metric": METRIC, "value": value, "unit": "ip/s", "impl": "reference",
        "n_gpus": world, "steps": reps, "warmup": warm,
        "warmup_note": "one untimed iteration per slab (one whole-configuration step) before the timed steps; "
                       "steps = --steps unless the estimated run exceeds EPFEM_REF_BUDGET_S (180 s)",
        "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "n_int": n_int, "plastic_fraction": npl / n_int if n_int else 0.0,
                   "same_config": True},
        "cpu_baseline": {"value": value, "unit": "ip/s", "cores": W, "kind": "port", "host_nproc": cores,
                         "sample": sample, "wall_s": wall},
        "e2e": {"value": value, "unit": "ip/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def measured_traffic(config, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel` from
    the committed ncu capture (profiles/traffic.json), or None."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "traffic.json")) as f:
            return json.load(f).get(config, {}).get(kernel)
    except (OSError, ValueError):
        return None


def run_slabs(args, rank, world, dev, cfg):
    """N GPUs: one z-slab (y-slab in 2D) of the configuration's mesh per rank,
    interface-layer exchange over NCCL each step (paper_1805_04155_b200/dist.py).
    Strong scaling: the total work is the whole mesh."""
    import torch
    import torch.distributed as dist

    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.dist import DistributedTangent, make_plan
    from paper_1805_04155_b200.synthetic import displacement, plastic_fraction
    plan = make_plan(cfg.family, cfg.dim, cfg.n, world, rank)
    eng = DistributedTangent(plan, cfg.material, dev)
    u = torch.from_numpy(displacement(plan.mesh.coord, cfg.seed)).to(dev)
    E1 = eng.cache.strains(u)
    p0, p1 = plan.own_points
    E1 = E1[p0:p1].contiguous()
    # global amplitude: bisection on the all-reduced plastic count
    target = cfg.target if args.target is None else args.target
    n_own = torch.tensor([p1 - p0], dtype=torch.float64, device=dev)
    dist.all_reduce(n_own)

    def gfrac(s):
        f = torch.tensor([plastic_fraction(s * E1, eng.mat_own) * (p1 - p0)], dtype=torch.float64,
                         device=dev)
        dist.all_reduce(f)
        return float(f) / float(n_own)

    lo, hi = 0.0, 1.0
    while gfrac(hi) < target and hi < 1e12:
        lo, hi = hi, hi * 4.0
    for _ in range(40):
        mid = 0.5 * (lo + hi)
        lo, hi = (mid, hi) if gfrac(mid) < target else (lo, mid)
    E = (hi * E1).contiguous()
    Ep0 = torch.zeros_like(E)
    Hard0 = torch.zeros_like(E) if cfg.model == "vm" else None
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        eng.step(E, Ep0, Hard0)
    torch.cuda.synchronize(dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            eng.step(E, Ep0, Hard0)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    dist.barrier()
    t = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_per_step = float(t) / args.steps
    n_total = float(n_own)

    # e2e: every step uploads this rank's E / Ep / Hard from pinned host memory
    # and downloads its S, flag bytes and owned K rows (max over ranks).  As in
    # e2e_section, steps are pipelined: the upload of step i+1 (h2d stream) and
    # the download of step i (d2h stream, from a device staging copy, since the
    # engine's outputs are rewritten by the next step) overlap the compute.
    e2e = None
    if not args.no_e2e:
        host_in = [x for x in (E, Ep0, Hard0) if x is not None]
        h_in = [torch.empty_like(x, device="cpu").pin_memory() for x in host_in]
        for h, x in zip(h_in, host_in):
            h.copy_(x)
        d_in = [[torch.empty_like(x) for x in host_in] for _ in range(2)]
        S_, f_, K_ = eng.step(E, Ep0, Hard0)
        stage = [[torch.empty_like(y) for y in (S_, f_, K_)] for _ in range(2)]
        h_out = [[torch.empty_like(y, device="cpu").pin_memory() for y in (S_, f_, K_)] for _ in range(2)]
        bi = sum(x.numel() * x.element_size() for x in host_in)
        bo = sum(y.numel() * y.element_size() for y in h_out[0])
        h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_used = [torch.cuda.Event() for _ in range(2)]
        ev_st = [torch.cuda.Event() for _ in range(2)]
        ev_out = [torch.cuda.Event() for _ in range(2)]
        used = [False, False]

        def e2e_step(i):
            b = i % 2
            if used[b]:
                h2d_s.wait_event(ev_used[b])   # step i-2 has consumed d_in[b]
                stream.wait_event(ev_out[b])   # stage[b] has been downloaded
            with torch.cuda.stream(h2d_s):
                for d, h in zip(d_in[b], h_in):
                    d.copy_(h, non_blocking=True)
                ev_in[b].record(h2d_s)
            stream.wait_event(ev_in[b])
            outs = eng.step(*(d_in[b] + [None] * (3 - len(d_in[b]))))
            ev_used[b].record(stream)
            for d, y in zip(stage[b], outs):
                d.copy_(y, non_blocking=True)
            ev_st[b].record(stream)
            d2h_s.wait_event(ev_st[b])
            with torch.cuda.stream(d2h_s):
                for h, y in zip(h_out[b], stage[b]):
                    h.copy_(y, non_blocking=True)
                ev_out[b].record(d2h_s)
            used[b] = True
        for i in range(max(2, args.warmup)):
            e2e_step(i)
        torch.cuda.synchronize(dev)
        dist.barrier()
        k2 = max(4, min(args.steps, 10))
        ev0.record(stream)
        h2d_s.wait_event(ev0)
        d2h_s.wait_event(ev0)
        for i in range(k2):
            e2e_step(i)
        stream.wait_stream(d2h_s)
        stream.wait_stream(h2d_s)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        t2 = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
        dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        tb = torch.tensor([bi, bo], dtype=torch.float64, device=dev)
        dist.all_reduce(tb)
        ms2 = float(t2) / k2
        e2e = {"value": n_total / (ms2 * 1e-3), "unit": "ip/s", "h2d_bytes_per_step": int(tb[0]),
               "d2h_bytes_per_step": int(tb[1]), "ms_per_step": ms2,
               "how": "per rank: H2D of own E/Ep/Hard, step, D2H of own S/flags/K rows (pipelined across steps "
                      "over two buffer sets and three streams); all ranks summed"}
    # our kernel launches per step on this rank (dist.py DistributedTangent.step): the fused update (two launches
    # when the top layer goes first), the halo deltas (ranks with a halo), the row stream; summed over ranks
    top = max(plan.halo_elems, plan.mesh.n_elements - plan.layer_elems)
    n_launch = (2 if (rank + 1 < world and top > plan.halo_elems) else 1) + (1 if plan.halo_elems else 0) + 1
    launches = torch.tensor([float(n_launch * args.steps)], dtype=torch.float64, device=dev)
    dist.all_reduce(launches)
    npl = torch.tensor([float((eng.flags[p0:p1] & 1).sum())], dtype=torch.float64, device=dev)
    dist.all_reduce(npl)
    # whole-job algorithmic bytes from the owned shares, against
    # world x the per-GPU HBM peak
    v0, v1 = eng.own_values
    n0, n1 = plan.own_nodes
    e_own = (p1 - p0) // max(1, eng.cache.info.n_q)
    cnt = torch.tensor([float(v1 - v0), float(n1 - n0), float(e_own)], dtype=torch.float64, device=dev)
    dist.all_reduce(cnt)
    cons_b, asm_b = algorithmic_bytes(cfg, int(n_total), int(npl), int(cnt[0]), int(cnt[1]), int(cnt[2]),
                                      eng.cache.info.n_p)
    hbm_peak, peak_src = load_peaks()
    step_gbs = (cons_b + asm_b) / (ms_per_step * 1e-3) / 1e9
    if rank == 0:
        line = {
            "metric": METRIC, "value": n_total / (ms_per_step * 1e-3), "unit": "ip/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "element": f"{cfg.family} {cfg.dim}D",
                       "mesh": f"{cfg.n}^{cfg.dim}", "model": cfg.model, "n_int": int(n_total),
                       "plastic_fraction": float(npl) / n_total,
                       "parallelism": f"slab x{world} (one halo cell layer, NCCL interface exchange)",
                       "l2": "inputs larger than L2"},
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "kernel": "whole step (fused update + halo deltas + row stream)",
                         "achieved": step_gbs, "peak": hbm_peak * world, "unit": "GB/s",
                         "frac": step_gbs / (hbm_peak * world), "traffic": None,
                         "algorithmic_bytes": cons_b + asm_b, "peak_source": peak_src + f" x {world} GPUs"},
            "clocks": clk.summary(),
            "e2e": e2e,
        }
        print(json.dumps(line), flush=True)
    dist.destroy_process_group()


def measure_step(name, args, dev, local, world, target=None):
    """Workload + timed steps of one configuration on this GPU.  Returns
    (line fields, context for the e2e / side sections)."""
    import torch

    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, make_workload
    cfg = CONFIGS[name]
    wl = make_workload(cfg, target=target, device=dev)
    cache, mat = wl.cache, wl.mat
    n_int, nnz = cache.n_int, cache.nnz
    stream = torch.cuda.Stream(dev)
    eng = P.TangentEngine(cache, mat, stream=stream)
    E = wl.E.contiguous()
    # plastic history of the previous time step: zero (BASELINE configs), but
    # passed as real arrays and read every step like the reference does
    # (evaluate_constitutive reads prev.Ep / prev.Hard, solver.cpp:24)
    Ep0 = torch.zeros_like(E) if cfg.model != "elastic" else None
    Hard0 = torch.zeros_like(E) if cfg.model == "vm" else None
    hbm_peak, peak_src = load_peaks()
    elastic = cfg.model == "elastic"
    if elastic:
        # cfg1: the timed region is K5, the elastic assembly into the pattern
        Kout = torch.empty((nnz,), dtype=torch.float64, device=dev)

        def launch():
            with torch.cuda.stream(stream):
                P.api._check(P.api.L.lib().epfem_assemble_elastic(eng.ctx.handle, cache.handle,
                                                                 P.api._ptr(Kout)))
        launches_per_step = 1
    else:
        with torch.cuda.stream(stream):
            eng.capture(E, Ep0, Hard0)

        def launch():
            eng.replay()
        launches_per_step = 2  # fused update + row stream (one CUDA graph)

    for _ in range(args.warmup):
        launch()
    torch.cuda.synchronize(dev)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            launch()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    t_ms = ev0.elapsed_time(ev1)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        t = torch.tensor([t_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_ms = float(t)
    ms_per_step = t_ms / args.steps

    info = cache.info
    flags = eng.flags if not elastic else None
    n_plastic = int((flags & 1).sum().item()) if not elastic else 0
    n_smooth = int(((flags >> 1) & 1).sum().item()) if cfg.model == "dp" else None
    n_apex = int(((flags >> 2) & 1).sum().item()) if cfg.model == "dp" else None
    cons_b, asm_b = algorithmic_bytes(cfg, n_int, n_plastic, nnz, info.n_nodes, info.n_elements, info.n_p)
    step_bytes = cons_b + asm_b if not elastic else asm_b
    # per-kernel device time, each half of the step launched alone on the
    # stream (the same kernels the graph replays), CUDA events around it
    k_ms, k_gbs = {}, {}
    KF, KR = "k_newton_fused (constitutive + element delta)", "k_row_stream (K = K_elast + sum dK_e)"
    if not elastic:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        lib = P.api.L.lib()
        C_ = P.api.C
        tot_c = tot_t = 0.0
        reps = max(args.steps, 5)
        for _ in range(reps):
            evs[0].record(stream)
            P.api._check(lib.epfem_constitutive_delta(eng.ctx.handle, cache.handle, C_.byref(eng._mv),
                                                      P.api._ptr(E), P.api._ptr(Ep0),
                                                      P.api._ptr(Hard0), C_.byref(eng._out)))
            evs[1].record(stream)
            P.api._check(lib.epfem_assemble_rows(eng.ctx.handle, cache.handle, P.api._ptr(eng.K)))
            evs[2].record(stream)
            torch.cuda.synchronize(dev)
            tot_c += evs[0].elapsed_time(evs[1])
            tot_t += evs[1].elapsed_time(evs[2])
        k_ms = {KF: tot_c / reps, KR: tot_t / reps}
        k_gbs = {KF: cons_b / (tot_c / reps * 1e-3) / 1e9, KR: asm_b / (tot_t / reps * 1e-3) / 1e9}
        if tot_t >= tot_c:
            dom_bytes, dom_ms, dom = asm_b, tot_t / reps, KR
        else:
            dom_bytes, dom_ms, dom = cons_b, tot_c / reps, KF
    else:
        dom_bytes, dom_ms, dom = asm_b, ms_per_step, "k_elastic_p1 (K5, P1 meshes)"
    achieved = dom_bytes / (dom_ms * 1e-3) / 1e9
    step_gbs = step_bytes / (ms_per_step * 1e-3) / 1e9
    fp64 = None
    fma_pt = FMA_PER_PLASTIC_POINT.get((cfg.family, cfg.dim))
    if not elastic and fma_pt and k_ms:
        fp_peak, fp_src = load_fp64_peak()
        flops = 2.0 * fma_pt * n_plastic
        tf = flops / (k_ms[KF] * 1e-3) / 1e12
        fp64 = {"bound": "fp64", "kernel": KF, "achieved": tf, "peak": fp_peak, "unit": "TFLOP/s",
                "frac": tf / fp_peak, "algorithmic_flops": flops,
                "how": f"2 x {fma_pt} FMA (optimal element-delta contraction, SURVEY 8(d)) per plastic point / "
                       f"the fused kernel's CUDA-event time", "peak_source": fp_src}
    working_set = step_bytes + (8 * nnz if not elastic else 0)
    l2 = (f"inputs larger than L2 (working set {working_set / 1e9:.2f} GB > 126 MB)" if working_set > 126e6 else
          f"L2-RESIDENT: the working set ({working_set / 1e6:.0f} MB) fits the 126 MB L2, so this is an L2 "
          f"number, not an HBM one (no flush between steps)")
    line = {
        "value": world * n_int / (ms_per_step * 1e-3), "ms_per_step": ms_per_step,
        "config": {"workload": name, "element": f"{cfg.family} {cfg.dim}D", "mesh": f"{cfg.n}^{cfg.dim}",
                   "model": cfg.model, "n_int": n_int, "nnz": nnz, "n_dofs": info.n_dofs,
                   "plastic_fraction": n_plastic / n_int if n_int else 0.0,
                   **({"smooth_points": n_smooth, "apex_points": n_apex} if cfg.model == "dp" else {}),
                   "strain_scale": wl.scale, "l2": l2,
                   "parallelism": f"replica x{world}" if world > 1 else "single GPU"},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm_peak,
                     "unit": "GB/s", "frac": achieved / hbm_peak,
                     "traffic": measured_traffic(name, dom),
                     "traffic_source": "profiles/traffic.json (ncu --set full, bytes per launch)",
                     "algorithmic_bytes": dom_bytes, "kernel_ms": dom_ms, "peak_source": peak_src},
        "roofline_step": {"algorithmic_bytes": step_bytes, "achieved": step_gbs, "frac": step_gbs / hbm_peak},
        "roofline_fp64": fp64,
        "kernels_ms": k_ms,
        "kernels_algorithmic_gbs": k_gbs,
        "clocks": clk.summary(),
    }
    ctx = dict(cfg=cfg, wl=wl, cache=cache, mat=mat, eng=eng, E=E, Ep0=Ep0, Hard0=Hard0, stream=stream,
               elastic=elastic, Kout=Kout if elastic else None, ev=(ev0, ev1))
    return line, ctx


def side_sections(args, dev, c):
    """SURVEY §8(f) ranks 1-2 beside the step: the step from nodal
    displacements (strains fused) and the step with its internal forces."""
    import gc

    import torch

    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import displacement
    cfg, wl, cache, mat, stream = c["cfg"], c["wl"], c["cache"], c["mat"], c["stream"]
    E, Ep0, Hard0 = c["E"], c["Ep0"], c["Hard0"]
    ev0, ev1 = c["ev"]
    u = (wl.scale * torch.from_numpy(displacement(wl.mesh.coord, cfg.seed)).to(dev)).contiguous()
    Etmp = torch.empty_like(E)
    eng_u = P.TangentEngine(cache, mat, stream=stream)
    with torch.cuda.stream(stream):
        eng_u.capture_u(u, Ep0, Hard0)
    g2 = torch.cuda.CUDAGraph()
    s2 = torch.cuda.Stream(dev)
    s2.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(s2):
        eng2 = P.TangentEngine(cache, mat, stream=s2)
        lib_ = P.api.L.lib()
        P.api._check(lib_.epfem_strains(eng2.ctx.handle, cache.handle, P.api._ptr(u), P.api._ptr(Etmp)))
        eng2.step(Etmp, Ep0, Hard0)
        with torch.cuda.graph(g2, stream=s2):
            eng2.ctx.set_stream(torch.cuda.current_stream(dev))
            P.api._check(lib_.epfem_strains(eng2.ctx.handle, cache.handle, P.api._ptr(u), P.api._ptr(Etmp)))
            eng2.step(Etmp, Ep0, Hard0)
    torch.cuda.current_stream(dev).wait_stream(s2)

    def t_graph(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        return ev0.elapsed_time(ev1) / args.steps

    def run2():
        with torch.cuda.stream(stream):
            g2.replay()
    t_u = t_graph(eng_u.replay)
    t_2 = t_graph(run2)
    n_int = cache.n_int
    from_u = {"newton_step_u_ms": t_u, "strains_plus_newton_step_ms": t_2, "value_from_u": n_int / (t_u * 1e-3),
              "how": "epfem_newton_step_u (E = B u inside the fused kernel, never stored) vs "
                     "epfem_strains + epfem_newton_step, each one CUDA graph"}
    del g2, eng2, eng_u, Etmp, u
    gc.collect()
    torch.cuda.empty_cache()

    def graph_of(fn):
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(torch.cuda.current_stream(dev))
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(gs):
            fn(gs)
            with torch.cuda.graph(gr, stream=gs):
                fn(torch.cuda.current_stream(dev))
        torch.cuda.current_stream(dev).wait_stream(gs)
        return gr
    Fbuf = torch.empty((cache.info.n_dofs,), dtype=torch.float64, device=dev)
    eng_f = P.TangentEngine(cache, mat, stream=stream)

    def step_f(st):
        eng_f.ctx.set_stream(st)
        eng_f.step_f(E, Ep0, Hard0, Fbuf)
    gf = graph_of(step_f)

    def t_replay(gr):
        for _ in range(3):
            with torch.cuda.stream(stream):
                gr.replay()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                gr.replay()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        return ev0.elapsed_time(ev1) / args.steps
    t_f = t_replay(gf)
    with_f = {"newton_step_f_ms": t_f, "value_with_forces": n_int / (t_f * 1e-3),
              "how": "epfem_newton_step_f (the step, then K9 in two passes: element force records, "
                     "per-node fold), one CUDA graph"}
    del gf, eng_f, Fbuf
    gc.collect()
    torch.cuda.empty_cache()
    return from_u, with_f


def e2e_section(args, dev, local, world, c):
    """The reference-facing call with HOST buffers: E, Ep, Hard in (pinned,
    H2D every step), S, flag bytes and K values out (D2H every step); the
    packed D stays on the device (its consumer, the tangent assembly, runs
    inside the same call)."""
    import torch

    import paper_1805_04155_b200 as P
    cache, mat, stream, eng = c["cache"], c["mat"], c["stream"], c["eng"]
    E, Ep0, Hard0, elastic = c["E"], c["Ep0"], c["Hard0"], c["elastic"]
    n_int, nnz = cache.n_int, cache.nnz
    host_in = [E] + [x for x in (Ep0, Hard0) if x is not None]
    h_in = [torch.empty_like(x, device="cpu").pin_memory() for x in host_in]
    for h, x in zip(h_in, host_in):
        h.copy_(x)
    # Steps are pipelined over two buffer sets and three streams: the upload
    # of step i+1 (h2d stream) and the download of step i (d2h stream)
    # overlap on the full-duplex PCIe link while the compute stream runs the
    # hot path; every step still moves all its own bytes.
    nbuf = 1 if elastic else 2
    d_in = [[torch.empty_like(x) for x in host_in] for _ in range(nbuf)]
    if elastic:
        outs = [[torch.empty((nnz,), dtype=torch.float64).pin_memory()]]
        engines = [None]
        Kout = c["Kout"]
    else:
        outs = [[torch.empty((n_int, 6), dtype=torch.float64).pin_memory(),
                 torch.empty((n_int,), dtype=torch.uint8).pin_memory(),
                 torch.empty((nnz,), dtype=torch.float64).pin_memory()] for _ in range(nbuf)]
        engines = [eng] + [P.TangentEngine(cache, mat, stream=stream) for _ in range(nbuf - 1)]
    ctx = P.Context(local, stream=stream, synchronous=False)
    h2d_s, d2h_s = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_in = [torch.cuda.Event() for _ in range(nbuf)]
    ev_comp = [torch.cuda.Event() for _ in range(nbuf)]
    ev_out = [torch.cuda.Event() for _ in range(nbuf)]
    used = [False] * nbuf

    def e2e_step(i):
        b = i % nbuf
        if elastic:
            with torch.cuda.stream(stream):
                P.api._check(P.api.L.lib().epfem_assemble_elastic(ctx.handle, cache.handle, P.api._ptr(Kout)))
                outs[0][0].copy_(Kout, non_blocking=True)
            return
        if used[b]:
            h2d_s.wait_event(ev_comp[b])     # inputs of buffer b consumed
            stream.wait_event(ev_out[b])     # outputs of buffer b downloaded
        with torch.cuda.stream(h2d_s):
            for d, h in zip(d_in[b], h_in):
                d.copy_(h, non_blocking=True)
            ev_in[b].record(h2d_s)
        stream.wait_event(ev_in[b])
        ep = d_in[b][1] if Ep0 is not None else None
        hd = d_in[b][2] if Hard0 is not None else None
        S, flags, D, K = engines[b].step(d_in[b][0], ep, hd)
        ev_comp[b].record(stream)
        d2h_s.wait_event(ev_comp[b])
        with torch.cuda.stream(d2h_s):
            outs[b][0].copy_(S, non_blocking=True)
            outs[b][1].copy_(flags, non_blocking=True)
            outs[b][2].copy_(K, non_blocking=True)
            ev_out[b].record(d2h_s)
        used[b] = True

    for i in range(2):
        e2e_step(i)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_steps = max(4, min(args.steps, 12))
    e0.record(stream)
    h2d_s.wait_event(e0)
    d2h_s.wait_event(e0)
    for i in range(e2e_steps):
        e2e_step(i)
    stream.wait_stream(d2h_s)
    stream.wait_stream(h2d_s)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    e_ms = e0.elapsed_time(e1) / e2e_steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t)
    h2d = 0 if elastic else sum(x.numel() * 8 for x in h_in)
    d2h = sum(o.numel() * o.element_size() for o in outs[0])
    return {"value": world * n_int / (e_ms * 1e-3), "unit": "ip/s", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": e_ms,
            "how": "epfem_newton_step with host E/Ep/Hard in and S/flags/K out every step; "
                   "H2D, compute, D2H on three streams, double-buffered across steps"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="cfg4")
    ap.add_argument("--extra", default=None,
                    help="comma-separated extra configurations timed in the same run (lean lines; "
                         "default cfg5,cfg3 for the cfg4 headline at N=1, 'none' to skip)")
    ap.add_argument("--target", type=float, default=None, help="plastic fraction override")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--ref-reps", type=int, default=None,
                    help="--impl reference: timed iterations per slab (default: --steps, within a time budget)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-side", action="store_true", help="skip the from-displacements / with-forces timings")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    # stdout carries exactly one JSON line: Python's prints keep the original stdout, while anything native
    # libraries printf to fd 1 (NCCL's version banner at NCCL_DEBUG=VERSION / WARN) goes to stderr
    sys.stdout.flush()
    sys.stdout = os.fdopen(os.dup(1), "w", buffering=1)
    os.dup2(2, 1)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return run_reference(args, rank, world)

    import gc

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # EPFEM_BENCH_SLABS=1: run the slab (multi-GPU) data path even at world
    # size 1 (one-GPU check of the N>1 code under torchrun)
    slabs = world > 1 or os.environ.get("EPFEM_BENCH_SLABS") == "1"
    if slabs:
        dist.init_process_group("nccl", device_id=dev)

    from paper_1805_04155_b200 import build as B
    B.build()
    from paper_1805_04155_b200.synthetic import CONFIGS
    cfg = CONFIGS[args.config]
    if slabs and cfg.model != "elastic":
        return run_slabs(args, rank, world, dev, cfg)
    if args.extra is None:
        extra = ["cfg5", "cfg3"] if (args.config == "cfg4" and world == 1) else []
    else:
        extra = [x for x in args.extra.split(",") if x and x != "none"]

    line, c = measure_step(args.config, args, dev, local, world, target=args.target)
    from_u = with_f = None
    if not c["elastic"] and not args.no_side:
        from_u, with_f = side_sections(args, dev, c)
    e2e = None if args.no_e2e else e2e_section(args, dev, local, world, c)
    scale = c["wl"].scale
    del c
    gc.collect()
    torch.cuda.empty_cache()
    extras = {}
    for name in extra:
        xl, xc = measure_step(name, args, dev, local, world)
        del xc
        gc.collect()
        torch.cuda.empty_cache()
        extras[name] = {k: xl[k] for k in ("value", "ms_per_step", "config", "roofline", "roofline_step",
                                           "roofline_fp64", "kernels_ms", "kernels_algorithmic_gbs", "clocks",
                                           "gpu_launches")}
        line["gpu_launches"] += xl["gpu_launches"]

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(args.config, scale)

    if rank == 0:
        out = {"metric": METRIC, "value": line["value"], "unit": "ip/s", "n_gpus": world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": line["ms_per_step"],
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
               "dtype": "f64", "data": "synthetic (seeded smooth displacement fields, SURVEY §8(d))"}
        out.update({k: v for k, v in line.items() if k not in ("value", "ms_per_step")})
        out["e2e"] = e2e
        out["cpu_baseline"] = cpu
        out["step_from_displacements"] = from_u
        out["step_with_internal_forces"] = with_f
        if extras:
            out["extra_configs"] = extras
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
