"""Multi-rank slab partition on CPU with gloo, world_size 2.

The per-rank compute is the CPU oracle (test-only stand-in for the kernels);
what is tested is the product's host logic in paper_1805_04155_b200/dist.py:
the balanced split, the extended slab with its halo layer, the ownership
ranges, the contiguous global row/value ranges and the interface exchange of
(flags, packed D).  The concatenation of every rank's owned rows must equal
the single-domain K: pattern bit-exact, values to 1e-12 row-scaled.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from helpers import row_scaled_error

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASES = [("Q2", 2, 8, "vm"), ("Q1", 3, 4, "vm"), ("P2", 3, 3, "dp"), ("P1", 2, 7, "vm")]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _material(O, model):
    if model == "vm":
        K, G = O.elastic_moduli(206900.0, 0.29)
        return K, G, 1.0e4, 450.0
    K, G = O.elastic_moduli(1.0e7, 0.48)
    eta, c = O.dp_parameters(450.0, math.pi / 9.0)
    return K, G, eta, c


def _evaluate(O, model, E, G, K, p1, p2):
    if model == "vm":
        return O.constitutive_vm(E, None, None, G, K, p1, p2)
    return O.constitutive_dp(E, None, G, K, p1, p2)


def _pack(DS):
    from paper_1805_04155_b200._lib import D_COL, D_ROW
    D = np.zeros((DS.shape[0], 24))
    blocks = DS.reshape(-1, 6, 6).transpose(0, 2, 1)
    D[:, :21] = blocks[:, D_ROW, D_COL]
    return D


def _unpack(D):
    from paper_1805_04155_b200._lib import D_COL, D_ROW
    full = np.zeros((D.shape[0], 6, 6))
    for k, (i, j) in enumerate(zip(D_ROW, D_COL)):
        full[:, i, j] = D[:, k]
        full[:, j, i] = D[:, k]
    return full.transpose(0, 2, 1).reshape(-1, 36)


def _strain_scale(O, model, E1, G, K, p1, p2, target=0.4):
    if model == "vm":
        crit = O.constitutive_vm(E1, None, None, G, K, p1, 0.0)["crit"]
        return p2 / np.quantile(crit, 1.0 - target)
    s = 1.0
    for _ in range(80):
        f = O.constitutive_dp(s * E1, None, G, K, p1, p2)["plastic"].mean()
        if abs(f - target) < 0.08:
            break
        s *= 1.2 if f < target else 0.85
    return s


def _worker(rank, world, port, case, q):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle as O
        from paper_1805_04155_b200.dist import exchange_interface, make_plan
        from paper_1805_04155_b200.synthetic import displacement
        family, dim, n, model = case
        K, G, p1, p2 = _material(O, model)
        plan = make_plan(family, dim, n, world, rank)
        m = plan.mesh
        oc = O.Cache(family, dim, m.coord, m.elem, G, K)
        # strains of the extended slab from the global displacement field
        u = displacement(m.coord, 7)
        E1 = oc.strains(u)
        # one global strain scale, agreed by all ranks (rank 0 decides on its slab)
        s = torch.tensor([_strain_scale(O, model, E1, G, K, p1, p2)], dtype=torch.float64)
        dist.broadcast(s, 0)
        E = float(s) * E1
        n_ext = m.n_int
        flags = torch.zeros(n_ext, dtype=torch.uint8)
        D = torch.zeros((n_ext, 24), dtype=torch.float64)
        p0, pe = plan.own_points
        res = _evaluate(O, model, E[p0:pe], G, K, p1, p2)
        flags[p0:pe] = torch.from_numpy(res["plastic"].astype(np.uint8))
        D[p0:pe] = torch.from_numpy(_pack(res["DS"]))
        exchange_interface(plan, flags, D)
        # the received halo layer equals what this rank would compute itself
        h0, h1 = plan.halo_points
        if h1 > h0:
            mine = _evaluate(O, model, E[h0:h1], G, K, p1, p2)
            assert np.array_equal(flags[h0:h1].numpy(), mine["plastic"].astype(np.uint8))
            assert np.array_equal(D[h0:h1].numpy()[mine["plastic"].astype(bool)],
                                  _pack(mine["DS"])[mine["plastic"].astype(bool)])
        Kt = oc.tangent(_unpack(D.numpy()), flags.numpy())
        r0, r1 = plan.own_rows
        v0, v1 = Kt.indptr[r0], Kt.indptr[r1]
        rows = dict(rank=rank, global_rows=plan.global_rows,
                    indptr=Kt.indptr[r0:r1 + 1] - v0,
                    cols=Kt.indices[v0:v1].astype(np.int64) + dim * plan.node_offset,
                    vals=Kt.data[v0:v1], base=oc.K_elast().data[v0:v1],
                    plastic=int(flags[p0:pe].sum()), scale=float(s))
        q.put(rows)
    except Exception as exc:  # pragma: no cover - reported to the parent
        import traceback
        q.put(dict(rank=rank, error=traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def test_split_layers():
    from paper_1805_04155_b200.dist import split_layers
    assert split_layers(100, 8) == [(0, 13), (13, 26), (26, 39), (39, 52), (52, 64), (64, 76),
                                    (76, 88), (88, 100)]
    assert split_layers(160, 8)[3] == (60, 80)
    with pytest.raises(ValueError):
        split_layers(3, 4)


@pytest.mark.parametrize("world", [2, 3])
def test_plans_tile_the_global_rows(world):
    from paper_1805_04155_b200.dist import make_plan
    from paper_1805_04155_b200.mesh import structured_mesh
    for family, dim, n in [("Q2", 2, 9), ("Q1", 3, 5), ("P2", 3, 4)]:
        full = structured_mesh(family, dim, n, n, n if dim == 3 else 0)
        nxt = 0
        for r in range(world):
            p = make_plan(family, dim, n, world, r)
            g0, g1 = p.global_rows
            assert g0 == nxt and g1 > g0
            nxt = g1
            # the extended slab is a contiguous, identically ordered node range
            lo = p.node_offset
            assert np.array_equal(full.coord[lo:lo + p.mesh.n_nodes], p.mesh.coord)
            e_lo = p.ext_layers[0] * p.layer_elems
            assert np.array_equal(full.elem[e_lo:e_lo + p.mesh.n_elements] - lo, p.mesh.elem)
        assert nxt == dim * full.n_nodes


@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}{c[1]}d-{c[3]}" for c in CASES])
def test_two_rank_gloo_assembly_matches_single_domain(case, oracle):
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    errs = [p["error"] for p in parts if "error" in p]
    assert not errs, errs[0]
    parts.sort(key=lambda d: d["rank"])
    # single-domain reference with the same strain scale
    import sys
    sys.path.insert(0, ROOT)
    from paper_1805_04155_b200.mesh import structured_mesh
    from paper_1805_04155_b200.synthetic import displacement
    family, dim, n, model = case
    O = oracle
    K, G, p1, p2 = _material(O, model)
    full = structured_mesh(family, dim, n, n, n if dim == 3 else 0)
    oc = O.Cache(family, dim, full.coord, full.elem, G, K)
    E = parts[0]["scale"] * oc.strains(displacement(full.coord, 7))
    res = _evaluate(O, model, E, G, K, p1, p2)
    assert sum(p["plastic"] for p in parts) == int(res["plastic"].sum()) > 0
    Kref = oc.tangent(res["DS"], res["plastic"])
    indptr = [np.zeros(1, np.int64)]
    cols, vals, base = [], [], []
    off = 0
    for p in parts:
        indptr.append(p["indptr"][1:] + off)
        off += p["indptr"][-1]
        cols.append(p["cols"])
        vals.append(p["vals"])
        base.append(p["base"])
    indptr = np.concatenate(indptr)
    assert np.array_equal(indptr, Kref.indptr)
    assert np.array_equal(np.concatenate(cols), Kref.indices.astype(np.int64))
    got = np.concatenate(vals)
    assert row_scaled_error(got, Kref.data, Kref.indptr, oc.K_elast().data) <= 1e-12
