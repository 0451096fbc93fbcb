"""Multi-GPU data path under real NCCL.

* world 1 with the C-ABI exchange (epfem_ctx_attach_nccl: NCCL loaded at run
  time, a one-rank communicator, the exchange a no-op): the slab path equals
  the single-GPU step bit for bit.  Runs on any GPU box.
* world 2 and 4 (needs that many GPUs; skipped otherwise): one process per
  GPU over NCCL, both exchanges (torch.distributed P2P and the C-ABI's own
  communicator); the owned K rows of all ranks, concatenated, are bitwise the
  single-GPU K and the flags / S per point match.
The same exchange logic runs on gloo at world 2 in tests/test_dist.py.
"""
import os
import sys
import tempfile

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _single_gpu(name, n, dev):
    import paper_1805_04155_b200 as P
    from paper_1805_04155_b200.synthetic import CONFIGS, calibrate, displacement
    cfg = CONFIGS[name]
    mesh = cfg.mesh(n)
    mat = cfg.material(mesh.n_int)
    gc = P.build_assembly_cache(P.Mesh.from_structured(mesh, dev), mat)
    E1 = gc.strains(torch.from_numpy(displacement(mesh.coord, cfg.seed)).to(dev))
    s, _ = calibrate(E1, mat, 0.35)
    E = (s * E1).contiguous()
    eng = P.TangentEngine(gc, mat)
    S, f, D, K = eng.step(E)
    eng.sync()
    return E, S.cpu().numpy(), f.cpu().numpy(), K.cpu().numpy(), gc


def test_capi_exchange_world1_equals_single_gpu(cuda):
    from paper_1805_04155_b200.dist import DistributedTangent, make_plan
    from paper_1805_04155_b200.synthetic import CONFIGS
    name, n = "cfg4", 6
    E, S, f, K, gc = _single_gpu(name, n, cuda)
    plan = make_plan("Q1", 3, n, 1, 0)
    dt = DistributedTangent(plan, CONFIGS[name].material, cuda, exchange="capi")
    S2, f2, K2 = dt.step(E)
    dt.ctx.sync()
    assert np.array_equal(f2.cpu().numpy(), f) and np.array_equal(S2.cpu().numpy(), S)
    assert np.array_equal(K2.cpu().numpy().view(np.uint64), K.view(np.uint64))


def _rank_main(rank, world, name, n, exchange, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    sys.path.insert(0, ROOT)
    import torch.distributed as dist

    from paper_1805_04155_b200.dist import DistributedTangent, make_plan
    from paper_1805_04155_b200.synthetic import CONFIGS
    dev = torch.device("cuda", rank)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    cfg = CONFIGS[name]
    E = torch.from_numpy(np.load(os.path.join(out_dir, "E.npy"))).to(dev)
    plan = make_plan(cfg.family, cfg.dim, n, world, rank)
    dt = DistributedTangent(plan, cfg.material, dev, exchange=exchange)
    nq = plan.n_q
    k0, k1 = plan.own_layers
    q0, q1 = k0 * plan.layer_elems * nq, k1 * plan.layer_elems * nq
    S, f, K = dt.step(E[q0:q1].contiguous())
    torch.cuda.synchronize(dev)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), S=S.cpu().numpy(), f=f.cpu().numpy(), K=K.cpu().numpy(),
             rows=np.array(plan.global_rows))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("exchange", ["torch", "capi"])
def test_nccl_ranks_equal_single_gpu(cuda, world, exchange):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs (this box has {torch.cuda.device_count()})")
    import torch.multiprocessing as mp
    name, n = "cfg4", 8
    E, S, f, K, gc = _single_gpu(name, n, cuda)
    rp = gc.row_ptr.cpu().numpy()
    with tempfile.TemporaryDirectory() as d:
        np.save(os.path.join(d, "E.npy"), E.cpu().numpy())
        port = 29500 + (os.getpid() % 1000)
        mp.start_processes(_rank_main, args=(world, name, n, exchange, port, d), nprocs=world, join=True,
                           start_method="spawn")
        q = 0
        rows = 0
        for r in range(world):
            z = np.load(os.path.join(d, f"r{r}.npz"))
            nq = z["S"].shape[0]
            assert np.array_equal(z["f"], f[q:q + nq]) and np.array_equal(z["S"], S[q:q + nq])
            g0, g1 = z["rows"]
            assert np.array_equal(z["K"].view(np.uint64), K[rp[g0]:rp[g1]].view(np.uint64))
            q += nq
            rows += g1 - g0
        assert q == f.size and rows == gc.info.n_dofs
