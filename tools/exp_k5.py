"""Timing experiment: K5 (elastic assembly into the pattern) per config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1805_04155_b200 as P  # noqa: E402
from paper_1805_04155_b200.synthetic import CONFIGS  # noqa: E402

dev = torch.device("cuda", 0)
for name in sys.argv[1:]:
    cfg = CONFIGS[name]
    mesh = cfg.mesh(None)
    mat = cfg.material(mesh.n_int)
    cache = P.build_assembly_cache(P.Mesh.from_structured(mesh, dev), mat)
    K = torch.empty((cache.nnz,), dtype=torch.float64, device=dev)
    ctx = P.Context(0, synchronous=False)
    lib = P.api.L.lib()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(3):
        P.api._check(lib.epfem_assemble_elastic(ctx.handle, cache.handle, P.api._ptr(K)))
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(5):
        P.api._check(lib.epfem_assemble_elastic(ctx.handle, cache.handle, P.api._ptr(K)))
    ev[1].record()
    torch.cuda.synchronize()
    print(name, os.environ.get("EPFEM_K5", "rows"), f"{ev[0].elapsed_time(ev[1]) / 5:.4f} ms")
    del cache, K
    torch.cuda.empty_cache()
