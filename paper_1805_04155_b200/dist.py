"""Multi-GPU slab partition of one mesh.

The mesh is cut along its LAST axis (z in 3D, y in 2D) into `world` slabs of
whole cell layers.  Node numbering is last-axis-major (mesh.cpp:164-168), so
every slab's nodes — and therefore its K rows and K values — are one
contiguous range of the global arrays.

Ownership: rank r owns the node planes of its slab EXCEPT the top one, which
belongs to rank r+1 (the last rank also owns the top plane of the mesh).
Rank r's rows couple to the elements of the layer just below its slab, so
each rank builds its assembly cache on an *extended* slab = its own cell
layers + one halo layer below (r > 0).  With the extended mesh every owned
row has its full global column set, locally.

Per Newton iteration:
  1. constitutive update + element deltas on the rank's own elements (K1 +
     pass 1, fused);
  2. interface exchange: rank r sends the flag bytes + packed tangents of
     its TOP cell layer to rank r+1, which receives them as the plastic data
     of its halo layer (one grouped send/recv between neighbours: NCCL over
     NVLink on GPUs, gloo in the CPU tests);
  3. element deltas of the halo layer from the received data, then the row
     stream over the extended slab; the owned rows are complete and written
     exactly once.
Step 1 is the fused kernel of the single-GPU step restricted to the rank's
own elements (epfem_newton_range), so a 1-rank run is bitwise the fused step.
The exchange carries the producer-side data of the interface layer rather
than partial K rows, so every rank assembles its rows with the single-GPU
kernels and no remap/add kernel is needed; its volume, n_layer_points x
(192 + 1) B, is of the same order as the partial-row exchange.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .mesh import StructuredMesh, quad_count, structured_mesh


def split_layers(n_layers: int, world: int) -> list[tuple[int, int]]:
    """Balanced contiguous split of n_layers cell layers over `world` ranks."""
    if world < 1 or world > n_layers:
        raise ValueError(f"cannot split {n_layers} cell layers over {world} ranks")
    base, extra = divmod(n_layers, world)
    out, k = [], 0
    for r in range(world):
        step = base + (1 if r < extra else 0)
        out.append((k, k + step))
        k += step
    return out


@dataclass
class SlabPlan:
    """Rank r's piece of a structured mesh and the maps back to the global one."""

    rank: int
    world: int
    own_layers: tuple[int, int]      # cell layers [k0, k1) owned by this rank
    ext_layers: tuple[int, int]      # [k0 - halo, k1): own layers + halo layer below
    mesh: StructuredMesh             # extended slab, numbered as its own mesh
    node_offset: int                 # global id of the extended slab's node 0
    own_nodes: tuple[int, int]       # local node range owned (rows written by this rank)
    halo_elems: int                  # leading elements of the extended mesh that belong to r-1
    layer_elems: int                 # elements per cell layer
    n_q: int

    @property
    def dim(self) -> int:
        return self.mesh.dim

    @property
    def own_points(self) -> tuple[int, int]:
        """Local integration-point range evaluated by this rank."""
        return self.halo_elems * self.n_q, self.mesh.n_elements * self.n_q

    @property
    def halo_points(self) -> tuple[int, int]:
        return 0, self.halo_elems * self.n_q

    @property
    def send_points(self) -> tuple[int, int]:
        """Local points of the top cell layer (sent to rank + 1)."""
        n = self.mesh.n_elements * self.n_q
        return n - self.layer_elems * self.n_q, n

    @property
    def own_rows(self) -> tuple[int, int]:
        return self.dim * self.own_nodes[0], self.dim * self.own_nodes[1]

    @property
    def global_rows(self) -> tuple[int, int]:
        d = self.dim
        return d * (self.node_offset + self.own_nodes[0]), d * (self.node_offset + self.own_nodes[1])


def _plane_index(mesh: StructuredMesh) -> np.ndarray:
    """Fine-grid index along the slab axis of every node."""
    return mesh.fine[:, 2] if mesh.dim == 3 else mesh.fine[:, 1]


def make_plan(family: str, dim: int, n: int, world: int, rank: int) -> SlabPlan:
    """Plan for an n^dim unit-cube/square structured mesh."""
    splits = split_layers(n, world)
    k0, k1 = splits[rank]
    halo = 1 if rank > 0 else 0
    e0 = k0 - halo
    ext = structured_mesh(family, dim, n, n, n if dim == 3 else 0, slab=(e0, k1))
    plane = _plane_index(ext)
    lo = int(np.searchsorted(plane, 2 * k0, side="left"))
    hi = int(np.searchsorted(plane, 2 * k1, side="left"))
    if rank == world - 1:
        hi = ext.n_nodes
    # global node id of the extended slab's first node: nodes of the full mesh
    # strictly below fine plane 2*e0
    if e0 == 0:
        node_offset = 0
    else:
        below = structured_mesh(family, dim, n, n, n if dim == 3 else 0, slab=(0, e0))
        node_offset = int(np.searchsorted(_plane_index(below), 2 * e0, side="left"))
    per_layer = ext.n_elements // (k1 - e0)
    nq = quad_count(ext.elem_type)
    return SlabPlan(rank, world, (k0, k1), (e0, k1), ext, node_offset, (lo, hi),
                    halo * per_layer, per_layer, nq)


def finish_exchange(pending):
    """Complete exchange_interface(..., wait=False): wait (a stream wait for
    NCCL) and copy any staged receive buffers into place."""
    reqs, recv = pending
    for req in reqs:
        req.wait()
    for dst, buf in recv:
        if dst.data_ptr() != buf.data_ptr():
            dst.copy_(buf)


def exchange_interface(plan: SlabPlan, flags, D, group=None, wait=True):
    """Send the top layer's (flags, D) to rank + 1 and receive the halo
    layer's from rank - 1, in place (torch tensors on the process group's
    device: CUDA with NCCL, CPU with gloo).  wait=False returns the pending
    exchange for finish_exchange()."""
    import torch.distributed as dist
    ops = []
    s0, s1 = plan.send_points
    h0, h1 = plan.halo_points
    if plan.rank + 1 < plan.world:
        ops.append(dist.P2POp(dist.isend, flags[s0:s1].contiguous(), plan.rank + 1, group))
        ops.append(dist.P2POp(dist.isend, D[s0:s1].contiguous(), plan.rank + 1, group))
    recv = []
    if plan.rank > 0:
        fb = flags[h0:h1]
        db = D[h0:h1]
        rf = fb if fb.is_contiguous() else fb.contiguous()
        rd = db if db.is_contiguous() else db.contiguous()
        ops.append(dist.P2POp(dist.irecv, rf, plan.rank - 1, group))
        ops.append(dist.P2POp(dist.irecv, rd, plan.rank - 1, group))
        recv = [(fb, rf), (db, rd)]
    reqs = dist.batch_isend_irecv(ops) if ops else []
    if not wait:
        return reqs, recv
    finish_exchange((reqs, recv))


class DistributedTangent:
    """GPU data path of one rank: K1 on own points, interface exchange over
    the process group (NCCL), tangent assembly on the extended slab."""

    def __init__(self, plan: SlabPlan, mat_factory, device, group=None, exchange: str = "torch"):
        """exchange: "torch" = torch.distributed P2P (NCCL on its own stream,
        overlapping the interior update; gloo on the CPU); "capi" = the
        C-ABI's own NCCL communicator (epfem_ctx_attach_nccl /
        epfem_exchange_interface, the path a C++ caller uses), ordered on
        the context's stream."""
        import torch

        from . import api
        self.plan = plan
        self.group = group
        self.exchange = exchange
        self.device = device
        n_ext = plan.mesh.n_int
        self.mat_ext = mat_factory(n_ext)
        self.cache = api.build_assembly_cache(api.Mesh.from_structured(plan.mesh, device), self.mat_ext)
        p0, p1 = plan.own_points
        # own points' material = the extended field's [p0, p1) slice (per-point
        # arrays sliced, not rebuilt)
        self.mat_own = self.mat_ext.slice(p0, p1)
        self.ctx = api.Context(device.index or 0, synchronous=False)
        self.S = torch.empty((n_ext, 6), dtype=torch.float64, device=device)
        self.flags = torch.zeros((n_ext,), dtype=torch.uint8, device=device)
        self.D = torch.zeros((n_ext, 24), dtype=torch.float64, device=device)
        self.K = torch.empty((self.cache.nnz,), dtype=torch.float64, device=device)
        r0, r1 = plan.own_rows
        rp = self.cache.row_ptr
        self.own_values = (int(rp[r0]), int(rp[r1]))
        if exchange == "capi":
            self._attach_nccl()

    def _attach_nccl(self):
        """One NCCL communicator for the C-ABI exchange: rank 0's unique id
        broadcast over the process group, then epfem_ctx_attach_nccl."""
        import ctypes as C

        import torch.distributed as dist

        from . import api
        uid = C.create_string_buffer(128)
        if self.plan.rank == 0:
            api._check(api.L.lib().epfem_nccl_unique_id(uid))
        obj = [bytes(uid.raw)]
        if self.plan.world > 1:
            dist.broadcast_object_list(obj, src=0, group=self.group)
        uid = C.create_string_buffer(obj[0], 128)
        api._check(api.L.lib().epfem_ctx_attach_nccl(self.ctx.handle, uid, self.plan.world, self.plan.rank))

    def _exchange_capi(self):
        from . import api
        s0, s1 = self.plan.send_points
        h0, h1 = self.plan.halo_points
        if self.plan.rank + 1 >= self.plan.world:
            s0 = s1 = 0
        if self.plan.rank == 0:
            h0 = h1 = 0
        self.ctx.use_current_stream()
        api._check(api.L.lib().epfem_exchange_interface(self.ctx.handle, api._ptr(self.flags), api._ptr(self.D),
                                                        s0, s1, h0, h1))

    def step(self, E_own, Ep_own=None, Hard_own=None):
        """One Newton iteration of this rank: fused constitutive update +
        element deltas on its own elements (epfem_newton_range), interface
        exchange, deltas of the halo elements from the received flags + D
        (epfem_delta_range), then the row stream over the extended slab.
        The top cell layer (the data rank + 1 needs) is updated first, so the
        NCCL exchange — which torch runs on its own stream after the work
        already queued — overlaps the update of the interior layers.
        Returns this rank's S, flag bytes and owned K values."""
        n_e = self.plan.mesh.n_elements
        top = max(self.plan.halo_elems, n_e - self.plan.layer_elems)
        if self.exchange == "capi":
            if self.plan.rank + 1 < self.plan.world and top > self.plan.halo_elems:
                self.update_own(E_own, Ep_own, Hard_own, (top, n_e))
                self._exchange_capi()
                self.update_own(E_own, Ep_own, Hard_own, (self.plan.halo_elems, top))
            else:
                self.update_own(E_own, Ep_own, Hard_own)
                self._exchange_capi()
            return self.assemble()
        if self.plan.rank + 1 < self.plan.world and top > self.plan.halo_elems:
            self.update_own(E_own, Ep_own, Hard_own, (top, n_e))
            reqs = exchange_interface(self.plan, self.flags, self.D, self.group, wait=False)
            self.update_own(E_own, Ep_own, Hard_own, (self.plan.halo_elems, top))
            finish_exchange(reqs)
        else:
            self.update_own(E_own, Ep_own, Hard_own)
            exchange_interface(self.plan, self.flags, self.D, self.group)
        return self.assemble()

    def update_own(self, E_own, Ep_own=None, Hard_own=None, elems=None):
        """epfem_newton_range on own elements [e0, e1) (default: all own)."""
        import ctypes as C

        from . import api
        h_e, n_e = self.plan.halo_elems, self.plan.mesh.n_elements
        e0, e1 = elems if elems is not None else (h_e, n_e)
        nq = self.plan.n_q
        p0, q0, q1 = self.plan.own_points[0], e0 * nq, e1 * nq  # extended-mesh points
        o0, o1 = q0 - p0, q1 - p0                                # offsets in the own arrays
        out = api.L.ConstitutiveOut()
        out.S, out.flags, out.D = (api._ptr(self.S[q0:q1]), api._ptr(self.flags[q0:q1]),
                                   api._ptr(self.D[q0:q1]))
        mat = self.mat_own if (o0, o1) == (0, self.mat_own.n_int) else self._mat_part(o0, o1)
        mv = mat.view()
        sl = (lambda x: None if x is None else x[o0:o1])
        self.ctx.use_current_stream()
        api._check(api.L.lib().epfem_newton_range(
            self.ctx.handle, self.cache.handle, C.byref(mv), api._ptr(sl(E_own)), api._ptr(sl(Ep_own)),
            api._ptr(sl(Hard_own)), C.byref(out), e0, e1))

    def _mat_part(self, o0, o1):
        """The own material of own points [o0, o1) (per-point arrays sliced)."""
        cache = self.__dict__.setdefault("_mat_parts", {})
        if (o0, o1) not in cache:
            cache[(o0, o1)] = self.mat_own.slice(o0, o1)
        return cache[(o0, o1)]

    def assemble(self):
        from . import api
        lib = api.L.lib()
        self.ctx.use_current_stream()
        h_e = self.plan.halo_elems
        if h_e:
            api._check(lib.epfem_delta_range(self.ctx.handle, self.cache.handle, self.cache.n_int,
                                             api._ptr(self.D), api._ptr(self.flags), 0, h_e))
        api._check(lib.epfem_assemble_rows(self.ctx.handle, self.cache.handle, api._ptr(self.K)))
        p0, p1 = self.plan.own_points
        v0, v1 = self.own_values
        return self.S[p0:p1], self.flags[p0:p1], self.K[v0:v1]
