// K2 + K6: the per-iteration tangent  K = K_elast + sum_{plastic q} B_q^T w_q (D_q - C_q) B_q
// (assembly.cpp:262-289), as two deterministic passes without atomics.
//
// Pass 1 (element delta, k_elem_delta_staged here; fused into the
// constitutive kernel by epfem_newton_step, see constitutive.cu).  Phase 1:
// one thread per (element, point) of the CTA's elements issues that point's
// loads (J^-1, w, packed D) independently of every other point and stages
//     dphi_p = J^-1 ghat_p (all nodes),  Dw = w (D - C)   (plane-strain rows in 2D)
// in shared memory.  Phase 2: one thread per (element, node a, block chunk)
// loops over the element's plastic points reading only shared memory:
//     T_a = B_a^T Dw,   block(a, b) += T_a B_b        (registers)
// and writes the symmetric element delta dK_e (blocks a <= b) to the
// per-element workspace and the plastic-point bitmask to emask[e].
//
// Pass 2 (k_row_stream): one CTA per range of NPC consecutive nodes = one
// contiguous value range of K (a node's dim rows are contiguous and nodes are
// numbered in row order).  One TMA bulk copy brings K_elast[range] into a
// shared-memory image while the threads stage the range's (element, node)
// items; each warp adds the plastic items' block rows of dK_e for its nodes
// at the cached slots (one warp per node: a single writer per row); one TMA
// bulk store writes the image to K[range].  Rows without plastic
// contributions are therefore bitwise copies of K_elast.
#include "rows.cuh"

namespace epfem_gpu {

namespace {

template <int DIM, int NP, int NQ, int MODE>
__global__ void __launch_bounds__(DeltaCfg<DIM, NP, NQ>::THREADS) k_elem_delta_staged(GatherArgs a) {
  pdl_trigger();
  using Cfg = DeltaCfg<DIM, NP, NQ>;
  constexpr int EPB = Cfg::EPB;
  constexpr int NS = Cfg::NS, REC = Cfg::REC;
  __shared__ double s_st[EPB][NQ][REC];
  __shared__ unsigned s_mask[EPB];

  const int tid = threadIdx.x;
  const int64_t e0 = a.e_begin + (int64_t)blockIdx.x * EPB;
  if (tid < EPB) s_mask[tid] = 0u;
  __syncthreads();
  for (int k = tid; k < EPB * NQ; k += blockDim.x) {
    const int le = k / NQ, q = k - le * NQ;
    const int64_t e = e0 + le;
    if (e >= a.e_end) continue;
    const int64_t m = e * NQ + q;
    if (MODE != G_ELASTIC && !(__ldg(a.flags + m) & 1)) continue;
    atomicOr(&s_mask[le], 1u << q);
    double* st = s_st[le][q];
    stage_geometry<DIM, NP>(st, a.inv + m * Cfg::D2, a.gradhat, q);
    if (MODE == G_ELASTIC) {
      stage_c<DIM>(st + NP * DIM, __ldg(a.weight + m), a, m);
      continue;
    }
    // packed-D loads first (independent), then the staged products
    double dv[NS][NS];
#pragma unroll
    for (int r = 0; r < NS; ++r)
#pragma unroll
      for (int c = r; c < NS; ++c) {
        const int ri = arow<DIM>(r), ci = arow<DIM>(c);
        dv[r][c] = MODE == G_TANGENT_PACKED ? __ldg(a.D + m * EPFEM_D_STRIDE + pk_index(ri, ci))
                                            : __ldg(a.D + m * 36 + ci * 6 + ri);
      }
    stage_dw<DIM>(st + NP * DIM, __ldg(a.weight + m), a, m, [&](int ri, int ci) {
      int r = ri, c = ci;
      if constexpr (DIM == 2) {
        r = ri == 3 ? 2 : ri;
        c = ci == 3 ? 2 : ci;
      }
      return dv[r][c];
    });
  }
  __syncthreads();
  if (tid < EPB && e0 + tid < a.e_end) a.emask[e0 + tid] = s_mask[tid];
  delta_phase2<DIM, NP, NQ>(s_st, s_mask, tid, e0, a.e_end, a.scratch);
}

// k_delta_warp (2D): pass 1 from a finished constitutive update (flags +
// packed D or reference DS), warp-owned elements like k_newton_warp: lane
// (element, q) stages dphi and w (D - C) of its point when plastic, the
// ballot gives the element masks, phase-2 lanes build uniform chunks and the
// element records leave through TMA bulk stores.  Same FMA sequence as the
// fused kernel, hence identical bits.
template <int NP, int NQ, int MODE>
__global__ void __launch_bounds__(WarpCfg<2, NP, NQ>::THREADS) k_delta_warp(GatherArgs a) {
  pdl_trigger();
  constexpr int DIM = 2;
  using W = WarpCfg<DIM, NP, NQ>;
  constexpr int EPW = W::EPW, REC = W::REC, NS = W::NS;
  constexpr unsigned QMASK = NQ >= 32 ? 0xffffffffu : (1u << NQ) - 1u;
  constexpr int RECB = W::NB * W::D2;
  __shared__ double s_st[W::WPB][EPW * NQ * REC];
  __shared__ __align__(16) double s_out[W::WPB][EPW * RECB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e0 = a.e_begin + ((int64_t)blockIdx.x * W::WPB + w) * EPW;
  if (e0 >= a.e_end) return;  // warp-uniform
  double* st_w = s_st[w];
  bool plastic = false;
  if (lane < EPW * NQ) {
    const int le = lane / NQ, q = lane - le * NQ;
    const int64_t e = e0 + le;
    if (e < a.e_end) {
      const int64_t m = e * NQ + q;
      plastic = MODE == G_ELASTIC || (__ldg(a.flags + m) & 1) != 0;
      if (MODE == G_ELASTIC) {
        double* st = st_w + lane * REC;
        stage_geometry<DIM, NP>(st, a.inv + m * W::D2, a.gradhat, q);
        stage_c<DIM>(st + NP * DIM, __ldg(a.weight + m), a, m);
      } else if (plastic) {
        double* st = st_w + lane * REC;
        double dv[NS][NS];
#pragma unroll
        for (int r = 0; r < NS; ++r)
#pragma unroll
          for (int c = r; c < NS; ++c) {
            const int ri = arow<DIM>(r), ci = arow<DIM>(c);
            dv[r][c] = MODE == G_TANGENT_PACKED ? __ldg(a.D + m * EPFEM_D_STRIDE + pk_index(ri, ci))
                                                : __ldg(a.D + m * 36 + ci * 6 + ri);
          }
        stage_geometry<DIM, NP>(st, a.inv + m * W::D2, a.gradhat, q);
        stage_dw<DIM>(st + NP * DIM, __ldg(a.weight + m), a, m, [&](int ri, int ci) {
          const int r = ri == 3 ? 2 : ri, c = ci == 3 ? 2 : ci;
          return dv[r][c];
        });
      }
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, plastic);
  __syncwarp();
  if (lane < EPW && e0 + lane < a.e_end) a.emask[e0 + lane] = (bal >> (lane * NQ)) & QMASK;
  // phase 2 by row pairs (as k_newton_warp)
  constexpr int PL2 = 2 * ((NP + 1) / 2);
  for (int t = lane; t < EPW * PL2; t += 32) {
    const int le = t / PL2, k = t - (t / PL2) * PL2;
    const unsigned mask = (bal >> (le * NQ)) & QMASK;
    if (e0 + le < a.e_end && mask)
      delta_pairs2<NP>(st_w + le * NQ * REC, mask, k / 2, k % 2, REC, s_out[w] + le * RECB);
  }
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    int n = 0;
    for (int le = 0; le < EPW; ++le)
      if (e0 + le < a.e_end && ((bal >> (le * NQ)) & QMASK)) {
        tma_store_1d(a.scratch + (size_t)(e0 + le) * RECB, s_out[w] + le * RECB,
                     (unsigned)(RECB * sizeof(double)));
        ++n;
      }
    if (n) tma_store_wait_read();
  }
}

// k_delta_mma: the tensor-core phase 2 (delta_mma_warp) behind the same
// pass-1 staging as k_delta_warp, EPW = 32 / NQ elements per warp.
template <int DIM, int NP, int NQ, int MODE>
__global__ void __launch_bounds__(MmaCfg<DIM, NP, NQ>::THREADS) k_delta_mma(GatherArgs a) {
  pdl_trigger();
  using M = MmaCfg<DIM, NP, NQ>;
  constexpr int EPW = M::EPW, REC = M::REC, NS = M::NS;
  constexpr unsigned QMASK = NQ >= 32 ? 0xffffffffu : (1u << NQ) - 1u;
  __shared__ double s_st[M::WPB][EPW * NQ * REC];
  __shared__ __align__(16) double s_out[M::WPB][M::OUTB * M::RECB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e0 = a.e_begin + ((int64_t)blockIdx.x * M::WPB + w) * EPW;
  if (e0 >= a.e_end) return;  // warp-uniform
  double* st_w = s_st[w];
  bool plastic = false;
  if (lane < EPW * NQ) {
    const int le = lane / NQ, q = lane - le * NQ;
    const int64_t e = e0 + le;
    if (e < a.e_end) {
      const int64_t m = e * NQ + q;
      plastic = MODE == G_ELASTIC || (__ldg(a.flags + m) & 1) != 0;
      if (MODE == G_ELASTIC) {
        double* st = st_w + lane * REC;
        stage_geometry<DIM, NP>(st, a.inv + m * M::D2, a.gradhat, q);
        stage_c<DIM>(st + NP * DIM, __ldg(a.weight + m), a, m);
      } else if (plastic) {
        double* st = st_w + lane * REC;
        double dv[NS][NS];
#pragma unroll
        for (int r = 0; r < NS; ++r)
#pragma unroll
          for (int c = r; c < NS; ++c) {
            const int ri = arow<DIM>(r), ci = arow<DIM>(c);
            dv[r][c] = MODE == G_TANGENT_PACKED ? __ldg(a.D + m * EPFEM_D_STRIDE + pk_index(ri, ci))
                                                : __ldg(a.D + m * 36 + ci * 6 + ri);
          }
        stage_geometry<DIM, NP>(st, a.inv + m * M::D2, a.gradhat, q);
        stage_dw<DIM>(st + NP * DIM, __ldg(a.weight + m), a, m, [&](int ri, int ci) {
          int r = ri, c = ci;
          if constexpr (DIM == 2) {
            r = ri == 3 ? 2 : ri;
            c = ci == 3 ? 2 : ci;
          }
          return dv[r][c];
        });
      }
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, plastic);
  __syncwarp();
  if (lane < EPW && e0 + lane < a.e_end) a.emask[e0 + lane] = (bal >> (lane * NQ)) & QMASK;
  delta_mma_warp<DIM, NP, NQ>(st_w, s_out[w], bal, e0, a.e_end, a.scratch, lane);
}

constexpr int kStreamThreads = 256;

// one CTA per node range (rows.cuh); programmatic dependent launch: the
// K_elast load and node offsets overlap the producer's tail
template <int DIM, int NP, int NQ>
__global__ void __launch_bounds__(kStreamThreads) k_row_stream(GatherArgs a, int npc) {
  extern __shared__ __align__(128) double img_raw[];
  __shared__ uint64_t s_bar;
  if (threadIdx.x == 0) {
    mbar_init(&s_bar, 1);
    mbar_init_fence();
  }
  __syncthreads();
  row_range<DIM, NP, NQ, kStreamThreads, false>(a, npc, blockIdx.x, img_raw, &s_bar, 0u,
                                               [] { asm volatile("griddepcontrol.wait;" ::: "memory"); });
}

__global__ void k_range_span(int64_t n_nodes, int npc, int d2, const int64_t* __restrict__ nbr_ptr,
                             const int64_t* __restrict__ n2e_ptr, int* out) {
  int m = 0, mi = 0;
  const int64_t n_ranges = (n_nodes + npc - 1) / npc;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_ranges;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = r * npc, n1 = min(n0 + (int64_t)npc, n_nodes);
    m = max(m, (int)((nbr_ptr[n1] - nbr_ptr[n0]) * d2));
    mi = max(mi, (int)(n2e_ptr[n1] - n2e_ptr[n0]));
  }
  atomicMax(out, m);
  atomicMax(out + 1, mi);
}

// largest element touching each node chunk (items are sorted, so a node's
// last item holds its largest element)
__global__ void k_chunk_emax(int64_t n_nodes, int np, int64_t nodes_per_chunk,
                             const int64_t* __restrict__ n2e_ptr, const int32_t* __restrict__ n2e,
                             unsigned long long* emax) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n_nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t hi = n2e_ptr[a + 1];
    if (hi > n2e_ptr[a]) atomicMax(emax + a / nodes_per_chunk, (unsigned long long)(n2e[hi - 1] / np));
  }
}

}  // namespace

// Split the nodes into n_chunks ranges aligned to the row-stream CTA size and
// the elements so that element chunk k holds exactly the elements the rows of
// node chunk k need beyond chunks < k (monotone by construction).
int plan_chunks(int64_t n_nodes, int64_t n_elements, int np, const int64_t* n2e_ptr,
                const int32_t* n2e, int npc, int n_chunks, int64_t* nchunk, int64_t* echunk,
                cudaStream_t st) {
  int64_t per = ((n_nodes + n_chunks - 1) / n_chunks + npc - 1) / npc * npc;
  if (per < npc) per = npc;
  n_chunks = (int)((n_nodes + per - 1) / per);
  unsigned long long* d = nullptr;
  unsigned long long h[64];
  // returns -1 (message set) on failure: the chunk count is the success value
  if (cudaMalloc(&d, sizeof(unsigned long long) * n_chunks) != cudaSuccess ||
      cudaMemsetAsync(d, 0, sizeof(unsigned long long) * n_chunks, st) != cudaSuccess)
    return cuda_fail(cudaGetLastError(), "plan_chunks"), -1;
  k_chunk_emax<<<256, 256, 0, st>>>(n_nodes, np, per, n2e_ptr, n2e, d);
  if (cudaMemcpyAsync(h, d, sizeof(unsigned long long) * n_chunks, cudaMemcpyDeviceToHost, st) !=
          cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess) {
    cudaFree(d);
    return cuda_fail(cudaGetLastError(), "plan_chunks"), -1;
  }
  cudaFree(d);
  nchunk[0] = 0;
  echunk[0] = 0;
  int64_t run = 0;
  for (int k = 0; k < n_chunks; ++k) {
    nchunk[k + 1] = std::min<int64_t>(n_nodes, (int64_t)(k + 1) * per);
    run = std::max<int64_t>(run, (int64_t)h[k] + 1);
    echunk[k + 1] = k + 1 == n_chunks ? n_elements : std::min<int64_t>(run, n_elements);
  }
  return n_chunks;
}

size_t tangent_workspace_doubles(int family, int dim, int64_t n_elements) {
  size_t nb = 0;
  dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int NP = ET<decltype(F)::value, decltype(D)::value>::NP;
    nb = (size_t)NP * (NP + 1) / 2 * decltype(D)::value * decltype(D)::value;
  });
  return nb * (size_t)n_elements;
}

// Nodes per CTA for the row stream: the largest power of two <= 64 whose
// widest value range and item list fit the shared-memory budget.
int plan_row_stream(int64_t n_nodes, int dim, const int64_t* nbr_ptr, const int64_t* n2e_ptr,
                    cudaStream_t st, int* npc_out, int* span_out, int* items_out, int budget_bytes) {
  // bytes of dynamic smem per CTA and the starting node count; EPFEM_ROW_KB /
  // EPFEM_ROW_NPC override them for tuning runs (budget_bytes > 0: the
  // caller's budget, e.g. one warp's slice in the one-launch step)
  int budget = (dim == 2 ? 100 : 40) * 1024;  // measured optimum (2D: 32 nodes, Q1 hex: 16)
  int npc = 32;
  if (const char* v = getenv("EPFEM_ROW_KB")) budget = atoi(v) * 1024;
  if (budget_bytes > 0) budget = budget_bytes;
  if (const char* v = getenv("EPFEM_ROW_NPC")) npc = atoi(v);
  int* d = nullptr;
  EPFEM_CUDA_TRY(cudaMalloc(&d, 2 * sizeof(int)));
  int h[2] = {0, 0};
  for (;;) {
    EPFEM_CUDA_TRY(cudaMemsetAsync(d, 0, 2 * sizeof(int), st));
    k_range_span<<<256, 256, 0, st>>>(n_nodes, npc, dim * dim, nbr_ptr, n2e_ptr, d);
    EPFEM_CUDA_TRY(cudaMemcpyAsync(h, d, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
    EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
    const size_t bytes = 8 * ((size_t)h[0] + 2) + 4 * ((size_t)h[1] + 2 * (npc + 1));
    if (bytes <= (size_t)budget || npc == 1) break;
    npc /= 2;
  }
  cudaFree(d);
  *npc_out = npc;
  *span_out = h[0];
  *items_out = h[1];
  return 0;
}

int launch_row_stream(int family, int dim, const GatherArgs& a, cudaStream_t st) {
  if (a.n_nodes == 0) return 0;
  int rc = 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    const int64_t rblocks = (a.n_end - a.n_begin + a.npc - 1) / a.npc;
    if (rblocks <= 0) return;
    const size_t smem = row_range_smem(a);
    auto kern = k_row_stream<DIM, NP, NQ>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) { rc = cuda_fail(e, "cudaFuncSetAttribute"); return; }
    }
    // Programmatic dependent launch: the CTAs may start while the producer
    // of the workspace (fused / delta kernel) drains; they load K_elast and
    // the item lists, then block in griddepcontrol.wait until the producer
    // grid has completed and flushed (a no-op after a normal launch).
    static const bool pdl = getenv("EPFEM_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)rblocks);
    cfg.blockDim = dim3(kStreamThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, a.npc);
    if (e != cudaSuccess) rc = cuda_fail(e, "row stream launch");
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  if (rc) return rc;
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

int launch_delta(int family, int dim, int mode, const GatherArgs& a, cudaStream_t st) {
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    using Cfg = DeltaCfg<DIM, NP, NQ>;
    // same kernel family as the fused step (constitutive.cu): the tensor-core
    // phase 2 only with EPFEM_FUSED=mma
    static const int mma = [] {
      const char* v = getenv("EPFEM_FUSED");
      return (v && v[0] == 'm') ? 2 : 0;
    }();
    if (mma == 2 && mode != G_ELASTIC) {
      if (a.n_elements > 0) {
        using M = MmaCfg<DIM, NP, NQ>;
        const int64_t per = (int64_t)M::EPW * M::WPB;
        const unsigned blocks = (unsigned)((a.e_end - a.e_begin + per - 1) / per);
        if (mode == G_TANGENT_PACKED)
          k_delta_mma<DIM, NP, NQ, G_TANGENT_PACKED><<<blocks, M::THREADS, 0, st>>>(a);
        else
          k_delta_mma<DIM, NP, NQ, G_TANGENT_DS36><<<blocks, M::THREADS, 0, st>>>(a);
      }
      return;
    }
    if constexpr (DIM == 2) {
      if (a.n_elements > 0) {
        using W = WarpCfg<DIM, NP, NQ>;
        const int64_t per = (int64_t)W::EPW * W::WPB;
        const unsigned blocks = (unsigned)((a.e_end - a.e_begin + per - 1) / per);
        if (mode == G_TANGENT_PACKED)
          k_delta_warp<NP, NQ, G_TANGENT_PACKED><<<blocks, W::THREADS, 0, st>>>(a);
        else if (mode == G_ELASTIC)
          k_delta_warp<NP, NQ, G_ELASTIC><<<blocks, W::THREADS, 0, st>>>(a);
        else
          k_delta_warp<NP, NQ, G_TANGENT_DS36><<<blocks, W::THREADS, 0, st>>>(a);
      }
      return;
    }
    if (a.n_elements > 0) {
      const int64_t blocks = (a.e_end - a.e_begin + Cfg::EPB - 1) / Cfg::EPB;
      if (mode == G_TANGENT_PACKED)
        k_elem_delta_staged<DIM, NP, NQ, G_TANGENT_PACKED><<<(unsigned)blocks, Cfg::THREADS, 0, st>>>(a);
      else if (mode == G_ELASTIC)
        k_elem_delta_staged<DIM, NP, NQ, G_ELASTIC><<<(unsigned)blocks, Cfg::THREADS, 0, st>>>(a);
      else
        k_elem_delta_staged<DIM, NP, NQ, G_TANGENT_DS36><<<(unsigned)blocks, Cfg::THREADS, 0, st>>>(a);
    }
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

int launch_tangent(int family, int dim, int mode, const GatherArgs& a, cudaStream_t st) {
  if (a.n_nodes == 0) return 0;
  if (int rc = launch_delta(family, dim, mode, a, st)) return rc;
  return launch_row_stream(family, dim, a, st);
}

}  // namespace epfem_gpu
