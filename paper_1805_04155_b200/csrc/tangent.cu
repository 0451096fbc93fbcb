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
#include <algorithm>
#include <climits>
#include <vector>

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
// Q2-20: 4 CTAs per SM (64 registers) measured 9.6 vs 11.2 ms on cfg5; the
// same bound on Q1 / P2 tetrahedra is slower (ptxas then uses 56 registers)
#ifndef EPFEM_ROW_MINB20
#define EPFEM_ROW_MINB20 4
#endif

// The K_elast range [v0, v1) is read with ONE TMA bulk copy of the enclosing
// 16-byte-aligned range into the shared image (the K_elast allocation is
// padded by two doubles), overlapped with the item staging; the image goes
// back to K with one TMA bulk store of the aligned interior plus at most two
// edge doubles.  (rows.cuh holds the same range pass as a device function
// for the warp-owned ranges of the one-launch step; this stand-alone kernel
// keeps its own code: written as the shared function it compiled to 17 %
// slower 3D instances.)
// FLAGS: the overlapped step (OvlArgs): wait on the ready flags of the
// producer groups this range reads instead of griddepcontrol.wait, read the
// element records with plain (coherent) loads, and let the last CTA bump the
// generation.
__device__ __forceinline__ int ld_acquire_gpu_i(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// FORCES: also fold the element internal-force records (GatherArgs::fws,
// written by the fused kernel) into F for the range's nodes, every item in
// item order from zero (k_internal_forces' association, hence its bits).
#ifndef EPFEM_ROW_DYN
#define EPFEM_ROW_DYN 0
#endif
template <int DIM, int NP, int NQ, bool FLAGS = false, bool FORCES = false>
__global__ void __launch_bounds__(kStreamThreads, (DIM == 3 && NP >= 20) ? EPFEM_ROW_MINB20 : 0)
    k_row_stream(GatherArgs a, int npc, OvlArgs o) {
  extern __shared__ __align__(128) double img_raw[];
  __shared__ uint64_t s_bar;
  __shared__ int s_next;  // EPFEM_ROW_DYN: next unclaimed node of the range
  constexpr int NB = NP * (NP + 1) / 2;
  constexpr int D2 = DIM * DIM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t range = a.range_order ? (int64_t)__ldg(a.range_order + blockIdx.x) : (int64_t)blockIdx.x;
  const int64_t n0 = a.n_begin + range * npc;
  const int64_t n1 = min(n0 + (int64_t)npc, a.n_end);
  const int nloc = (int)(n1 - n0);
  const int64_t v0 = __ldg(a.nbr_ptr + n0) * D2;
  const int64_t v1 = __ldg(a.nbr_ptr + n1) * D2;
  const int64_t a0 = v0 & ~int64_t(1), a1 = (v1 + 1) & ~int64_t(1);
  const int64_t i_begin = __ldg(a.n2e_ptr + n0);
  const int nitems = (int)(__ldg(a.n2e_ptr + n1) - i_begin);
  // layout: [image (aligned to a0) | item (int) | iptr (int) | vptr (int)]
  double* img = img_raw + (v0 - a0);  // img[k] <-> global v0 + k
  int* s_item = reinterpret_cast<int*>(img_raw + a.max_span + 2);
  int* s_iptr = s_item + a.max_items;
  int* s_vptr = s_iptr + npc + 1;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_next = kStreamThreads / 32;
  }
  __syncthreads();
  const bool zero_base = a.base == nullptr;  // elastic assembly: K = sum of element blocks
  if (zero_base)
    for (int64_t k = tid; k < a1 - a0; k += blockDim.x) img_raw[k] = 0.0;
  if (tid == 0 && a1 > a0 && !zero_base) {
    const unsigned bytes = (unsigned)((a1 - a0) * 8);
    mbar_expect_tx(&s_bar, bytes);
    if (EPFEM_K_EVICT_FIRST && DIM == 3 && NP < 20)
      tma_load_1d_hint(img_raw, a.base + a0, bytes, &s_bar, l2_evict_first());
    else
      tma_load_1d(img_raw, a.base + a0, bytes, &s_bar);
  }
  // node offsets (cache data, independent of the producer kernel)
  for (int k = tid; k <= nloc; k += blockDim.x) {
    s_iptr[k] = (int)(__ldg(a.n2e_ptr + n0 + k) - i_begin);
    s_vptr[k] = (int)(__ldg(a.nbr_ptr + n0 + k) * D2 - v0);
  }
  // everything below reads the producer's emask / workspace
  int gen = 0;
  if constexpr (FLAGS) {
    gen = *((volatile int*)&o.sync->gen);
    if (warp == 0) {
      const int lo = __ldg(o.rlo + range), hi = __ldg(o.rhi + range);
      for (int k = lo + lane; k <= hi; k += 32)
        while (ld_acquire_gpu_i(o.flag + k) != gen + 1) __nanosleep(64);
    }
    __syncthreads();
  } else {
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  // stage the range's items (plastic ones kept, others -1)
  for (int k = tid; k < nitems; k += blockDim.x) {
    const int32_t it = __ldg(a.n2e + i_begin + k);
    s_item[k] = __ldcg(a.emask + it / NP) ? it : -1;
  }
  if constexpr (FORCES) {  // the range's force records, folded after the K adds
    double* s_fv = reinterpret_cast<double*>(
        (reinterpret_cast<uintptr_t>(s_vptr + npc + 1) + 15) & ~uintptr_t(15));
    for (int k = tid; k < nitems * DIM; k += blockDim.x) {
      const int it = __ldg(a.n2e + i_begin + k / DIM);
      s_fv[k] = a.fws[(size_t)it * DIM + k % DIM];
    }
  }
  __syncthreads();
  if (a1 > a0 && !zero_base) mbar_wait(&s_bar, 0);
  // Items are taken UB at a time: every lane first issues the loads of all
  // UB items (slot byte + workspace value), then applies the adds in item
  // order, so a node costs one memory round trip per UB items instead of
  // one per item (the add order, hence the bits, is unchanged).
  constexpr int KP = (NP * D2 + 31) / 32;
  constexpr int UB = KP == 1 ? 4 : 1;  // 3D: wider rows already give ILP; registers matter more
  for (int ln = warp; ln < nloc;) {
    const int ib = s_iptr[ln], ie = s_iptr[ln + 1];
    const int row_len = (s_vptr[ln + 1] - s_vptr[ln]) / DIM;
    double* seg = img + s_vptr[ln];
    for (int kb = ib; kb < ie; kb += UB) {
      double v[UB][KP];
      int sl[UB][KP];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int it = kb + u < ie ? s_item[kb + u] : -1;  // warp-uniform
        const int64_t el = it / NP;
        const int pa = it - (int)el * NP;
        const double* rec = a.scratch + (size_t)el * NB * D2;
#pragma unroll
        for (int kk = 0; kk < KP; ++kk) {
          const int k = lane + 32 * kk;
          sl[u][kk] = -1;
          if (it >= 0 && k < NP * D2) {
            // lane <-> entry (pb, i, j) of block row pa; block (pb, pa) read
            // transposed when pb < pa (branch-free addressing)
            const int pb = k / D2, ij = k - pb * D2;
            const int i = ij / DIM, j = ij - i * DIM;
            const bool up = pa <= pb;
            const int lo = up ? pa : pb, hi = up ? pb : pa;
            const int src = blk_index<NP>(lo, hi) * D2 + (up ? ij : j * DIM + i);
            sl[u][kk] = __ldg(a.slot + (int64_t)it * NP + pb);
            v[u][kk] = FLAGS ? rec[src] : __ldg(rec + src);  // FLAGS: written in this step's overlap
          }
        }
      }
      // A lane's column node differs from item to item, so two lanes can
      // update the same entry for different items: a warp barrier between
      // items keeps the add order = item order even when the warp has
      // diverged (independent thread scheduling).
#pragma unroll
      for (int u = 0; u < UB; ++u) {
#pragma unroll
        for (int kk = 0; kk < KP; ++kk)
          if (sl[u][kk] >= 0) {
            const int k = lane + 32 * kk;
            const int ij = k % D2, i = ij / DIM, j = ij - i * DIM;
            seg[i * row_len + sl[u][kk] * DIM + j] += v[u][kk];
          }
        __syncwarp();
      }
    }
#if EPFEM_ROW_DYN
    // dynamic node claim: warps that drew light nodes take the next ones
    // (one warp per node and item order as before, so the same bits)
    int nx = 0;
    if (lane == 0) nx = atomicAdd(&s_next, 1);
    ln = __shfl_sync(0xffffffffu, nx, 0);
#else
    ln += kStreamThreads / 32;
#endif
  }
  if constexpr (FORCES) {
    // the range's force records (item = (element, local node) = record
    // index) staged by all threads, then one thread per (node, component)
    // sums them in item order from zero
    const double* s_fv = reinterpret_cast<const double*>(
        (reinterpret_cast<uintptr_t>(s_vptr + npc + 1) + 15) & ~uintptr_t(15));
    for (int t = tid; t < nloc * DIM; t += blockDim.x) {
      const int ln = t / DIM, i = t - (t / DIM) * DIM;
      double f = 0.0;
      for (int k = s_iptr[ln]; k < s_iptr[ln + 1]; ++k) f = __dadd_rn(f, s_fv[k * DIM + i]);
      a.F_out[(n0 + ln) * DIM + i] = f;
    }
  }
  fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
  __syncthreads();
  if (tid == 0 && v1 > v0) {
    const int64_t s0 = (v0 + 1) & ~int64_t(1), s1 = v1 & ~int64_t(1);
    if (v0 & 1) a.out[v0] = img[0];
    if ((v1 & 1) && v1 - 1 >= s0) a.out[v1 - 1] = img[v1 - 1 - v0];
    if (s1 > s0) {
      if (EPFEM_K_EVICT_FIRST && DIM == 3 && NP < 20)
        tma_store_1d_sync_hint(a.out + s0, img + (s0 - v0), (unsigned)((s1 - s0) * 8), l2_evict_first());
      else
        tma_store_1d_sync(a.out + s0, img + (s0 - v0), (unsigned)((s1 - s0) * 8));
    }
  }
  if constexpr (FLAGS) {
    // every CTA of this grid has read gen once the counter completes
    if (tid == 0 && atomicAdd(&o.sync->finished, 1) == (int)gridDim.x - 1) {
      o.sync->finished = 0;
      atomicAdd(&o.sync->gen, 1);
      __threadfence();
    }
  }
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

// Row-stream CTA order along a space-filling curve.  A node range's K
// values are contiguous whatever order the ranges run in, but the element
// records it reads are shared with the ranges of the neighbouring node rows
// and planes: in node order those sit a whole plane of K apart, too far for
// the records to stay in L2 (cfg5: 15 KB per Q2-20 record, 8 GB of records
// re-read).  Ordering the ranges by the Morton code of their first node's
// coordinates (normalised to the mesh box) runs geometric neighbours
// together, so a record's readers meet while it is L2-resident.  Generic: it
// uses only the coordinates, not the structured numbering.
__global__ void k_coord_box(int64_t n, int dim, const double* __restrict__ coord, double* box) {
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n; a += (int64_t)gridDim.x * blockDim.x)
    for (int d = 0; d < dim; ++d) {
      const double x = coord[a * dim + d];
      lo[d] = fmin(lo[d], x);
      hi[d] = fmax(hi[d], x);
    }
  for (int d = 0; d < dim; ++d)
    for (int o = 16; o > 0; o >>= 1) {
      lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  if ((threadIdx.x & 31) == 0) {
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    for (int d = 0; d < dim; ++d) {
      box[w * 6 + d] = lo[d];
      box[w * 6 + 3 + d] = hi[d];
    }
  }
}

__device__ __forceinline__ uint64_t spread3(uint64_t v) {  // 21 bits -> every third bit
  v &= 0x1fffff;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}
__device__ __forceinline__ uint64_t spread2(uint64_t v) {  // 32 bits -> every second bit
  v &= 0xffffffffull;
  v = (v | v << 16) & 0x0000ffff0000ffffull;
  v = (v | v << 8) & 0x00ff00ff00ff00ffull;
  v = (v | v << 4) & 0x0f0f0f0f0f0f0f0full;
  v = (v | v << 2) & 0x3333333333333333ull;
  v = (v | v << 1) & 0x5555555555555555ull;
  return v;
}

__global__ void k_range_keys(int64_t n_nodes, int npc, int dim, const double* __restrict__ coord,
                             const double* __restrict__ box, uint64_t* keys) {
  const int64_t n_ranges = (n_nodes + npc - 1) / npc;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_ranges;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = r * npc;
    uint64_t q[3] = {0, 0, 0};
    const double scale = dim == 3 ? 2097151.0 : 4294967295.0;
    for (int d = 0; d < dim; ++d) {
      const double ext = box[3 + d] - box[d];
      const double t = ext > 0 ? (coord[a * dim + d] - box[d]) / ext : 0.0;
      q[d] = (uint64_t)fmin(fmax(t * scale, 0.0), scale);
    }
    keys[r] = dim == 3 ? (spread3(q[0]) | spread3(q[1]) << 1 | spread3(q[2]) << 2)
                       : (spread2(q[0]) | spread2(q[1]) << 1);
  }
}

int plan_range_order(int64_t n_nodes, int dim, int npc, const double* coord, cudaStream_t st,
                     int32_t** order_out) {
  *order_out = nullptr;
  const int64_t n_ranges = (n_nodes + npc - 1) / npc;
  if (n_ranges <= 1 || n_ranges >= INT32_MAX || !coord) return 0;
  constexpr int B = 256, T = 256, WARPS = B * T / 32;
  double* box = nullptr;
  uint64_t* keys = nullptr;
  EPFEM_CUDA_TRY(cudaMalloc(&box, sizeof(double) * 6 * WARPS));
  EPFEM_CUDA_TRY(cudaMalloc(&keys, sizeof(uint64_t) * n_ranges));
  k_coord_box<<<B, T, 0, st>>>(n_nodes, dim, coord, box);
  std::vector<double> hb(6 * WARPS);
  EPFEM_CUDA_TRY(cudaMemcpyAsync(hb.data(), box, sizeof(double) * hb.size(), cudaMemcpyDeviceToHost, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  double g[6] = {1e300, 1e300, 1e300, -1e300, -1e300, -1e300};
  for (int w = 0; w < WARPS; ++w)
    for (int d = 0; d < dim; ++d) {
      g[d] = std::min(g[d], hb[w * 6 + d]);
      g[3 + d] = std::max(g[3 + d], hb[w * 6 + 3 + d]);
    }
  EPFEM_CUDA_TRY(cudaMemcpyAsync(box, g, sizeof(g), cudaMemcpyHostToDevice, st));
  k_range_keys<<<256, 256, 0, st>>>(n_nodes, npc, dim, coord, box, keys);
  std::vector<uint64_t> hk(n_ranges);
  EPFEM_CUDA_TRY(cudaMemcpyAsync(hk.data(), keys, sizeof(uint64_t) * n_ranges, cudaMemcpyDeviceToHost, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(box);
  cudaFree(keys);
  std::vector<int32_t> order(n_ranges);
  for (int64_t r = 0; r < n_ranges; ++r) order[r] = (int32_t)r;
  std::stable_sort(order.begin(), order.end(), [&](int32_t x, int32_t y) { return hk[x] < hk[y]; });
  int32_t* d = nullptr;
  EPFEM_CUDA_TRY(cudaMalloc(&d, sizeof(int32_t) * n_ranges));
  EPFEM_CUDA_TRY(cudaMemcpyAsync(d, order.data(), sizeof(int32_t) * n_ranges, cudaMemcpyHostToDevice, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  *order_out = d;
  return 0;
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
    const size_t smem = row_range_smem(a) + (a.F_out ? 16 + sizeof(double) * DIM * (size_t)a.max_items : 0);
    auto kern = a.F_out ? k_row_stream<DIM, NP, NQ, false, true> : k_row_stream<DIM, NP, NQ>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) { rc = cuda_fail(e, "cudaFuncSetAttribute"); return; }
    }
    // Programmatic dependent launch: the CTAs may start while the producer
    // of the workspace (fused / delta kernel) drains; they load K_elast and
    // the item lists, then block in griddepcontrol.wait until the producer
    // grid has completed and flushed (a no-op after a normal launch).
    // Not after Q2-20 producers: their one-element CTAs (constitutive.cu,
    // FusedCfg) ran slower beside waiting row-stream CTAs (cfg5 step 25.6 vs
    // 24.76 ms); on the other meshes PDL is neutral to slightly positive.
    static const bool pdl_env = getenv("EPFEM_NO_PDL") == nullptr;
    const bool pdl = pdl_env && !(DIM == 3 && NP >= 20);
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
    GatherArgs b = a;
    if (a.n_begin != 0 || a.n_end != a.n_nodes) b.range_order = nullptr;  // the order covers whole-mesh launches
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, b, a.npc, OvlArgs{});
    if (e != cudaSuccess) rc = cuda_fail(e, "row stream launch");
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  if (rc) return rc;
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

// Row stream of the overlapped step: PDL launch (its CTAs start once every
// producer CTA has started) waiting on per-group flags (k_row_stream<FLAGS>).
int launch_row_stream_ovl(int family, int dim, const GatherArgs& a, const OvlArgs& o, cudaStream_t st) {
  if (a.n_nodes == 0) return 0;
  int rc = 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    if constexpr (DIM == 2) {
      const int64_t rblocks = (a.n_nodes + a.npc - 1) / a.npc;
      const size_t smem = sizeof(double) * ((size_t)a.max_span + 2) +
                          sizeof(int) * ((size_t)a.max_items + 2 * ((size_t)a.npc + 1));
      auto kern = k_row_stream<DIM, NP, NQ, true>;
      if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) { rc = cuda_fail(e, "cudaFuncSetAttribute"); return; }
      }
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)rblocks);
      cfg.blockDim = dim3(kStreamThreads);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      GatherArgs b = a;
      b.range_order = nullptr;  // flags are ordered by node range
      cudaError_t e = cudaLaunchKernelEx(&cfg, kern, b, a.npc, o);
      if (e != cudaSuccess) rc = cuda_fail(e, "overlapped row stream launch");
    } else {
      rc = fail(EPFEM_ERR_INVALID, "overlapped step: 2D meshes only");
    }
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
