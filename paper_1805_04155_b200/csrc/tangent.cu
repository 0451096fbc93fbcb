// K2 + K6: the per-iteration tangent  K = K_elast + sum_{plastic q} B_q^T w_q (D_q - C_q) B_q
// (assembly.cpp:186-213), as two deterministic passes without atomics.
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

#include "delta.cuh"

#ifndef EPFEM_K_EVICT_FIRST
#define EPFEM_K_EVICT_FIRST 1  // 3D Q1 / P2: K_elast and K streamed through L2 with evict_first (measured
                               // cfg3 row stream 3.08 -> 2.97 ms, cfg4 3.76 -> 3.66; neutral or worse in 2D / Q2-20)
#endif

namespace epfem_gpu {

namespace {

// CTA shape of the standalone element-delta kernel: DeltaCfg's, except for Q1
// hexahedra, which take the fused kernel's 16 elements on 128 threads (one
// thread per point in phase 1)
#ifndef EPFEM_DELTA_EPB_Q1
#define EPFEM_DELTA_EPB_Q1 16
#endif
template <int DIM, int NP, int NQ, int MODE>
struct StagedCfg : DeltaCfg<DIM, NP, NQ> {
  using Base = DeltaCfg<DIM, NP, NQ>;
  // (the elastic assembly keeps delta_phase2, written for DeltaCfg's shape)
  static constexpr bool Q1 = DIM == 3 && NP == 8 && EPFEM_DELTA_EPB_Q1 > 0 && MODE != G_ELASTIC;
  static constexpr int EPB = Q1 ? EPFEM_DELTA_EPB_Q1 : Base::EPB;
  static constexpr int THREADS = Q1 ? ((EPB * NQ + 31) / 32) * 32 : Base::THREADS;
};

template <int DIM, int NP, int NQ, int MODE>
__global__ void __launch_bounds__(StagedCfg<DIM, NP, NQ, MODE>::THREADS) k_elem_delta_staged(GatherArgs a) {
  pdl_trigger();
  using Cfg = StagedCfg<DIM, NP, NQ, MODE>;
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
  if constexpr (DIM == 3 && UseCyc3<NP>::value && MODE != G_ELASTIC) {
    // the fused kernels' phase 2 (cyclic row pairs), so the records match
    // theirs bit for bit
    using PC = Pair3Cfg<NP, NQ>;
    for (int t = tid; t < EPB * PC::PL; t += blockDim.x) {
      const int le = t / PC::PL;
      const int64_t e = e0 + le;
      if (e < a.e_end && s_mask[le])
        delta_rowpair3<NP, NQ>(&s_st[le][0][0], s_mask[le], t - le * PC::PL, a.scratch + (size_t)e * Cfg::NB * Cfg::D2);
    }
  } else {
    static_assert(EPB == DeltaCfg<DIM, NP, NQ>::EPB, "delta_phase2 uses DeltaCfg's shape");
    delta_phase2<DIM, NP, NQ>(s_st, s_mask, tid, e0, a.e_end, a.scratch);
  }
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

constexpr int kStreamThreads = 256;  // the most threads of a row-stream CTA
// Threads per row-stream CTA (a warp per node at a time).  Measured on B200
// with the row-task add loop (32 registers): Q1 hexahedra 8 nodes on 128 threads
// 3.34 ms against 3.48 ms for 16 nodes on 256 (cfg4); P2 tetrahedra 4 nodes on
// 128 threads 2.79 against 2.84 ms (cfg3); Q2-20 and 2D stay at 256 threads
// (cfg5 9.06 against 9.54 ms at 128).  EPFEM_ROW_THREADS overrides (tuning).
static int row_stream_threads(int dim, int np) {
  static const int env = [] {
    const char* v = getenv("EPFEM_ROW_THREADS");
    return v ? atoi(v) : 0;
  }();
  if (env >= 32 && env <= kStreamThreads && env % 32 == 0) return env;
  return (dim == 3 && np < 20) ? 128 : kStreamThreads;
}
// Q2-20: 4 CTAs per SM (64 registers) measured 9.6 vs 11.2 ms on cfg5; the
// same bound on Q1 / P2 tetrahedra is slower (ptxas then uses 56 registers)
#ifndef EPFEM_ROW_MINB20
#define EPFEM_ROW_MINB20 4
#endif
// Q1 hexahedra: the items' block rows are copied into a per-warp double buffer in
// shared memory with cp.async one plastic item ahead of its adds (the slot
// bytes one item ahead in registers), so a node's record reads overlap the
// adds of its previous item instead of costing one memory round trip each
#ifndef EPFEM_ROW_ASYNC
#define EPFEM_ROW_ASYNC 1
#endif
#ifndef EPFEM_ROW_ASYNC20
#define EPFEM_ROW_ASYNC20 1
#endif
// element types whose row stream takes the async item ring (measured: Q1
// cfg4 rows 3.70 -> 3.55 ms, Q2-20 cfg5 9.44 -> 9.21 ms; P2 tetrahedra
// slower, 3.00 -> 3.05 ms: the ring's shared memory costs a CTA per SM)
#ifndef EPFEM_ROW_ASYNC10
#define EPFEM_ROW_ASYNC10 1
#endif
__host__ __device__ constexpr bool async_row_stream(int np) {
  return np == 8 || (EPFEM_ROW_ASYNC20 && np == 20) || (EPFEM_ROW_ASYNC10 && np == 10);
}
#ifndef EPFEM_ROW_STAGES
#define EPFEM_ROW_STAGES 2  // items in flight + 1
#endif

// The K_elast range [v0, v1) is read with ONE TMA bulk copy of the enclosing
// 16-byte-aligned range into the shared image (the K_elast allocation is
// padded by two doubles), overlapped with the item staging; the image goes
// back to K with one TMA bulk store of the aligned interior plus at most two
// edge doubles.
template <int DIM, int NP, int NQ>
__global__ void __launch_bounds__(kStreamThreads, (DIM == 3 && NP >= 20) ? EPFEM_ROW_MINB20 : 0)
    k_row_stream(GatherArgs a, int npc) {
  extern __shared__ __align__(128) double img_raw[];
  __shared__ uint64_t s_bar;
  constexpr int NB = NP * (NP + 1) / 2;
  constexpr int D2 = DIM * DIM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  const int64_t range = blockIdx.x;
  const int64_t n0 = a.n_begin + range * npc;
  const int64_t n1 = min(n0 + (int64_t)npc, a.n_end);
  const int nloc = (int)(n1 - n0);
  const int64_t v0 = __ldg(a.nbr_ptr + n0) * D2;
  const int64_t v1 = __ldg(a.nbr_ptr + n1) * D2;
  const int64_t a0 = v0 & ~int64_t(1), a1 = (v1 + 1) & ~int64_t(1);
  const int64_t i_begin = __ldg(a.n2e_ptr + n0);
  const int nitems = (int)(__ldg(a.n2e_ptr + n1) - i_begin);
  EPFEM_CHECK(nloc >= 0 && nloc <= npc && v1 - v0 <= a.max_span && nitems <= a.max_items);
  // layout: [image (aligned to a0) | item (int) | iptr (int) | vptr (int)]
  double* img = img_raw + (v0 - a0);  // img[k] <-> global v0 + k
  int* s_item = reinterpret_cast<int*>(img_raw + a.max_span + 2);
  int* s_iptr = s_item + a.max_items;
  int* s_vptr = s_iptr + npc + 1;
  if (tid == 0) {
    mbar_init(&s_bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
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
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // stage the range's items (plastic ones kept, others -1)
  for (int k = tid; k < nitems; k += blockDim.x) {
    const int32_t it = __ldg(a.n2e + i_begin + k);
    s_item[k] = __ldcg(a.emask + it / NP) ? it : -1;
  }
  __syncthreads();
  if (a1 > a0 && !zero_base) mbar_wait(&s_bar, 0);
  // Items are taken UB at a time: every lane first issues the loads of all
  // UB items (slot byte + workspace value), then applies the adds in item
  // order, so a node costs one memory round trip per UB items instead of
  // one per item (the add order, hence the bits, is unchanged).
  constexpr int KP = (NP * D2 + 31) / 32;
  constexpr int UB = KP == 1 ? 4 : 1;  // 3D: wider rows already give ILP; registers matter more
  constexpr bool ASYNC = EPFEM_ROW_ASYNC && KP > 1 && async_row_stream(NP);
  if constexpr (ASYNC) {
    // per-warp ring of STAGES buffers after the node offsets (16-byte
    // aligned): an item's block row (NP * D2 doubles) and its NP slot bytes
    constexpr int STAGES = EPFEM_ROW_STAGES;
    constexpr int SLW = (NP + 7) / 8;                   // doubles holding the NP slot bytes
    constexpr int BUF = ((NP * D2 + 1) / 2) * 2 + ((SLW + 1) / 2) * 2;  // doubles (even: 16-byte steps)
    double* wbuf = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(s_vptr + npc + 1) + 15) & ~uintptr_t(15)) +
                   warp * STAGES * BUF;
    // lane <-> row task t = (pb, i): the three entries (i, 0..2) of block
    // (pa, pb), contiguous in the buffer and in the K row (one slot lookup and
    // one address per task instead of per entry)
    constexpr int NTASK = NP * DIM, TR = (NTASK + 31) / 32;
    static_assert(DIM == 3, "row tasks are written for dim 3");
    // NP % 4 != 0 (P2 tetrahedra): an item's slot bytes are not 4-byte aligned,
    // so each lane loads its task's slot byte into a register when the item's
    // copies are issued, one item ahead of the adds (two stages)
    constexpr bool SLOT_REG = NP % 4 != 0;
    static_assert(!SLOT_REG || STAGES == 2, "register slots are written for one item in flight");
    int sl_cur[TR], sl_nxt[TR];
#pragma unroll
    for (int rr = 0; rr < TR; ++rr) sl_cur[rr] = sl_nxt[rr] = 0;
    // copy item `it`'s block row and slots into buffer `buf` (one commit group)
    auto issue = [&](int it, double* buf, int* sl_reg) {
      const int64_t el = it / NP;
      const int pa = it - (int)el * NP;
      const double* rec = a.scratch + (size_t)el * NB * D2;
#pragma unroll
      for (int rr = 0; rr < TR; ++rr) {
        const int t = lane + 32 * rr;
        if (t < NTASK) {
          const int pb = t / DIM, i = t - pb * DIM;
          const bool up = pa <= pb;
          const int lo = up ? pa : pb, hi = up ? pb : pa;
          // block (pb, pa) is read transposed when pb < pa
          const double* src = rec + blk_index<NP>(lo, hi) * D2 + (up ? DIM * i : i);
          const int step = up ? 1 : DIM;
          double* dst = buf + DIM * t;
          cp_async8(dst, src);
          cp_async8(dst + 1, src + step);
          cp_async8(dst + 2, src + 2 * step);
          if constexpr (SLOT_REG) sl_reg[rr] = __ldg(a.slot + (int64_t)it * NP + pb);
        }
      }
      // the NP slot bytes in 4-byte words (NP % 4 == 0: 4-byte aligned source), on the last lanes
      if (!SLOT_REG && lane >= 32 - NP / 4) {
        const int w = lane - (32 - NP / 4);
        cp_async4(reinterpret_cast<uint8_t*>(buf + NP * D2 + (NP * D2) % 2) + 4 * w, a.slot + (int64_t)it * NP + 4 * w);
      }
      cp_async_commit();
    };
    for (int ln = warp; ln < nloc; ln += nwarps) {
      const int ie = s_iptr[ln + 1];
      const int row_len = (s_vptr[ln + 1] - s_vptr[ln]) / DIM;
      double* seg = img + s_vptr[ln];
      auto next = [&](int k) {  // the node's next plastic item at or after k (warp-uniform)
        while (k < ie && s_item[k] < 0) ++k;
        return k;
      };
      int kb = next(s_iptr[ln]);
      if (kb >= ie) continue;
      // prologue: STAGES - 1 items in flight (empty groups past the node's end)
      int kiss = kb;
#pragma unroll
      for (int s = 0; s < STAGES - 1; ++s) {
        if (kiss < ie) {
          issue(s_item[kiss], wbuf + s * BUF, sl_cur);
          kiss = next(kiss + 1);
        } else {
          cp_async_commit();
        }
      }
      int r = 0;
      while (kb < ie) {
        const int w = (r + STAGES - 1) % STAGES;
        if (kiss < ie) {
          issue(s_item[kiss], wbuf + w * BUF, sl_nxt);
          kiss = next(kiss + 1);
        } else {
          cp_async_commit();
        }
        cp_async_wait_n<STAGES - 1>();  // item kb's group is complete
        __syncwarp();
        const double* cur = wbuf + r * BUF;
        const uint8_t* sls = reinterpret_cast<const uint8_t*>(cur + NP * D2 + (NP * D2) % 2);
#pragma unroll
        for (int rr = 0; rr < TR; ++rr) {
          const int t = lane + 32 * rr;
          if (t < NTASK) {
            const int pb = t / DIM, i = t - pb * DIM;
            const int sl = SLOT_REG ? sl_cur[rr] : sls[pb];
            EPFEM_CHECK(sl < row_len / DIM && s_vptr[ln] + i * row_len + sl * DIM + DIM - 1 < s_vptr[ln + 1]);
            double* p = seg + i * row_len + sl * DIM;
            const double* c3 = cur + DIM * t;
            p[0] += c3[0];
            p[1] += c3[1];
            p[2] += c3[2];
          }
        }
        if constexpr (SLOT_REG) {
#pragma unroll
          for (int rr = 0; rr < TR; ++rr) sl_cur[rr] = sl_nxt[rr];
        }
        // every lane's adds of this item are done (add order = item order)
        // and the buffer is free before the next copy into it
        __syncwarp();
        r = (r + 1) % STAGES;
        kb = next(kb + 1);
      }
    }
  }
  if constexpr (!ASYNC && DIM == 3) {
    // tetrahedra: the same row tasks with the loads into registers (the ring's
    // shared memory would cost a resident CTA)
    constexpr int NTASK = NP * DIM, TR = (NTASK + 31) / 32;
    for (int ln = warp; ln < nloc; ln += nwarps) {
      const int ib = s_iptr[ln], ie = s_iptr[ln + 1];
      const int row_len = (s_vptr[ln + 1] - s_vptr[ln]) / DIM;
      double* seg = img + s_vptr[ln];
      for (int kb = ib; kb < ie; ++kb) {
        const int it = s_item[kb];  // warp-uniform
        if (it < 0) continue;
        const int64_t el = it / NP;
        const int pa = it - (int)el * NP;
        const double* rec = a.scratch + (size_t)el * NB * D2;
        double v[TR][DIM];
        int sl[TR];
#pragma unroll
        for (int rr = 0; rr < TR; ++rr) {
          const int t = lane + 32 * rr;
          if (t < NTASK) {
            const int pb = t / DIM, i = t - pb * DIM;
            const bool up = pa <= pb;
            const int lo = up ? pa : pb, hi = up ? pb : pa;
            const double* src = rec + blk_index<NP>(lo, hi) * D2 + (up ? DIM * i : i);
            const int step = up ? 1 : DIM;
            sl[rr] = __ldg(a.slot + (int64_t)it * NP + pb);
#pragma unroll
            for (int j = 0; j < DIM; ++j) v[rr][j] = __ldg(src + j * step);
          }
        }
#pragma unroll
        for (int rr = 0; rr < TR; ++rr) {
          const int t = lane + 32 * rr;
          if (t < NTASK) {
            const int i = t % DIM;
            EPFEM_CHECK(sl[rr] < row_len / DIM && s_vptr[ln] + i * row_len + sl[rr] * DIM + DIM - 1 < s_vptr[ln + 1]);
            double* p = seg + i * row_len + sl[rr] * DIM;
#pragma unroll
            for (int j = 0; j < DIM; ++j) p[j] += v[rr][j];
          }
        }
        __syncwarp();  // add order = item order (see below)
      }
    }
  }
  for (int ln = (ASYNC || DIM == 3) ? nloc : warp; ln < nloc;) {

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
            v[u][kk] = __ldg(rec + src);
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
            // single writer: warp ln owns node ln's dim rows [vptr[ln], vptr[ln + 1])
            EPFEM_CHECK(sl[u][kk] < row_len / DIM &&
                        s_vptr[ln] + i * row_len + sl[u][kk] * DIM + j < s_vptr[ln + 1]);
            seg[i * row_len + sl[u][kk] * DIM + j] += v[u][kk];
          }
        __syncwarp();
      }
    }
    // (claiming nodes dynamically from a shared counter gave the same bits
    // and measured no faster: warp imbalance inside a range is not the limit)
    ln += nwarps;
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

}  // namespace

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
int plan_row_stream(int64_t n_nodes, int dim, int np, const int64_t* nbr_ptr, const int64_t* n2e_ptr,
                    cudaStream_t st, int* npc_out, int* span_out, int* items_out, int budget_bytes) {
  // bytes of dynamic smem per CTA and the starting node count; EPFEM_ROW_KB /
  // EPFEM_ROW_NPC override them for tuning runs (budget_bytes > 0: the
  // caller's budget)
  int budget = (dim == 2 ? 100 : 40) * 1024;  // measured optimum (2D: 32 nodes; Q2-20: 8)
  int npc = 32;
  if (dim == 3 && np == 8) npc = 8;        // Q1 hexahedra: 8 nodes on 128 threads (row_stream_threads)
  else if (dim == 3 && np < 20) npc = 4;   // tetrahedra: 4 nodes on 128 threads
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

// dynamic shared memory of one node range: image + items + node offsets
static size_t row_range_smem(const GatherArgs& a, int async_buf, int threads) {
  return sizeof(double) * ((size_t)a.max_span + 2) + sizeof(int) * ((size_t)a.max_items + 2 * ((size_t)a.npc + 1)) +
         (async_buf ? 16 + sizeof(double) * (threads / 32) * EPFEM_ROW_STAGES * (size_t)async_buf : 0);
}

int launch_row_stream(int family, int dim, const GatherArgs& a, cudaStream_t st) {
  if (a.n_nodes == 0) return 0;
  int rc = 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    const int64_t rblocks = (a.n_end - a.n_begin + a.npc - 1) / a.npc;
    if (rblocks <= 0) return;
    constexpr int KP = (NP * DIM * DIM + 31) / 32;
    constexpr int SLW = (NP + 7) / 8;
    const int threads = row_stream_threads(DIM, NP);
    const size_t smem = row_range_smem(
        a, (EPFEM_ROW_ASYNC && KP > 1 && async_row_stream(NP)) ? ((NP * DIM * DIM + 1) / 2) * 2 + ((SLW + 1) / 2) * 2 : 0,
        threads);
    auto kern = k_row_stream<DIM, NP, NQ>;
    if (smem + 1024 > 48 * 1024) {  // the static mbarrier and the reserved 1 KB count against the 48 KB default
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
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, a, a.npc);
    if (e != cudaSuccess)
      rc = cuda_fail(e, ("row stream launch: " + std::to_string(rblocks) + " CTAs, " + std::to_string(smem) +
                         " B shared memory").c_str());
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
      auto go = [&](auto m) {
        using SC = StagedCfg<DIM, NP, NQ, decltype(m)::value>;
        const int64_t blocks = (a.e_end - a.e_begin + SC::EPB - 1) / SC::EPB;
        k_elem_delta_staged<DIM, NP, NQ, decltype(m)::value><<<(unsigned)blocks, SC::THREADS, 0, st>>>(a);
      };
      if (mode == G_TANGENT_PACKED) go(IC<G_TANGENT_PACKED>{});
      else if (mode == G_ELASTIC) go(IC<G_ELASTIC>{});
      else go(IC<G_TANGENT_DS36>{});
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
