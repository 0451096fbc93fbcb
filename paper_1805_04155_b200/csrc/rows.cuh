// Pass 2 of the tangent (K2 + K6) for one range of consecutive nodes as a
// device function: the warp-owned ranges of the one-launch Newton step
// (k_newton_mega, constitutive.cu).  Same algorithm as the stand-alone row
// stream k_row_stream (tangent.cu), which keeps its own code for codegen
// reasons (see there).
//
// One CTA owns the nodes [n0, n1) = one contiguous value range of K (a node's
// dim rows are contiguous and nodes are numbered in row order).  ONE TMA bulk
// copy brings the enclosing 16-byte-aligned range of K_elast into a shared
// image (the K_elast allocation is padded by two doubles) while the threads
// stage the range's (element, node) items; each warp adds the plastic items'
// block rows of dK_e for its nodes at the cached slots (one warp per node: a
// single writer per row, no atomics); ONE TMA bulk store writes the image to
// K[range] (plus at most two unaligned edge doubles).  Rows without plastic
// contributions are therefore bitwise copies of K_elast.
//
// `wait()` runs after everything that does not depend on the producer of
// the workspace (K_elast load issued, node offsets staged) and before the
// first emask / workspace read: griddepcontrol.wait after a programmatic
// dependent launch, or the per-group ready flags of the one-launch step.
// FRESH = the workspace was written earlier in the SAME launch: plain weak
// loads after the acquire, never the read-only (.nc) path.
#pragma once

#include "delta.cuh"

#ifndef EPFEM_K_EVICT_FIRST
#define EPFEM_K_EVICT_FIRST 1  // 3D Q1 / P2: K_elast and K streamed through L2 with evict_first (measured
                               // cfg3 row stream 3.08 -> 2.97 ms, cfg4 3.76 -> 3.66; neutral or worse in 2D / Q2-20)
#endif

namespace epfem_gpu {

// dynamic shared memory of one node range: image + items + node offsets
inline size_t row_range_smem(const GatherArgs& a) {
  return sizeof(double) * ((size_t)a.max_span + 2) + sizeof(int) * ((size_t)a.max_items + 2 * ((size_t)a.npc + 1));
}

// s_bar: the CTA's mbarrier, initialised by the caller (mbar_init(s_bar, 1)
// + fence); `parity` = the phase this range's K_elast load completes.
// Returns true when the range used the barrier (a phase completed).
// NTHREADS = 32: one warp owns the range (tid = its lane; warp barriers
// only, and the bulk store is only waited for until its source is read).
template <int DIM, int NP, int NQ, int NTHREADS, bool FRESH, class Wait>
__device__ __forceinline__ bool row_range(const GatherArgs& a, int npc, int64_t range, double* img_raw,
                                          uint64_t* s_bar, unsigned parity, Wait&& wait,
                                          int tid = threadIdx.x) {
  constexpr int NB = NP * (NP + 1) / 2;
  constexpr int D2 = DIM * DIM;
  constexpr bool HINT = EPFEM_K_EVICT_FIRST && DIM == 3 && NP < 20;
  constexpr bool WARP = NTHREADS == 32;
  auto sync = [] {
    if constexpr (WARP) __syncwarp(); else __syncthreads();
  };
  const int lane = tid & 31, warp = tid >> 5;
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
  const bool zero_base = a.base == nullptr;  // elastic assembly: K = sum of element blocks
  // staging loops stride by the runtime block size (a compile-time stride
  // gets them unrolled: +14 registers on the 3D instances, one CTA per SM less)
  const int nthr = WARP ? 32 : (int)blockDim.x;
  if (zero_base)
    for (int64_t k = tid; k < a1 - a0; k += nthr) img_raw[k] = 0.0;
  if (tid == 0 && a1 > a0 && !zero_base) {
    const unsigned bytes = (unsigned)((a1 - a0) * 8);
    mbar_expect_tx(s_bar, bytes);
    if (HINT)
      tma_load_1d_hint(img_raw, a.base + a0, bytes, s_bar, l2_evict_first());
    else
      tma_load_1d(img_raw, a.base + a0, bytes, s_bar);
  }
  // node offsets (cache data, independent of the producer)
  for (int k = tid; k <= nloc; k += nthr) {
    s_iptr[k] = (int)(__ldg(a.n2e_ptr + n0 + k) - i_begin);
    s_vptr[k] = (int)(__ldg(a.nbr_ptr + n0 + k) * D2 - v0);
  }
  // everything below reads the producer's emask / workspace
  wait();
  // stage the range's items (plastic ones kept, others -1)
  for (int k = tid; k < nitems; k += nthr) {
    const int32_t it = __ldg(a.n2e + i_begin + k);
    s_item[k] = __ldcg(a.emask + it / NP) ? it : -1;
  }
  sync();
  const bool used_bar = a1 > a0 && !zero_base;
  if (used_bar) mbar_wait(s_bar, parity);
  // Items are taken UB at a time: every lane first issues the loads of all
  // UB items (slot byte + workspace value), then applies the adds in item
  // order, so a node costs one memory round trip per UB items instead of
  // one per item (the add order, hence the bits, is unchanged).
  constexpr int KP = (NP * D2 + 31) / 32;
  constexpr int UB = KP == 1 ? 4 : 1;  // 3D: wider rows already give ILP; registers matter more
  for (int ln = warp; ln < nloc; ln += NTHREADS / 32) {
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
            // FRESH: a weak (L1-cacheable, coherent after the acquire) load,
            // never the read-only .nc path
            v[u][kk] = FRESH ? rec[src] : __ldg(rec + src);
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
  }
  fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
  sync();
  if (tid == 0 && v1 > v0) {
    const int64_t s0 = (v0 + 1) & ~int64_t(1), s1 = v1 & ~int64_t(1);
    if (v0 & 1) a.out[v0] = img[0];
    if ((v1 & 1) && v1 - 1 >= s0) a.out[v1 - 1] = img[v1 - 1 - v0];
    if (s1 > s0) {
      if (WARP) {
        tma_store_1d(a.out + s0, img + (s0 - v0), (unsigned)((s1 - s0) * 8));
        tma_store_wait_read();
      } else if (HINT)
        tma_store_1d_sync_hint(a.out + s0, img + (s0 - v0), (unsigned)((s1 - s0) * 8), l2_evict_first());
      else
        tma_store_1d_sync(a.out + s0, img + (s0 - v0), (unsigned)((s1 - s0) * 8));
    }
  }
  return used_bar;
}

}  // namespace epfem_gpu
