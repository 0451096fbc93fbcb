// K2 + K6: the per-iteration tangent  K = K_elast + sum_{plastic q} B_q^T w_q (D_q - C_q) B_q
// (assembly.cpp:262-289), as two deterministic passes without atomics.
//
// Pass 1, k_elem_delta (element-centric; one thread per symmetric node-pair
// block (a <= b) of an element, several elements per CTA).  For every element
// with at least one plastic integration point the per-point work is done ONCE
// per (element, point) and shared through shared memory:
//     dphi_p = J^-1 ghat_p            (all nodes)
//     Dw     = w (D - C)              (plane-strain rows {0,1,3} in 2D)
//     T_p    = B_p^T Dw               (all nodes)
//     block(a,b) += T_a B_b           (each thread, in registers)
// The symmetric element matrix dK_e (NB = NP(NP+1)/2 blocks of dim x dim)
// goes to a per-element workspace record and the element's plastic-point
// bitmask to emask[e].  Shared buffers are double-buffered on the point
// index, so a point costs two CTA barriers.
//
// Pass 2, k_row_stream (row-centric; one CTA per range of NPC consecutive
// nodes = one contiguous value range of K, because a node's dim rows are
// contiguous and nodes are numbered in row order).  The CTA streams
// K_elast[range] into a shared-memory image, each warp adds the plastic
// items' block rows of dK_e for its nodes at the cached slots (one warp per
// node: no two writers per row), and the image is streamed out to K[range].
// Rows without plastic contributions are copied bitwise.
#include "kernels.cuh"

namespace epfem_gpu {

namespace {

template <int NP>
__host__ __device__ constexpr int blk_index(int a, int b) {  // a <= b
  return a * (2 * NP - a + 1) / 2 + (b - a);
}

// Voigt operators as constant tables for runtime indices (voigt.hpp:49-74).
static __constant__ double c_vol[36] = {1, 1, 1, 0, 0, 0, 1, 1, 1, 0, 0, 0, 1, 1, 1, 0, 0, 0,
                                        0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
static __constant__ double c_dev[36] = {
    1.0 - 1.0 / 3.0, -1.0 / 3.0, -1.0 / 3.0, 0, 0, 0, -1.0 / 3.0, 1.0 - 1.0 / 3.0, -1.0 / 3.0, 0,
    0, 0, -1.0 / 3.0, -1.0 / 3.0, 1.0 - 1.0 / 3.0, 0, 0, 0, 0, 0, 0, 0.5, 0, 0, 0, 0, 0, 0, 0.5,
    0, 0, 0, 0, 0, 0, 0.5};

constexpr int kDeltaThreads = 256;

template <int DIM, int NP, int NQ, int MODE>
__global__ void __launch_bounds__(kDeltaThreads) k_elem_delta(GatherArgs a) {
  constexpr int NS = DIM == 3 ? 6 : 3;
  constexpr int NB = NP * (NP + 1) / 2;
  constexpr int EPB = NB >= kDeltaThreads ? 1 : kDeltaThreads / NB;  // elements per CTA
  static_assert(NB >= NP + NS, "phase-1 thread mapping");
  __shared__ double s_dphi[2][EPB][NP][DIM];
  __shared__ double s_dw[2][EPB][NS][NS];
  __shared__ double s_T[2][EPB][NP][DIM][NS];
  __shared__ double s_ghat[NQ * NP * DIM];
  __shared__ unsigned s_mask[EPB];
  __shared__ unsigned s_union;

  const int tid = threadIdx.x;
  const int le = tid / NB;        // local element
  const int t = tid - le * NB;    // block index inside the element
  const int64_t e = (int64_t)blockIdx.x * EPB + le;
  const bool live = le < EPB && e < a.n_elements;

  if (tid < EPB) s_mask[tid] = 0u;
  if (tid == 0) s_union = 0u;
  __syncthreads();
  for (int k = tid; k < EPB * NQ; k += blockDim.x) {
    const int l = k / NQ, q = k - l * NQ;
    const int64_t el = (int64_t)blockIdx.x * EPB + l;
    if (el < a.n_elements && (__ldg(a.flags + el * NQ + q) & 1)) {
      atomicOr(&s_mask[l], 1u << q);
      atomicOr(&s_union, 1u << q);
    }
  }
  for (int k = tid; k < NQ * NP * DIM; k += blockDim.x) s_ghat[k] = __ldg(a.gradhat + k);
  __syncthreads();
  if (tid < EPB) {
    const int64_t el = (int64_t)blockIdx.x * EPB + tid;
    if (el < a.n_elements) a.emask[el] = s_mask[tid];
  }
  unsigned todo = s_union;  // CTA-uniform
  if (!todo) return;

  int pa = 0, r = t;  // this thread's block (pa, pb), pa <= pb
  while (pa < NP - 1 && r >= NP - pa) {
    r -= NP - pa;
    ++pa;
  }
  const int pb = pa + r;
  const unsigned mask = live ? s_mask[le] : 0u;
  const bool uniform_c = a.shear == nullptr && a.bulk == nullptr;
  double blk[DIM][DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int j = 0; j < DIM; ++j) blk[i][j] = 0.0;

  int buf = 0;
  while (todo) {
    const int q = __ffs(todo) - 1;
    todo &= todo - 1u;
    const bool on = (mask >> q) & 1u;
    const int64_t m = e * NQ + q;
    // phase 1: geometry (threads 0..NP-1) and one row of Dw per thread (NP..NP+NS-1)
    if (on) {
      if (t < NP) {
        const double* Ji = a.inv + m * DIM * DIM;
        double J[DIM * DIM];
#pragma unroll
        for (int k = 0; k < DIM * DIM; ++k) J[k] = __ldg(Ji + k);
        const double* g = s_ghat + (q * NP + t) * DIM;
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < DIM; ++j) s += J[j * DIM + i] * g[j];
          s_dphi[buf][le][t][i] = s;
        }
      } else if (t < NP + NS) {
        const int rr = t - NP;
        const int ri = (DIM == 2 && rr == 2) ? 3 : rr;  // assembly row -> Voigt row
        const double w = __ldg(a.weight + m);
        double G2 = 0.0, Km = 0.0;
        if (!uniform_c) {
          G2 = 2.0 * (a.shear ? __ldg(a.shear + m) : a.shear_u);
          Km = a.bulk ? __ldg(a.bulk + m) : a.bulk_u;
        }
#pragma unroll
        for (int c = 0; c < NS; ++c) {
          const int ci = (DIM == 2 && c == 2) ? 3 : c;
          const double d = MODE == G_TANGENT_PACKED
                               ? __ldg(a.D + m * EPFEM_D_STRIDE + pk_index_rt(ri, ci))
                               : __ldg(a.D + m * 36 + ci * 6 + ri);
          const double cel = uniform_c ? a.Cu[pk_index_rt(ri, ci)]
                                       : Km * c_vol[ri * 6 + ci] + G2 * c_dev[ri * 6 + ci];
          s_dw[buf][le][rr][c] = w * (d - cel);
        }
      }
    }
    __syncthreads();
    // phase 2: T_p = B_p^T Dw, thread <-> (p, column c)
    if (on) {
      for (int k = t; k < NP * NS; k += NB) {
        const int p = k / NS, c = k - p * NS;
        const double* g = s_dphi[buf][le][p];
        double(*Dw)[NS] = s_dw[buf][le];
        if constexpr (DIM == 3) {
          // B rows e11,e22,e33,2e12,2e23,2e31 (assembly.cpp:162-171)
          s_T[buf][le][p][0][c] = g[0] * Dw[0][c] + g[1] * Dw[3][c] + g[2] * Dw[5][c];
          s_T[buf][le][p][1][c] = g[1] * Dw[1][c] + g[0] * Dw[3][c] + g[2] * Dw[4][c];
          s_T[buf][le][p][2][c] = g[2] * Dw[2][c] + g[1] * Dw[4][c] + g[0] * Dw[5][c];
        } else {
          // rows e11, e22, 2e12 (assembly.cpp:173-176)
          s_T[buf][le][p][0][c] = g[0] * Dw[0][c] + g[1] * Dw[2][c];
          s_T[buf][le][p][1][c] = g[1] * Dw[1][c] + g[0] * Dw[2][c];
        }
      }
    }
    __syncthreads();
    // phase 3: block (pa, pb) += T_pa B_pb.  The next point writes the other
    // buffer, so no barrier is needed before it.
    if (on && live) {
      const double* h = s_dphi[buf][le][pb];
      const double h0 = h[0], h1 = h[1], h2 = DIM == 3 ? h[DIM - 1] : 0.0;
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        const double* T = s_T[buf][le][pa][i];
        if constexpr (DIM == 3) {
          blk[i][0] += T[0] * h0 + T[3] * h1 + T[5] * h2;
          blk[i][1] += T[1] * h1 + T[3] * h0 + T[4] * h2;
          blk[i][DIM - 1] += T[2] * h2 + T[4] * h1 + T[5] * h0;
        } else {
          blk[i][0] += T[0] * h0 + T[2] * h1;
          blk[i][1] += T[1] * h1 + T[2] * h0;
        }
      }
    }
    buf ^= 1;
  }
  if (live && mask) {
    double* out = a.scratch + ((size_t)e * NB + t) * DIM * DIM;
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) out[i * DIM + j] = blk[i][j];
  }
}

// Pass 1 for small elements (NP <= 8): one lane per (element, node a).  A
// group of GW = pow2ceil(NP) lanes holds one element; each lane forms its own
// dphi_a, receives the others by shuffles, builds Dw and T_a = B_a^T Dw in
// registers and accumulates the whole block row a.  It writes the blocks
// (a, b >= a) of the symmetric record.  No barriers, only the element's own
// plastic points are visited (warp-uniform loop over the union of the groups'
// masks).
template <int NP>
struct LaneGroup {
  static constexpr int GW = NP <= 2 ? 2 : NP <= 4 ? 4 : 8;
};

template <int DIM, int NP, int NQ, int MODE>
__global__ void __launch_bounds__(256) k_elem_delta_lane(GatherArgs a) {
  constexpr int NS = DIM == 3 ? 6 : 3;
  constexpr int GW = LaneGroup<NP>::GW;
  constexpr int EPW = 32 / GW;
  constexpr int D2 = DIM * DIM;
  constexpr int NB = NP * (NP + 1) / 2;
  constexpr int RV[3] = {0, 1, 3};  // 2D assembly rows -> Voigt rows
  __shared__ double s_ghat[NQ * NP * DIM];
  for (int k = threadIdx.x; k < NQ * NP * DIM; k += blockDim.x) s_ghat[k] = __ldg(a.gradhat + k);
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const int g = lane / GW, p = lane - g * GW;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t e = warp * EPW + g;
  const bool elem_ok = e < a.n_elements;
  const bool node_ok = elem_ok && p < NP;
  const unsigned full = 0xffffffffu;
  const unsigned gmask = (GW == 32 ? full : ((1u << GW) - 1u));

  // plastic-point bitmask of this lane's element
  unsigned mask = 0u;
#pragma unroll
  for (int q0 = 0; q0 < NQ; q0 += GW) {
    const bool f = elem_ok && q0 + p < NQ && (__ldg(a.flags + e * NQ + q0 + p) & 1);
    const unsigned b = __ballot_sync(full, f);
    mask |= ((b >> (g * GW)) & gmask) << q0;
  }
  if (elem_ok && p == 0) a.emask[e] = mask;
  unsigned todo = __reduce_or_sync(full, mask);
  if (!todo) return;

  const bool uniform_c = a.shear == nullptr && a.bulk == nullptr;
  double blk[NP][DIM][DIM];
#pragma unroll
  for (int b = 0; b < NP; ++b)
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) blk[b][i][j] = 0.0;

  while (todo) {
    const int q = __ffs(todo) - 1;
    todo &= todo - 1u;
    const bool on = node_ok && ((mask >> q) & 1u);
    const int64_t m = e * NQ + q;
    double gself[DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i) gself[i] = 0.0;
    double w = 0.0;
    if (on) {
      const double* Ji = a.inv + m * D2;
      const double* gh = s_ghat + (q * NP + p) * DIM;
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < DIM; ++j) s += __ldg(Ji + j * DIM + i) * gh[j];
        gself[i] = s;
      }
      w = __ldg(a.weight + m);
    }
    // Dw = w (D - C) on the assembly rows, then T_a = B_a^T Dw
    double T[DIM][NS];
    if (on) {
      double Dw[NS][NS];
      double G2 = 0.0, Km = 0.0;
      if (!uniform_c) {
        G2 = 2.0 * (a.shear ? __ldg(a.shear + m) : a.shear_u);
        Km = a.bulk ? __ldg(a.bulk + m) : a.bulk_u;
      }
#pragma unroll
      for (int r = 0; r < NS; ++r)
#pragma unroll
        for (int c = r; c < NS; ++c) {
          const int ri = DIM == 3 ? r : RV[r], ci = DIM == 3 ? c : RV[c];
          const double d = MODE == G_TANGENT_PACKED
                               ? __ldg(a.D + m * EPFEM_D_STRIDE + pk_index(ri, ci))
                               : __ldg(a.D + m * 36 + ci * 6 + ri);
          const double vol = (ri < 3 && ci < 3) ? 1.0 : 0.0;
          const double dev = ((ri == ci) ? (ri < 3 ? 1.0 : 0.5) : 0.0) - vol / 3.0;
          const double cel = uniform_c ? a.Cu[pk_index(ri, ci)] : Km * vol + G2 * dev;
          Dw[r][c] = Dw[c][r] = w * (d - cel);
        }
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        if constexpr (DIM == 3) {
          T[0][c] = gself[0] * Dw[0][c] + gself[1] * Dw[3][c] + gself[2] * Dw[5][c];
          T[1][c] = gself[1] * Dw[1][c] + gself[0] * Dw[3][c] + gself[2] * Dw[4][c];
          T[DIM - 1][c] = gself[2] * Dw[2][c] + gself[1] * Dw[4][c] + gself[0] * Dw[5][c];
        } else {
          T[0][c] = gself[0] * Dw[0][c] + gself[1] * Dw[2][c];
          T[1][c] = gself[1] * Dw[1][c] + gself[0] * Dw[2][c];
        }
      }
    }
    // block row: blk[b] += T_a B_b with dphi_b shuffled from lane b
#pragma unroll
    for (int b = 0; b < NP; ++b) {
      double h[DIM];
#pragma unroll
      for (int i = 0; i < DIM; ++i) h[i] = __shfl_sync(full, gself[i], g * GW + b);
      if (on) {
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          if constexpr (DIM == 3) {
            blk[b][i][0] += T[i][0] * h[0] + T[i][3] * h[1] + T[i][5] * h[2];
            blk[b][i][1] += T[i][1] * h[1] + T[i][3] * h[0] + T[i][4] * h[2];
            blk[b][i][DIM - 1] += T[i][2] * h[2] + T[i][4] * h[1] + T[i][5] * h[0];
          } else {
            blk[b][i][0] += T[i][0] * h[0] + T[i][2] * h[1];
            blk[b][i][1] += T[i][1] * h[1] + T[i][2] * h[0];
          }
        }
      }
    }
  }
  if (node_ok && mask) {
    double* rec = a.scratch + (size_t)e * NB * D2;
#pragma unroll
    for (int b = 0; b < NP; ++b) {
      if (b >= p) {
        double* o = rec + blk_index<NP>(p, b) * D2;
#pragma unroll
        for (int i = 0; i < DIM; ++i)
#pragma unroll
          for (int j = 0; j < DIM; ++j) o[i * DIM + j] = blk[b][i][j];
      }
    }
  }
}

// Pass 1, staged form (default).  Phase 1: one thread per (element, point)
// of the CTA's elements issues that point's loads (J^-1, w, packed D) with no
// dependence on any other point, and stages dphi_p for all nodes and the
// packed Dw = w (D - C) in shared memory.  Phase 2: one thread per (element,
// node a, block chunk) loops over the element's plastic points reading only
// shared memory: T_a = B_a^T Dw, block(a, b) += T_a B_b for the b of its
// chunk, in registers.  Two CTA barriers in total.
template <int DIM, int NP>
struct StagedCfg {
  static constexpr int BCH = DIM == 2 ? 1 : (NP <= 4 ? 1 : (NP <= 10 ? 2 : 4));
  static constexpr int CS = (NP + BCH - 1) / BCH;  // blocks per chunk
};

template <int DIM, int NP, int NQ, int MODE>
__global__ void __launch_bounds__(256) k_elem_delta_staged(GatherArgs a) {
  constexpr int NS = DIM == 3 ? 6 : 3;
  constexpr int NSP = NS * (NS + 1) / 2;
  constexpr int D2 = DIM * DIM;
  constexpr int NB = NP * (NP + 1) / 2;
  constexpr int REC = NP * DIM + NSP;
  constexpr int BCH = StagedCfg<DIM, NP>::BCH, CS = StagedCfg<DIM, NP>::CS;
  constexpr int BUDGET = 5120;  // doubles of staged data per CTA (40 KB)
  constexpr int E1 = 256 / (NP * BCH), E2 = BUDGET / (NQ * REC);
  constexpr int EPB = (E1 < E2 ? E1 : E2) > 0 ? (E1 < E2 ? E1 : E2) : 1;
  constexpr int RV[6] = {0, 1, DIM == 3 ? 2 : 3, 3, 4, 5};  // assembly row -> Voigt row
  __shared__ double s_st[EPB][NQ][REC];
  __shared__ unsigned s_mask[EPB];

  const int tid = threadIdx.x;
  const int64_t e0 = (int64_t)blockIdx.x * EPB;
  if (tid < EPB) s_mask[tid] = 0u;
  __syncthreads();
  const bool uniform_c = a.shear == nullptr && a.bulk == nullptr;
  // phase 1
  for (int k = tid; k < EPB * NQ; k += blockDim.x) {
    const int le = k / NQ, q = k - le * NQ;
    const int64_t e = e0 + le;
    if (e >= a.n_elements) continue;
    const int64_t m = e * NQ + q;
    if (!(__ldg(a.flags + m) & 1)) continue;
    atomicOr(&s_mask[le], 1u << q);
    double J[D2];
#pragma unroll
    for (int t = 0; t < D2; ++t) J[t] = __ldg(a.inv + m * D2 + t);
    const double w = __ldg(a.weight + m);
    double dv[NSP];
    {
      int k2 = 0;
#pragma unroll
      for (int r = 0; r < NS; ++r)
#pragma unroll
        for (int c = r; c < NS; ++c, ++k2) {
          const int ri = RV[r], ci = RV[c];
          dv[k2] = MODE == G_TANGENT_PACKED ? __ldg(a.D + m * EPFEM_D_STRIDE + pk_index(ri, ci))
                                            : __ldg(a.D + m * 36 + ci * 6 + ri);
        }
    }
    double* st = s_st[le][q];
#pragma unroll 4
    for (int p = 0; p < NP; ++p) {
      const double* gh = a.gradhat + (q * NP + p) * DIM;
      double g[DIM];
#pragma unroll
      for (int j = 0; j < DIM; ++j) g[j] = __ldg(gh + j);
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < DIM; ++j) s += J[j * DIM + i] * g[j];
        st[p * DIM + i] = s;
      }
    }
    double G2 = 0.0, Km = 0.0;
    if (!uniform_c) {
      G2 = 2.0 * (a.shear ? __ldg(a.shear + m) : a.shear_u);
      Km = a.bulk ? __ldg(a.bulk + m) : a.bulk_u;
    }
    int k2 = 0;
#pragma unroll
    for (int r = 0; r < NS; ++r)
#pragma unroll
      for (int c = r; c < NS; ++c, ++k2) {
        const int ri = RV[r], ci = RV[c];
        const double vol = (ri < 3 && ci < 3) ? 1.0 : 0.0;
        const double dev = ((ri == ci) ? (ri < 3 ? 1.0 : 0.5) : 0.0) - vol / 3.0;
        const double cel = uniform_c ? a.Cu[pk_index(ri, ci)] : Km * vol + G2 * dev;
        st[NP * DIM + k2] = w * (dv[k2] - cel);
      }
  }
  __syncthreads();
  if (tid < EPB && e0 + tid < a.n_elements) a.emask[e0 + tid] = s_mask[tid];
  // phase 2
  if (tid >= EPB * NP * BCH) return;
  const int le = tid / (NP * BCH);
  const int rr = tid - le * (NP * BCH);
  const int pa = rr / BCH, ch = rr - pa * BCH;
  const int b0 = ch * CS;
  const int64_t e = e0 + le;
  if (e >= a.n_elements) return;
  unsigned mask = s_mask[le];
  if (!mask) return;
  double blk[CS][DIM][DIM];
#pragma unroll
  for (int b = 0; b < CS; ++b)
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) blk[b][i][j] = 0.0;
  while (mask) {
    const int q = __ffs(mask) - 1;
    mask &= mask - 1u;
    const double* st = s_st[le][q];
    const double* dw = st + NP * DIM;
    auto Dw = [&](int r, int c) {  // compile-time indices after unrolling
      const int lo = r < c ? r : c, hi = r < c ? c : r;
      return dw[lo * NS - lo * (lo - 1) / 2 + (hi - lo)];
    };
    double ga[DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i) ga[i] = st[pa * DIM + i];
    double T[DIM][NS];
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      if constexpr (DIM == 3) {
        // B rows e11,e22,e33,2e12,2e23,2e31 (assembly.cpp:162-171)
        T[0][c] = ga[0] * Dw(0, c) + ga[1] * Dw(3, c) + ga[2] * Dw(5, c);
        T[1][c] = ga[1] * Dw(1, c) + ga[0] * Dw(3, c) + ga[2] * Dw(4, c);
        T[DIM - 1][c] = ga[2] * Dw(2, c) + ga[1] * Dw(4, c) + ga[0] * Dw(5, c);
      } else {
        // rows e11, e22, 2e12 (assembly.cpp:173-176)
        T[0][c] = ga[0] * Dw(0, c) + ga[1] * Dw(2, c);
        T[1][c] = ga[1] * Dw(1, c) + ga[0] * Dw(2, c);
      }
    }
#pragma unroll
    for (int bb = 0; bb < CS; ++bb) {
      const int b = b0 + bb;
      if (b >= NP) break;
      const double* h = st + b * DIM;
      const double h0 = h[0], h1 = h[1], h2 = DIM == 3 ? h[DIM - 1] : 0.0;
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        if constexpr (DIM == 3) {
          blk[bb][i][0] += T[i][0] * h0 + T[i][3] * h1 + T[i][5] * h2;
          blk[bb][i][1] += T[i][1] * h1 + T[i][3] * h0 + T[i][4] * h2;
          blk[bb][i][DIM - 1] += T[i][2] * h2 + T[i][4] * h1 + T[i][5] * h0;
        } else {
          blk[bb][i][0] += T[i][0] * h0 + T[i][2] * h1;
          blk[bb][i][1] += T[i][1] * h1 + T[i][2] * h0;
        }
      }
    }
  }
  double* rec = a.scratch + (size_t)e * NB * D2;
#pragma unroll
  for (int bb = 0; bb < CS; ++bb) {
    const int b = b0 + bb;
    if (b >= NP) break;
    if (b >= pa) {
      double* o = rec + blk_index<NP>(pa, b) * D2;
#pragma unroll
      for (int i = 0; i < DIM; ++i)
#pragma unroll
        for (int j = 0; j < DIM; ++j) o[i * DIM + j] = blk[bb][i][j];
    }
  }
}

template <int DIM, int NP, int NQ>
constexpr int staged_epb() {
  constexpr int NS = DIM == 3 ? 6 : 3;
  constexpr int REC = NP * DIM + NS * (NS + 1) / 2;
  constexpr int E1 = 256 / (NP * StagedCfg<DIM, NP>::BCH), E2 = 5120 / (NQ * REC);
  return (E1 < E2 ? E1 : E2) > 0 ? (E1 < E2 ? E1 : E2) : 1;
}

constexpr int kStreamThreads = 256;

// --- TMA bulk-copy / mbarrier helpers (sm_90+ PTX, used on sm_100a) --------
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// global -> shared, completion counted on the mbarrier (bytes % 16 == 0)
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// shared -> global bulk store, then wait for completion
__device__ __forceinline__ void tma_store_1d_sync(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// The K_elast range [v0, v1) is read with ONE TMA bulk copy of the enclosing
// 16-byte-aligned range into the shared image (the K_elast allocation is
// padded by two doubles), overlapped with the item staging; the image goes
// back to K with one TMA bulk store of the aligned interior plus at most two
// edge doubles.
template <int DIM, int NP, int NQ>
__global__ void __launch_bounds__(kStreamThreads) k_row_stream(GatherArgs a, int npc) {
  extern __shared__ __align__(128) double img_raw[];
  __shared__ uint64_t s_bar;
  constexpr int NB = NP * (NP + 1) / 2;
  constexpr int D2 = DIM * DIM;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n0 = (int64_t)blockIdx.x * npc;
  const int64_t n1 = min(n0 + (int64_t)npc, a.n_nodes);
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
  }
  __syncthreads();
  if (tid == 0 && a1 > a0) {
    const unsigned bytes = (unsigned)((a1 - a0) * 8);
    mbar_expect_tx(&s_bar, bytes);
    tma_load_1d(img_raw, a.base + a0, bytes, &s_bar);
  }
  // stage the range's items (plastic ones kept, others -1) and node offsets
  for (int k = tid; k < nitems; k += blockDim.x) {
    const int32_t it = __ldg(a.n2e + i_begin + k);
    s_item[k] = __ldg(a.emask + it / NP) ? it : -1;
  }
  for (int k = tid; k <= nloc; k += blockDim.x) {
    s_iptr[k] = (int)(__ldg(a.n2e_ptr + n0 + k) - i_begin);
    s_vptr[k] = (int)(__ldg(a.nbr_ptr + n0 + k) * D2 - v0);
  }
  __syncthreads();
  if (a1 > a0) mbar_wait(&s_bar, 0);
  for (int ln = warp; ln < nloc; ln += kStreamThreads / 32) {
    const int ib = s_iptr[ln], ie = s_iptr[ln + 1];
    const int row_len = (s_vptr[ln + 1] - s_vptr[ln]) / DIM;
    double* seg = img + s_vptr[ln];
    for (int k0 = ib; k0 < ie; ++k0) {
      const int it = s_item[k0];  // warp-uniform
      if (it < 0) continue;
      const int64_t el = it / NP;
      const int pa = it - (int)el * NP;
      const double* rec = a.scratch + (size_t)el * NB * D2;
      // lane <-> entry (pb, i, j) of block row pa; block (pb, pa) read
      // transposed when pb < pa (branch-free addressing)
      for (int k = lane; k < NP * D2; k += 32) {
        const int pb = k / D2, ij = k - pb * D2;
        const int i = ij / DIM, j = ij - i * DIM;
        const bool up = pa <= pb;
        const int lo = up ? pa : pb, hi = up ? pb : pa;
        const int src = blk_index<NP>(lo, hi) * D2 + (up ? ij : j * DIM + i);
        const int slot = __ldg(a.slot + (int64_t)it * NP + pb);
        seg[i * row_len + slot * DIM + j] += __ldg(rec + src);
      }
      __syncwarp();
    }
  }
  fence_proxy_async_smem();  // generic-proxy smem writes -> visible to the bulk store
  __syncthreads();
  if (tid == 0 && v1 > v0) {
    const int64_t s0 = (v0 + 1) & ~int64_t(1), s1 = v1 & ~int64_t(1);
    if (v0 & 1) a.out[v0] = img[0];
    if ((v1 & 1) && v1 - 1 >= s0) a.out[v1 - 1] = img[v1 - 1 - v0];
    if (s1 > s0) tma_store_1d_sync(a.out + s0, img + (s0 - v0), (unsigned)((s1 - s0) * 8));
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
// widest value range fits the shared-memory budget (two CTAs per SM).
int plan_row_stream(int64_t n_nodes, int dim, const int64_t* nbr_ptr, const int64_t* n2e_ptr,
                    cudaStream_t st, int* npc_out, int* span_out, int* items_out) {
  const int budget = 100 * 1024;  // bytes of dynamic smem: two CTAs per SM
  int* d = nullptr;
  EPFEM_CUDA_TRY(cudaMalloc(&d, 2 * sizeof(int)));
  int npc = 64, h[2] = {0, 0};
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

int launch_tangent(int family, int dim, int mode, const GatherArgs& a, cudaStream_t st) {
  if (a.n_nodes == 0) return 0;
  int rc = 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    constexpr int NB = NP * (NP + 1) / 2;
    constexpr int EPB = NB >= kDeltaThreads ? 1 : kDeltaThreads / NB;
    constexpr int threads = ((EPB * NB + 31) / 32) * 32;
    // pass-1 variant: staged (default), 'lane' or 'cta' via EPFEM_DELTA (A/B runs)
    static const char variant = [] {
      const char* v = getenv("EPFEM_DELTA");
      return v ? v[0] : 's';
    }();
    if (a.n_elements > 0) {
      bool done = false;
      if (variant == 's') {
        constexpr int SEPB = staged_epb<DIM, NP, NQ>();
        const int64_t blocks = (a.n_elements + SEPB - 1) / SEPB;
        if (mode == G_TANGENT_PACKED)
          k_elem_delta_staged<DIM, NP, NQ, G_TANGENT_PACKED><<<(unsigned)blocks, 256, 0, st>>>(a);
        else
          k_elem_delta_staged<DIM, NP, NQ, G_TANGENT_DS36><<<(unsigned)blocks, 256, 0, st>>>(a);
        done = true;
      }
      if constexpr (NP <= 8) {
        if (!done && variant == 'l') {
          constexpr int EPW = 32 / LaneGroup<NP>::GW;
          const int64_t warps = (a.n_elements + EPW - 1) / EPW;
          const int64_t blocks = (warps + 7) / 8;
          if (mode == G_TANGENT_PACKED)
            k_elem_delta_lane<DIM, NP, NQ, G_TANGENT_PACKED><<<(unsigned)blocks, 256, 0, st>>>(a);
          else
            k_elem_delta_lane<DIM, NP, NQ, G_TANGENT_DS36><<<(unsigned)blocks, 256, 0, st>>>(a);
          done = true;
        }
      }
      if (!done) {
        const int64_t blocks = (a.n_elements + EPB - 1) / EPB;
        if (mode == G_TANGENT_PACKED)
          k_elem_delta<DIM, NP, NQ, G_TANGENT_PACKED><<<(unsigned)blocks, threads, 0, st>>>(a);
        else
          k_elem_delta<DIM, NP, NQ, G_TANGENT_DS36><<<(unsigned)blocks, threads, 0, st>>>(a);
      }
    }
    const int64_t rblocks = (a.n_nodes + a.npc - 1) / a.npc;
    const size_t smem = sizeof(double) * ((size_t)a.max_span + 2) +
                        sizeof(int) * ((size_t)a.max_items + 2 * ((size_t)a.npc + 1));
    auto kern = k_row_stream<DIM, NP, NQ>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) { rc = cuda_fail(e, "cudaFuncSetAttribute"); return; }
    }
    kern<<<(unsigned)rblocks, kStreamThreads, smem, st>>>(a, a.npc);
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  if (rc) return rc;
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace epfem_gpu
