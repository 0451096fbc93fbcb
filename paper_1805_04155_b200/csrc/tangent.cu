// K2 + K6: the per-iteration tangent  K = K_elast + sum_{plastic q} B_q^T w_q (D_q - C_q) B_q
// (assembly.cpp:262-289), as two deterministic passes without atomics.
//
// Pass 1, k_elem_delta (element-centric, one thread per symmetric node-pair
// block (a <= b) of an element): for every element with at least one plastic
// integration point, the per-point work is done ONCE per (element, point):
// dphi_p = J^-1 ghat_p for all nodes, Dw = w (D - C) (reduced to the plane-
// strain rows in 2D), T_a = B_a^T Dw for all nodes, then each thread adds
// T_a B_b to its block in registers.  The symmetric element matrix dK_e
// (NB = NP(NP+1)/2 blocks of dim x dim) goes to a per-element workspace
// record, and the element's plastic-point bitmask to emask[e].  Elements with
// no plastic point write only their (zero) mask.
//
// Pass 2, k_row_gather (row-centric, one warp per node a = the contiguous
// value segment of its dim rows): the warp reads emask of the node's items;
// with none plastic it copies K_elast[seg] -> K[seg] bitwise; otherwise it
// adds every plastic item's block row a of dK_e (transposed blocks for b < a)
// into a shared-memory image of the segment at the cached slots, then streams
// K[seg] = K_elast[seg] + image.
#include "kernels.cuh"

namespace epfem_gpu {

namespace {

template <int NP>
__host__ __device__ constexpr int blk_index(int a, int b) {  // a <= b
  return a * (2 * NP - a + 1) / 2 + (b - a);
}

__device__ __forceinline__ double t_iota(int i) { return i < 3 ? 1.0 : 0.0; }
__device__ __forceinline__ double t_dev(int i, int j) {
  return ((i == j) ? (i < 3 ? 1.0 : 0.5) : 0.0) - t_iota(i) * t_iota(j) / 3.0;
}
__device__ __forceinline__ double t_cel(double K, double G, int i, int j) {
  return K * (t_iota(i) * t_iota(j)) + 2.0 * G * t_dev(i, j);
}

constexpr int kDeltaThreads = 256;

template <int DIM, int NP, int NQ, int MODE>
__global__ void __launch_bounds__(kDeltaThreads) k_elem_delta(GatherArgs a) {
  constexpr int NS = DIM == 3 ? 6 : 3;
  constexpr int NSP = NS * (NS + 1) / 2;
  constexpr int NB = NP * (NP + 1) / 2;
  constexpr int EPB = NB >= kDeltaThreads ? 1 : kDeltaThreads / NB;  // elements per CTA
  constexpr int R[6] = {0, 1, DIM == 3 ? 2 : 3, 3, 4, 5};          // assembly rows
  __shared__ double s_dphi[EPB][NP][DIM];
  __shared__ double s_dw[EPB][NSP];
  __shared__ double s_T[EPB][NP][DIM][NS];
  __shared__ double s_ghat[NQ * NP * DIM];
  __shared__ unsigned s_mask[EPB];
  __shared__ int s_any;

  const int tid = threadIdx.x;
  const int le = tid / NB;           // local element
  const int t = tid - le * NB;       // block index inside the element
  const int64_t e = (int64_t)blockIdx.x * EPB + le;
  const bool live = le < EPB && e < a.n_elements;

  for (int k = tid; k < NQ * NP * DIM; k += blockDim.x) s_ghat[k] = __ldg(a.gradhat + k);
  if (tid < EPB) s_mask[tid] = 0u;
  if (tid == 0) s_any = 0;
  __syncthreads();
  // plastic-point bitmask of each element
  for (int k = tid; k < EPB * NQ; k += blockDim.x) {
    const int l = k / NQ, q = k - l * NQ;
    const int64_t el = (int64_t)blockIdx.x * EPB + l;
    if (el < a.n_elements && (__ldg(a.flags + el * NQ + q) & 1)) {
      atomicOr(&s_mask[l], 1u << q);
      s_any = 1;
    }
  }
  __syncthreads();
  if (tid < EPB) {
    const int64_t el = (int64_t)blockIdx.x * EPB + tid;
    if (el < a.n_elements) a.emask[el] = s_mask[tid];
  }
  if (!s_any) return;  // CTA-uniform

  // this thread's block (pa, pb), pa <= pb
  int pa = 0, pb = 0;
  {
    int r = t;
    while (pa < NP && r >= NP - pa) {
      r -= NP - pa;
      ++pa;
    }
    pb = pa + r;
  }
  const unsigned mask = live ? s_mask[le] : 0u;
  double blk[DIM][DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int j = 0; j < DIM; ++j) blk[i][j] = 0.0;

  const double Gu = a.shear_u, Ku = a.bulk_u;
  for (int q = 0; q < NQ; ++q) {
    const bool on = (mask >> q) & 1u;
    const int64_t m = e * NQ + q;
    // phase 1: geometry and effective material block
    if (on) {
      if (t < NP) {
        const double* Ji = a.inv + m * DIM * DIM;
        double J[DIM * DIM];
#pragma unroll
        for (int k = 0; k < DIM * DIM; ++k) J[k] = __ldg(Ji + k);
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < DIM; ++j) s += J[j * DIM + i] * s_ghat[(q * NP + t) * DIM + j];
          s_dphi[le][t][i] = s;
        }
      }
      for (int k = t; k < NSP; k += NB) {
        // k -> (r, c), r <= c, row-major upper triangle of the NS x NS block
        int r = 0, rem = k;
        while (rem >= NS - r) {
          rem -= NS - r;
          ++r;
        }
        const int c = r + rem;
        const int ri = R[r], ci = R[c];
        const double Gm = a.shear ? __ldg(a.shear + m) : Gu;
        const double Km = a.bulk ? __ldg(a.bulk + m) : Ku;
        double d;
        if (MODE == G_TANGENT_PACKED) d = __ldg(a.D + m * EPFEM_D_STRIDE + pk_index_rt(ri, ci));
        else d = __ldg(a.D + m * 36 + ci * 6 + ri);
        s_dw[le][k] = __ldg(a.weight + m) * (d - t_cel(Km, Gm, ri, ci));
      }
    }
    __syncthreads();
    // phase 2: T_p = B_p^T Dw for every node p
    if (on) {
      for (int k = t; k < NP * DIM; k += NB) {
        const int p = k / DIM, i = k - p * DIM;
        const double* g = s_dphi[le][p];
        auto Dw = [&](int r, int c) {
          const int lo = r < c ? r : c, hi = r < c ? c : r;
          return s_dw[le][lo * NS - lo * (lo - 1) / 2 + (hi - lo)];
        };
#pragma unroll
        for (int c = 0; c < NS; ++c) {
          double v;
          if constexpr (DIM == 3) {
            // B rows e11,e22,e33,2e12,2e23,2e31 (assembly.cpp:162-171)
            if (i == 0) v = g[0] * Dw(0, c) + g[1] * Dw(3, c) + g[2] * Dw(5, c);
            else if (i == 1) v = g[1] * Dw(1, c) + g[0] * Dw(3, c) + g[2] * Dw(4, c);
            else v = g[2] * Dw(2, c) + g[1] * Dw(4, c) + g[0] * Dw(5, c);
          } else {
            // rows e11, e22, 2e12 (assembly.cpp:173-176)
            if (i == 0) v = g[0] * Dw(0, c) + g[1] * Dw(2, c);
            else v = g[1] * Dw(1, c) + g[0] * Dw(2, c);
          }
          s_T[le][p][i][c] = v;
        }
      }
    }
    __syncthreads();
    // phase 3: block (pa, pb) += T_pa B_pb
    if (on && live) {
      const double* h = s_dphi[le][pb];
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        const double* T = s_T[le][pa][i];
        if constexpr (DIM == 3) {
          blk[i][0] += T[0] * h[0] + T[3] * h[1] + T[5] * h[2];
          blk[i][1] += T[1] * h[1] + T[3] * h[0] + T[4] * h[2];
          blk[i][2] += T[2] * h[2] + T[4] * h[1] + T[5] * h[0];
        } else {
          blk[i][0] += T[0] * h[0] + T[2] * h[1];
          blk[i][1] += T[1] * h[1] + T[2] * h[0];
        }
      }
    }
    // the next iteration's phase 1 rewrites s_dphi/s_dw only after this
    // barrier, so phase 3 readers are done
    __syncthreads();
  }
  if (live && mask) {
    double* out = a.scratch + ((size_t)e * NB + t) * DIM * DIM;
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) out[i * DIM + j] = blk[i][j];
  }
}

constexpr int kRowWarps = 8;

template <int DIM, int NP, int NQ>
__global__ void __launch_bounds__(32 * kRowWarps) k_row_gather(GatherArgs a) {
  extern __shared__ double smem[];
  constexpr int NB = NP * (NP + 1) / 2;
  constexpr int D2 = DIM * DIM;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* acc = smem + (size_t)wib * a.max_seg;
  const int64_t node = (int64_t)blockIdx.x * kRowWarps + wib;
  if (node >= a.n_nodes) return;

  const int64_t i0 = __ldg(a.n2e_ptr + node);
  const int nit = (int)(__ldg(a.n2e_ptr + node + 1) - i0);
  const int64_t nb0 = __ldg(a.nbr_ptr + node);
  const int nn = (int)(__ldg(a.nbr_ptr + node + 1) - nb0);
  const int seg_len = D2 * nn;
  const int64_t sb = nb0 * D2;
  const double* __restrict__ base = a.base + sb;
  double* __restrict__ out = a.out + sb;

  // which of the node's items (element, local index) carry plastic points
  unsigned plastic_items = 0u;
  bool any_plastic = false;
  for (int c = 0; c < nit; c += 32) {
    bool pl = false;
    if (c + lane < nit) {
      const int32_t item = __ldg(a.n2e + i0 + c + lane);
      pl = __ldg(a.emask + item / NP) != 0u;
    }
    const unsigned bal = __ballot_sync(0xffffffffu, pl);
    if (c == 0) plastic_items = bal;
    any_plastic |= bal != 0u;
  }
  if (!any_plastic) {
    for (int k = lane; k < seg_len; k += 32) out[k] = __ldg(base + k);
    return;
  }
  const bool full_scan = nit > 32;  // rare high-valence node: re-read the masks
  for (int k = lane; k < seg_len; k += 32) acc[k] = 0.0;
  __syncwarp();
  const int row_len = DIM * nn;
  for (int it = 0; it < nit; ++it) {
    if (!full_scan && !((plastic_items >> it) & 1u)) continue;
    const int32_t item = __ldg(a.n2e + i0 + it);
    const int64_t e = item / NP;
    if (full_scan && __ldg(a.emask + e) == 0u) continue;
    const int pa = item - (int)e * NP;
    const double* rec = a.scratch + (size_t)e * NB * D2;
    for (int k = lane; k < NP * D2; k += 32) {
      const int pb = k / D2, ij = k - pb * D2;
      const int i = ij / DIM, j = ij - i * DIM;
      const int slot = __ldg(a.slot + (int64_t)item * NP + pb);
      double v;
      if (pa <= pb) v = __ldg(rec + blk_index<NP>(pa, pb) * D2 + i * DIM + j);
      else v = __ldg(rec + blk_index<NP>(pb, pa) * D2 + j * DIM + i);
      acc[i * row_len + slot * DIM + j] += v;
    }
    __syncwarp();
  }
  for (int k = lane; k < seg_len; k += 32) out[k] = __ldg(base + k) + acc[k];
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

int launch_tangent(int family, int dim, int mode, const GatherArgs& a, cudaStream_t st) {
  if (a.n_nodes == 0) return 0;
  int rc = 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    constexpr int NB = NP * (NP + 1) / 2;
    constexpr int EPB = NB >= kDeltaThreads ? 1 : kDeltaThreads / NB;
    constexpr int threads = ((EPB * NB + 31) / 32) * 32;
    if (a.n_elements > 0) {
      const int64_t blocks = (a.n_elements + EPB - 1) / EPB;
      if (mode == G_TANGENT_PACKED)
        k_elem_delta<DIM, NP, NQ, G_TANGENT_PACKED><<<(unsigned)blocks, threads, 0, st>>>(a);
      else
        k_elem_delta<DIM, NP, NQ, G_TANGENT_DS36><<<(unsigned)blocks, threads, 0, st>>>(a);
    }
    const int64_t rblocks = (a.n_nodes + kRowWarps - 1) / kRowWarps;
    const size_t smem = sizeof(double) * (size_t)a.max_seg * kRowWarps;
    auto kern = k_row_gather<DIM, NP, NQ>;
    if (smem > 48 * 1024) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) { rc = cuda_fail(e, "cudaFuncSetAttribute"); return; }
    }
    kern<<<(unsigned)rblocks, 32 * kRowWarps, smem, st>>>(a);
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  if (rc) return rc;
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace epfem_gpu
