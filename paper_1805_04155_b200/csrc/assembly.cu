// Assembly kernels (sm_100a): geometry, CSR pattern + element->slot map
// (one-time), and the per-iteration row-block gather that writes every value
// of K exactly once without atomics.
//
// Layout in HBM (all device-resident, built once per mesh):
//   inv[m*DIM*DIM + j*DIM + i]  J^-1(i,j) at integration point m (column-major
//                               like the reference's JacobianData::inv)
//   weight[m]                   |det J| * w_q
//   n2e_ptr/n2e                 node -> (element, local node) items, sorted
//   nbr_ptr                     node -> sorted neighbour nodes (the CSR column
//                               set shared by the node's dim rows); the dim rows
//                               of node a form ONE contiguous value segment
//                               starting at row_ptr[dim*a] = dim*dim*nbr_ptr[a]
//                               of length dim*dim*(nbr_ptr[a+1]-nbr_ptr[a])
//   slot[(e*NP+pa)*NP+pb]       uint8 position of node elem(pb,e) inside the
//                               column set of node elem(pa,e)
//
// Row-block gather (k_gather): one warp owns node a, i.e. the contiguous
// value segment of its dim rows.  Lanes are split into G = 32/NP groups; a
// group takes one (element, local index pa) item of node a and its lane pb
// accumulates the dim x dim block (a, elem(pb,e)) over the element's
// integration points in registers:
//     block += B_a^T [w (D - C)] B_b      (tangent, plastic points only)
//     block += B_a^T [w C] B_b            (elastic assembly, every point)
// dphi_p = J^-1 ghat_p is formed per lane and dphi_a shuffled from lane pa.
// Blocks are then added into a per-warp shared-memory image of the segment
// (groups take turns, so there are no conflicts), and the warp streams
//     K[seg] = K_elast[seg] + acc
// with coalesced loads/stores.  Nodes with no plastic point in any adjacent
// element skip the arithmetic and copy K_elast bitwise.
#include <cub/cub.cuh>

#include "delta.cuh"

namespace epfem_gpu {

// ---------------------------------------------------------------------------
// Geometry: det J, J^-1, weight (assembly.cpp:20-61, 237-241)
template <int DIM, int NP, int NQ>
__global__ void k_jacobians(int64_t n_e, const int32_t* __restrict__ elem,
                            const double* __restrict__ coord,
                            const double* __restrict__ gradhat,
                            const double* __restrict__ wq, double* __restrict__ det_out,
                            double* __restrict__ inv_out, double* __restrict__ weight,
                            DevErr* err) {
  const int64_t n_int = n_e * NQ;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < n_int;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = m / NQ;
    const int q = (int)(m - e * NQ);
    const int32_t* en = elem + e * NP;
    double* inv = inv_out + m * DIM * DIM;
    const double det = point_geometry<DIM, NP>(
        [&](int p, int j) { return __ldg(coord + (int64_t)DIM * __ldg(en + p) + j); }, gradhat, q, inv);
    if (!(det > 0.0)) raise_dev(err, EPFEM_ERR_DEGENERATE, (unsigned long long)e);
    det_out[m] = det;
    weight[m] = __dmul_rn(fabs(det), __ldg(wq + q));
  }
}

// ---------------------------------------------------------------------------
// Pattern construction (K3) and element->slot map (K4), one time per mesh.

__global__ void k_count_nodes(int64_t n_items, const int32_t* __restrict__ elem,
                              int64_t* __restrict__ cnt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_items;
       t += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + elem[t]), 1ull);
}

__global__ void k_fill_n2e(int64_t n_items, const int32_t* __restrict__ elem,
                           const int64_t* __restrict__ ptr, int64_t* __restrict__ cursor,
                           int32_t* __restrict__ n2e) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_items;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int32_t node = elem[t];
    const unsigned long long pos =
        atomicAdd(reinterpret_cast<unsigned long long*>(cursor + node), 1ull);
    n2e[ptr[node] + (int64_t)pos] = (int32_t)t;  // item = e*NP + p
  }
}

// Deterministic order: items of a node sorted ascending (= element order).
__global__ void k_sort_n2e(int64_t n_nodes, const int64_t* __restrict__ ptr,
                           int32_t* __restrict__ n2e) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n_nodes;
       a += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = ptr[a], e = ptr[a + 1];
    for (int64_t i = b + 1; i < e; ++i) {
      const int32_t v = n2e[i];
      int64_t j = i - 1;
      while (j >= b && n2e[j] > v) {
        n2e[j + 1] = n2e[j];
        --j;
      }
      n2e[j + 1] = v;
    }
  }
}

// All (node_a, node_b) pairs of every element as 64-bit keys.
template <int NP>
__global__ void k_pair_keys(int64_t n_e, const int32_t* __restrict__ elem,
                            uint64_t* __restrict__ keys) {
  const int64_t n = n_e * NP * NP;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / (NP * NP);
    const int r = (int)(t - e * NP * NP);
    const uint32_t a = (uint32_t)elem[e * NP + r / NP], b = (uint32_t)elem[e * NP + r % NP];
    keys[t] = ((uint64_t)a << 32) | b;
  }
}

__global__ void k_count_nbr(int64_t n_unique, const uint64_t* __restrict__ ukeys,
                            int64_t* __restrict__ cnt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_unique;
       t += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(reinterpret_cast<unsigned long long*>(cnt + (ukeys[t] >> 32)), 1ull);
}

__global__ void k_max_nbr(int64_t n_nodes, const int64_t* __restrict__ nbr_ptr, int* out) {
  int m = 0;
  for (int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; a < n_nodes;
       a += (int64_t)gridDim.x * blockDim.x)
    m = max(m, (int)(nbr_ptr[a + 1] - nbr_ptr[a]));
  atomicMax(out, m);
}

// row_ptr and col_idx from the node-level neighbour lists; one thread per
// (node, local row i, neighbour slot s).
__global__ void k_fill_csr(int64_t n_nodes, int dim, const int64_t* __restrict__ nbr_ptr,
                           const uint64_t* __restrict__ ukeys, int64_t* __restrict__ row_ptr,
                           int32_t* __restrict__ col_idx) {
  for (int64_t a = (int64_t)blockIdx.x * blockDim.y + threadIdx.y; a < n_nodes;
       a += (int64_t)gridDim.x * blockDim.y) {
    const int m = (int)(nbr_ptr[a + 1] - nbr_ptr[a]);
    const int64_t base = nbr_ptr[a] * dim * dim;
    if (threadIdx.x < dim) row_ptr[(int64_t)dim * a + threadIdx.x] = base + (int64_t)threadIdx.x * dim * m;
    for (int s = threadIdx.x; s < m; s += blockDim.x) {
      const int32_t b = (int32_t)(ukeys[nbr_ptr[a] + s] & 0xffffffffull);
      for (int i = 0; i < dim; ++i)
        for (int j = 0; j < dim; ++j)
          col_idx[base + (int64_t)i * dim * m + (int64_t)s * dim + j] = dim * b + j;
    }
  }
}

template <int NP>
__global__ void k_slot_map(int64_t n_e, const int32_t* __restrict__ elem,
                           const int64_t* __restrict__ nbr_ptr,
                           const uint64_t* __restrict__ ukeys, uint8_t* __restrict__ slot) {
  const int64_t n = n_e * NP * NP;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / (NP * NP);
    const int r = (int)(t - e * NP * NP);
    const int32_t a = elem[e * NP + r / NP], b = elem[e * NP + r % NP];
    int64_t lo = nbr_ptr[a], hi = nbr_ptr[a + 1] - 1;
    const uint64_t key = ((uint64_t)(uint32_t)a << 32) | (uint32_t)b;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (ukeys[mid] < key) lo = mid + 1;
      else hi = mid;
    }
    slot[t] = (uint8_t)(lo - nbr_ptr[a]);
  }
}

// ---------------------------------------------------------------------------
// Row-block gather: K5 (elastic), K2+K6 (tangent, packed D or reference DS).
constexpr int kGatherWarps = 8;

__device__ __forceinline__ double c_iota(int i) { return i < 3 ? 1.0 : 0.0; }
__device__ __forceinline__ double c_dev(int i, int j) {
  return ((i == j) ? (i < 3 ? 1.0 : 0.5) : 0.0) - c_iota(i) * c_iota(j) / 3.0;
}
__device__ __forceinline__ double c_el(double K, double G, int i, int j) {
  return K * (c_iota(i) * c_iota(j)) + 2.0 * G * c_dev(i, j);
}

template <int DIM, int NP, int NQ, int MODE>
__global__ void __launch_bounds__(32 * kGatherWarps) k_gather(GatherArgs a) {
  extern __shared__ double smem[];
  constexpr int NS = DIM == 3 ? 6 : 3;
  constexpr int G = 32 / NP;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double* acc = smem + (size_t)wib * a.max_seg;
  const int64_t node = (int64_t)blockIdx.x * kGatherWarps + wib;
  if (node >= a.n_nodes) return;

  const int64_t i0 = a.n2e_ptr[node];
  const int nit = (int)(a.n2e_ptr[node + 1] - i0);
  const int64_t nb0 = a.nbr_ptr[node];
  const int nn = (int)(a.nbr_ptr[node + 1] - nb0);
  const int seg_len = DIM * DIM * nn;
  const int64_t sb = nb0 * DIM * DIM;

  if (MODE != G_ELASTIC) {
    bool any = false;
    for (int t = lane; t < nit * NQ; t += 32) {
      const int it = t / NQ, q = t - it * NQ;
      const int32_t item = __ldg(a.n2e + i0 + it);
      const int64_t e = item / NP;
      any |= (__ldg(a.flags + e * NQ + q) & 1) != 0;
    }
    if (!__any_sync(0xffffffffu, any)) {
      for (int k = lane; k < seg_len; k += 32) a.out[sb + k] = __ldg(a.base + sb + k);
      return;
    }
  }
  for (int k = lane; k < seg_len; k += 32) acc[k] = 0.0;
  __syncwarp();

  const int g = lane / NP, p = lane - (lane / NP) * NP;
  const bool in_group = g < G;
  for (int ib = 0; ib < nit; ib += G) {
    const int it = ib + g;
    const bool valid = in_group && it < nit;
    int64_t e = 0;
    int pa = 0, slot = 0;
    if (valid) {
      const int32_t item = __ldg(a.n2e + i0 + it);
      e = item / NP;
      pa = item - (int)e * NP;
      slot = __ldg(a.slot + ((int64_t)item) * NP + p);
    }
    double blk[DIM][DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) blk[i][j] = 0.0;

    for (int q = 0; q < NQ; ++q) {
      const int64_t m = e * NQ + q;
      bool contrib = valid;
      if (MODE != G_ELASTIC && valid) contrib = (__ldg(a.flags + m) & 1) != 0;
      if (!__any_sync(0xffffffffu, contrib)) continue;
      double h[DIM];
      double w = 0.0;
      if (contrib) {
        const double* Ji = a.inv + m * DIM * DIM;
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          double s = 0.0;
#pragma unroll
          for (int j = 0; j < DIM; ++j) s += __ldg(Ji + j * DIM + i) * __ldg(a.gradhat + (q * NP + p) * DIM + j);
          h[i] = s;
        }
        w = __ldg(a.weight + m);
      } else {
#pragma unroll
        for (int i = 0; i < DIM; ++i) h[i] = 0.0;
      }
      double ga[DIM];
      const int src = (in_group ? g : 0) * NP + pa;
#pragma unroll
      for (int i = 0; i < DIM; ++i) ga[i] = __shfl_sync(0xffffffffu, h[i], src);
      if (!contrib) continue;

      // effective material block Dw = w * (D - C) or w * C, reduced to the
      // assembly rows (2D: Voigt rows {0,1,3}, assembly.cpp:16,123-124)
      const double Gm = a.shear ? __ldg(a.shear + m) : a.shear_u;
      const double Km = a.bulk ? __ldg(a.bulk + m) : a.bulk_u;
      constexpr int R[6] = {0, 1, DIM == 3 ? 2 : 3, 3, 4, 5};
      double Dw[NS][NS];
#pragma unroll
      for (int r = 0; r < NS; ++r)
#pragma unroll
        for (int c = r; c < NS; ++c) {
          const int ri = R[r], ci = R[c];
          double v;
          if (MODE == G_ELASTIC) {
            v = c_el(Km, Gm, ri, ci);
          } else if (MODE == G_TANGENT_PACKED) {
            v = __ldg(a.D + m * EPFEM_D_STRIDE + pk_index(ri, ci)) - c_el(Km, Gm, ri, ci);
          } else {
            v = __ldg(a.D + m * 36 + ci * 6 + ri) - c_el(Km, Gm, ri, ci);
          }
          Dw[r][c] = w * v;
          Dw[c][r] = w * v;
        }
      if constexpr (DIM == 3) {
        // T = B_a^T Dw  (B rows e11,e22,e33,2e12,2e23,2e31; assembly.cpp:86-95)
        double T[3][6];
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          T[0][c] = ga[0] * Dw[0][c] + ga[1] * Dw[3][c] + ga[2] * Dw[5][c];
          T[1][c] = ga[1] * Dw[1][c] + ga[0] * Dw[3][c] + ga[2] * Dw[4][c];
          T[2][c] = ga[2] * Dw[2][c] + ga[1] * Dw[4][c] + ga[0] * Dw[5][c];
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          blk[i][0] += T[i][0] * h[0] + T[i][3] * h[1] + T[i][5] * h[2];
          blk[i][1] += T[i][1] * h[1] + T[i][3] * h[0] + T[i][4] * h[2];
          blk[i][2] += T[i][2] * h[2] + T[i][4] * h[1] + T[i][5] * h[0];
        }
      } else {
        // 2D rows e11, e22, 2e12 (assembly.cpp:96-100)
        double T[2][3];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          T[0][c] = ga[0] * Dw[0][c] + ga[1] * Dw[2][c];
          T[1][c] = ga[1] * Dw[1][c] + ga[0] * Dw[2][c];
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          blk[i][0] += T[i][0] * h[0] + T[i][2] * h[1];
          blk[i][1] += T[i][1] * h[1] + T[i][2] * h[0];
        }
      }
    }
    // groups take turns adding into the segment image (slots are distinct
    // within one element, but two elements may share a neighbour)
    const int row_len = DIM * nn;
#pragma unroll 1
    for (int gg = 0; gg < G; ++gg) {
      if (valid && g == gg) {
#pragma unroll
        for (int i = 0; i < DIM; ++i)
#pragma unroll
          for (int j = 0; j < DIM; ++j) acc[i * row_len + slot * DIM + j] += blk[i][j];
      }
      __syncwarp();
    }
  }
  if (MODE == G_ELASTIC) {
    for (int k = lane; k < seg_len; k += 32) a.out[sb + k] = acc[k];
  } else {
    for (int k = lane; k < seg_len; k += 32) a.out[sb + k] = __ldg(a.base + sb + k) + acc[k];
  }
}

// ---------------------------------------------------------------------------
// K8 strains E = B u, one thread per integration point (assembly.cpp:135-146)
template <int DIM, int NP, int NQ>
__global__ void k_strains(int64_t n_e, const int32_t* __restrict__ elem,
                          const double* __restrict__ inv, const double* __restrict__ gradhat,
                          const double* __restrict__ u, double* __restrict__ E) {
  const int64_t n_int = n_e * NQ;
  for (int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; m < n_int;
       m += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = m / NQ;
    const int q = (int)(m - e * NQ);
    double Ji[DIM * DIM];
#pragma unroll
    for (int k = 0; k < DIM * DIM; ++k) Ji[k] = __ldg(inv + m * DIM * DIM + k);
    double s[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll 4
    for (int p = 0; p < NP; ++p) {
      const int32_t node = __ldg(elem + e * NP + p);
      double d[DIM], uu[DIM];
      point_dphi<DIM>(Ji, gradhat + (q * NP + p) * DIM, d);
#pragma unroll
      for (int i = 0; i < DIM; ++i) uu[i] = __ldg(u + (int64_t)DIM * node + i);
      strain_accumulate<DIM>(d, uu, s);
    }
    double2* o = reinterpret_cast<double2*>(E + 6 * m);
    o[0] = make_double2(s[0], s[1]);
    o[1] = make_double2(s[2], s[3]);
    o[2] = make_double2(s[4], s[5]);
  }
}

// K9 internal forces F = B^T (w S), one thread per node gathering its items.
// K9 F = B^T (w S) in two passes (assembly.cpp:215-225).  Pass 1, thread per
// (element, node p): the element's force record F_e[p] = sum_q w_q B_p(q)^T
// S_q from zero in point order, with explicit roundings (dphi as
// stage_geometry, delta.cuh).  Pass 2, thread per node: F[a] = the records of
// the node's items summed from zero in item order.  The fused forces step
// (epfem_newton_step_f) forms the same records in its constitutive kernel and
// folds them in the row stream: the same bits.
template <int DIM, int NP, int NQ>
__global__ void k_elem_forces(int64_t n_e, const double* __restrict__ inv, const double* __restrict__ weight,
                              const double* __restrict__ gradhat, const double* __restrict__ S,
                              double* __restrict__ fws) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_e * NP;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = t / NP;
    const int p = (int)(t - e * NP);
    double fe[DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i) fe[i] = 0.0;
    for (int q = 0; q < NQ; ++q) {
      const int64_t m = e * NQ + q;
      double g[DIM];
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        double s = __dmul_rn(__ldg(inv + m * DIM * DIM + i), __ldg(gradhat + (q * NP + p) * DIM));
#pragma unroll
        for (int j = 1; j < DIM; ++j)
          s = __fma_rn(__ldg(inv + m * DIM * DIM + j * DIM + i), __ldg(gradhat + (q * NP + p) * DIM + j), s);
        g[i] = s;
      }
      const double w = __ldg(weight + m);
      const double* s6 = S + 6 * m;
      if constexpr (DIM == 3) {
        fe[0] = __fma_rn(w, __fma_rn(g[2], s6[5], __fma_rn(g[1], s6[3], __dmul_rn(g[0], s6[0]))), fe[0]);
        fe[1] = __fma_rn(w, __fma_rn(g[2], s6[4], __fma_rn(g[0], s6[3], __dmul_rn(g[1], s6[1]))), fe[1]);
        fe[2] = __fma_rn(w, __fma_rn(g[0], s6[5], __fma_rn(g[1], s6[4], __dmul_rn(g[2], s6[2]))), fe[2]);
      } else {
        fe[0] = __fma_rn(w, __fma_rn(g[1], s6[3], __dmul_rn(g[0], s6[0])), fe[0]);
        fe[1] = __fma_rn(w, __fma_rn(g[0], s6[3], __dmul_rn(g[1], s6[1])), fe[1]);
      }
    }
#pragma unroll
    for (int i = 0; i < DIM; ++i) fws[t * DIM + i] = fe[i];
  }
}

template <int DIM>
__global__ void k_fold_forces(int64_t n_nodes, const int64_t* __restrict__ n2e_ptr, const int32_t* __restrict__ n2e,
                              const double* __restrict__ fws, double* __restrict__ F) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_nodes * DIM;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = t / DIM;
    const int i = (int)(t - a * DIM);
    double f = 0.0;
    for (int64_t k = n2e_ptr[a]; k < n2e_ptr[a + 1]; ++k) f = __dadd_rn(f, __ldg(fws + (int64_t)n2e[k] * DIM + i));
    F[t] = f;
  }
}

// ---------------------------------------------------------------------------
// K5 for one-point P1 elements (cfg1), thread per node: the node's two (three)
// K rows are formed from its elements in item order, each element block with
// delta.cuh's explicit-rounding sequence (Dw = w C, T_a = B_a^T Dw, block =
// T_a B_b), into a shared-memory image laid out exactly like K[v0, v1) of the
// CTA's nodes (a node's rows are contiguous and nodes are numbered in row
// order), which the CTA then writes out coalesced.  One launch, one wave on
// cfg1 (66,049 nodes): the warp-per-node gather it replaces spent its time in
// per-node dependent load chains.
template <int DIM, int NP>
__global__ void k_elastic_p1(GatherArgs a) {
  extern __shared__ double img[];
  constexpr int NS = DIM == 3 ? 6 : 3, D2 = DIM * DIM;
  const int64_t first = (int64_t)blockIdx.x * blockDim.x;
  const int64_t last = min(first + (int64_t)blockDim.x, a.n_nodes);
  const int64_t v0 = __ldg(a.nbr_ptr + first) * D2, v1 = __ldg(a.nbr_ptr + last) * D2;
  for (int64_t k = threadIdx.x; k < v1 - v0; k += blockDim.x) img[k] = 0.0;
  __syncthreads();
  const int64_t node = first + threadIdx.x;
  if (node < last) {
    const int64_t nb0 = __ldg(a.nbr_ptr + node);
    const int row_len = DIM * (int)(__ldg(a.nbr_ptr + node + 1) - nb0);
    double* seg = img + (nb0 * D2 - v0);
    const bool uniform_c = a.shear == nullptr && a.bulk == nullptr;
    for (int64_t t = __ldg(a.n2e_ptr + node); t < __ldg(a.n2e_ptr + node + 1); ++t) {
      const int32_t item = __ldg(a.n2e + t);
      const int64_t e = item / NP;  // one point per element: m = e
      const int pa = item - (int)e * NP;
      double J[D2];
#pragma unroll
      for (int k = 0; k < D2; ++k) J[k] = __ldg(a.inv + e * D2 + k);
      const double w = __ldg(a.weight + e);
      double G2 = 0.0, Km = 0.0;
      if (!uniform_c) {
        G2 = 2.0 * (a.shear ? __ldg(a.shear + e) : a.shear_u);
        Km = a.bulk ? __ldg(a.bulk + e) : a.bulk_u;
      }
      double dw[NS][NS];
#pragma unroll
      for (int r = 0; r < NS; ++r)
#pragma unroll
        for (int c = r; c < NS; ++c) {  // stage_c (delta.cuh)
          const int ri = arow<DIM>(r), ci = arow<DIM>(c);
          const double vol = (ri < 3 && ci < 3) ? 1.0 : 0.0;
          const double dev = ((ri == ci) ? (ri < 3 ? 1.0 : 0.5) : 0.0) - vol / 3.0;
          const double cel = uniform_c ? a.Cu[pk_index(ri, ci)] : __fma_rn(G2, dev, __dmul_rn(Km, vol));
          dw[r][c] = dw[c][r] = __dmul_rn(w, cel);
        }
      double d[NP][DIM];
#pragma unroll
      for (int p = 0; p < NP; ++p) point_dphi<DIM>(J, a.gradhat + p * DIM, d[p]);
      double ga[DIM];
#pragma unroll
      for (int i = 0; i < DIM; ++i) ga[i] = d[0][i];
#pragma unroll
      for (int p = 1; p < NP; ++p)
        if (p == pa)
#pragma unroll
          for (int i = 0; i < DIM; ++i) ga[i] = d[p][i];
      double T[DIM][NS];  // delta_phase2's T_a
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        if constexpr (DIM == 3) {
          T[0][c] = __fma_rn(ga[2], dw[5][c], __fma_rn(ga[1], dw[3][c], __dmul_rn(ga[0], dw[0][c])));
          T[1][c] = __fma_rn(ga[2], dw[4][c], __fma_rn(ga[0], dw[3][c], __dmul_rn(ga[1], dw[1][c])));
          T[DIM - 1][c] = __fma_rn(ga[0], dw[5][c], __fma_rn(ga[1], dw[4][c], __dmul_rn(ga[2], dw[2][c])));
        } else {
          T[0][c] = __fma_rn(ga[1], dw[2][c], __dmul_rn(ga[0], dw[0][c]));
          T[1][c] = __fma_rn(ga[0], dw[2][c], __dmul_rn(ga[1], dw[1][c]));
        }
      }
#pragma unroll
      for (int pb = 0; pb < NP; ++pb) {
        const int sl = __ldg(a.slot + (int64_t)item * NP + pb);
        const double h0 = d[pb][0], h1 = d[pb][1], h2 = DIM == 3 ? d[pb][DIM - 1] : 0.0;
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          double b[DIM];
          if constexpr (DIM == 3) {
            b[0] = __fma_rn(T[i][5], h2, __fma_rn(T[i][3], h1, __fma_rn(T[i][0], h0, 0.0)));
            b[1] = __fma_rn(T[i][4], h2, __fma_rn(T[i][3], h0, __fma_rn(T[i][1], h1, 0.0)));
            b[DIM - 1] = __fma_rn(T[i][5], h0, __fma_rn(T[i][4], h1, __fma_rn(T[i][2], h2, 0.0)));
          } else {
            b[0] = __fma_rn(T[i][2], h1, __fma_rn(T[i][0], h0, 0.0));
            b[1] = __fma_rn(T[i][2], h0, __fma_rn(T[i][1], h1, 0.0));
          }
#pragma unroll
          for (int j = 0; j < DIM; ++j) seg[i * row_len + sl * DIM + j] += b[j];
        }
      }
    }
  }
  __syncthreads();
  for (int64_t k = threadIdx.x; k < v1 - v0; k += blockDim.x) a.out[v0 + k] = img[k];
}

// ---------------------------------------------------------------------------
// Host launchers (called from capi.cu)

static inline int grid_for(int64_t n, int threads, int num_sms) {
  int64_t b = (n + threads - 1) / threads;
  // one unit per thread (the kernels' grid-stride loops cover grids past the
  // launch limit): a grid capped at 32 CTAs per SM measured no faster (K8) or
  // slower (K9 1.94 vs 1.87 ms on cfg4)
  (void)num_sms;
  const int64_t cap = (int64_t)INT32_MAX;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

int launch_jacobians(int family, int dim, int64_t n_e, const int32_t* elem, const double* coord,
                     const double* gradhat, const double* wq, double* det, double* inv,
                     double* weight, DevErr* err, cudaStream_t st, int num_sms) {
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    k_jacobians<DIM, NP, NQ><<<grid_for(n_e * NQ, 256, num_sms), 256, 0, st>>>(
        n_e, elem, coord, gradhat, wq, det, inv, weight, err);
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

// Builds node->element items, neighbour lists, CSR pattern and slot map.
// Synchronous (sizes are needed on the host).
int build_pattern(int family, int dim, int64_t n_nodes, int64_t n_e, const int32_t* elem,
                  cudaStream_t st, int num_sms, PatternOut* o) {
  const int NPr = node_count(family, dim);
  const int64_t n_items = n_e * NPr;
  if (n_items >= (int64_t)INT32_MAX)
    return fail(EPFEM_ERR_UNSUPPORTED, "build_assembly_cache: n_elements * n_p exceeds int32");
  // node -> element items
  EPFEM_CUDA_TRY(cudaMalloc(&o->n2e_ptr, sizeof(int64_t) * (n_nodes + 1)));
  EPFEM_CUDA_TRY(cudaMalloc(&o->n2e, sizeof(int32_t) * std::max<int64_t>(n_items, 1)));
  int64_t* cnt = nullptr;
  EPFEM_CUDA_TRY(cudaMalloc(&cnt, sizeof(int64_t) * (n_nodes + 1)));
  EPFEM_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (n_nodes + 1), st));
  k_count_nodes<<<grid_for(n_items, 256, num_sms), 256, 0, st>>>(n_items, elem, cnt);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, o->n2e_ptr, n_nodes + 1, st);
  void* tmp = nullptr;
  EPFEM_CUDA_TRY(cudaMalloc(&tmp, tmp_bytes));
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, o->n2e_ptr, n_nodes + 1, st);
  cudaFree(tmp);
  EPFEM_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (n_nodes + 1), st));
  k_fill_n2e<<<grid_for(n_items, 256, num_sms), 256, 0, st>>>(n_items, elem, o->n2e_ptr, cnt, o->n2e);
  k_sort_n2e<<<grid_for(n_nodes, 128, num_sms), 128, 0, st>>>(n_nodes, o->n2e_ptr, o->n2e);
  cudaFree(cnt);

  // (a, b) pairs -> sorted unique keys
  const int64_t n_pairs = n_items * NPr;
  uint64_t *keys = nullptr, *keys_alt = nullptr, *ukeys = nullptr;
  EPFEM_CUDA_TRY(cudaMalloc(&keys, sizeof(uint64_t) * n_pairs));
  EPFEM_CUDA_TRY(cudaMalloc(&keys_alt, sizeof(uint64_t) * n_pairs));
  dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int NP = ET<decltype(F)::value, decltype(D)::value>::NP;
    k_pair_keys<NP><<<grid_for(n_pairs, 256, num_sms), 256, 0, st>>>(n_e, elem, keys);
  });
  EPFEM_CUDA_TRY(cudaGetLastError());
  int node_bits = 1;
  while (node_bits < 32 && ((int64_t)1 << node_bits) < n_nodes) ++node_bits;
  cub::DoubleBuffer<uint64_t> db(keys, keys_alt);
  tmp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, n_pairs, 0, 32 + node_bits, st);
  EPFEM_CUDA_TRY(cudaMalloc(&tmp, tmp_bytes));
  cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, db, n_pairs, 0, 32 + node_bits, st);
  cudaFree(tmp);
  uint64_t* sorted = db.Current();
  uint64_t* spare = db.Alternate();
  ukeys = spare;
  int64_t* d_nu = nullptr;
  EPFEM_CUDA_TRY(cudaMalloc(&d_nu, sizeof(int64_t)));
  tmp_bytes = 0;
  cub::DeviceSelect::Unique(nullptr, tmp_bytes, sorted, ukeys, d_nu, n_pairs, st);
  EPFEM_CUDA_TRY(cudaMalloc(&tmp, tmp_bytes));
  cub::DeviceSelect::Unique(tmp, tmp_bytes, sorted, ukeys, d_nu, n_pairs, st);
  cudaFree(tmp);
  int64_t n_unique = 0;
  EPFEM_CUDA_TRY(cudaMemcpyAsync(&n_unique, d_nu, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(d_nu);
  cudaFree(sorted);  // ukeys lives in the other buffer

  EPFEM_CUDA_TRY(cudaMalloc(&cnt, sizeof(int64_t) * (n_nodes + 1)));
  EPFEM_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int64_t) * (n_nodes + 1), st));
  k_count_nbr<<<grid_for(n_unique, 256, num_sms), 256, 0, st>>>(n_unique, ukeys, cnt);
  EPFEM_CUDA_TRY(cudaMalloc(&o->nbr_ptr, sizeof(int64_t) * (n_nodes + 1)));
  tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, o->nbr_ptr, n_nodes + 1, st);
  EPFEM_CUDA_TRY(cudaMalloc(&tmp, tmp_bytes));
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, o->nbr_ptr, n_nodes + 1, st);
  cudaFree(tmp);
  cudaFree(cnt);
  int* d_max = nullptr;
  EPFEM_CUDA_TRY(cudaMalloc(&d_max, sizeof(int)));
  EPFEM_CUDA_TRY(cudaMemsetAsync(d_max, 0, sizeof(int), st));
  k_max_nbr<<<grid_for(n_nodes, 256, num_sms), 256, 0, st>>>(n_nodes, o->nbr_ptr, d_max);
  EPFEM_CUDA_TRY(cudaMemcpyAsync(&o->max_nbr, d_max, sizeof(int), cudaMemcpyDeviceToHost, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(d_max);
  if (o->max_nbr > 255) {
    cudaFree(ukeys);
    return fail(EPFEM_ERR_UNSUPPORTED,
                "build_assembly_cache: node valence above 255 is not supported");
  }
  o->nnz = n_unique * dim * dim;
  const int64_t n_dofs = n_nodes * dim;
  EPFEM_CUDA_TRY(cudaMalloc(&o->row_ptr, sizeof(int64_t) * (n_dofs + 1)));
  EPFEM_CUDA_TRY(cudaMalloc(&o->col_idx, sizeof(int32_t) * std::max<int64_t>(o->nnz, 1)));
  EPFEM_CUDA_TRY(cudaMemcpyAsync(o->row_ptr + n_dofs, &o->nnz, sizeof(int64_t), cudaMemcpyHostToDevice, st));
  {
    dim3 blk(32, 8);
    k_fill_csr<<<grid_for(n_nodes, 8, num_sms), blk, 0, st>>>(n_nodes, dim, o->nbr_ptr, ukeys,
                                                              o->row_ptr, o->col_idx);
  }
  EPFEM_CUDA_TRY(cudaMalloc(&o->slot, std::max<int64_t>(n_pairs, 1)));
  dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int NP = ET<decltype(F)::value, decltype(D)::value>::NP;
    k_slot_map<NP><<<grid_for(n_pairs, 256, num_sms), 256, 0, st>>>(n_e, elem, o->nbr_ptr,
                                                                   ukeys, o->slot);
  });
  EPFEM_CUDA_TRY(cudaGetLastError());
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFree(ukeys);
  return 0;
}

int launch_gather(int family, int dim, int mode, const GatherArgs& a, cudaStream_t st) {
  if (a.n_nodes == 0) return 0;
  const int64_t blocks = (a.n_nodes + kGatherWarps - 1) / kGatherWarps;
  const size_t smem = sizeof(double) * (size_t)a.max_seg * kGatherWarps;
  int rc = 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    auto launch = [&](auto kern) {
      if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) { rc = cuda_fail(e, "cudaFuncSetAttribute"); return; }
      }
      kern<<<(unsigned)blocks, 32 * kGatherWarps, smem, st>>>(a);
    };
    if (mode == G_ELASTIC) launch(k_gather<DIM, NP, NQ, G_ELASTIC>);
    else if (mode == G_TANGENT_PACKED) launch(k_gather<DIM, NP, NQ, G_TANGENT_PACKED>);
    else launch(k_gather<DIM, NP, NQ, G_TANGENT_DS36>);
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  if (rc) return rc;
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

// K5 for P1 meshes (k_elastic_p1); block size by dimension so that the
// image (at most threads x max_seg doubles) fits the shared memory.
int launch_elastic_p1(int family, int dim, const GatherArgs& a, cudaStream_t st) {
  if (a.n_nodes == 0) return 0;
  if (family != EPFEM_P1) return fail(EPFEM_ERR_INVALID, "elastic_p1: P1 elements only");
  const int threads = dim == 2 ? 128 : 32;
  const size_t smem = sizeof(double) * (size_t)a.max_seg * threads;
  const int64_t blocks = (a.n_nodes + threads - 1) / threads;
  auto run = [&](auto kern) -> int {
    if (smem > 48 * 1024)
      EPFEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    kern<<<(unsigned)blocks, threads, smem, st>>>(a);
    EPFEM_CUDA_TRY(cudaGetLastError());
    return 0;
  };
  return dim == 2 ? run(k_elastic_p1<2, 3>) : run(k_elastic_p1<3, 4>);
}

int launch_strains(int family, int dim, int64_t n_e, const int32_t* elem, const double* inv,
                   const double* gradhat, const double* u, double* E, cudaStream_t st,
                   int num_sms) {
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    k_strains<DIM, NP, NQ><<<grid_for(n_e * NQ, 256, num_sms), 256, 0, st>>>(n_e, elem, inv,
                                                                            gradhat, u, E);
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

int launch_internal_forces(int family, int dim, int64_t n_nodes, int64_t n_e, const int64_t* n2e_ptr,
                           const int32_t* n2e, const double* inv, const double* weight,
                           const double* gradhat, const double* S, double* fws, double* F_out,
                           cudaStream_t st, int num_sms) {
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    if (n_e > 0)
      k_elem_forces<DIM, NP, NQ><<<grid_for(n_e * NP, 256, num_sms), 256, 0, st>>>(n_e, inv, weight, gradhat, S,
                                                                                    fws);
    k_fold_forces<DIM><<<grid_for(n_nodes * DIM, 256, num_sms), 256, 0, st>>>(n_nodes, n2e_ptr, n2e, fws, F_out);
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace epfem_gpu
