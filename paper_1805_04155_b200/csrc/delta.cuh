// Element tangent-delta building blocks shared by the standalone pass
// (tangent.cu) and the fused constitutive + delta kernel (constitutive.cu).
// All multiply-adds are explicit __fma_rn so both translation units (one is
// compiled with --fmad=false) produce identical bits.
//
//   staged record per (element, point), REC doubles in shared memory:
//     [ dphi_p (NP x DIM) | Dw = w (D - C), packed upper triangle (NSP) ]
//   workspace record per element (global), NB = NP(NP+1)/2 blocks of dim x dim:
//     block (a, b), a <= b, at blk_index(a, b) * dim^2, row-major
//
// Phase 2 computes only the symmetric blocks (a, b >= a).  Block row a is cut
// into chunks of CS blocks; one thread owns one (a, chunk): it forms
// T_a = B_a^T Dw once per plastic point and adds T_a B_b for the b of its
// chunk.  FMA per plastic point: NT*|T| + NB*|block| (vs NP*|T| + NP^2*|block|
// for full block rows), and no thread holds more than CS blocks.
#pragma once

#include "kernels.cuh"
#include "tma.cuh"

namespace epfem_gpu {

template <int NP>
__host__ __device__ constexpr int blk_index(int a, int b) {  // a <= b
  return a * (2 * NP - a + 1) / 2 + (b - a);
}

// (row a, first column c0) of phase-2 slot k of an element, chunks of CS
template <int NP, int CS>
__device__ __forceinline__ void chunk_of(int k, int& a, int& c0) {
  a = 0;
  while ((NP - a + CS - 1) / CS <= k) {
    k -= (NP - a + CS - 1) / CS;
    ++a;
  }
  c0 = a + k * CS;
}

template <int DIM, int NP, int NQ>
struct DeltaCfg {
  static constexpr int NS = DIM == 3 ? 6 : 3;
  static constexpr int NSP = NS * (NS + 1) / 2;
  static constexpr int D2 = DIM * DIM;
  static constexpr int NB = NP * (NP + 1) / 2;
  static constexpr int REC = NP * DIM + NSP;
// Q2-20 (cfg5) phase 2: chunks of 4 blocks at <= 128 registers (4 CTAs/SM)
// measured 16.0 ms vs 18.9 ms for chunks of 5 at ptxas' 164 registers; 3, 6
// and 7 blocks, sub-passes and 5 CTAs/SM were all slower (B200 sweep)
#ifndef EPFEM_CS20
#define EPFEM_CS20 4
#endif
#ifndef EPFEM_SUB20
#define EPFEM_SUB20 0
#endif
#ifndef EPFEM_MINB20
#define EPFEM_MINB20 4
#endif
  static constexpr int CS = (DIM == 3 && NP >= 20) ? EPFEM_CS20 : 4;  // blocks per phase-2 thread
  static constexpr int nt() {
    int s = 0;
    for (int a = 0; a < NP; ++a) s += (NP - a + CS - 1) / CS;
    return s;
  }
  static constexpr int NT = nt();                        // phase-2 threads per element
  static constexpr int TPE = NQ > NT ? NQ : NT;           // threads per element
#ifndef EPFEM_DELTA_MAXT
#define EPFEM_DELTA_MAXT 128
#endif
  static constexpr int MAXT = EPFEM_DELTA_MAXT;
  static constexpr int BUDGET = 5120;                     // doubles of staged records per CTA
  static constexpr int E1 = MAXT / TPE, E2 = BUDGET / (NQ * REC);
  static constexpr int EPB = (E1 < E2 ? E1 : E2) > 0 ? (E1 < E2 ? E1 : E2) : 1;
  static constexpr int THREADS = ((EPB * TPE + 31) / 32) * 32;
  // CTA-kernel phase 2 sub-pass width and minimum CTAs per SM (measured on
  // B200: 3D Q1 / P2 tet with row-pair phase 2 at <= 128 registers; Q2-20 with
  // whole chunks and ptxas' own register choice; 2D: 1024 threads per SM)
#ifndef EPFEM_MINB3
#define EPFEM_MINB3 4
#endif
  static constexpr int SUB = (DIM == 3 && NP < 20) ? 2 : (DIM == 3 ? EPFEM_SUB20 : 0);
  static constexpr int MINB = DIM == 2 ? 1024 / THREADS : (NP < 20 ? EPFEM_MINB3 : EPFEM_MINB20);
};

// assembly row r -> Voigt row (2D plane strain uses {0,1,3}, assembly.cpp:16)
template <int DIM>
__device__ __forceinline__ constexpr int arow(int r) {
  return (DIM == 2 && r == 2) ? 3 : r;
}

// Geometry at one integration point from the element's nodal coordinates
// (jacobians, assembly.cpp:20-61): J(i, j) = sum_p ghat_i(p, q) x_p(j) in
// node order, det J by the first-row cofactor expansion and J^-1 by Eigen's
// cofactor inverse (compute_inverse_size3), each product and sum rounded
// separately in the reference's evaluation order (the reference's Release
// x86-64 build has no FMA).  Used by the one-time geometry kernel and, with
// the same bits, by kernels that form J^-1 on the fly.  `inv` is column-major
// dim x dim like JacobianData::inv; returns det J.  `xs(p, j)` gives
// coordinate j of local node p.
template <int DIM, int NP, class X>
__device__ __forceinline__ double point_geometry(X&& xs, const double* __restrict__ gradhat, int q, double* inv) {
  double J[DIM][DIM];
#pragma unroll
  for (int i = 0; i < DIM; ++i)
#pragma unroll
    for (int j = 0; j < DIM; ++j) J[i][j] = 0.0;
#pragma unroll 4
  for (int p = 0; p < NP; ++p) {
    double x[DIM], g[DIM];
#pragma unroll
    for (int j = 0; j < DIM; ++j) x[j] = xs(p, j);
#pragma unroll
    for (int i = 0; i < DIM; ++i) g[i] = __ldg(gradhat + (q * NP + p) * DIM + i);
#pragma unroll
    for (int i = 0; i < DIM; ++i)
#pragma unroll
      for (int j = 0; j < DIM; ++j) J[i][j] = __dadd_rn(J[i][j], __dmul_rn(g[i], x[j]));
  }
  auto mul = [](double a, double b) { return __dmul_rn(a, b); };
  auto sub = [](double a, double b) { return __dsub_rn(a, b); };
  double det;
  if constexpr (DIM == 3) {
    det = __dadd_rn(sub(mul(J[0][0], sub(mul(J[1][1], J[2][2]), mul(J[1][2], J[2][1]))),
                        mul(J[0][1], sub(mul(J[1][0], J[2][2]), mul(J[1][2], J[2][0])))),
                    mul(J[0][2], sub(mul(J[1][0], J[2][1]), mul(J[1][1], J[2][0]))));
    double cof[3][3];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        const int i1 = (i + 1) % 3, i2 = (i + 2) % 3, j1 = (j + 1) % 3, j2 = (j + 2) % 3;
        cof[i][j] = sub(mul(J[i1][j1], J[i2][j2]), mul(J[i1][j2], J[i2][j1]));
      }
    const double d2 = __dadd_rn(__dadd_rn(mul(cof[0][0], J[0][0]), mul(cof[1][0], J[1][0])), mul(cof[2][0], J[2][0]));
    const double invdet = __drcp_rn(d2);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) inv[j * 3 + i] = mul(cof[j][i], invdet);
  } else {
    det = sub(mul(J[0][0], J[1][1]), mul(J[1][0], J[0][1]));
    const double invdet = __drcp_rn(det);
    inv[0] = mul(J[1][1], invdet);
    inv[1] = mul(-J[1][0], invdet);
    inv[2] = mul(-J[0][1], invdet);
    inv[3] = mul(J[0][0], invdet);
  }
  return det;
}

// dphi_p = J^-1 ghat_p for every node of the element at point q.
template <int DIM, int NP, bool INV_IN_SMEM = false>
__device__ __forceinline__ void stage_geometry(double* st, const double* inv_m,
                                               const double* __restrict__ gradhat, int q) {
  double J[DIM * DIM];
#pragma unroll
  for (int t = 0; t < DIM * DIM; ++t) J[t] = INV_IN_SMEM ? inv_m[t] : __ldg(inv_m + t);
#pragma unroll 4
  for (int p = 0; p < NP; ++p) {
    const double* gh = gradhat + (q * NP + p) * DIM;
    double g[DIM];
#pragma unroll
    for (int j = 0; j < DIM; ++j) g[j] = __ldg(gh + j);
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      double s = __dmul_rn(J[i], g[0]);
#pragma unroll
      for (int j = 1; j < DIM; ++j) s = __fma_rn(J[j * DIM + i], g[j], s);
      st[p * DIM + i] = s;
    }
  }
}

// K8 at one point: E = sum_p B_p u_p (assembly.cpp:135-146) from the
// physical gradients dphi (as stage_geometry computes them) and the element's
// nodal displacements; explicit roundings so every translation unit (K8
// alone, the fused strain + Newton kernel) produces the same bits.  2D fills
// Voigt rows {0, 1, 3}.
template <int DIM>
__device__ __forceinline__ void strain_accumulate(const double* d, const double* uu, double* s) {
  if constexpr (DIM == 3) {
    s[0] = __fma_rn(d[0], uu[0], s[0]);
    s[1] = __fma_rn(d[1], uu[1], s[1]);
    s[2] = __fma_rn(d[2], uu[2], s[2]);
    s[3] = __fma_rn(d[0], uu[1], __fma_rn(d[1], uu[0], s[3]));
    s[4] = __fma_rn(d[1], uu[2], __fma_rn(d[2], uu[1], s[4]));
    s[5] = __fma_rn(d[0], uu[2], __fma_rn(d[2], uu[0], s[5]));
  } else {
    s[0] = __fma_rn(d[0], uu[0], s[0]);
    s[1] = __fma_rn(d[1], uu[1], s[1]);
    s[3] = __fma_rn(d[0], uu[1], __fma_rn(d[1], uu[0], s[3]));
  }
}
// dphi_p at point q (same arithmetic as stage_geometry)
template <int DIM>
__device__ __forceinline__ void point_dphi(const double* J, const double* __restrict__ gh, double* d) {
  double g[DIM];
#pragma unroll
  for (int j = 0; j < DIM; ++j) g[j] = __ldg(gh + j);
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    double t = __dmul_rn(J[i], g[0]);
#pragma unroll
    for (int j = 1; j < DIM; ++j) t = __fma_rn(J[j * DIM + i], g[j], t);
    d[i] = t;
  }
}

// Dw(r, c) = w (D(R r, R c) - C(R r, R c)) packed upper triangle.  Dfun gives
// the tangent entry D(i, j) in Voigt indices.
template <int DIM, class Dfun>
__device__ __forceinline__ void stage_dw(double* dwst, double w, const GatherArgs& a, int64_t m,
                                         Dfun&& Dv) {
  constexpr int NS = DIM == 3 ? 6 : 3;
  const bool uniform_c = a.shear == nullptr && a.bulk == nullptr;
  double G2 = 0.0, Km = 0.0;
  if (!uniform_c) {
    G2 = 2.0 * (a.shear ? __ldg(a.shear + m) : a.shear_u);
    Km = a.bulk ? __ldg(a.bulk + m) : a.bulk_u;
  }
  int k = 0;
#pragma unroll
  for (int r = 0; r < NS; ++r)
#pragma unroll
    for (int c = r; c < NS; ++c, ++k) {
      const int ri = arow<DIM>(r), ci = arow<DIM>(c);
      const double vol = (ri < 3 && ci < 3) ? 1.0 : 0.0;
      const double dev = ((ri == ci) ? (ri < 3 ? 1.0 : 0.5) : 0.0) - vol / 3.0;
      const double cel = uniform_c ? a.Cu[pk_index(ri, ci)] : __fma_rn(G2, dev, __dmul_rn(Km, vol));
      dwst[k] = __dmul_rn(w, __dsub_rn(Dv(ri, ci), cel));
    }
}

// Elastic assembly (K5) through the same two passes: Dw = w C, packed upper
// triangle in assembly rows (stage_dw with D - C replaced by C).
template <int DIM>
__device__ __forceinline__ void stage_c(double* dwst, double w, const GatherArgs& a, int64_t m) {
  constexpr int NS = DIM == 3 ? 6 : 3;
  const bool uniform_c = a.shear == nullptr && a.bulk == nullptr;
  double G2 = 0.0, Km = 0.0;
  if (!uniform_c) {
    G2 = 2.0 * (a.shear ? __ldg(a.shear + m) : a.shear_u);
    Km = a.bulk ? __ldg(a.bulk + m) : a.bulk_u;
  }
  int k = 0;
#pragma unroll
  for (int r = 0; r < NS; ++r)
#pragma unroll
    for (int c = r; c < NS; ++c, ++k) {
      const int ri = arow<DIM>(r), ci = arow<DIM>(c);
      const double vol = (ri < 3 && ci < 3) ? 1.0 : 0.0;
      const double dev = ((ri == ci) ? (ri < 3 ? 1.0 : 0.5) : 0.0) - vol / 3.0;
      const double cel = uniform_c ? a.Cu[pk_index(ri, ci)] : __fma_rn(G2, dev, __dmul_rn(Km, vol));
      dwst[k] = __dmul_rn(w, cel);
    }
}

// Phase 2: thread (element le, row a, chunk starting at block c0 >= a)
// accumulates the blocks (a, b), c0 <= b < c0 + CS, over the element's
// plastic points from the staged records, then writes them to the workspace.
template <int DIM, int NP, int NQ>
__device__ __forceinline__ void delta_phase2(
    const double (*s_st)[NQ][DeltaCfg<DIM, NP, NQ>::REC], const unsigned* s_mask, int tid,
    int64_t e0, int64_t n_elements, double* __restrict__ scratch) {
  using Cfg = DeltaCfg<DIM, NP, NQ>;
  constexpr int NS = Cfg::NS, D2 = Cfg::D2, NB = Cfg::NB, CS = Cfg::CS, NT = Cfg::NT;
  if (tid >= Cfg::EPB * NT) return;
  const int le = tid / NT;
  int k = tid - le * NT, a = 0;
  while ((NP - a + CS - 1) / CS <= k) {
    k -= (NP - a + CS - 1) / CS;
    ++a;
  }
  const int c0 = a + k * CS;
  const int nb = NP - c0 < CS ? NP - c0 : CS;
  const int64_t e = e0 + le;
  if (e >= n_elements) return;
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
    for (int i = 0; i < DIM; ++i) ga[i] = st[a * DIM + i];
    double T[DIM][NS];  // T_a = B_a^T Dw
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      if constexpr (DIM == 3) {
        // B rows e11,e22,e33,2e12,2e23,2e31 (assembly.cpp:86-95)
        T[0][c] = __fma_rn(ga[2], Dw(5, c), __fma_rn(ga[1], Dw(3, c), __dmul_rn(ga[0], Dw(0, c))));
        T[1][c] = __fma_rn(ga[2], Dw(4, c), __fma_rn(ga[0], Dw(3, c), __dmul_rn(ga[1], Dw(1, c))));
        T[DIM - 1][c] =
            __fma_rn(ga[0], Dw(5, c), __fma_rn(ga[1], Dw(4, c), __dmul_rn(ga[2], Dw(2, c))));
      } else {
        // rows e11, e22, 2e12 (assembly.cpp:96-100)
        T[0][c] = __fma_rn(ga[1], Dw(2, c), __dmul_rn(ga[0], Dw(0, c)));
        T[1][c] = __fma_rn(ga[0], Dw(2, c), __dmul_rn(ga[1], Dw(1, c)));
      }
    }
#pragma unroll
    for (int bb = 0; bb < CS; ++bb) {
      if (bb < nb) {
        const double* h = st + (c0 + bb) * DIM;
        const double h0 = h[0], h1 = h[1], h2 = DIM == 3 ? h[DIM - 1] : 0.0;
#pragma unroll
        for (int i = 0; i < DIM; ++i) {
          if constexpr (DIM == 3) {
            blk[bb][i][0] = __fma_rn(T[i][5], h2, __fma_rn(T[i][3], h1, __fma_rn(T[i][0], h0, blk[bb][i][0])));
            blk[bb][i][1] = __fma_rn(T[i][4], h2, __fma_rn(T[i][3], h0, __fma_rn(T[i][1], h1, blk[bb][i][1])));
            blk[bb][i][DIM - 1] =
                __fma_rn(T[i][5], h0, __fma_rn(T[i][4], h1, __fma_rn(T[i][2], h2, blk[bb][i][DIM - 1])));
          } else {
            blk[bb][i][0] = __fma_rn(T[i][2], h1, __fma_rn(T[i][0], h0, blk[bb][i][0]));
            blk[bb][i][1] = __fma_rn(T[i][2], h0, __fma_rn(T[i][1], h1, blk[bb][i][1]));
          }
        }
      }
    }
  }
  double* rec = scratch + (size_t)e * NB * D2;
#pragma unroll
  for (int bb = 0; bb < CS; ++bb) {
    if (bb < nb) {
      double* o = rec + blk_index<NP>(a, c0 + bb) * D2;
#pragma unroll
      for (int i = 0; i < DIM; ++i)
#pragma unroll
        for (int j = 0; j < DIM; ++j) o[i * DIM + j] = blk[bb][i][j];
    }
  }
}

// ---------------------------------------------------------------------------
// Warp-synchronous variant (2D): a warp owns EPW whole elements, so phase 1
// and phase 2 meet at a __syncwarp instead of a CTA barrier, and the plastic
// masks come from one __ballot_sync.  CS is the smallest chunk that fits the
// most elements in a warp; every phase-2 lane runs exactly CS blocks (blocks
// past the row end are computed on a clamped column and dropped), so the
// block loop has no divergent branch.  Same FMA sequence per block as
// delta_phase2, hence identical bits.
template <int DIM, int NP, int NQ>
struct WarpCfg {
  static constexpr int NS = DIM == 3 ? 6 : 3;
  static constexpr int NSP = NS * (NS + 1) / 2;
  static constexpr int D2 = DIM * DIM;
  static constexpr int NB = NP * (NP + 1) / 2;
  static constexpr int REC = NP * DIM + NSP;
  static constexpr int nt(int cs) {
    int s = 0;
    for (int a = 0; a < NP; ++a) s += (NP - a + cs - 1) / cs;
    return s;
  }
  static constexpr int epw(int cs) {
    const int t = NQ > nt(cs) ? NQ : nt(cs);
    return 32 / t;
  }
  static constexpr int best_cs() {
    int best = NP, be = 0;
    for (int cs = 1; cs <= NP; ++cs)
      if (epw(cs) > be) {
        be = epw(cs);
        best = cs;
      }
    return best;
  }
  static constexpr int CS = best_cs();
  static constexpr int NT = nt(CS);
  static constexpr int EPW = epw(CS);  // elements per warp
#ifndef EPFEM_WARP_WPB
#define EPFEM_WARP_WPB 4
#endif
  static constexpr int WPB = EPFEM_WARP_WPB;  // warps per CTA
  static constexpr int THREADS = 32 * WPB;
};

// Blocks (a, c0 .. c0 + CS - 1) of one element from its staged records
// st_e[q * REC], accumulated over the plastic points in `mask`, written to
// the element's workspace record.
#ifndef EPFEM_SUBCHUNK
#define EPFEM_SUBCHUNK 0
#endif
template <int DIM, int NP, int CS, int REC>
__device__ __forceinline__ void delta_chunk_uniform1(const double* st_e, unsigned mask, int a, int c0,
                                                     double* __restrict__ rec);
// CS blocks in passes of SUB (fewer live accumulators; T_a is recomputed per pass)
template <int DIM, int NP, int CS, int REC, int SUB_ = EPFEM_SUBCHUNK>
__device__ __forceinline__ void delta_chunk_uniform(const double* st_e, unsigned mask, int a, int c0,
                                                    double* __restrict__ rec) {
  constexpr int SUB = SUB_ > 0 && SUB_ < CS ? SUB_ : CS;
#pragma unroll 1
  for (int s0 = 0; s0 < CS; s0 += SUB)
    if (c0 + s0 < NP) delta_chunk_uniform1<DIM, NP, SUB, REC>(st_e, mask, a, c0 + s0, rec);
}
template <int DIM, int NP, int CS, int REC>
__device__ __forceinline__ void delta_chunk_uniform1(const double* st_e, unsigned mask, int a, int c0,
                                                     double* __restrict__ rec) {
  constexpr int NS = DIM == 3 ? 6 : 3, D2 = DIM * DIM;
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
    const double* st = st_e + q * REC;
    const double* dw = st + NP * DIM;
    auto Dw = [&](int r, int c) {
      const int lo = r < c ? r : c, hi = r < c ? c : r;
      return dw[lo * NS - lo * (lo - 1) / 2 + (hi - lo)];
    };
    double ga[DIM];
#pragma unroll
    for (int i = 0; i < DIM; ++i) ga[i] = st[a * DIM + i];
    double T[DIM][NS];
#pragma unroll
    for (int c = 0; c < NS; ++c) {
      if constexpr (DIM == 3) {
        T[0][c] = __fma_rn(ga[2], Dw(5, c), __fma_rn(ga[1], Dw(3, c), __dmul_rn(ga[0], Dw(0, c))));
        T[1][c] = __fma_rn(ga[2], Dw(4, c), __fma_rn(ga[0], Dw(3, c), __dmul_rn(ga[1], Dw(1, c))));
        T[DIM - 1][c] =
            __fma_rn(ga[0], Dw(5, c), __fma_rn(ga[1], Dw(4, c), __dmul_rn(ga[2], Dw(2, c))));
      } else {
        T[0][c] = __fma_rn(ga[1], Dw(2, c), __dmul_rn(ga[0], Dw(0, c)));
        T[1][c] = __fma_rn(ga[0], Dw(2, c), __dmul_rn(ga[1], Dw(1, c)));
      }
    }
#pragma unroll
    for (int bb = 0; bb < CS; ++bb) {
      const int b = c0 + bb < NP ? c0 + bb : NP - 1;  // clamped: result dropped below
      const double* h = st + b * DIM;
      const double h0 = h[0], h1 = h[1], h2 = DIM == 3 ? h[DIM - 1] : 0.0;
#pragma unroll
      for (int i = 0; i < DIM; ++i) {
        if constexpr (DIM == 3) {
          blk[bb][i][0] = __fma_rn(T[i][5], h2, __fma_rn(T[i][3], h1, __fma_rn(T[i][0], h0, blk[bb][i][0])));
          blk[bb][i][1] = __fma_rn(T[i][4], h2, __fma_rn(T[i][3], h0, __fma_rn(T[i][1], h1, blk[bb][i][1])));
          blk[bb][i][DIM - 1] =
              __fma_rn(T[i][5], h0, __fma_rn(T[i][4], h1, __fma_rn(T[i][2], h2, blk[bb][i][DIM - 1])));
        } else {
          blk[bb][i][0] = __fma_rn(T[i][2], h1, __fma_rn(T[i][0], h0, blk[bb][i][0]));
          blk[bb][i][1] = __fma_rn(T[i][2], h0, __fma_rn(T[i][1], h1, blk[bb][i][1]));
        }
      }
    }
  }
#pragma unroll
  for (int bb = 0; bb < CS; ++bb) {
    if (c0 + bb < NP) {
      EPFEM_CHECK(a <= c0 + bb && blk_index<NP>(a, c0 + bb) < NP * (NP + 1) / 2);
      double* o = rec + blk_index<NP>(a, c0 + bb) * D2;
#pragma unroll
      for (int i = 0; i < DIM; ++i)
#pragma unroll
        for (int j = 0; j < DIM; ++j) o[i * DIM + j] = blk[bb][i][j];
    }
  }
}



// ---------------------------------------------------------------------------
// 3D warp phase 2 by row pairs: lane (element, pair p, component i) owns row
// i of the block rows a = p and a' = NP - 1 - p (a <= a'), i.e. (NP - a) +
// (a + 1) = NP + 1 blocks whatever p is (balanced), and forms its own T rows
// T_a[i][:] and T_a'[i][:] once per plastic point: every T entry and every
// block entry is computed exactly once (the optimal n_p n_s g + n_p(n_p+1)/2 g
// dim FMA per point).  Per-entry FMA sequences are those of delta_phase2, so
// the bits are identical.  Accumulators are written straight to the element
// record (no shared-memory staging of outputs).
template <int NP, int NQ>
struct Pair3Cfg {
  static constexpr int DIM = 3, NS = 6, NSP = 21, D2 = 9;
  static constexpr int NB = NP * (NP + 1) / 2;
  static constexpr int REC = NP * DIM + NSP;
  static constexpr int NPAIR = (NP + 1) / 2;
  static constexpr int PL = 3 * NPAIR;          // phase-2 lanes per element
  static constexpr int EPW = 32 / NQ;           // elements per warp (phase 1)
  static constexpr int EPR = 32 / PL;           // elements per phase-2 round
  static constexpr int NBLK = NP + 1;           // blocks per lane (a != a'); NP - a for a == a'
  static constexpr int WPB = 4;
  static constexpr int THREADS = 32 * WPB;
};

template <int NP, int NQ>
__device__ __forceinline__ void delta_pairs3(const double* st_e, unsigned mask, int p, int i,
                                             double* __restrict__ rec) {
  using C = Pair3Cfg<NP, NQ>;
  constexpr int NS = C::NS, REC = C::REC, D2 = C::D2, NBLK = C::NBLK;
  const int a0 = p, a1 = NP - 1 - p;
  const bool twin = a1 != a0;
  // T row i: sum over the B column (node, i) nonzeros in delta_phase2's order
  const int d0 = i, d1 = i == 2 ? 4 : 3, d2 = i == 0 ? 5 : (i == 1 ? 4 : 5);
  const int e1 = i == 0 ? 1 : (i == 1 ? 0 : 1), e2 = i == 0 ? 2 : (i == 1 ? 2 : 0);
  auto pk = [](int r, int c) {
    const int lo = r < c ? r : c, hi = r < c ? c : r;
    return lo * NS - lo * (lo - 1) / 2 + (hi - lo);
  };
  double acc[NBLK][3];
#pragma unroll
  for (int k = 0; k < NBLK; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
  while (mask) {
    const int q = __ffs(mask) - 1;
    mask &= mask - 1u;
    const double* st = st_e + q * REC;
    const double* dw = st + NP * 3;
    double T0[NS], T1[NS];
    {
      const double* g0 = st + a0 * 3;
      const double* g1 = st + a1 * 3;
      const double gA0 = g0[d0], gA1 = g0[e1], gA2 = g0[e2];
      const double gB0 = g1[d0], gB1 = g1[e1], gB2 = g1[e2];
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        const double w0 = dw[pk(d0, c)], w1 = dw[pk(d1, c)], w2 = dw[pk(d2, c)];
        T0[c] = __fma_rn(gA2, w2, __fma_rn(gA1, w1, __dmul_rn(gA0, w0)));
        T1[c] = __fma_rn(gB2, w2, __fma_rn(gB1, w1, __dmul_rn(gB0, w0)));
      }
    }
    // blocks (a0, b) for b = a0 .. NP-1, then (a1, b) for b = a1 .. NP-1
#pragma unroll
    for (int k = 0; k < NBLK; ++k) {
      const bool first = k < NP - a0;
      const int b = first ? a0 + k : a1 + (k - (NP - a0));
      const bool ok = first || (twin && k - (NP - a0) < NP - a1);
      const double* T = first ? T0 : T1;
      const double* h = st + (ok ? b : NP - 1) * 3;
      const double h0 = h[0], h1 = h[1], h2 = h[2];
      acc[k][0] = __fma_rn(T[5], h2, __fma_rn(T[3], h1, __fma_rn(T[0], h0, acc[k][0])));
      acc[k][1] = __fma_rn(T[4], h2, __fma_rn(T[3], h0, __fma_rn(T[1], h1, acc[k][1])));
      acc[k][2] = __fma_rn(T[5], h0, __fma_rn(T[4], h1, __fma_rn(T[2], h2, acc[k][2])));
    }
  }
#pragma unroll
  for (int k = 0; k < NBLK; ++k) {
    const bool first = k < NP - a0;
    const int b = first ? a0 + k : a1 + (k - (NP - a0));
    const bool ok = first || (twin && k - (NP - a0) < NP - a1);
    if (!ok) continue;
    EPFEM_CHECK(blk_index<NP>(first ? a0 : a1, b) < C::NB && b < NP);
    double* o = rec + blk_index<NP>(first ? a0 : a1, b) * D2 + i * 3;
    o[0] = acc[k][0];
    o[1] = acc[k][1];
    o[2] = acc[k][2];
  }
}

// Cyclic row pairs (even NP: Q1 hexahedra, P2 tetrahedra).  delta_pairs3's
// lane (pair p, component i) needs T_a for its first NP - p blocks and T_a'
// after that; with p a per-lane value every block selects its T row (12 FSEL
// per block).  Here a symmetric block {a, b} is owned by the row from which b
// lies 0 .. H = NP / 2 steps ahead cyclically (b - a mod NP in [0, H), or
// = H with a < H), and lane r in [0, H) owns rows r and r + H: blocks
// (r, r + k mod NP) for k = 0 .. H with T_r, then (r + H, r + H + k mod NP)
// for k = 0 .. H - 1 with T_{r+H}.  The T row of every block is a constant,
// the same NP + 1 blocks per lane and the same (optimal) FMA count.  A block
// whose column node precedes its row node is the transpose of a stored
// (a <= b) block: the lane writes its row i as that block's column i.  The
// standalone element-delta kernel (k_elem_delta_staged) uses the same
// function, so fused and separate paths give the same bits.
#ifndef EPFEM_CYC3
#define EPFEM_CYC3 1
#endif
template <int NP>
struct UseCyc3 {
  static constexpr bool value = EPFEM_CYC3 && NP % 2 == 0 && NP < 20;  // Q2-20 keeps its chunks
};
template <int NP, int NQ>
__device__ __forceinline__ void delta_cyc3(const double* st_e, unsigned mask, int r, int i,
                                           double* __restrict__ rec) {
  static_assert(NP % 2 == 0, "cyclic row pairs need an even node count");
  using C = Pair3Cfg<NP, NQ>;
  constexpr int NS = C::NS, REC = C::REC, D2 = C::D2, NBLK = C::NBLK, H = NP / 2;
  const int R0 = r, R1 = r + H;
  const int d0 = i, d1 = i == 2 ? 4 : 3, d2 = i == 0 ? 5 : (i == 1 ? 4 : 5);
  const int e1 = i == 0 ? 1 : (i == 1 ? 0 : 1), e2 = i == 0 ? 2 : (i == 1 ? 2 : 0);
  auto pk = [](int a, int b) {
    const int lo = a < b ? a : b, hi = a < b ? b : a;
    return lo * NS - lo * (lo - 1) / 2 + (hi - lo);
  };
  // column node of block k (k <= H: row R0, else row R1)
  auto col = [&](int k) {
    const int c = k <= H ? R0 + k : R1 + (k - H - 1);
    return c >= NP ? c - NP : c;
  };
  double acc[NBLK][3];
#pragma unroll
  for (int k = 0; k < NBLK; ++k) acc[k][0] = acc[k][1] = acc[k][2] = 0.0;
  while (mask) {
    const int q = __ffs(mask) - 1;
    mask &= mask - 1u;
    const double* st = st_e + q * REC;
    const double* dw = st + NP * 3;
    double T0[NS], T1[NS];
    {
      const double* g0 = st + R0 * 3;
      const double* g1 = st + R1 * 3;
      const double gA0 = g0[d0], gA1 = g0[e1], gA2 = g0[e2];
      const double gB0 = g1[d0], gB1 = g1[e1], gB2 = g1[e2];
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        const double w0 = dw[pk(d0, c)], w1 = dw[pk(d1, c)], w2 = dw[pk(d2, c)];
        T0[c] = __fma_rn(gA2, w2, __fma_rn(gA1, w1, __dmul_rn(gA0, w0)));
        T1[c] = __fma_rn(gB2, w2, __fma_rn(gB1, w1, __dmul_rn(gB0, w0)));
      }
    }
#pragma unroll
    for (int k = 0; k < NBLK; ++k) {
      const double* T = k <= H ? T0 : T1;
      const double* h = st + col(k) * 3;
      const double h0 = h[0], h1 = h[1], h2 = h[2];
      acc[k][0] = __fma_rn(T[5], h2, __fma_rn(T[3], h1, __fma_rn(T[0], h0, acc[k][0])));
      acc[k][1] = __fma_rn(T[4], h2, __fma_rn(T[3], h0, __fma_rn(T[1], h1, acc[k][1])));
      acc[k][2] = __fma_rn(T[5], h0, __fma_rn(T[4], h1, __fma_rn(T[2], h2, acc[k][2])));
    }
  }
#pragma unroll
  for (int k = 0; k < NBLK; ++k) {
    const int a = k <= H ? R0 : R1, b = col(k);
    if (b >= a) {
      EPFEM_CHECK(blk_index<NP>(a, b) < C::NB);
      double* o = rec + blk_index<NP>(a, b) * D2 + i * 3;
      o[0] = acc[k][0];
      o[1] = acc[k][1];
      o[2] = acc[k][2];
    } else {  // block (b, a) = this block transposed: row i here is its column i
      EPFEM_CHECK(blk_index<NP>(b, a) < C::NB);
      double* o = rec + blk_index<NP>(b, a) * D2 + i;
      o[0] = acc[k][0];
      o[3] = acc[k][1];
      o[6] = acc[k][2];
    }
  }
}
// The 3D row-pair phase 2 of one (element, lane k < PL) task.
template <int NP, int NQ>
__device__ __forceinline__ void delta_rowpair3(const double* st_e, unsigned mask, int k,
                                               double* __restrict__ rec) {
  if constexpr (UseCyc3<NP>::value)
    delta_cyc3<NP, NQ>(st_e, mask, k / 3, k % 3, rec);
  else
    delta_pairs3<NP, NQ>(st_e, mask, k / 3, k % 3, rec);
}

// 2D row pairs (delta_pairs3's scheme with dim 2): lane (element, pair p,
// component i) owns row i of block rows p and NP - 1 - p; 2 * ceil(NP / 2)
// lanes per element (8 for Q2-8), NP + 1 blocks per lane, optimal FMA count.
// Per-entry sequences are delta_phase2's, so the bits are identical.
template <int NP>
__device__ __forceinline__ void delta_pairs2(const double* st_e, unsigned mask, int p, int i, int REC,
                                             double* __restrict__ rec) {
  constexpr int NS = 3, D2 = 4, NBLK = NP + 1;
  const int a0 = p, a1 = NP - 1 - p;
  const bool twin = a1 != a0;
  // T row i (delta_phase2): i = 0: g0 Dw(0, c) then g1 Dw(2, c); i = 1: g1 Dw(1, c) then g0 Dw(2, c)
  auto pk = [](int r, int c) {
    const int lo = r < c ? r : c, hi = r < c ? c : r;
    return lo * NS - lo * (lo - 1) / 2 + (hi - lo);
  };
  double acc[NBLK][2];
#pragma unroll
  for (int k = 0; k < NBLK; ++k) acc[k][0] = acc[k][1] = 0.0;
  while (mask) {
    const int q = __ffs(mask) - 1;
    mask &= mask - 1u;
    const double* st = st_e + q * REC;
    const double* dw = st + NP * 2;
    double T0[NS], T1[NS];
    {
      const double gA0 = st[a0 * 2 + i], gA1 = st[a0 * 2 + (1 - i)];
      const double gB0 = st[a1 * 2 + i], gB1 = st[a1 * 2 + (1 - i)];
#pragma unroll
      for (int c = 0; c < NS; ++c) {
        const double w0 = dw[pk(i, c)], w1 = dw[pk(2, c)];
        T0[c] = __fma_rn(gA1, w1, __dmul_rn(gA0, w0));
        T1[c] = __fma_rn(gB1, w1, __dmul_rn(gB0, w0));
      }
    }
#pragma unroll
    for (int k = 0; k < NBLK; ++k) {
      const bool first = k < NP - a0;
      const int b = first ? a0 + k : a1 + (k - (NP - a0));
      const bool ok = first || (twin && k - (NP - a0) < NP - a1);
      const double* T = first ? T0 : T1;
      const double* h = st + (ok ? b : NP - 1) * 2;
      const double h0 = h[0], h1 = h[1];
      acc[k][0] = __fma_rn(T[2], h1, __fma_rn(T[0], h0, acc[k][0]));
      acc[k][1] = __fma_rn(T[2], h0, __fma_rn(T[1], h1, acc[k][1]));
    }
  }
#pragma unroll
  for (int k = 0; k < NBLK; ++k) {
    const bool first = k < NP - a0;
    const int b = first ? a0 + k : a1 + (k - (NP - a0));
    const bool ok = first || (twin && k - (NP - a0) < NP - a1);
    if (!ok) continue;
    double* o = rec + blk_index<NP>(first ? a0 : a1, b) * D2 + i * 2;
    o[0] = acc[k][0];
    o[1] = acc[k][1];
  }
}

// ---------------------------------------------------------------------------
// Tensor-core phase 2: dK_e = sum_q B_q^T (Dw_q B_q) on the FP64 tensor pipe
// (mma.sync m8n8k4 f64, SASS DMMA.8x8x4; B200 runs it at the vector-FP64
// rate but each instruction is 256 FMA, so the warp issues ~10x fewer
// instructions and holds 2 accumulators per 8x8 tile instead of whole
// blocks).  The element's dofs (node-major, dim per node) are cut into 8-dof
// tiles; only upper tiles (I <= J) are formed.  Per plastic point and k-step
// lane (g = lane / 4, t = lane % 4) supplies A[g][t] = B[4ks + t][8I + g] and
// Y[t][g] = (Dw B)[4ks + t][8J + g]; rows past NS and dofs past NDOF are 0.
// The warp owns one element at a time (warp-uniform loop over its plastic
// points), so there is no per-lane chunking.  Records are the same symmetric
// block layout as delta_phase2; a diagonal block split across two tiles
// (3D nodes whose dofs straddle an 8-dof boundary) gets its lower entries
// mirrored from the upper tile.
template <int DIM, int NP, int NQ>
struct MmaCfg {
  static constexpr int NS = DIM == 3 ? 6 : 3;
  static constexpr int NSP = NS * (NS + 1) / 2;
  static constexpr int D2 = DIM * DIM;
  static constexpr int NB = NP * (NP + 1) / 2;
  static constexpr int REC = NP * DIM + NSP;  // staged doubles per point (as delta_phase2)
  static constexpr int RECB = NB * D2;        // workspace doubles per element
  static constexpr int NDOF = DIM * NP;
  static constexpr int NT8 = (NDOF + 7) / 8;
  static constexpr int NSYM = NT8 * (NT8 + 1) / 2;
  static constexpr int KS = (NS + 3) / 4;
  static constexpr int TPP = NSYM <= 12 ? NSYM : 12;  // tiles per pass (accumulator budget)
  static constexpr int NPASS = (NSYM + TPP - 1) / TPP;
  static constexpr int EPW = 32 / NQ;                 // elements per warp (phase 1 lanes)
  static constexpr int OUTB = EPW * RECB * 8 <= 4096 ? EPW : 2;  // output record buffers per warp
  // warps per CTA: keeps the static shared memory (staged records + output
  // buffers) under 48 KB
  static constexpr int WPB = DIM == 2 ? 4 : (NQ >= 27 ? 1 : 2);
  static constexpr int THREADS = 32 * WPB;
  static constexpr int tile_i(int s) {
    int i = 0;
    while (s >= NT8 - i) {
      s -= NT8 - i;
      ++i;
    }
    return i;
  }
  static constexpr int tile_j(int s) {
    int i = 0;
    while (s >= NT8 - i) {
      s -= NT8 - i;
      ++i;
    }
    return i + s;
  }
};

__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// B[k][(node, comp)] of the strain-displacement operator from the node's
// physical gradient g (assembly.cpp:86-100 row order)
template <int DIM>
__device__ __forceinline__ double b_entry(int k, int comp, const double* g) {
  // 2 bits per (k, comp): index into g, 3 = structural zero
  // 3D rows k: (g0,-,-) (-,g1,-) (-,-,g2) (g1,g0,-) (-,g2,g1) (g2,-,g0); 2D: (g0,-) (-,g1) (g1,g0)
  constexpr unsigned long long T3 = 0x39bc6fdfcull;
  constexpr unsigned long long T2 = 0x17cull;
  const int idx = DIM == 3 ? (int)((T3 >> (2 * (k * 3 + comp))) & 3u) : (int)((T2 >> (2 * (k * 2 + comp))) & 3u);
  return idx == 0 ? g[0] : idx == 1 ? g[1] : (DIM == 3 && idx == 2) ? g[DIM - 1] : 0.0;
}

// (Dw B)[k][(node, j)] = sum_m Dw[k][d_m(j)] g[e_m(j)], fixed order
template <int DIM>
__device__ __forceinline__ double y_entry(int k, int j, const double* g, const double* dw) {
  constexpr int NS = DIM == 3 ? 6 : 3;
  auto pk = [](int r, int c) {
    const int lo = r < c ? r : c, hi = r < c ? c : r;
    return lo * NS - lo * (lo - 1) / 2 + (hi - lo);
  };
  if constexpr (DIM == 3) {
    // j=0: (0,g0) (3,g1) (5,g2); j=1: (1,g1) (3,g0) (4,g2); j=2: (2,g2) (4,g1) (5,g0)
    const int d1 = j == 2 ? 4 : 3, d2 = j == 0 ? 5 : (j == 1 ? 4 : 5);
    const double gj = j == 0 ? g[0] : j == 1 ? g[1] : g[2];
    const double ge1 = j == 0 ? g[1] : j == 1 ? g[0] : g[1];
    const double ge2 = j == 0 ? g[2] : j == 1 ? g[2] : g[0];
    double s = __dmul_rn(dw[pk(k, j)], gj);
    s = __fma_rn(dw[pk(k, d1)], ge1, s);
    return __fma_rn(dw[pk(k, d2)], ge2, s);
  } else {
    // j=0: (0,g0) (2,g1); j=1: (1,g1) (2,g0)
    const double gj = j == 0 ? g[0] : g[1];
    const double go = j == 0 ? g[1] : g[0];
    return __fma_rn(dw[pk(k, 2)], go, __dmul_rn(dw[pk(k, j)], gj));
  }
}

// Phase 2 of IL elements on the tensor pipe, interleaved so that IL * TPP
// independent accumulator chains hide the DMMA latency: staged records
// st_w + le * NQ * REC (plastic points in masks[le]) -> symmetric block
// records recs[le] (shared memory).
template <int DIM, int NP, int NQ, int IL>
__device__ __forceinline__ void delta_mma_elements(const double* st_w, const unsigned* masks,
                                                   double* const* recs, int lane) {
  using M = MmaCfg<DIM, NP, NQ>;
  constexpr int NT8 = M::NT8, NDOF = M::NDOF, NS = M::NS, REC = M::REC, D2 = M::D2;
  const int g = lane >> 2, t = lane & 3;
  unsigned any = 0;
#pragma unroll
  for (int l = 0; l < IL; ++l) any |= masks[l];
#pragma unroll 1
  for (int pass = 0; pass < M::NPASS; ++pass) {
    double acc[IL][M::TPP][2];
#pragma unroll
    for (int l = 0; l < IL; ++l)
#pragma unroll
      for (int s = 0; s < M::TPP; ++s) acc[l][s][0] = acc[l][s][1] = 0.0;
    unsigned mk = any;
    while (mk) {
      const int q = __ffs(mk) - 1;
      mk &= mk - 1u;
#pragma unroll
      for (int l = 0; l < IL; ++l) {
        if (!((masks[l] >> q) & 1u)) continue;  // warp-uniform
        const double* st = st_w + (l * NQ + q) * REC;
        const double* dw = st + NP * DIM;
        double gv[NT8][DIM];
#pragma unroll
        for (int T = 0; T < NT8; ++T) {
          const int dof = 8 * T + g;
          const int node = dof < NDOF ? dof / DIM : 0;
#pragma unroll
          for (int c = 0; c < DIM; ++c) gv[T][c] = st[node * DIM + c];
        }
#pragma unroll
        for (int ks = 0; ks < M::KS; ++ks) {
          const int k = 4 * ks + t;
          double av[NT8], yv[NT8];
#pragma unroll
          for (int T = 0; T < NT8; ++T) {
            const int dof = 8 * T + g;
            const bool ok = dof < NDOF && k < NS;
            const int comp = dof % DIM;
            av[T] = ok ? b_entry<DIM>(k, comp, gv[T]) : 0.0;
            yv[T] = ok ? y_entry<DIM>(k, comp, gv[T], dw) : 0.0;
          }
#pragma unroll
          for (int s = 0; s < M::TPP; ++s) {
            const int sg = pass * M::TPP + s;
            if (sg < M::NSYM) dmma884(acc[l][s][0], acc[l][s][1], av[M::tile_i(sg)], yv[M::tile_j(sg)]);
          }
        }
      }
    }
#pragma unroll
    for (int l = 0; l < IL; ++l) {
      if (!masks[l]) continue;
      double* rec = recs[l];
#pragma unroll
      for (int s = 0; s < M::TPP; ++s) {
        const int sg = pass * M::TPP + s;
        if (sg >= M::NSYM) continue;
        const int I = M::tile_i(sg), J = M::tile_j(sg);
        const int row = 8 * I + g;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int col = 8 * J + 2 * t + e;
          if (row >= NDOF || col >= NDOF) continue;
          const int an = row / DIM, i = row % DIM, bn = col / DIM, jj = col % DIM;
          if (an < bn) {
            rec[blk_index<NP>(an, bn) * D2 + i * DIM + jj] = acc[l][s][e];
          } else if (an == bn) {
            rec[blk_index<NP>(an, an) * D2 + i * DIM + jj] = acc[l][s][e];
            if (I < J) rec[blk_index<NP>(an, an) * D2 + jj * DIM + i] = acc[l][s][e];
          }
        }
      }
    }
  }
}

// Phase 2 + workspace store for the EPW elements of a warp (after the staged
// records and the ballot `bal` of plastic points are in place).  2D: all EPW
// elements interleaved (EPW * RECB fits the output buffers); 3D: one at a
// time through OUTB = 2 rotating buffers.
template <int DIM, int NP, int NQ>
__device__ __forceinline__ void delta_mma_warp(const double* st_w, double* out_w, unsigned bal, int64_t e0,
                                               int64_t e_end, double* __restrict__ scratch, int lane) {
  using M = MmaCfg<DIM, NP, NQ>;
  constexpr unsigned QMASK = NQ >= 32 ? 0xffffffffu : (1u << NQ) - 1u;
  if constexpr (M::RECB % 2 != 0) {
    // records not 16-byte multiples (P2 tet: 495 doubles): no bulk copies,
    // one element at a time through the first buffer, coalesced lane stores
#pragma unroll 1
    for (int le = 0; le < M::EPW; ++le) {
      const unsigned mask = e0 + le < e_end ? (bal >> (le * NQ)) & QMASK : 0u;
      if (!mask) continue;  // warp-uniform
      double* rec = out_w;
      delta_mma_elements<DIM, NP, NQ, 1>(st_w + le * NQ * M::REC, &mask, &rec, lane);
      __syncwarp();
      double* dst = scratch + (size_t)(e0 + le) * M::RECB;
      for (int k = lane; k < M::RECB; k += 32) dst[k] = rec[k];
      __syncwarp();
    }
  } else if constexpr (M::OUTB == M::EPW) {
    unsigned masks[M::EPW];
    double* recs[M::EPW];
#pragma unroll
    for (int le = 0; le < M::EPW; ++le) {
      masks[le] = e0 + le < e_end ? (bal >> (le * NQ)) & QMASK : 0u;
      recs[le] = out_w + le * M::RECB;
    }
    if (!bal) return;
    delta_mma_elements<DIM, NP, NQ, M::EPW>(st_w, masks, recs, lane);
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      for (int le = 0; le < M::EPW; ++le)
        if (masks[le])
          tma_store_1d(scratch + (size_t)(e0 + le) * M::RECB, recs[le], (unsigned)(M::RECB * sizeof(double)));
      tma_store_wait_read();
    }
  } else {
    int issued = 0;
#pragma unroll 1
    for (int le = 0; le < M::EPW; ++le) {
      const unsigned mask = e0 + le < e_end ? (bal >> (le * NQ)) & QMASK : 0u;
      if (!mask) continue;  // warp-uniform
      double* rec = out_w + (issued % M::OUTB) * M::RECB;
      if (issued >= M::OUTB) {  // the buffer's previous bulk store must have read it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(M::OUTB - 1) : "memory");
        __syncwarp();
      }
      delta_mma_elements<DIM, NP, NQ, 1>(st_w + le * NQ * M::REC, &mask, &rec, lane);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        tma_store_1d(scratch + (size_t)(e0 + le) * M::RECB, rec, (unsigned)(M::RECB * sizeof(double)));
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
      ++issued;
    }
    if (issued && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

}  // namespace epfem_gpu
