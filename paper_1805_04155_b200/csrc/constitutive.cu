// K1: per-integration-point constitutive update (sm_100a), standalone and
// fused with the element tangent delta (epfem_newton_step).
//
// One thread per integration point.  Reads E, Ep_prev [, Hard_prev] (48 B
// each, AoS like the reference's 6 x n_int column-major Mat) and writes
//   * S (48 B) at every point,
//   * one flag byte (plastic / smooth / apex),
//   * the packed 21-entry tangent (192 B incl. pad = 6 full sectors) ONLY at
//     plastic points — elastic points reuse the cached elastic operator,
// plus the optional reference-layout outputs (full DS, masks, Ep, Hard, crit)
// when the caller asks for them.
//
// This file is compiled with --fmad=false and evaluates every expression in
// the reference's operation order (constitutive.cpp:90-196, voigt.hpp:11-51),
// so S, D and — what parity requires bit-exactly — the plastic/elastic
// decision (crit <= 0 is elastic, constitutive.cpp:117,169,172) reproduce the
// oracle's bits.  The kernel is HBM-bound, so the lost FMA contraction costs
// nothing measurable; the fused delta math uses explicit __fma_rn (delta.cuh).
//
// k_newton_fused: a CTA owns EPB whole elements (their points are
// contiguous, m = e * NQ + q).  Phase 1 = the point update above; at plastic
// points the thread also stages dphi and w (D - C) for the element delta
// straight from registers (D is never re-read).  Phase 2 builds dK_e
// (delta.cuh).  The row stream (tangent.cu) then assembles K.
#include <algorithm>
#include <climits>
#include <type_traits>

#include "delta.cuh"

namespace epfem_gpu {

namespace {

// k_newton_fused's CTA shape: DeltaCfg's, except for Q1 hexahedra with the
// row-pair phase 2.  There a CTA owns EPB_Q1 = 16 elements on 128 threads =
// one thread per point, so no thread idles in phase 1, and phase 2's 12 row-pair
// lanes per element run in rounds over the CTA (the loop is strided).  Measured
// on B200, cfg4: 3.50 ms vs 3.88 ms for DeltaCfg's 10 elements on 120 threads,
// where a quarter of the warp samples waited at the phase barrier (threads with
// no point); 8 and 12 elements per CTA took 3.66 / 3.65 ms.  (For P2
// tetrahedra the same shape does not beat the warp kernel: 3.87 vs 3.70 ms.)
#ifndef EPFEM_EPB_Q1
#define EPFEM_EPB_Q1 16
#endif
// Q2-20: one element per 32-thread CTA (27 points on 27 lanes, then its 60
// phase-2 chunks in two rounds over the warp) at up to 16 CTAs/SM (128
// registers; shared memory admits 13).  Measured on B200, cfg5: fused 15.33 vs
// 16.04 ms for DeltaCfg's 2 elements on 128 threads (54 of them busy in phase
// 1); 2 elements on 64 threads: 15.69 ms; 1 element on 64 threads (its 60 chunks in
// one round, 8 CTAs/SM): 16.03 ms.  The row stream after it is launched
// without PDL (tangent.cu): its early CTAs slowed this many-CTA grid (step
// 25.6 ms with PDL, 24.76 ms without).  EPFEM_EPB_Q20=0 restores DeltaCfg.
#ifndef EPFEM_EPB_Q20
#define EPFEM_EPB_Q20 1
#endif
#ifndef EPFEM_THREADS_Q20
#define EPFEM_THREADS_Q20 32
#endif
#ifndef EPFEM_MINB_Q20
#define EPFEM_MINB_Q20 16
#endif
#ifndef EPFEM_Q1_DWQUAD
#define EPFEM_Q1_DWQUAD 1
#endif
template <int DIM, int NP, int NQ>
struct FusedCfg : DeltaCfg<DIM, NP, NQ> {
  using Base = DeltaCfg<DIM, NP, NQ>;
  static constexpr bool Q1 = DIM == 3 && NP == 8 && EPFEM_EPB_Q1 > 0;
  static constexpr bool Q20 = DIM == 3 && NP == 20 && EPFEM_EPB_Q20 > 0;
  static constexpr int EPB = Q1 ? EPFEM_EPB_Q1 : (Q20 ? EPFEM_EPB_Q20 : Base::EPB);
  static constexpr int THREADS = Q1 ? ((EPB * NQ + 31) / 32) * 32 : (Q20 ? EPFEM_THREADS_Q20 : Base::THREADS);
  static constexpr int MINB = Q20 ? EPFEM_MINB_Q20 : Base::MINB;
  static constexpr bool ROUNDS = THREADS < EPB * Base::NT;  // chunk phase 2 needs more than one pass
};

__device__ __forceinline__ double iota(int i) { return i < 3 ? 1.0 : 0.0; }
__device__ __forceinline__ double vol(int i, int j) { return iota(i) * iota(j); }
// DEV = diag(1,1,1,1/2,1/2,1/2) - VOL/3 (voigt.hpp:24-31)
__device__ __forceinline__ double devop(int i, int j) {
  return ((i == j) ? (i < 3 ? 1.0 : 0.5) : 0.0) - vol(i, j) / 3.0;
}
// C = K VOL + 2G DEV (voigt.hpp:33-36)
__device__ __forceinline__ double cel(double K, double G, int i, int j) {
  return K * vol(i, j) + 2.0 * G * devop(i, j);
}

// Streamed per-point inputs: three 16-byte read-only loads per 48-byte record
// (a lane's three loads share the lines the first one brings into L1; an
// L1::no_allocate variant measured slower, cfg2 fused 0.237 vs 0.215 ms).
__device__ __forceinline__ double2 ld_stream2(const double2* p) { return __ldg(p); }
__device__ __forceinline__ void load6(const double* p, int64_t q, double* v) {
  const double2* p2 = reinterpret_cast<const double2*>(p + 6 * q);
  const double2 a = ld_stream2(p2), b = ld_stream2(p2 + 1), c = ld_stream2(p2 + 2);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y;
}
__device__ __forceinline__ void store6(double* p, int64_t q, const double* v) {
  double2* p2 = reinterpret_cast<double2*>(p + 6 * q);
  p2[0] = make_double2(v[0], v[1]);
  p2[1] = make_double2(v[2], v[3]);
  p2[2] = make_double2(v[4], v[5]);
}
// Tangent block producer: f(i, j) gives D(i, j).  Writes the packed block
// (plastic points) and/or the reference 36-entry block.
template <class F>
__device__ __forceinline__ void write_tangent(const ConstArgs& a, int64_t q, bool plastic, F f) {
  if (a.D && plastic) {
    // entry k holds D(PR[k], PC[k]) (epfem_gpu.h); stored pairwise as soon as
    // computed so the block never lives in registers as a whole
    constexpr int PR[24] = {0, 0, 0, 1, 1, 3, 0, 0, 0, 1, 1, 1, 2, 2, 2, 2, 3, 3, 4, 4, 5, 0, 0, 0};
    constexpr int PC[24] = {0, 1, 3, 1, 3, 3, 2, 4, 5, 2, 4, 5, 2, 3, 4, 5, 4, 5, 4, 5, 5, 0, 0, 0};
    double2* d2 = reinterpret_cast<double2*>(a.D + (int64_t)EPFEM_D_STRIDE * q);
#pragma unroll
    for (int k = 0; k < EPFEM_D_STRIDE / 2; ++k) {
      const double x = 2 * k < 21 ? f(PR[2 * k], PC[2 * k]) : 0.0;
      const double y = 2 * k + 1 < 21 ? f(PR[2 * k + 1], PC[2 * k + 1]) : 0.0;
      d2[k] = make_double2(x, y);
    }
  }
  if (a.DS) {
    double2* d2 = reinterpret_cast<double2*>(a.DS + 36 * q);
#pragma unroll
    for (int k = 0; k < 18; ++k) {
      const int i0 = (2 * k) % 6, j0 = (2 * k) / 6;  // column-major 6x6
      const int i1 = (2 * k + 1) % 6, j1 = (2 * k + 1) / 6;
      d2[k] = make_double2(f(i0, j0), f(i1, j1));
    }
  }
}

struct NoSink {
  template <class F>
  __device__ __forceinline__ void operator()(F&&) const {}
};

// Where a point's E / Ep / Hard come from: global memory (grid-stride
// kernels) or a shared-memory tile filled by TMA (pipelined fused kernel).
struct GlobalIn {  // pointers by value: never take the address of the kernel arguments
  const double* E;
  const double* Ep;
  const double* H;
  __device__ __forceinline__ void e(int64_t q, double* v) const { load6(E, q, v); }
  __device__ __forceinline__ void ep(int64_t q, double* v) const { load6(Ep, q, v); }
  __device__ __forceinline__ void hard(int64_t q, double* v) const { load6(H, q, v); }
};
// E from registers (strain-fused kernel), Ep / Hard from global memory
struct RegEIn {
  const double* e6;
  const double* Ep;
  const double* H;
  __device__ __forceinline__ void e(int64_t, double* v) const {
#pragma unroll
    for (int i = 0; i < 6; ++i) v[i] = e6[i];
  }
  __device__ __forceinline__ void ep(int64_t q, double* v) const { load6(Ep, q, v); }
  __device__ __forceinline__ void hard(int64_t q, double* v) const { load6(H, q, v); }
};
// K8 at point m of element e for the strain-fused kernels: dphi of every
// node into the staged record st (for phase 2), E = B u into e6 (and E_out).
template <int DIM, int NP>
__device__ __forceinline__ void strain_point(const GatherArgs& g, int64_t e, int q, int64_t m, double* st,
                                             double* e6) {
  constexpr int D2 = DIM * DIM;
  double J[D2];
#pragma unroll
  for (int k = 0; k < D2; ++k) J[k] = __ldg(g.inv + m * D2 + k);
#pragma unroll
  for (int k = 0; k < 6; ++k) e6[k] = 0.0;
#pragma unroll 4
  for (int p = 0; p < NP; ++p) {
    const int32_t node = __ldg(g.elem + e * NP + p);
    double d[DIM], uu[DIM];
    point_dphi<DIM>(J, g.gradhat + (q * NP + p) * DIM, d);
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      uu[i] = __ldg(g.u + (int64_t)DIM * node + i);
      st[p * DIM + i] = d[i];
    }
    strain_accumulate<DIM>(d, uu, e6);
  }
  if (g.E_out) {
    double2* o = reinterpret_cast<double2*>(g.E_out + 6 * m);
    o[0] = make_double2(e6[0], e6[1]);
    o[1] = make_double2(e6[2], e6[3]);
    o[2] = make_double2(e6[4], e6[5]);
  }
}

// The return map at point q (constitutive.cpp:76-196).  `sink(f)` is called
// at plastic points with the tangent functor f(i, j) = D(i, j).  Returns the
// plastic flag.
// `ssink(s6)` (optional) receives the stress at every point (the fused
// internal-forces step stages w S for F = B^T (w S)).
struct NoSSink {
  __device__ __forceinline__ void operator()(const double*) const {}
};
template <int MODEL, class In, class Sink, class SSink = NoSSink>
__device__ __forceinline__ bool eval_point(const ConstArgs& a, int64_t q, const In& in, Sink& sink,
                                           SSink ssink = SSink{}) {
  const double G = a.G ? __ldg(a.G + q) : a.Gu;
  const double K = a.K ? __ldg(a.K + q) : a.Ku;
  double e[6], ep[6];
  in.e(q, e);
  if (a.Ep) in.ep(q, ep);
  else
#pragma unroll
    for (int i = 0; i < 6; ++i) ep[i] = 0.0;
  double etr[6], de[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) etr[i] = e[i] - ep[i];
  // dev_e = DEV * e_tr, summed in column order
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    double s = devop(i, 0) * etr[0];
#pragma unroll
    for (int k = 1; k < 6; ++k) s = s + devop(i, k) * etr[k];
    de[i] = s;
  }
  const double tr = (etr[0] + etr[1]) + etr[2];

  if (MODEL == EPFEM_MODEL_ELASTIC) {
    // S = C E (constitutive.cpp:76-88), evaluated on E itself
    double s6[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) {
      double s = cel(K, G, i, 0) * e[0];
#pragma unroll
      for (int k = 1; k < 6; ++k) s = s + cel(K, G, i, k) * e[k];
      s6[i] = s;
    }
    if (a.S) store6(a.S, q, s6);
    ssink(s6);
    if (a.flags) a.flags[q] = 0;
    if (a.pm) a.pm[q] = 0;
    if (a.sm) a.sm[q] = 0;
    if (a.am) a.am[q] = 0;
    const double z6[6] = {0, 0, 0, 0, 0, 0};
    if (a.Ep_out) store6(a.Ep_out, q, z6);
    if (a.Hard_out) store6(a.Hard_out, q, z6);
    write_tangent(a, q, false, [&](int i, int j) { return cel(K, G, i, j); });
    return false;
  } else if (MODEL == EPFEM_MODEL_VON_MISES) {
    // radial return with linear kinematic hardening (constitutive.cpp:105-134)
    const double am = a.p1 ? __ldg(a.p1 + q) : a.p1u;
    const double Y = a.p2 ? __ldg(a.p2 + q) : a.p2u;
    double h[6];
    if (a.Hard) in.hard(q, h);
    else
#pragma unroll
      for (int i = 0; i < 6; ++i) h[i] = 0.0;
    const double ktr = K * tr;
    double sig[6], s[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) sig[i] = ktr * iota(i) + 2.0 * G * de[i];
#pragma unroll
    for (int i = 0; i < 6; ++i) s[i] = 2.0 * G * de[i] - h[i];
    const double n1 = s[0] * s[0] + s[1] * s[1] + s[2] * s[2];
    const double n2 = s[3] * s[3] + s[4] * s[4] + s[5] * s[5];
    const double ns = sqrt(n1 + 2.0 * n2);
    const double crit = ns - Y;
    if (a.crit) a.crit[q] = crit;
    const bool plastic = !(crit <= 0.0);
    if (a.flags) a.flags[q] = plastic ? EPFEM_FLAG_PLASTIC : 0;
    if (a.pm) a.pm[q] = plastic;
    if (a.sm) a.sm[q] = 0;
    if (a.am) a.am[q] = 0;
    if (!plastic) {
      if (a.S) store6(a.S, q, sig);
      ssink(sig);
      if (a.Ep_out) store6(a.Ep_out, q, ep);
      if (a.Hard_out) store6(a.Hard_out, q, h);
      write_tangent(a, q, false, [&](int i, int j) { return cel(K, G, i, j); });
      return false;
    }
    double nh[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) nh[i] = s[i] / ns;
    const double denom = 2.0 * G + am;
    const double lam = crit / denom;
    double out[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) out[i] = sig[i] - 2.0 * G * lam * nh[i];
    if (a.S) store6(a.S, q, out);
    ssink(out);
    const double c4 = 4.0 * G * G / denom;
    const double cy = c4 * Y / ns;
    auto f = [&](int i, int j) {
      return cel(K, G, i, j) - c4 * devop(i, j) + cy * (devop(i, j) - nh[i] * nh[j]);
    };
    write_tangent(a, q, true, f);
    sink(f);
    if (a.Hard_out) {
#pragma unroll
      for (int i = 0; i < 6; ++i) out[i] = h[i] + (am * lam) * nh[i];
      store6(a.Hard_out, q, out);
    }
    if (a.Ep_out) {
#pragma unroll
      for (int i = 0; i < 6; ++i) out[i] = ep[i] + lam * (i < 3 ? nh[i] : nh[i] * 2.0);
      store6(a.Ep_out, q, out);
    }
    return true;
  } else {
    // Drucker-Prager perfect plasticity (constitutive.cpp:152-194)
    const double eta = a.p1 ? __ldg(a.p1 + q) : a.p1u;
    const double c = a.p2 ? __ldg(a.p2 + q) : a.p2u;
    const double sqrt2 = sqrt(2.0);
    double dot = etr[0] * de[0];
#pragma unroll
    for (int i = 1; i < 6; ++i) dot = dot + etr[i] * de[i];
    const double ne = sqrt(fmax(0.0, dot));
    const double rho = 2.0 * G * ne;
    const double p = K * tr;
    const double da = K * eta * eta;
    const double dsm = G + da;
    const double crit1 = rho / sqrt2 + eta * p - c;
    const double crit2 = eta * p - da * rho / (G * sqrt2) - c;
    double sig[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) sig[i] = p * iota(i) + 2.0 * G * de[i];
    const double z6[6] = {0, 0, 0, 0, 0, 0};
    if (a.Hard_out) store6(a.Hard_out, q, z6);  // evaluate_constitutive keeps Hard = 0 for DP
    if (crit1 <= 0.0) {
      if (a.flags) a.flags[q] = 0;
      if (a.pm) a.pm[q] = 0;
      if (a.sm) a.sm[q] = 0;
      if (a.am) a.am[q] = 0;
      if (a.S) store6(a.S, q, sig);
      ssink(sig);
      if (a.Ep_out) store6(a.Ep_out, q, ep);
      write_tangent(a, q, false, [&](int i, int j) { return cel(K, G, i, j); });
      return false;
    }
    if (crit2 <= 0.0) {
      if (a.flags) a.flags[q] = EPFEM_FLAG_PLASTIC | EPFEM_FLAG_SMOOTH;
      if (a.pm) a.pm[q] = 1;
      if (a.sm) a.sm[q] = 1;
      if (a.am) a.am[q] = 0;
      if (ne <= 0.0) {
        raise_dev(a.err, EPFEM_ERR_ZERO_DEVIATOR, (unsigned long long)q);
        return false;
      }
      const double lam = crit1 / dsm;
      double nh[6], mh[6], out[6];
#pragma unroll
      for (int i = 0; i < 6; ++i) nh[i] = de[i] / ne;
#pragma unroll
      for (int i = 0; i < 6; ++i) mh[i] = sqrt2 * G * nh[i] + K * eta * iota(i);
#pragma unroll
      for (int i = 0; i < 6; ++i) out[i] = sig[i] - lam * mh[i];
      if (a.S) store6(a.S, q, out);
      ssink(out);
      const double c1 = 2.0 * sqrt2 * G * G * lam / rho;
      auto f = [&](int i, int j) {
        return cel(K, G, i, j) - c1 * (devop(i, j) - nh[i] * nh[j]) - mh[i] * mh[j] / dsm;
      };
      write_tangent(a, q, true, f);
      sink(f);
      if (a.Ep_out) {
#pragma unroll
        for (int i = 0; i < 6; ++i) {
          const double nst = i < 3 ? nh[i] : nh[i] * 2.0;
          out[i] = ep[i] + lam * ((sqrt2 / 2.0) * nst + (eta / 3.0) * iota(i));
        }
        store6(a.Ep_out, q, out);
      }
      return true;
    }
    if (a.flags) a.flags[q] = EPFEM_FLAG_PLASTIC | EPFEM_FLAG_APEX;
    if (a.pm) a.pm[q] = 1;
    if (a.sm) a.sm[q] = 0;
    if (a.am) a.am[q] = 1;
    double out[6];
#pragma unroll
    for (int i = 0; i < 6; ++i) out[i] = (c / eta) * iota(i);
    if (a.S) store6(a.S, q, out);
    ssink(out);
    auto f = [&](int, int) { return 0.0; };
    write_tangent(a, q, true, f);
    sink(f);
    if (a.Ep_out) {
      const double sh = c / (3.0 * K * eta);
#pragma unroll
      for (int i = 0; i < 6; ++i) out[i] = e[i] - sh * iota(i);
      store6(a.Ep_out, q, out);
    }
    return true;
  }
}

// LEAN: the hot-path instance (S, flags, packed D only); the reference-layout
// outputs are compiled out so the kernel keeps its registers low.
template <int MODEL, bool LEAN>
__global__ void __launch_bounds__(256) k_constitutive(ConstArgs a) {
  if (LEAN) {
    a.DS = nullptr;
    a.Ep_out = a.Hard_out = nullptr;
    a.pm = a.sm = a.am = nullptr;
    a.crit = nullptr;
  }
  NoSink none;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < a.n; q += stride)
    eval_point<MODEL>(a, q, GlobalIn{a.E, a.Ep, a.Hard}, none);
}

// minBlocks: 1024 threads/SM in 2D (caps at 64 registers, measured faster); 0 in 3D
// leaves ptxas its own heuristic (126 registers; an explicit 1 gives 144 and
// is ~15% slower on cfg4).
template <int MODEL, int DIM, int NP, int NQ, bool FROM_U = false>
__global__ void __launch_bounds__(FusedCfg<DIM, NP, NQ>::THREADS, FusedCfg<DIM, NP, NQ>::MINB)
    k_newton_fused(ConstArgs c, GatherArgs g) {
  pdl_trigger();
  using Cfg = FusedCfg<DIM, NP, NQ>;
  constexpr int EPB = Cfg::EPB;
  __shared__ double s_st[EPB][NQ][Cfg::REC];
  __shared__ unsigned s_mask[EPB];
  c.DS = nullptr;  // hot path: S, flags, packed D only
  c.Ep_out = c.Hard_out = nullptr;
  c.pm = c.sm = c.am = nullptr;
  c.crit = nullptr;

  const int tid = threadIdx.x;
  const int64_t e0 = g.e_begin + (int64_t)blockIdx.x * EPB;
  if (tid < EPB) s_mask[tid] = 0u;
  __syncthreads();
  for (int k = tid; k < EPB * NQ; k += blockDim.x) {
    const int le = k / NQ, q = k - le * NQ;
    const int64_t e = e0 + le;
    if (e >= g.e_end) continue;
    const int64_t m = e * NQ + q;
    double* st = s_st[le][q];
    if constexpr (FROM_U) {
      double e6[6];
      strain_point<DIM, NP>(g, e, q, m, st, e6);
      auto stage = [&](auto&& f) {
        atomicOr(&s_mask[le], 1u << q);
        stage_dw<DIM>(st + NP * DIM, __ldg(g.weight + m), g, m, f);
      };
      eval_point<MODEL>(c, m, RegEIn{e6, c.Ep, c.Hard}, stage);
    } else {
      auto stage = [&](auto&& f) {
        atomicOr(&s_mask[le], 1u << q);
        stage_geometry<DIM, NP>(st, g.inv + m * Cfg::D2, g.gradhat, q);
        stage_dw<DIM>(st + NP * DIM, __ldg(g.weight + m), g, m, f);
      };
      eval_point<MODEL>(c, m, GlobalIn{c.E, c.Ep, c.Hard}, stage);
    }
  }
  __syncthreads();
  if (tid < EPB && e0 + tid < g.e_end) g.emask[e0 + tid] = s_mask[tid];
  // 3D (not Q2-20): phase 2 by balanced row pairs (delta_pairs3): every T
  // entry and block entry computed once (cfg4: 1,404 instead of 2,592 FMA per
  // plastic point)
  if constexpr (DIM == 3 && NP < 20) {
    using PC = Pair3Cfg<NP, NQ>;
    for (int t = tid; t < EPB * PC::PL; t += blockDim.x) {
      const int le = t / PC::PL, k = t - (t / PC::PL) * PC::PL;
      const int64_t e = e0 + le;
      const unsigned mask = s_mask[le];
      EPFEM_CHECK(!(e < g.e_end) || e < g.n_elements);
      if (e < g.e_end && mask) {
        if constexpr (Cfg::Q1 && EPFEM_Q1_DWQUAD && UseCyc3<NP>::value) {
          // Lane order inside an element: quads (r, i), (r + 1, i), (r, i + 1), (r + 1, i + 1) for
          // components {0, 1}, then the four row pairs of component 2.  The Dw loads (address by i)
          // are then "aabb / aaaa" per quad: one shared-memory wavefront instead of two
          // (profiles/r2_l1tex.md); the B-column loads stay at two.
          const int r = k < 8 ? 2 * (k >> 2) + (k & 1) : k - 8, ci = k < 8 ? (k >> 1) & 1 : 2;
          delta_cyc3<NP, NQ>(&s_st[le][0][0], mask, r, ci, g.scratch + (size_t)e * Cfg::NB * Cfg::D2);
        } else {
          delta_rowpair3<NP, NQ>(&s_st[le][0][0], mask, k, g.scratch + (size_t)e * Cfg::NB * Cfg::D2);
        }
      }
    }
    return;
  }
  // phase 2: uniform chunks (no divergent block branch) in sub-passes of SUB
  if constexpr (Cfg::ROUNDS) {
    for (int t = tid; t < EPB * Cfg::NT; t += blockDim.x) {
      const int le = t / Cfg::NT;
      const int64_t e = e0 + le;
      const unsigned mask = s_mask[le];
      if (e < g.e_end && mask) {
        int a, c0;
        chunk_of<NP, Cfg::CS>(t - le * Cfg::NT, a, c0);
        delta_chunk_uniform<DIM, NP, Cfg::CS, Cfg::REC, Cfg::SUB>(&s_st[le][0][0], mask, a, c0,
                                                                  g.scratch + (size_t)e * Cfg::NB * Cfg::D2);
      }
    }
  } else if (tid < EPB * Cfg::NT) {
    const int le = tid / Cfg::NT;
    const int64_t e = e0 + le;
    const unsigned mask = s_mask[le];
    if (e < g.e_end && mask) {
      int a, c0;
      chunk_of<NP, Cfg::CS>(tid - le * Cfg::NT, a, c0);
      delta_chunk_uniform<DIM, NP, Cfg::CS, Cfg::REC, Cfg::SUB>(&s_st[le][0][0], mask, a, c0,
                                                                g.scratch + (size_t)e * Cfg::NB * Cfg::D2);
    }
  }
}

// k_newton_warp (2D): the fused kernel with warp-owned elements (WarpCfg,
// delta.cuh).  Lane l < EPW * NQ updates point q = l % NQ of element l / NQ;
// the warp's plastic masks are one ballot; phase-2 lane l < EPW * NT builds
// chunk l % NT of element l / NT.  No CTA barrier anywhere.  (Measured on
// B200, cfg2: a persistent grid-stride version is ~10% slower, and adding a
// cp.async prefetch of the next group's inputs slower still.)
#ifndef EPFEM_WARP_MINB
#define EPFEM_WARP_MINB 5
#endif
// One warp's group of EPW elements starting at e0: st_w = the warp's staged
// records (EPW * NQ * REC doubles), out_w = its element-record buffer
// (EPW * RECB doubles, 16-byte aligned).
template <int MODEL, int NP, int NQ, bool FROM_U>
__device__ __forceinline__ void newton_warp_group(ConstArgs c, const GatherArgs& g, int64_t e0, double* st_w,
                                                  double* out_w, int lane) {
  constexpr int DIM = 2;
  using W = WarpCfg<DIM, NP, NQ>;
  static_assert(W::EPW * NQ <= 32 && W::EPW * W::NT <= 32, "warp mapping");
  constexpr int EPW = W::EPW, REC = W::REC;
  constexpr unsigned QMASK = NQ >= 32 ? 0xffffffffu : (1u << NQ) - 1u;
  constexpr int RECB = W::NB * W::D2;  // doubles per element workspace record
  c.DS = nullptr;  // hot path: S, flags, packed D only
  c.Ep_out = c.Hard_out = nullptr;
  c.pm = c.sm = c.am = nullptr;
  c.crit = nullptr;
  if (e0 >= g.e_end) return;  // warp-uniform
  bool plastic = false;
  if (lane < EPW * NQ) {
    const int le = lane / NQ, q = lane - le * NQ;
    const int64_t e = e0 + le;
    if (e < g.e_end) {
      const int64_t m = e * NQ + q;
      double* st = st_w + lane * REC;
      if constexpr (FROM_U) {
        // K8 fused: dphi of every node (staged for phase 2 right away) and
        // E = B u from the element's nodal displacements, in registers
        double J[W::D2];
        {
          const double2* p2 = reinterpret_cast<const double2*>(g.inv + m * W::D2);
#pragma unroll
          for (int k = 0; k < W::D2 / 2; ++k) {
            const double2 v = __ldg(p2 + k);
            J[2 * k] = v.x;
            J[2 * k + 1] = v.y;
          }
        }
        double e6[6] = {0, 0, 0, 0, 0, 0};
#pragma unroll 4
        for (int p = 0; p < NP; ++p) {
          const int32_t node = __ldg(g.elem + e * NP + p);
          double d[DIM], uu[DIM];
          point_dphi<DIM>(J, g.gradhat + (q * NP + p) * DIM, d);
#pragma unroll
          for (int i = 0; i < DIM; ++i) {
            uu[i] = __ldg(g.u + (int64_t)DIM * node + i);
            st[p * DIM + i] = d[i];
          }
          strain_accumulate<DIM>(d, uu, e6);
        }
        if (g.E_out) {
          double2* o = reinterpret_cast<double2*>(g.E_out + 6 * m);
          o[0] = make_double2(e6[0], e6[1]);
          o[1] = make_double2(e6[2], e6[3]);
          o[2] = make_double2(e6[4], e6[5]);
        }
        const double wq = __ldg(g.weight + m);
        auto stage = [&](auto&& f) { stage_dw<DIM>(st + NP * DIM, wq, g, m, f); };
        plastic = eval_point<MODEL>(c, m, RegEIn{e6, c.Ep, c.Hard}, stage);
      } else {
        // J^-1 and w are loaded with E / Ep / Hard, before the return map, so
        // plastic points do not pay a second dependent memory round trip
        double jinv[W::D2];
        {
          const double2* p2 = reinterpret_cast<const double2*>(g.inv + m * W::D2);
#pragma unroll
          for (int k = 0; k < W::D2 / 2; ++k) {
            const double2 v = ld_stream2(p2 + k);
            jinv[2 * k] = v.x;
            jinv[2 * k + 1] = v.y;
          }
        }
        const double wq = __ldg(g.weight + m);
        auto stage = [&](auto&& f) {
          stage_geometry<DIM, NP, true>(st, jinv, g.gradhat, q);
          stage_dw<DIM>(st + NP * DIM, wq, g, m, f);
        };
        plastic = eval_point<MODEL>(c, m, GlobalIn{c.E, c.Ep, c.Hard}, stage);
      }
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, plastic);
  __syncwarp();
  if (lane < EPW && e0 + lane < g.e_end) g.emask[e0 + lane] = (bal >> (lane * NQ)) & QMASK;
  // phase 2 by row pairs: lane (element, pair, component), 2 ceil(NP/2) lanes per element
  constexpr int PL2 = 2 * ((NP + 1) / 2);
  for (int t = lane; t < EPW * PL2; t += 32) {  // one round except for P1 (EPW = 10)
    const int le = t / PL2, k = t - (t / PL2) * PL2;
    const unsigned mask = (bal >> (le * NQ)) & QMASK;
    if (e0 + le < g.e_end && mask)
      delta_pairs2<NP>(st_w + le * NQ * REC, mask, k / 2, k % 2, REC, out_w + le * RECB);
  }
  // the workspace records leave through the TMA unit: whole 1-KB-class
  // records instead of 8-byte scattered stores from every lane
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    int n = 0;
    for (int le = 0; le < EPW; ++le)
      if (e0 + le < g.e_end && ((bal >> (le * NQ)) & QMASK)) {
        tma_store_1d(g.scratch + (size_t)(e0 + le) * RECB, out_w + le * RECB, (unsigned)(RECB * sizeof(double)));
        ++n;
      }
    if (n) tma_store_wait_read();
  }
}

template <int MODEL, int NP, int NQ, bool FROM_U = false>
__global__ void __launch_bounds__(WarpCfg<2, NP, NQ>::THREADS, EPFEM_WARP_MINB)
    k_newton_warp(ConstArgs c, GatherArgs g) {
  pdl_trigger();
  using W = WarpCfg<2, NP, NQ>;
  __shared__ double s_st[W::WPB][W::EPW * NQ * W::REC];
  __shared__ __align__(16) double s_out[W::WPB][W::EPW * W::NB * W::D2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e0 = g.e_begin + ((int64_t)blockIdx.x * W::WPB + w) * W::EPW;
  newton_warp_group<MODEL, NP, NQ, FROM_U>(c, g, e0, s_st[w], s_out[w], lane);
}

// k_newton_warp3 (3D): warp-owned elements (EPW = 32 / NQ, all lanes busy in
// phase 1 for Q1), ballot masks, phase 2 by row pairs (delta_pairs3) in
// rounds of EPR elements.  No CTA barrier.
#ifndef EPFEM_WARP3_MINB
#define EPFEM_WARP3_MINB 4
#endif
template <int MODEL, int NP, int NQ, bool FROM_U = false>
__global__ void __launch_bounds__(Pair3Cfg<NP, NQ>::THREADS, EPFEM_WARP3_MINB)
    k_newton_warp3(ConstArgs c, GatherArgs g) {
  pdl_trigger();
  constexpr int DIM = 3;
  using W = Pair3Cfg<NP, NQ>;
  constexpr int EPW = W::EPW, REC = W::REC;
  constexpr unsigned QMASK = NQ >= 32 ? 0xffffffffu : (1u << NQ) - 1u;
  __shared__ double s_st[W::WPB][EPW * NQ * REC];
  c.DS = nullptr;  // hot path: S, flags, packed D only
  c.Ep_out = c.Hard_out = nullptr;
  c.pm = c.sm = c.am = nullptr;
  c.crit = nullptr;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e0 = g.e_begin + ((int64_t)blockIdx.x * W::WPB + w) * EPW;
  if (e0 >= g.e_end) return;  // warp-uniform
  double* st_w = s_st[w];
  bool plastic = false;
  if (lane < EPW * NQ) {
    const int le = lane / NQ, q = lane - le * NQ;
    const int64_t e = e0 + le;
    if (e < g.e_end) {
      const int64_t m = e * NQ + q;
      double* st = st_w + lane * REC;
      if constexpr (FROM_U) {
        double e6[6];
        strain_point<DIM, NP>(g, e, q, m, st, e6);
        auto stage = [&](auto&& f) { stage_dw<DIM>(st + NP * DIM, __ldg(g.weight + m), g, m, f); };
        plastic = eval_point<MODEL>(c, m, RegEIn{e6, c.Ep, c.Hard}, stage);
      } else {
        auto stage = [&](auto&& f) {
          stage_geometry<DIM, NP>(st, g.inv + m * W::D2, g.gradhat, q);
          stage_dw<DIM>(st + NP * DIM, __ldg(g.weight + m), g, m, f);
        };
        plastic = eval_point<MODEL>(c, m, GlobalIn{c.E, c.Ep, c.Hard}, stage);
      }
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, plastic);
  __syncwarp();
  if (lane < EPW && e0 + lane < g.e_end) g.emask[e0 + lane] = (bal >> (lane * NQ)) & QMASK;
#pragma unroll 1
  for (int r0 = 0; r0 < EPW; r0 += W::EPR) {
    if (lane < W::EPR * W::PL) {
      const int le = r0 + lane / W::PL, k = lane % W::PL;
      if (le < EPW && e0 + le < g.e_end) {
        const unsigned mask = (bal >> (le * NQ)) & QMASK;
        if (mask)
          delta_rowpair3<NP, NQ>(st_w + le * NQ * REC, mask, k, g.scratch + (size_t)(e0 + le) * W::NB * W::D2);
      }
    }
  }
}

// k_newton_mma: k_newton_warp's phase 1 (EPW = 32 / NQ elements per warp)
// followed by the tensor-core phase 2 (delta_mma_warp, delta.cuh).
#ifndef EPFEM_MMA_MINB
#define EPFEM_MMA_MINB 6
#endif
template <int MODEL, int DIM, int NP, int NQ>
__global__ void __launch_bounds__(MmaCfg<DIM, NP, NQ>::THREADS, DIM == 2 ? EPFEM_MMA_MINB : 0)
    k_newton_mma(ConstArgs c, GatherArgs g) {
  pdl_trigger();
  using M = MmaCfg<DIM, NP, NQ>;
  constexpr int EPW = M::EPW, REC = M::REC;
  constexpr unsigned QMASK = NQ >= 32 ? 0xffffffffu : (1u << NQ) - 1u;
  __shared__ double s_st[M::WPB][EPW * NQ * REC];
  __shared__ __align__(16) double s_out[M::WPB][M::OUTB * M::RECB];
  c.DS = nullptr;  // hot path: S, flags, packed D only
  c.Ep_out = c.Hard_out = nullptr;
  c.pm = c.sm = c.am = nullptr;
  c.crit = nullptr;

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t e0 = g.e_begin + ((int64_t)blockIdx.x * M::WPB + w) * EPW;
  if (e0 >= g.e_end) return;  // warp-uniform
  double* st_w = s_st[w];
  bool plastic = false;
  if (lane < EPW * NQ) {
    const int le = lane / NQ, q = lane - le * NQ;
    const int64_t e = e0 + le;
    if (e < g.e_end) {
      const int64_t m = e * NQ + q;
      double* st = st_w + lane * REC;
      auto stage = [&](auto&& f) {
        stage_geometry<DIM, NP>(st, g.inv + m * M::D2, g.gradhat, q);
        stage_dw<DIM>(st + NP * DIM, __ldg(g.weight + m), g, m, f);
      };
      plastic = eval_point<MODEL>(c, m, GlobalIn{c.E, c.Ep, c.Hard}, stage);
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, plastic);
  __syncwarp();
  if (lane < EPW && e0 + lane < g.e_end) g.emask[e0 + lane] = (bal >> (lane * NQ)) & QMASK;
  delta_mma_warp<DIM, NP, NQ>(st_w, s_out[w], bal, e0, g.e_end, g.scratch, lane);
}

// One fused launch over [g.e_begin, g.e_end): the kernel per element shape
// (2D: k_newton_warp; tetrahedra: k_newton_warp3; hexahedra: k_newton_fused;
// MMA: k_newton_mma, the FP64 tensor-pipe phase 2), instantiated per model.
template <class L>
void by_model(int model, L&& launch) {
  switch (model) {
    case EPFEM_MODEL_VON_MISES: launch(std::integral_constant<int, EPFEM_MODEL_VON_MISES>{}); break;
    case EPFEM_MODEL_DRUCKER_PRAGER: launch(std::integral_constant<int, EPFEM_MODEL_DRUCKER_PRAGER>{}); break;
    default: launch(std::integral_constant<int, EPFEM_MODEL_ELASTIC>{}); break;
  }
}

template <bool FROM_U>
int launch_fused_impl(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g, bool mma,
                      cudaStream_t st) {
  if (g.e_end <= g.e_begin) return 0;
  const int64_t n_e = g.e_end - g.e_begin;
  auto grid = [&](int64_t per) { return (unsigned)((n_e + per - 1) / per); };
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    if (!FROM_U && mma) {
      using M = MmaCfg<DIM, NP, NQ>;
      by_model(model, [&](auto md) {
        k_newton_mma<decltype(md)::value, DIM, NP, NQ><<<grid(M::EPW * M::WPB), M::THREADS, 0, st>>>(c, g);
      });
    } else if constexpr (DIM == 2) {
      using W = WarpCfg<DIM, NP, NQ>;
      by_model(model, [&](auto md) {
        k_newton_warp<decltype(md)::value, NP, NQ, FROM_U><<<grid(W::EPW * W::WPB), W::THREADS, 0, st>>>(c, g);
      });
    } else if constexpr (NP != 8 && NP != 20) {
      // tetrahedra: warp-owned elements (measured on cfg3: 3.61 vs 4.08 ms
      // for the CTA kernel; for Q1 hexahedra the CTA kernel is faster, 4.17
      // vs 4.73 ms)
      using W = Pair3Cfg<NP, NQ>;
      by_model(model, [&](auto md) {
        k_newton_warp3<decltype(md)::value, NP, NQ, FROM_U><<<grid(W::EPW * W::WPB), W::THREADS, 0, st>>>(c, g);
      });
    } else {
      using FC = FusedCfg<DIM, NP, NQ>;
      by_model(model, [&](auto md) {
        k_newton_fused<decltype(md)::value, DIM, NP, NQ, FROM_U><<<grid(FC::EPB), FC::THREADS, 0, st>>>(c, g);
      });
    }
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace

int launch_constitutive(int model, const ConstArgs& a, cudaStream_t st, int num_sms) {
  if (a.n == 0) return 0;
  // one point per thread: a grid capped at 16 CTAs per SM with a grid-stride
  // loop measured slower (cfg4 1.39 -> 1.21 ms at 25 % plastic, 4.27 -> 2.82 ms
  // at 100 %; cfg3 0.98 -> 0.82 ms; cfg5 1.79 -> 1.45 ms without the cap)
  (void)num_sms;
  const int threads = 256;
  int64_t blocks = (a.n + threads - 1) / threads;
  if (blocks > INT_MAX) blocks = INT_MAX;  // the kernel's loop covers the rest
  const bool lean = !a.DS && !a.Ep_out && !a.Hard_out && !a.pm && !a.sm && !a.am && !a.crit;
  switch (model) {
    case EPFEM_MODEL_ELASTIC:
      if (lean) k_constitutive<EPFEM_MODEL_ELASTIC, true><<<(int)blocks, threads, 0, st>>>(a);
      else k_constitutive<EPFEM_MODEL_ELASTIC, false><<<(int)blocks, threads, 0, st>>>(a);
      break;
    case EPFEM_MODEL_VON_MISES:
      if (lean) k_constitutive<EPFEM_MODEL_VON_MISES, true><<<(int)blocks, threads, 0, st>>>(a);
      else k_constitutive<EPFEM_MODEL_VON_MISES, false><<<(int)blocks, threads, 0, st>>>(a);
      break;
    case EPFEM_MODEL_DRUCKER_PRAGER:
      if (lean) k_constitutive<EPFEM_MODEL_DRUCKER_PRAGER, true><<<(int)blocks, threads, 0, st>>>(a);
      else k_constitutive<EPFEM_MODEL_DRUCKER_PRAGER, false><<<(int)blocks, threads, 0, st>>>(a);
      break;
    default: return fail(EPFEM_ERR_INVALID, "evaluate_constitutive: unknown material model");
  }
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

int launch_newton_fused_u(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g,
                          cudaStream_t st) {
  return launch_fused_impl<true>(model, family, dim, c, g, false, st);
}

// The DMMA phase 2 (k_newton_mma, mma.sync.m8n8k4.f64) is opt-in,
// EPFEM_FUSED=mma: parity-tested, and measured slower than the DFMA row
// pairs / chunks on B200 (cfg2 0.253 vs 0.211 ms, cfg4 14.7 vs 4.2 ms): the
// per-lane fragment gathers cost more issue slots than the DMMA saves.
int launch_newton_fused(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g,
                        cudaStream_t st) {
  static const bool mma = [] {
    const char* v = getenv("EPFEM_FUSED");
    return v && v[0] == 'm';
  }();
  return launch_fused_impl<false>(model, family, dim, c, g, mma, st);
}

}  // namespace epfem_gpu
