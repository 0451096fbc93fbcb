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
#include <map>
#include <mutex>
#include <climits>
#include <type_traits>

#include "rows.cuh"

#ifndef EPFEM_WARP_PAIRS
#define EPFEM_WARP_PAIRS 1  // 2D warp kernel: phase 2 by row pairs
#endif
#ifndef EPFEM_HALFPAIRS20
#define EPFEM_HALFPAIRS20 0  // Q2-20 CTA kernel with half row pairs (delta_pairs3_half): fewer FMA, but
                             // measured slower on cfg5 (21.1 vs 16.0 ms; shared-memory loads per FMA)
#endif
#ifndef EPFEM_CTA_PAIRS
#define EPFEM_CTA_PAIRS 1
#endif
#ifndef EPFEM_TSHARED
#define EPFEM_TSHARED 0  // 1: 3D CTA phase 2 with T_a shared through shared memory (measured slower: the per-point barriers)
#endif

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
// 1); 2 elements on 64 threads: 15.69 ms.  The row stream after it is launched
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
// Tuning hook for the 2D CTA kernel (EPFEM_FUSED=cta): EPB_2D elements on
// one thread per point at MINB_2D CTAs/SM, phase 2 in rounds.
#ifndef EPFEM_EPB_2D
#define EPFEM_EPB_2D 0
#endif
#ifndef EPFEM_MINB_2D
#define EPFEM_MINB_2D 4
#endif
template <int DIM, int NP, int NQ>
struct FusedCfg : DeltaCfg<DIM, NP, NQ> {
  using Base = DeltaCfg<DIM, NP, NQ>;
  static constexpr bool D2C = DIM == 2 && EPFEM_EPB_2D > 0;
  static constexpr bool Q1 = DIM == 3 && NP == 8 && EPFEM_CTA_PAIRS && !EPFEM_TSHARED && EPFEM_EPB_Q1 > 0;
  static constexpr bool Q20 = DIM == 3 && NP == 20 && !EPFEM_HALFPAIRS20 && !EPFEM_TSHARED && EPFEM_EPB_Q20 > 0;
  static constexpr int EPB = Q1 ? EPFEM_EPB_Q1 : (Q20 ? EPFEM_EPB_Q20 : (D2C ? EPFEM_EPB_2D : Base::EPB));
  static constexpr int THREADS = (Q1 || D2C) ? ((EPB * NQ + 31) / 32) * 32 : (Q20 ? EPFEM_THREADS_Q20 : Base::THREADS);
  static constexpr int MINB = Q20 ? EPFEM_MINB_Q20 : (D2C ? EPFEM_MINB_2D : Base::MINB);
  static constexpr bool ROUNDS = THREADS < EPB * Base::NT;  // chunk phase 2 needs more than one pass
};

__device__ __forceinline__ double iota(int i) { return i < 3 ? 1.0 : 0.0; }
__device__ __forceinline__ double vol(int i, int j) { return iota(i) * iota(j); }
// DEV = diag(1,1,1,1/2,1/2,1/2) - VOL/3 (voigt.hpp:62-69)
__device__ __forceinline__ double devop(int i, int j) {
  return ((i == j) ? (i < 3 ? 1.0 : 0.5) : 0.0) - vol(i, j) / 3.0;
}
// C = K VOL + 2G DEV (voigt.hpp:72-74)
__device__ __forceinline__ double cel(double K, double G, int i, int j) {
  return K * vol(i, j) + 2.0 * G * devop(i, j);
}

// Streamed per-point inputs.  EPFEM_LOAD_NA=1 skips L1 allocation
// (ld.global.nc.L1::no_allocate) to keep the reference tables L1-resident:
// measured slower (cfg2 fused 0.237 vs 0.215 ms): a lane's three 16-byte
// loads share lines that the first one brought into L1.
#ifndef EPFEM_LOAD_NA
#define EPFEM_LOAD_NA 0
#endif
__device__ __forceinline__ double2 ld_stream2(const double2* p) {
#if EPFEM_LOAD_NA
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
#else
  return __ldg(p);
#endif
}
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

struct SmemIn {
  const double* E;
  const double* Ep;
  const double* H;
  int li;  // point index inside the tile
  __device__ __forceinline__ static void ld(const double* p, int li, double* v) {
    const double2* p2 = reinterpret_cast<const double2*>(p + 6 * li);
    const double2 a = p2[0], b = p2[1], c = p2[2];
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y;
  }
  __device__ __forceinline__ void e(int64_t, double* v) const { ld(E, li, v); }
  __device__ __forceinline__ void ep(int64_t, double* v) const { ld(Ep, li, v); }
  __device__ __forceinline__ void hard(int64_t, double* v) const { ld(H, li, v); }
};

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

// L2 prefetch of the per-point inputs of the elements [e_lo, e_hi) (E, Ep,
// Hard, J^-1, w: all contiguous per element range), issued one occupancy
// wave ahead by the fused kernels: the global-load latency of a CTA's first
// phase (the top stall of the 2D kernel) becomes an L2 hit.
template <int DIM, int NQ>
__device__ __forceinline__ void prefetch_elements(const ConstArgs& c, const GatherArgs& g, int64_t e_lo,
                                                  int64_t e_hi) {
  e_lo = max(e_lo, g.e_begin);
  e_hi = min(e_hi, g.e_end);
  if (e_hi <= e_lo) return;
  const int64_t m0 = e_lo * NQ, n = (e_hi - e_lo) * NQ;
  const int k = threadIdx.x;
  if (k == 0) l2_prefetch_bulk(c.E + 6 * m0, sizeof(double) * 6 * n);
  if (k == 1) l2_prefetch_bulk(c.Ep ? c.Ep + 6 * m0 : nullptr, sizeof(double) * 6 * n);
  if (k == 2) l2_prefetch_bulk(c.Hard ? c.Hard + 6 * m0 : nullptr, sizeof(double) * 6 * n);
  if (k == 3) l2_prefetch_bulk(g.inv + DIM * DIM * m0, sizeof(double) * DIM * DIM * n);
  if (k == 4) l2_prefetch_bulk(g.weight + m0, sizeof(double) * n);
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
  if (!FROM_U && g.pf_dist > 0) {
    const int64_t eb = g.e_begin + ((int64_t)blockIdx.x + g.pf_dist) * EPB;
    prefetch_elements<DIM, NQ>(c, g, eb, eb + EPB);
  }
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
#if EPFEM_TSHARED
  if constexpr (DIM == 3) {
    __shared__ double s_T[EPB][NP][DIM * Cfg::NS];
    delta_phase2_tshared<DIM, NP, NQ>(s_st, s_mask, s_T, tid, blockDim.x, e0, g.e_end, g.scratch);
    return;
  }
#endif
#if EPFEM_CTA_PAIRS
  // 3D (not Q2-20): phase 2 by balanced row pairs (delta_pairs3): every T
  // entry and block entry computed once (cfg4: 1,404 instead of 2,592 FMA per
  // plastic point)
  if constexpr (DIM == 3 && NP < 20) {
    using PC = Pair3Cfg<NP, NQ>;
    for (int t = tid; t < EPB * PC::PL; t += blockDim.x) {
      const int le = t / PC::PL, k = t - (t / PC::PL) * PC::PL;
      const int64_t e = e0 + le;
      const unsigned mask = s_mask[le];
      if (e < g.e_end && mask)
        delta_pairs3<NP, NQ>(&s_st[le][0][0], mask, k / 3, k % 3, g.scratch + (size_t)e * Cfg::NB * Cfg::D2);
    }
    return;
  }
#endif
#if EPFEM_HALFPAIRS20
  // Q2-20: row pairs split in halves (delta_pairs3_half): lane (element,
  // pair, half, component)
  if constexpr (DIM == 3 && NP >= 20) {
    constexpr int PL = 6 * ((NP + 1) / 2);
    for (int t = tid; t < EPB * PL; t += blockDim.x) {
      const int le = t / PL, k = t - (t / PL) * PL;
      const int64_t e = e0 + le;
      const unsigned mask = s_mask[le];
      if (e < g.e_end && mask)
        delta_pairs3_half<NP, NQ>(&s_st[le][0][0], mask, k / 6, k % 3, (k / 3) % 2,
                                  g.scratch + (size_t)e * Cfg::NB * Cfg::D2);
    }
    return;
  }
#endif
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
#ifndef EPFEM_EXP
#define EPFEM_EXP 0  // timing experiments only: 1 = no phase 2, 2 = phase 2 without FP64 work
#endif
#ifndef EPFEM_EARLY_GEOM
#define EPFEM_EARLY_GEOM 1
#endif
// One warp's group of EPW elements starting at e0: st_w = the warp's staged
// records (EPW * NQ * REC doubles), out_w = its element-record buffer
// (EPW * RECB doubles, 16-byte aligned).  MEGA: the records leave through
// plain coalesced stores (the one-launch step publishes them with a release
// flag right after; no async-proxy writes to order).
// FORCES (internal forces fused, epfem_newton_step_f): every point also
// stages dphi and (w, S11, S22, S12) after its record (stride REC + 4), and
// lane (element, node p) forms the element's internal-force record
// F_e[p] = sum_q w_q B_p(q)^T S_q (the explicit-rounding sequence of
// k_internal_forces) into g.fws; the row stream folds the records per node.
template <int MODEL, int NP, int NQ, bool FROM_U, bool MEGA, bool FORCES = false>
__device__ __forceinline__ void newton_warp_group(ConstArgs c, const GatherArgs& g, int64_t e0, double* st_w,
                                                  double* out_w, int lane) {
  constexpr int DIM = 2;
  using W = WarpCfg<DIM, NP, NQ>;
  static_assert(W::EPW * NQ <= 32 && W::EPW * W::NT <= 32, "warp mapping");
  static_assert(!(FORCES && FROM_U), "the forces step reads E");
  constexpr int EPW = W::EPW, REC0 = W::REC, REC = REC0 + (FORCES ? 4 : 0);
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
#if EPFEM_EARLY_GEOM
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
      if constexpr (FORCES) stage_geometry<DIM, NP, true>(st, jinv, g.gradhat, q);
      auto stage = [&](auto&& f) {
        if constexpr (!FORCES) stage_geometry<DIM, NP, true>(st, jinv, g.gradhat, q);
        stage_dw<DIM>(st + NP * DIM, wq, g, m, f);
      };
#else
      auto stage = [&](auto&& f) {
        stage_geometry<DIM, NP>(st, g.inv + m * W::D2, g.gradhat, q);
        stage_dw<DIM>(st + NP * DIM, __ldg(g.weight + m), g, m, f);
      };
#endif
      if constexpr (FORCES) {
        auto ss = [&](const double* s6) {
          st[REC0] = wq;
          st[REC0 + 1] = s6[0];
          st[REC0 + 2] = s6[1];
          st[REC0 + 3] = s6[3];
        };
        plastic = eval_point<MODEL>(c, m, GlobalIn{c.E, c.Ep, c.Hard}, stage, ss);
      } else {
        plastic = eval_point<MODEL>(c, m, GlobalIn{c.E, c.Ep, c.Hard}, stage);
      }
      }
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, plastic);
  __syncwarp();
  if (lane < EPW && e0 + lane < g.e_end) g.emask[e0 + lane] = (bal >> (lane * NQ)) & QMASK;
#if EPFEM_WARP_PAIRS
  // phase 2 by row pairs: lane (element, pair, component), 2 ceil(NP/2) lanes per element
  constexpr int PL2 = 2 * ((NP + 1) / 2);
  for (int t = lane; t < EPW * PL2; t += 32) {  // one round except for P1 (EPW = 10)
    const int le = t / PL2, k = t - (t / PL2) * PL2;
    const unsigned mask = (bal >> (le * NQ)) & QMASK;
    if (e0 + le < g.e_end && mask)
      delta_pairs2<NP>(st_w + le * NQ * REC, mask, k / 2, k % 2, REC, out_w + le * RECB);
  }
  if (false) {
#else
  if (EPFEM_EXP != 1 && lane < EPW * W::NT) {
#endif
    const int le = lane / W::NT;
    const int64_t e = e0 + le;
    const unsigned mask = (bal >> (le * NQ)) & QMASK;
    if (e < g.e_end && mask) {
      int a, c0;
      chunk_of<NP, W::CS>(lane - le * W::NT, a, c0);
      double* rec = out_w + le * RECB;  // staged, then one bulk store per element
      if (EPFEM_EXP == 2) {  // same stores, staged values instead of the products
        const double* st = st_w + le * NQ * REC;
        for (int bb = 0; bb < W::CS && c0 + bb < NP; ++bb)
          for (int k = 0; k < W::D2; ++k) rec[blk_index<NP>(a, c0 + bb) * W::D2 + k] = st[bb * 4 + k];
      } else {
        delta_chunk_uniform<DIM, NP, W::CS, REC>(st_w + le * NQ * REC, mask, a, c0, rec);
      }
    }
  }
  if constexpr (FORCES) {
    // element internal-force records: lane (element, node p), points in order
    for (int t = lane; t < EPW * NP; t += 32) {
      const int le = t / NP, p = t - (t / NP) * NP;
      if (e0 + le >= g.e_end) continue;
      double f0 = 0.0, f1 = 0.0;
#pragma unroll 1
      for (int q = 0; q < NQ; ++q) {
        const double* r = st_w + (le * NQ + q) * REC;
        const double g0 = r[p * 2], g1 = r[p * 2 + 1];
        const double w = r[REC0], s0 = r[REC0 + 1], s1 = r[REC0 + 2], s3 = r[REC0 + 3];
        f0 = __fma_rn(w, __fma_rn(g1, s3, __dmul_rn(g0, s0)), f0);
        f1 = __fma_rn(w, __fma_rn(g0, s3, __dmul_rn(g1, s1)), f1);
      }
      double2* o = reinterpret_cast<double2*>(g.fws + ((e0 + le) * NP + p) * DIM);
      *o = make_double2(f0, f1);
    }
  }
  // the workspace records leave through the TMA unit: whole 1-KB-class
  // records instead of 8-byte scattered stores from every lane
  if (MEGA) {
    __syncwarp();
    for (int le = 0; le < EPW; ++le)
      if (e0 + le < g.e_end && ((bal >> (le * NQ)) & QMASK)) {
        const double2* s2 = reinterpret_cast<const double2*>(out_w + le * RECB);
        double2* d2 = reinterpret_cast<double2*>(g.scratch + (size_t)(e0 + le) * RECB);
        for (int k = lane; k < RECB / 2; k += 32) d2[k] = s2[k];
      }
  } else if (EPFEM_EXP != 1) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      int n = 0;
      for (int le = 0; le < EPW; ++le)
        if (e0 + le < g.e_end && ((bal >> (le * NQ)) & QMASK)) {
          tma_store_1d(g.scratch + (size_t)(e0 + le) * RECB, out_w + le * RECB,
                       (unsigned)(RECB * sizeof(double)));
          ++n;
        }
      if (n) tma_store_wait_read();
    }
  }
}

template <int MODEL, int NP, int NQ, bool FROM_U = false, bool FORCES = false>
__global__ void __launch_bounds__(WarpCfg<2, NP, NQ>::THREADS, EPFEM_WARP_MINB)
    k_newton_warp(ConstArgs c, GatherArgs g) {
  pdl_trigger();
  using W = WarpCfg<2, NP, NQ>;
  __shared__ double s_st[W::WPB][W::EPW * NQ * (W::REC + (FORCES ? 4 : 0))];
  __shared__ __align__(16) double s_out[W::WPB][W::EPW * W::NB * W::D2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (!FROM_U && g.pf_dist > 0) {
    const int64_t eb = g.e_begin + ((int64_t)blockIdx.x + g.pf_dist) * W::WPB * W::EPW;
    prefetch_elements<2, NQ>(c, g, eb, eb + W::WPB * W::EPW);
  }
  const int64_t e0 = g.e_begin + ((int64_t)blockIdx.x * W::WPB + w) * W::EPW;
  newton_warp_group<MODEL, NP, NQ, FROM_U, false, FORCES>(c, g, e0, s_st[w], s_out[w], lane);
}

// k_newton_warp_pf (2D, EPFEM_FUSED=pf): k_newton_warp with two element
// groups per warp; at entry lane 0 starts TMA bulk copies of the SECOND
// group's E / Ep / Hard / J^-1 (contiguous: the group's points are) into
// shared memory, so their latency hides behind the whole first group.
constexpr int PFW = 3;  // warps per CTA (static shared memory < 48 KB)
template <int MODEL, int NP, int NQ>
__global__ void __launch_bounds__(32 * PFW, EPFEM_WARP_MINB * 4 / 3)
    k_newton_warp_pf(ConstArgs c, GatherArgs g) {
  pdl_trigger();
  constexpr int DIM = 2;
  using W = WarpCfg<DIM, NP, NQ>;
  constexpr int EPW = W::EPW, REC = W::REC, PPG = EPW * NQ, D2 = W::D2;
  constexpr unsigned QMASK = NQ >= 32 ? 0xffffffffu : (1u << NQ) - 1u;
  constexpr int RECB = W::NB * W::D2;
  constexpr int IN_E = 0, IN_EP = 6 * PPG, IN_H = 12 * PPG, IN_J = 18 * PPG, IN_SIZE = IN_J + D2 * PPG;
  __shared__ double s_st[PFW][EPW * NQ * REC];
  __shared__ __align__(16) double s_out[PFW][EPW * RECB];
  __shared__ __align__(128) double s_in[PFW][IN_SIZE];
  __shared__ uint64_t s_bar[PFW];
  c.DS = nullptr;  // hot path: S, flags, packed D only
  c.Ep_out = c.Hard_out = nullptr;
  c.pm = c.sm = c.am = nullptr;
  c.crit = nullptr;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t n_groups = (g.e_end - g.e_begin + EPW - 1) / EPW;
  const int64_t grp0 = 2 * ((int64_t)blockIdx.x * PFW + w);
  if (grp0 >= n_groups) return;  // warp-uniform
  const bool has2 = grp0 + 1 < n_groups;
  double* st_w = s_st[w];
  double* in_w = s_in[w];
  if (lane == 0) {
    mbar_init(&s_bar[w], 1);
    mbar_init_fence();
  }
  __syncwarp();
  if (has2 && lane == 0) {
    const int64_t p0 = (g.e_begin + (grp0 + 1) * EPW) * NQ;
    const unsigned np = (unsigned)min((int64_t)PPG, g.e_end * NQ - p0);
    unsigned total = np * 48u + np * 8u * D2;
    if (c.Ep) total += np * 48u;
    if (c.Hard) total += np * 48u;
    mbar_expect_tx(&s_bar[w], total);
    tma_load_1d(in_w + IN_E, c.E + 6 * p0, np * 48u, &s_bar[w]);
    if (c.Ep) tma_load_1d(in_w + IN_EP, c.Ep + 6 * p0, np * 48u, &s_bar[w]);
    if (c.Hard) tma_load_1d(in_w + IN_H, c.Hard + 6 * p0, np * 48u, &s_bar[w]);
    tma_load_1d(in_w + IN_J, g.inv + D2 * p0, np * 8u * D2, &s_bar[w]);
  }
  auto group = [&](int64_t grp, auto from_smem) {
    constexpr bool SM = decltype(from_smem)::value;
    const int64_t e0 = g.e_begin + grp * EPW;
    bool plastic = false;
    if (lane < PPG) {
      const int le = lane / NQ, q = lane - le * NQ;
      const int64_t e = e0 + le;
      if (e < g.e_end) {
        const int64_t m = e * NQ + q;
        double* st = st_w + lane * REC;
        double jinv[D2];
#pragma unroll
        for (int k = 0; k < D2; ++k) jinv[k] = SM ? in_w[IN_J + lane * D2 + k] : __ldg(g.inv + m * D2 + k);
        const double wq = __ldg(g.weight + m);
        auto stage = [&](auto&& f) {
          stage_geometry<DIM, NP, true>(st, jinv, g.gradhat, q);
          stage_dw<DIM>(st + NP * DIM, wq, g, m, f);
        };
        if constexpr (SM)
          plastic = eval_point<MODEL>(c, m, SmemIn{in_w + IN_E, in_w + IN_EP, in_w + IN_H, lane}, stage);
        else
          plastic = eval_point<MODEL>(c, m, GlobalIn{c.E, c.Ep, c.Hard}, stage);
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, plastic);
    __syncwarp();
    if (lane < EPW && e0 + lane < g.e_end) g.emask[e0 + lane] = (bal >> (lane * NQ)) & QMASK;
    if (lane < EPW * W::NT) {
      const int le = lane / W::NT;
      const unsigned mask = (bal >> (le * NQ)) & QMASK;
      if (e0 + le < g.e_end && mask) {
        int a, c0;
        chunk_of<NP, W::CS>(lane - le * W::NT, a, c0);
        delta_chunk_uniform<DIM, NP, W::CS, REC>(st_w + le * NQ * REC, mask, a, c0, s_out[w] + le * RECB);
      }
    }
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      int n = 0;
      for (int le = 0; le < EPW; ++le)
        if (e0 + le < g.e_end && ((bal >> (le * NQ)) & QMASK)) {
          tma_store_1d(g.scratch + (size_t)(e0 + le) * RECB, s_out[w] + le * RECB,
                       (unsigned)(RECB * sizeof(double)));
          ++n;
        }
      if (n) tma_store_wait_read();
    }
    __syncwarp();  // staged records and output buffers are reused by the next group
  };
  group(grp0, std::false_type{});
  if (has2) {
    mbar_wait(&s_bar[w], 0);
    group(grp0 + 1, std::true_type{});
  }
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
  if (!FROM_U && g.pf_dist > 0) {
    const int64_t eb = g.e_begin + ((int64_t)blockIdx.x + g.pf_dist) * W::WPB * EPW;
    prefetch_elements<DIM, NQ>(c, g, eb, eb + W::WPB * EPW);
  }
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
          delta_pairs3<NP, NQ>(st_w + le * NQ * REC, mask, k / 3, k % 3,
                               g.scratch + (size_t)(e0 + le) * W::NB * W::D2);
      }
    }
  }
}

// k_newton_ws (2D): the warp kernel split by role inside a persistent CTA.
// P producer warps run phase 1 (one group of EPW elements at a time, like
// k_newton_warp) into a private double-buffered slot of staged records and
// hand it over through an mbarrier; CW consumer warps run phase 2 from the
// slots and bulk-store the element records.  The producers never wait on
// phase-2 arithmetic, so their loads keep streaming while the consumers'
// FP64 work proceeds on the other warps.
#ifndef EPFEM_WS_P
#define EPFEM_WS_P 6
#endif
#ifndef EPFEM_WS_C
#define EPFEM_WS_C 2
#endif
#ifndef EPFEM_WS_MINB
#define EPFEM_WS_MINB 3
#endif
#ifndef EPFEM_WS_SUB
#define EPFEM_WS_SUB 3
#endif
template <int NP, int NQ>
struct WsCfg {
  using W = WarpCfg<2, NP, NQ>;
  static constexpr int P = EPFEM_WS_P, CW = EPFEM_WS_C, THREADS = 32 * (P + CW);
  static constexpr int SLOT = W::EPW * NQ * W::REC;  // doubles per staged slot
  static constexpr int RECB = W::NB * W::D2;
  static constexpr size_t SMEM = sizeof(double) * ((size_t)P * 2 * SLOT + (size_t)CW * W::EPW * RECB);
};
template <int MODEL, int NP, int NQ>
__global__ void __launch_bounds__(WsCfg<NP, NQ>::THREADS, EPFEM_WS_MINB)
    k_newton_ws(ConstArgs c, GatherArgs g) {
  pdl_trigger();
  constexpr int DIM = 2;
  using W = WarpCfg<DIM, NP, NQ>;
  using S = WsCfg<NP, NQ>;
  constexpr int P = S::P, CW = S::CW, EPW = W::EPW, REC = W::REC, SLOT = S::SLOT, RECB = S::RECB;
  constexpr unsigned QMASK = NQ >= 32 ? 0xffffffffu : (1u << NQ) - 1u;
  extern __shared__ __align__(128) double ws_smem[];
  double* slots = ws_smem;                 // [P][2][SLOT]
  double* outb = ws_smem + P * 2 * SLOT;   // [CW][EPW * RECB]
  __shared__ uint64_t full[P][2], empty[P][2];
  __shared__ unsigned s_bal[P][2];
  __shared__ long long s_e0[P][2];
  c.DS = nullptr;  // hot path: S, flags, packed D only
  c.Ep_out = c.Hard_out = nullptr;
  c.pm = c.sm = c.am = nullptr;
  c.crit = nullptr;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int p = 0; p < P; ++p)
      for (int b = 0; b < 2; ++b) {
        mbar_init(&full[p][b], 1);
        mbar_init(&empty[p][b], 1);
      }
    mbar_init_fence();
  }
  __syncthreads();
  const int64_t n_groups = (g.e_end - g.e_begin + EPW - 1) / EPW;
  if (w < P) {
    // ---- producer: phase 1
    const int64_t stride = (int64_t)gridDim.x * P;
    int it = 0;
    for (int64_t grp = (int64_t)blockIdx.x * P + w;; grp += stride, ++it) {
      const int b = it & 1;
      if (it >= 2) mbar_wait(&empty[w][b], ((it >> 1) & 1) ^ 1);
      if (grp >= n_groups) {
        if (lane == 0) {
          s_e0[w][b] = -1;
          mbar_arrive(&full[w][b]);
        }
        break;
      }
      double* st_w = slots + (w * 2 + b) * SLOT;
      const int64_t e0 = g.e_begin + grp * EPW;
      bool plastic = false;
      if (lane < EPW * NQ) {
        const int le = lane / NQ, q = lane - le * NQ;
        const int64_t e = e0 + le;
        if (e < g.e_end) {
          const int64_t m = e * NQ + q;
          double* st = st_w + lane * REC;
          auto stage = [&](auto&& f) {
            stage_geometry<DIM, NP>(st, g.inv + m * W::D2, g.gradhat, q);
            stage_dw<DIM>(st + NP * DIM, __ldg(g.weight + m), g, m, f);
          };
          plastic = eval_point<MODEL>(c, m, GlobalIn{c.E, c.Ep, c.Hard}, stage);
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, plastic);
      if (lane < EPW && e0 + lane < g.e_end) g.emask[e0 + lane] = (bal >> (lane * NQ)) & QMASK;
      if (lane == 0) {
        s_bal[w][b] = bal;
        s_e0[w][b] = e0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[w][b]);
    }
  } else {
    // ---- consumer: phase 2 for producers cw, cw + CW, ...
    const int cw = w - P;
    double* out_w = outb + cw * EPW * RECB;
    constexpr int NMY = (P + CW - 1) / CW;
    int its[NMY];
    unsigned done = 0;
    const int nmy = (P - cw + CW - 1) / CW;
#pragma unroll
    for (int k = 0; k < NMY; ++k) its[k] = 0;
    bool pending = false;  // bulk stores in flight from out_w
    while (done != (1u << nmy) - 1u) {
#pragma unroll
      for (int k = 0; k < NMY; ++k) {
        if (k >= nmy || ((done >> k) & 1u)) continue;
        const int p = cw + k * CW, b = its[k] & 1;
        mbar_wait(&full[p][b], (its[k] >> 1) & 1);
        const long long e0 = s_e0[p][b];
        if (e0 < 0) {
          done |= 1u << k;
          continue;
        }
        const unsigned bal = s_bal[p][b];
        if (pending) {  // out_w must have been read by the previous bulk stores
          if (lane == 0) tma_store_wait_read_only();
          __syncwarp();
          pending = false;
        }
        const double* st_w = slots + (p * 2 + b) * SLOT;
        if (lane < EPW * W::NT) {
          const int le = lane / W::NT;
          const unsigned mask = (bal >> (le * NQ)) & QMASK;
          if (e0 + le < g.e_end && mask) {
            int a, c0;
            chunk_of<NP, W::CS>(lane - le * W::NT, a, c0);
            delta_chunk_uniform<DIM, NP, W::CS, REC, EPFEM_WS_SUB>(st_w + le * NQ * REC, mask, a, c0,
                                                                     out_w + le * RECB);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&empty[p][b]);  // staged records consumed
          for (int le = 0; le < EPW; ++le)
            if (e0 + le < g.e_end && ((bal >> (le * NQ)) & QMASK)) {
              tma_store_1d(g.scratch + (size_t)(e0 + le) * RECB, out_w + le * RECB,
                           (unsigned)(RECB * sizeof(double)));
              pending = true;
            }
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        pending = __shfl_sync(0xffffffffu, pending, 0);
        ++its[k];
      }
    }
    if (lane == 0) tma_store_wait_read_only();
  }
}

template <int MODEL, int NP, int NQ>
static int launch_ws(const ConstArgs& c, const GatherArgs& g, cudaStream_t st) {
  using S = WsCfg<NP, NQ>;
  auto kern = k_newton_ws<MODEL, NP, NQ>;
  static int per_sm = -1, num_sms = 0;
  if (per_sm < 0) {
    EPFEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S::SMEM));
    EPFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, S::THREADS, S::SMEM));
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm < 1) per_sm = 1;
  }
  using W = WarpCfg<2, NP, NQ>;
  const int64_t n_groups = (g.e_end - g.e_begin + W::EPW - 1) / W::EPW;
  const int64_t need = (n_groups + S::P - 1) / S::P;
  const int64_t grid = std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)per_sm * num_sms));
  kern<<<(unsigned)grid, S::THREADS, S::SMEM, st>>>(c, g);
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
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

// Per-buffer shared-memory tile of the pipelined kernel (doubles): the
// group's E, Ep, Hard (6 per point), J^-1 (dim^2 per point, one extra point
// for the 16-byte alignment shift) and w (two extra).
template <int DIM, int NP, int NQ>
struct PipeTile {
  static constexpr int PPG = DeltaCfg<DIM, NP, NQ>::EPB * NQ;  // points per group
  static constexpr int D2 = DIM * DIM;
  static constexpr int r2(int n) { return (n + 1) & ~1; }
  static constexpr int OE = 0, OEP = OE + 6 * PPG, OH = OEP + 6 * PPG, OI = OH + 6 * PPG;
  static constexpr int OW = OI + r2((PPG + 1) * D2);
  static constexpr int SIZE = OW + r2(PPG + 2);
  static constexpr size_t BYTES = 2 * SIZE * sizeof(double);
};

// k_newton_pipe: the fused kernel made persistent and software-pipelined.
// Each CTA walks groups of EPB elements (grid-stride); one elected thread
// issues TMA bulk copies of the NEXT group's E / Ep / Hard / J^-1 / w into
// the other half of a double-buffered tile (mbarrier completion) while the
// CTA computes the current group from shared memory, so the point update
// never waits on a global load.  Outputs and arithmetic are identical to
// k_newton_fused.
template <int MODEL, int DIM, int NP, int NQ>
__global__ void __launch_bounds__(DeltaCfg<DIM, NP, NQ>::THREADS)
    k_newton_pipe(ConstArgs c, GatherArgs g, int64_t n_groups) {
  pdl_trigger();
  using Cfg = DeltaCfg<DIM, NP, NQ>;
  using Tile = PipeTile<DIM, NP, NQ>;
  constexpr int EPB = Cfg::EPB, PPG = Tile::PPG, D2 = Tile::D2;
  extern __shared__ __align__(128) double tiles[];
  __shared__ double s_st[EPB][NQ][Cfg::REC];
  __shared__ unsigned s_mask[EPB];
  __shared__ uint64_t s_bar[2];
  c.DS = nullptr;  // hot path: S, flags, packed D only
  c.Ep_out = c.Hard_out = nullptr;
  c.pm = c.sm = c.am = nullptr;
  c.crit = nullptr;
  const int tid = threadIdx.x;
  const int64_t n_int = g.e_end * NQ;
  const int64_t pbase = g.e_begin * NQ;

  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    mbar_init_fence();
  }
  __syncthreads();
  auto issue = [&](int64_t grp, int b) {  // one thread
    double* t = tiles + b * Tile::SIZE;
    const int64_t p0 = pbase + grp * PPG;
    const int np = (int)min((int64_t)PPG, n_int - p0);
    const int sh = (int)(p0 & 1);  // J^-1 / w source shifted down to a 16-byte boundary
    const unsigned be = (unsigned)np * 48u;
    const unsigned bi = (unsigned)(((np + sh) * D2 * 8 + 15) & ~15);
    const unsigned bw = (unsigned)(((np + sh) * 8 + 15) & ~15);
    unsigned total = be + bi + bw;
    if (c.Ep) total += be;
    if (c.Hard) total += be;
    mbar_expect_tx(&s_bar[b], total);
    tma_load_1d(t + Tile::OE, c.E + 6 * p0, be, &s_bar[b]);
    if (c.Ep) tma_load_1d(t + Tile::OEP, c.Ep + 6 * p0, be, &s_bar[b]);
    if (c.Hard) tma_load_1d(t + Tile::OH, c.Hard + 6 * p0, be, &s_bar[b]);
    tma_load_1d(t + Tile::OI, g.inv + (p0 - sh) * D2, bi, &s_bar[b]);
    tma_load_1d(t + Tile::OW, g.weight + (p0 - sh), bw, &s_bar[b]);
  };
  int64_t grp = blockIdx.x;
  if (tid == 0 && grp < n_groups) issue(grp, 0);
  for (int it = 0; grp < n_groups; grp += gridDim.x, ++it) {
    const int b = it & 1;
    const int64_t nxt = grp + gridDim.x;
    // buffer b^1 was released by the barrier that closed the previous iteration;
    // order those generic-proxy reads before the async-proxy (TMA) writes
    if (tid == 0 && nxt < n_groups) {
      fence_proxy_async_smem();
      issue(nxt, b ^ 1);
    }
    if (tid < EPB) s_mask[tid] = 0u;
    mbar_wait(&s_bar[b], (unsigned)(it >> 1) & 1u);
    __syncthreads();
    const double* t = tiles + b * Tile::SIZE;
    const int64_t e0 = g.e_begin + grp * EPB;
    const int sh = (int)((pbase + grp * PPG) & 1);
    for (int k = tid; k < PPG; k += blockDim.x) {
      const int le = k / NQ, q = k - le * NQ;
      const int64_t e = e0 + le;
      if (e >= g.e_end) continue;
      const int64_t m = e * NQ + q;
      double* st = s_st[le][q];
      auto stage = [&](auto&& f) {
        atomicOr(&s_mask[le], 1u << q);
        stage_geometry<DIM, NP, true>(st, t + Tile::OI + (k + sh) * D2, g.gradhat, q);
        stage_dw<DIM>(st + NP * DIM, t[Tile::OW + k + sh], g, m, f);
      };
      eval_point<MODEL>(c, m, SmemIn{t + Tile::OE, t + Tile::OEP, t + Tile::OH, k}, stage);
    }
    __syncthreads();
    if (tid < EPB && e0 + tid < g.e_end) g.emask[e0 + tid] = s_mask[tid];
    delta_phase2<DIM, NP, NQ>(s_st, s_mask, tid, e0, g.e_end, g.scratch);
    __syncthreads();
  }
}

}  // namespace

int launch_constitutive(int model, const ConstArgs& a, cudaStream_t st, int num_sms) {
  if (a.n == 0) return 0;
  const int threads = 256;
  int64_t blocks = (a.n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms * 16;  // grid-stride beyond 16 CTAs/SM
  if (blocks > cap) blocks = cap;
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

template <int MODEL, int DIM, int NP, int NQ>
static int launch_pipe(const ConstArgs& c, const GatherArgs& g, cudaStream_t st) {
  using Cfg = DeltaCfg<DIM, NP, NQ>;
  using Tile = PipeTile<DIM, NP, NQ>;
  auto kern = k_newton_pipe<MODEL, DIM, NP, NQ>;
  static int per_sm = -1, num_sms = 0;
  if (per_sm < 0) {
    EPFEM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)Tile::BYTES));
    EPFEM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, Cfg::THREADS,
                                                                 Tile::BYTES));
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm < 1) per_sm = 1;
  }
  const int64_t n_groups = (g.e_end - g.e_begin + Cfg::EPB - 1) / Cfg::EPB;
  const int64_t grid = std::min<int64_t>(n_groups, (int64_t)per_sm * num_sms);
  kern<<<(unsigned)grid, Cfg::THREADS, Tile::BYTES, st>>>(c, g, n_groups);
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

int launch_newton_fused_u(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g,
                          cudaStream_t st) {
  if (g.e_end <= g.e_begin) return 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    if constexpr (DIM == 3 && NP < 20 && NP != 8) {  // tetrahedra: warp kernel (as launch_newton_fused)
      using W = Pair3Cfg<NP, NQ>;
      const int64_t per = (int64_t)W::EPW * W::WPB;
      const unsigned blocks = (unsigned)((g.e_end - g.e_begin + per - 1) / per);
      switch (model) {
        case EPFEM_MODEL_VON_MISES:
          k_newton_warp3<EPFEM_MODEL_VON_MISES, NP, NQ, true><<<blocks, W::THREADS, 0, st>>>(c, g);
          break;
        case EPFEM_MODEL_DRUCKER_PRAGER:
          k_newton_warp3<EPFEM_MODEL_DRUCKER_PRAGER, NP, NQ, true><<<blocks, W::THREADS, 0, st>>>(c, g);
          break;
        default:
          k_newton_warp3<EPFEM_MODEL_ELASTIC, NP, NQ, true><<<blocks, W::THREADS, 0, st>>>(c, g);
          break;
      }
    } else if constexpr (DIM == 3) {  // hexahedra: CTA kernel
      using Cfg = FusedCfg<DIM, NP, NQ>;
      const unsigned blocks = (unsigned)((g.e_end - g.e_begin + Cfg::EPB - 1) / Cfg::EPB);
      switch (model) {
        case EPFEM_MODEL_VON_MISES:
          k_newton_fused<EPFEM_MODEL_VON_MISES, DIM, NP, NQ, true><<<blocks, Cfg::THREADS, 0, st>>>(c, g);
          break;
        case EPFEM_MODEL_DRUCKER_PRAGER:
          k_newton_fused<EPFEM_MODEL_DRUCKER_PRAGER, DIM, NP, NQ, true><<<blocks, Cfg::THREADS, 0, st>>>(c, g);
          break;
        default:
          k_newton_fused<EPFEM_MODEL_ELASTIC, DIM, NP, NQ, true><<<blocks, Cfg::THREADS, 0, st>>>(c, g);
          break;
      }
    }
    if constexpr (DIM == 2) {
      using W = WarpCfg<DIM, NP, NQ>;
      const int64_t per = (int64_t)W::EPW * W::WPB;
      const unsigned blocks = (unsigned)((g.e_end - g.e_begin + per - 1) / per);
      switch (model) {
        case EPFEM_MODEL_VON_MISES:
          k_newton_warp<EPFEM_MODEL_VON_MISES, NP, NQ, true><<<blocks, W::THREADS, 0, st>>>(c, g);
          break;
        case EPFEM_MODEL_DRUCKER_PRAGER:
          k_newton_warp<EPFEM_MODEL_DRUCKER_PRAGER, NP, NQ, true><<<blocks, W::THREADS, 0, st>>>(c, g);
          break;
        default:
          k_newton_warp<EPFEM_MODEL_ELASTIC, NP, NQ, true><<<blocks, W::THREADS, 0, st>>>(c, g);
          break;
      }
    }
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

// ---------------------------------------------------------------------------
// k_newton_mega (2D): the whole Newton step in ONE launch.  Every warp of a
// cooperative (all CTAs co-resident) persistent grid is an independent
// worker walking an ordered item list round-robin (worker w takes items w,
// w + W, w + 2W, ...): producer items are k_newton_warp's element groups
// (fused update + element deltas), consumer items are node ranges of the
// row stream (rows.cuh, one warp per range).  The list puts every range
// after all the groups it reads (plus a slack), so the smallest unfinished
// item can always progress (its worker's earlier items are finished and the
// groups it waits on have smaller positions): no deadlock.  The roles share
// the SMs, so the latency-bound update and the bandwidth-bound row stream
// overlap instead of running back to back, and the element records are
// still L2-resident when read.  A group is published with a release store
// of the launch generation (deferred to the worker's next item, so the
// fence finds its stores drained); a range waits with acquire loads.  The
// last CTA to finish bumps the generation: the launch is replayable (CUDA
// graphs) without a memset.  Same per-entry arithmetic and add order as the
// two-launch step, hence the same bits.
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <int NP, int NQ>
struct MegaCfg {
  using W = WarpCfg<2, NP, NQ>;
  static constexpr int ST = ((W::EPW * NQ * W::REC + 1) / 2) * 2;  // doubles (even: 16-B aligned)
  static constexpr int OUT = W::EPW * W::NB * W::D2;
  static constexpr int PRODUCER = ST + OUT;                        // doubles per warp
};

template <int MODEL, int NP, int NQ>
__global__ void __launch_bounds__(WarpCfg<2, NP, NQ>::THREADS, EPFEM_WARP_MINB)
    k_newton_mega(ConstArgs c, GatherArgs g, MegaArgs m, int slice) {
  using W = WarpCfg<2, NP, NQ>;
  using MC = MegaCfg<NP, NQ>;
  extern __shared__ __align__(128) double dyn[];
  __shared__ uint64_t s_bar[W::WPB];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t workers = (int64_t)gridDim.x * W::WPB;
  double* my = dyn + (size_t)w * slice;
  const int gen = *((volatile int*)&m.sync->gen);  // bumped only after every CTA has finished
  if (lane == 0) {
    mbar_init(&s_bar[w], 1);
    mbar_init_fence();
  }
  __syncwarp();
  unsigned parity = 0;
  int pending = -1;  // produced group not yet published
  auto publish = [&] {
    if (pending >= 0 && lane == 0) {
      __threadfence();
      st_release_gpu(m.flag + pending, gen + 1);
    }
    pending = -1;
  };
  for (int64_t t = (int64_t)blockIdx.x * W::WPB + w; t < m.n_items; t += workers) {
    const int item = __ldg(m.sched + t);
    if (item >= 0) {
      if (m.exp != 2) {
        newton_warp_group<MODEL, NP, NQ, false, true>(c, g, (int64_t)item * W::EPW, my, my + MC::ST, lane);
        __syncwarp();
      }
      publish();
      pending = item;
    } else {
      publish();
      if (m.exp == 1) continue;
      const int r = ~item;
      if (row_range<2, NP, NQ, 32, true>(
              g, g.npc, r, my, &s_bar[w], parity,
              [&] {
                if (m.exp == 0) {
                  const int lo = __ldg(m.rlo + r), hi = __ldg(m.rhi + r);
                  for (int k = lo + lane; k <= hi; k += 32)
                    while (ld_acquire_gpu(m.flag + k) != gen + 1) __nanosleep(32);
                }
                __syncwarp();
              },
              lane))
        parity ^= 1u;
    }
    // this worker's generic smem writes are next overwritten by TMA
    fence_proxy_async_smem();
    __syncwarp();
  }
  publish();
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&m.sync->finished, 1) == (int)gridDim.x - 1) {
      m.sync->finished = 0;
      atomicAdd(&m.sync->gen, 1);
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------------------
// k_newton_warp_ovl (2D): k_newton_warp made persistent for the overlapped
// step.  The grid is sized below full occupancy (EPFEM_OVL_CTAS per SM) so
// that the row stream's CTAs, launched with programmatic dependent launch,
// share the SMs with it; each warp walks the element groups (warp-strided,
// so groups complete roughly in order) and publishes every group with a
// release store of the step generation (deferred to its next group, so the
// fence finds the stores drained).  The trigger at entry lets the row
// stream launch as soon as every producer CTA is resident, which is what
// makes the row stream's flag waits deadlock-free.
template <int MODEL, int NP, int NQ>
__global__ void __launch_bounds__(WarpCfg<2, NP, NQ>::THREADS, EPFEM_WARP_MINB)
    k_newton_warp_ovl(ConstArgs c, GatherArgs g, OvlArgs o) {
  pdl_trigger();
  using W = WarpCfg<2, NP, NQ>;
  __shared__ double s_st[W::WPB][W::EPW * NQ * W::REC];
  __shared__ __align__(16) double s_out[W::WPB][W::EPW * W::NB * W::D2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int gen = *((volatile int*)&o.sync->gen);
  int pending = -1;
  for (int64_t grp = (int64_t)blockIdx.x * W::WPB + w; grp < o.n_groups; grp += (int64_t)gridDim.x * W::WPB) {
    newton_warp_group<MODEL, NP, NQ, false, true>(c, g, grp * W::EPW, s_st[w], s_out[w], lane);
    __syncwarp();
    if (pending >= 0 && lane == 0) {
      __threadfence();
      st_release_gpu(o.flag + pending, gen + 1);
    }
    pending = (int)grp;
  }
  if (pending >= 0 && lane == 0) {
    __threadfence();
    st_release_gpu(o.flag + pending, gen + 1);
  }
}

bool ovl_supported(int family, int dim, int* group_elems) {
  bool ok = false;
  dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    if constexpr (DIM == 2) {
      *group_elems = WarpCfg<2, NP, NQ>::EPW;
      ok = true;
    }
  });
  return ok;
}

int launch_newton_ovl(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g, const OvlArgs& o,
                      int ctas_per_sm, cudaStream_t st) {
  if (o.n_groups <= 0) return 0;
  int rc = 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    if constexpr (DIM == 2) {
      using W = WarpCfg<2, NP, NQ>;
      int dev = 0, sms = 148;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      const int64_t want = (o.n_groups + W::WPB - 1) / W::WPB;
      const unsigned grid = (unsigned)std::min<int64_t>(want, (int64_t)std::max(ctas_per_sm, 1) * sms);
      switch (model) {
        case EPFEM_MODEL_VON_MISES:
          k_newton_warp_ovl<EPFEM_MODEL_VON_MISES, NP, NQ><<<grid, W::THREADS, 0, st>>>(c, g, o);
          break;
        case EPFEM_MODEL_DRUCKER_PRAGER:
          k_newton_warp_ovl<EPFEM_MODEL_DRUCKER_PRAGER, NP, NQ><<<grid, W::THREADS, 0, st>>>(c, g, o);
          break;
        default: k_newton_warp_ovl<EPFEM_MODEL_ELASTIC, NP, NQ><<<grid, W::THREADS, 0, st>>>(c, g, o); break;
      }
    } else {
      rc = fail(EPFEM_ERR_INVALID, "overlapped step: 2D meshes only");
    }
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  if (rc) return rc;
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

// per node range: the first and last producer group whose elements touch it
__global__ void k_range_groups(int64_t n_nodes, int npc, int np, int group_elems,
                               const int64_t* __restrict__ n2e_ptr, const int32_t* __restrict__ n2e,
                               int32_t* rlo, int32_t* rhi) {
  const int64_t n_ranges = (n_nodes + npc - 1) / npc;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_ranges;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n0 = r * npc, n1 = min(n0 + (int64_t)npc, n_nodes);
    int lo = INT32_MAX, hi = -1;
    for (int64_t a = n0; a < n1; ++a) {
      const int64_t b = n2e_ptr[a], e = n2e_ptr[a + 1];
      if (e > b) {  // a node's items are sorted by element
        lo = min(lo, (int)(n2e[b] / np / group_elems));
        hi = max(hi, (int)(n2e[e - 1] / np / group_elems));
      }
    }
    rlo[r] = lo;
    rhi[r] = hi;
  }
}

// group_elems: elements per producer item (one warp group); slice_bytes:
// the per-warp shared-memory slice (at least the producer's, sized so that
// EPFEM_WARP_MINB CTAs fit an SM); workers: warps of the co-resident grid.
bool mega_supported(int family, int dim, int* group_elems, int* slice_bytes, int* workers) {
  bool ok = false;
  dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    if constexpr (DIM == 2) {
      using W = WarpCfg<2, NP, NQ>;
      *group_elems = W::EPW;
      const int per_warp = ((200 * 1024 / EPFEM_WARP_MINB) / W::WPB) & ~127;
      const int prod = (int)(MegaCfg<NP, NQ>::PRODUCER * sizeof(double));
      *slice_bytes = per_warp > prod ? per_warp : prod;
      if (const char* v = getenv("EPFEM_MEGA_SLICE")) *slice_bytes = atoi(v);  // tuning / debugging
      int per_sm = 0, dev = 0, sms = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      auto kern = k_newton_mega<EPFEM_MODEL_VON_MISES, NP, NQ>;
      const size_t smem = (size_t)*slice_bytes * W::WPB;
      if (smem > 48 * 1024 &&
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return;
      if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, W::THREADS, smem) != cudaSuccess ||
          per_sm <= 0)
        return;
      *workers = per_sm * sms * W::WPB;
      ok = true;
    }
  });
  cudaGetLastError();
  return ok;
}

int launch_range_groups(int64_t n_nodes, int npc, int np, int group_elems, const int64_t* n2e_ptr,
                        const int32_t* n2e, int32_t* rlo, int32_t* rhi, cudaStream_t st) {
  k_range_groups<<<256, 128, 0, st>>>(n_nodes, npc, np, group_elems, n2e_ptr, n2e, rlo, rhi);
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

int launch_newton_mega(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g, const MegaArgs& m,
                       int slice_bytes, int workers, cudaStream_t st) {
  if (m.n_items <= 0) return 0;
  int rc = 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    if constexpr (DIM == 2) {
      using W = WarpCfg<2, NP, NQ>;
      const size_t smem = (size_t)slice_bytes * W::WPB;
      const int slice = slice_bytes / (int)sizeof(double);
      auto run = [&](auto kern) {
        if (smem > 48 * 1024) {
          cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
          if (e != cudaSuccess) { rc = cuda_fail(e, "cudaFuncSetAttribute"); return; }
        }
        // cooperative: every CTA co-resident (the item walk relies on it)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)(workers / W::WPB));
        cfg.blockDim = dim3(W::THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaError_t e = cudaLaunchKernelEx(&cfg, kern, c, g, m, slice);
        if (e != cudaSuccess) rc = cuda_fail(e, "one-launch Newton step");
      };
      switch (model) {
        case EPFEM_MODEL_VON_MISES: run(k_newton_mega<EPFEM_MODEL_VON_MISES, NP, NQ>); break;
        case EPFEM_MODEL_DRUCKER_PRAGER: run(k_newton_mega<EPFEM_MODEL_DRUCKER_PRAGER, NP, NQ>); break;
        default: run(k_newton_mega<EPFEM_MODEL_ELASTIC, NP, NQ>); break;
      }
    } else {
      rc = fail(EPFEM_ERR_INVALID, "one-launch Newton step: 2D meshes only");
    }
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  if (rc) return rc;
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

// Fused internal-forces step (2D warp kernel with FORCES).
bool forces_fused_supported(int family, int dim) { return dim == 2 && family >= 0; }

int launch_newton_forces(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g, cudaStream_t st) {
  if (g.e_end <= g.e_begin) return 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    if constexpr (DIM == 2) {
      using W = WarpCfg<DIM, NP, NQ>;
      const int64_t per = (int64_t)W::EPW * W::WPB;
      const unsigned blocks = (unsigned)((g.e_end - g.e_begin + per - 1) / per);
      switch (model) {
        case EPFEM_MODEL_VON_MISES:
          k_newton_warp<EPFEM_MODEL_VON_MISES, NP, NQ, false, true><<<blocks, W::THREADS, 0, st>>>(c, g);
          break;
        case EPFEM_MODEL_DRUCKER_PRAGER:
          k_newton_warp<EPFEM_MODEL_DRUCKER_PRAGER, NP, NQ, false, true><<<blocks, W::THREADS, 0, st>>>(c, g);
          break;
        default: k_newton_warp<EPFEM_MODEL_ELASTIC, NP, NQ, false, true><<<blocks, W::THREADS, 0, st>>>(c, g); break;
      }
    }
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

// Prefetch distance of the fused kernels, in CTAs: EPFEM_PF occupancy waves
// times the CTAs resident on the device.  Opt-in (default 0): measured on
// B200 neutral in 2D (cfg2 0.210 vs 0.213 ms at half a wave) and slower in 3D
// (cfg3 4.34 vs 3.70 ms at one wave): the first-phase load stalls are
// queueing under load, not DRAM latency an L2 hit would remove.
static int prefetch_distance(const void* kern, int threads) {
  static const double waves = getenv("EPFEM_PF") ? atof(getenv("EPFEM_PF")) : 0.0;
  if (waves <= 0) return 0;
  static std::mutex mu;
  static std::map<const void*, int> resident;
  std::lock_guard<std::mutex> lock(mu);
  auto it = resident.find(kern);
  if (it == resident.end()) {
    int per_sm = 0, dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, 0) != cudaSuccess) per_sm = 0;
    cudaGetLastError();
    it = resident.emplace(kern, per_sm * sms).first;
  }
  return (int)(waves * it->second);
}

int launch_newton_fused(int model, int family, int dim, const ConstArgs& c, const GatherArgs& g,
                        cudaStream_t st) {
  if (g.e_end <= g.e_begin) return 0;
  // The TMA-pipelined variant measured slower than the plain one on B200
  // (cfg2: 0.255 vs 0.224 ms; the kernel is bound by FP64 dependency chains,
  // not load latency), so it is opt-in: EPFEM_FUSED=pipe.
  // EPFEM_FUSED=cta forces the CTA kernel in 2D (default there: k_newton_warp).
  static const bool pipe = [] {
    const char* v = getenv("EPFEM_FUSED");
    return v && v[0] == 'p' && v[1] == 'i';
  }();
  static const bool cta = [] {
    const char* v = getenv("EPFEM_FUSED");
    return v && v[0] == 'c' && v[1] == 't';
  }();
  // phase 2 on the tensor pipe (k_newton_mma): opt-in, EPFEM_FUSED=mma.
  // Correct (same parity tests) but measured slower on B200 for cfg2
  // (0.253 vs 0.211 ms): the per-lane fragment gathers cost more issue
  // slots than the DMMA saves.
  static const int mma = [] {
    const char* v = getenv("EPFEM_FUSED");
    return (v && v[0] == 'm') ? 2 : 0;
  }();
  // 3D tetrahedra: warp kernel with row-pair phase 2 by default (hexahedra
  // keep the CTA kernel); EPFEM_FUSED=cta forces the CTA kernel
  static const bool warp3 = [] {
    const char* v = getenv("EPFEM_FUSED");
    return !(v && v[0] == 'c' && v[1] == 't') && !getenv("EPFEM_NO_WARP3");
  }();
  // two groups per warp with TMA prefetch of the second (2D): EPFEM_FUSED=pf
  static const bool pf = [] {
    const char* v = getenv("EPFEM_FUSED");
    return v && v[0] == 'p' && v[1] == 'f';
  }();
  // warp-specialized producer / consumer kernel (2D): EPFEM_FUSED=ws
  static const bool ws = [] {
    const char* v = getenv("EPFEM_FUSED");
    return v && v[0] == 'w' && v[1] == 's';
  }();
  int rc = 0;
  bool ok = dispatch_element(family, dim, [&](auto F, auto D) {
    constexpr int DIM = decltype(D)::value;
    constexpr int NP = ET<decltype(F)::value, DIM>::NP, NQ = ET<decltype(F)::value, DIM>::NQ;
    using Cfg = DeltaCfg<DIM, NP, NQ>;
    if (pipe) {
      switch (model) {
        case EPFEM_MODEL_VON_MISES: rc = launch_pipe<EPFEM_MODEL_VON_MISES, DIM, NP, NQ>(c, g, st); break;
        case EPFEM_MODEL_DRUCKER_PRAGER:
          rc = launch_pipe<EPFEM_MODEL_DRUCKER_PRAGER, DIM, NP, NQ>(c, g, st);
          break;
        default: rc = launch_pipe<EPFEM_MODEL_ELASTIC, DIM, NP, NQ>(c, g, st); break;
      }
      return;
    }
    if (mma == 2) {
      using M = MmaCfg<DIM, NP, NQ>;
      const int64_t per = (int64_t)M::EPW * M::WPB;
      const unsigned blocks = (unsigned)((g.e_end - g.e_begin + per - 1) / per);
      switch (model) {
        case EPFEM_MODEL_VON_MISES:
          k_newton_mma<EPFEM_MODEL_VON_MISES, DIM, NP, NQ><<<blocks, M::THREADS, 0, st>>>(c, g);
          break;
        case EPFEM_MODEL_DRUCKER_PRAGER:
          k_newton_mma<EPFEM_MODEL_DRUCKER_PRAGER, DIM, NP, NQ><<<blocks, M::THREADS, 0, st>>>(c, g);
          break;
        default:
          k_newton_mma<EPFEM_MODEL_ELASTIC, DIM, NP, NQ><<<blocks, M::THREADS, 0, st>>>(c, g);
          break;
      }
      return;
    }
    // (measured: P2 tet cfg3 3.61 vs 4.08 ms; Q1 hex cfg4 4.73 vs 4.17 ms -> CTA kernel for Q1)
    if constexpr (DIM == 3 && NP < 20 && NP != 8) {
      if (warp3) {
        using W = Pair3Cfg<NP, NQ>;
        const int64_t per = (int64_t)W::EPW * W::WPB;
        const unsigned blocks = (unsigned)((g.e_end - g.e_begin + per - 1) / per);
        GatherArgs gp = g;
        gp.pf_dist = prefetch_distance((const void*)k_newton_warp3<EPFEM_MODEL_VON_MISES, NP, NQ>, W::THREADS);
        switch (model) {
          case EPFEM_MODEL_VON_MISES:
            k_newton_warp3<EPFEM_MODEL_VON_MISES, NP, NQ><<<blocks, W::THREADS, 0, st>>>(c, gp);
            break;
          case EPFEM_MODEL_DRUCKER_PRAGER:
            k_newton_warp3<EPFEM_MODEL_DRUCKER_PRAGER, NP, NQ><<<blocks, W::THREADS, 0, st>>>(c, gp);
            break;
          default:
            k_newton_warp3<EPFEM_MODEL_ELASTIC, NP, NQ><<<blocks, W::THREADS, 0, st>>>(c, gp);
            break;
        }
        return;
      }
    }
    if constexpr (DIM == 2) {
      if (pf) {
        using W = WarpCfg<DIM, NP, NQ>;
        const int64_t per = 2 * (int64_t)W::EPW * PFW;
        const unsigned blocks = (unsigned)((g.e_end - g.e_begin + per - 1) / per);
        switch (model) {
          case EPFEM_MODEL_VON_MISES:
            k_newton_warp_pf<EPFEM_MODEL_VON_MISES, NP, NQ><<<blocks, 32 * PFW, 0, st>>>(c, g);
            break;
          case EPFEM_MODEL_DRUCKER_PRAGER:
            k_newton_warp_pf<EPFEM_MODEL_DRUCKER_PRAGER, NP, NQ><<<blocks, 32 * PFW, 0, st>>>(c, g);
            break;
          default:
            k_newton_warp_pf<EPFEM_MODEL_ELASTIC, NP, NQ><<<blocks, 32 * PFW, 0, st>>>(c, g);
            break;
        }
        return;
      }
      if (ws) {
        switch (model) {
          case EPFEM_MODEL_VON_MISES: rc = launch_ws<EPFEM_MODEL_VON_MISES, NP, NQ>(c, g, st); break;
          case EPFEM_MODEL_DRUCKER_PRAGER: rc = launch_ws<EPFEM_MODEL_DRUCKER_PRAGER, NP, NQ>(c, g, st); break;
          default: rc = launch_ws<EPFEM_MODEL_ELASTIC, NP, NQ>(c, g, st); break;
        }
        return;
      }
      if (!cta) {
        using W = WarpCfg<DIM, NP, NQ>;
        const int64_t per = (int64_t)W::EPW * W::WPB;
        const unsigned blocks = (unsigned)((g.e_end - g.e_begin + per - 1) / per);
        GatherArgs gp = g;
        gp.pf_dist = prefetch_distance((const void*)k_newton_warp<EPFEM_MODEL_VON_MISES, NP, NQ>, W::THREADS);
        switch (model) {
          case EPFEM_MODEL_VON_MISES:
            k_newton_warp<EPFEM_MODEL_VON_MISES, NP, NQ><<<blocks, W::THREADS, 0, st>>>(c, gp);
            break;
          case EPFEM_MODEL_DRUCKER_PRAGER:
            k_newton_warp<EPFEM_MODEL_DRUCKER_PRAGER, NP, NQ><<<blocks, W::THREADS, 0, st>>>(c, gp);
            break;
          default:
            k_newton_warp<EPFEM_MODEL_ELASTIC, NP, NQ><<<blocks, W::THREADS, 0, st>>>(c, gp);
            break;
        }
        return;
      }
    }
    using FC = FusedCfg<DIM, NP, NQ>;
    const unsigned blocks = (unsigned)((g.e_end - g.e_begin + FC::EPB - 1) / FC::EPB);
    GatherArgs gp = g;
      gp.pf_dist = prefetch_distance((const void*)k_newton_fused<EPFEM_MODEL_VON_MISES, DIM, NP, NQ>, FC::THREADS);
      switch (model) {
      case EPFEM_MODEL_VON_MISES:
        k_newton_fused<EPFEM_MODEL_VON_MISES, DIM, NP, NQ><<<blocks, FC::THREADS, 0, st>>>(c, gp);
        break;
      case EPFEM_MODEL_DRUCKER_PRAGER:
        k_newton_fused<EPFEM_MODEL_DRUCKER_PRAGER, DIM, NP, NQ><<<blocks, FC::THREADS, 0, st>>>(c, gp);
        break;
      default:
        k_newton_fused<EPFEM_MODEL_ELASTIC, DIM, NP, NQ><<<blocks, FC::THREADS, 0, st>>>(c, gp);
        break;
    }
  });
  if (!ok) return fail(EPFEM_ERR_INVALID, "invalid element type");
  if (rc) return rc;
  EPFEM_CUDA_TRY(cudaGetLastError());
  return 0;
}

}  // namespace epfem_gpu
