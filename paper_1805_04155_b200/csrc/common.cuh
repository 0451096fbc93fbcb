// Shared definitions for the epfem B200 kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <cassert>

// EPFEM_DEBUG_CHECKS=1 (a test build, tools/variants.sh): device-side bounds
// and single-writer assertions on the scatter paths (compute-sanitizer is not
// available on this pool); off in the shipped library.
#ifndef EPFEM_DEBUG_CHECKS
#define EPFEM_DEBUG_CHECKS 0
#endif
#if EPFEM_DEBUG_CHECKS
#define EPFEM_CHECK(c) assert(c)
#else
#define EPFEM_CHECK(c) ((void)0)
#endif

#include <string>

#include "../../include/epfem_gpu.h"

namespace epfem_gpu {

// Element traits: nodes per element and quadrature points per element for
// the eight (family, dim) pairs (reference_elements.cpp:326-374).
template <int FAM, int DIM>
struct ET;
template <> struct ET<EPFEM_P1, 2> { static constexpr int NP = 3, NQ = 1; };
template <> struct ET<EPFEM_P2, 2> { static constexpr int NP = 6, NQ = 3; };
template <> struct ET<EPFEM_Q1, 2> { static constexpr int NP = 4, NQ = 4; };
template <> struct ET<EPFEM_Q2, 2> { static constexpr int NP = 8, NQ = 9; };
template <> struct ET<EPFEM_P1, 3> { static constexpr int NP = 4, NQ = 1; };
template <> struct ET<EPFEM_P2, 3> { static constexpr int NP = 10, NQ = 11; };
template <> struct ET<EPFEM_Q1, 3> { static constexpr int NP = 8, NQ = 8; };
template <> struct ET<EPFEM_Q2, 3> { static constexpr int NP = 20, NQ = 27; };

// Runtime (family, dim) -> compile-time dispatch.  F is a generic lambda
// taking (auto fam_tag, auto dim_tag) integral-constant tags.
template <int V>
struct IC { static constexpr int value = V; };

template <class F>
inline bool dispatch_element(int family, int dim, F&& f) {
  switch (family * 2 + (dim - 2)) {
    case EPFEM_P1 * 2 + 0: f(IC<EPFEM_P1>{}, IC<2>{}); return true;
    case EPFEM_P1 * 2 + 1: f(IC<EPFEM_P1>{}, IC<3>{}); return true;
    case EPFEM_P2 * 2 + 0: f(IC<EPFEM_P2>{}, IC<2>{}); return true;
    case EPFEM_P2 * 2 + 1: f(IC<EPFEM_P2>{}, IC<3>{}); return true;
    case EPFEM_Q1 * 2 + 0: f(IC<EPFEM_Q1>{}, IC<2>{}); return true;
    case EPFEM_Q1 * 2 + 1: f(IC<EPFEM_Q1>{}, IC<3>{}); return true;
    case EPFEM_Q2 * 2 + 0: f(IC<EPFEM_Q2>{}, IC<2>{}); return true;
    case EPFEM_Q2 * 2 + 1: f(IC<EPFEM_Q2>{}, IC<3>{}); return true;
  }
  return false;
}

int node_count(int family, int dim);
int quad_count(int family, int dim);

// Reference tables for one element type, computed on the host with the
// reference's formulas: gradhat[(q*np + p)*dim + d] = d(phi_p)/d(xi_d) at
// quadrature point q, weights[q] = reference quadrature weight.
struct HostTables {
  int dim = 0, np = 0, nq = 0;
  double gradhat[27 * 20 * 3];
  double weights[27];
};
bool make_tables(int family, int dim, HostTables* out);

// Packed symmetric tangent index: PK[i][j] -> entry of EPFEM_D_STRIDE block.
__host__ __device__ constexpr int pk_index(int i, int j) {
  // table in epfem_gpu.h (plane-strain entries first)
  constexpr int T[6][6] = {{0, 1, 6, 2, 7, 8},     {1, 3, 9, 4, 10, 11},
                           {6, 9, 12, 13, 14, 15}, {2, 4, 13, 5, 16, 17},
                           {7, 10, 14, 16, 18, 19}, {8, 11, 15, 17, 19, 20}};
  return T[i][j];
}

#ifdef __CUDACC__
// Same table for runtime (non-unrolled) indices: constant bank, no local memory.
static __constant__ signed char c_pk_table[36] = {0, 1, 6,  2,  7,  8,  1, 3,  9,  4,  10, 11,
                                                  6, 9, 12, 13, 14, 15, 2, 4,  13, 5,  16, 17,
                                                  7, 10, 14, 16, 18, 19, 8, 11, 15, 17, 19, 20};
__device__ __forceinline__ int pk_index_rt(int i, int j) { return c_pk_table[i * 6 + j]; }
#endif

// Latched device-side error word owned by a context.
struct DevErr {
  int code;            // first epfem_status raised on device (0 = none)
  int pad;
  unsigned long long index;  // smallest offending point / element index
};

#ifdef __CUDACC__
__device__ inline void raise_dev(DevErr* e, int code, unsigned long long idx) {
  atomicCAS(&e->code, 0, code);
  atomicMin(&e->index, idx);
}
#endif

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t err, const char* what);

#define EPFEM_CUDA_TRY(expr)                               \
  do {                                                     \
    cudaError_t _e = (expr);                               \
    if (_e != cudaSuccess) return cuda_fail(_e, #expr);    \
  } while (0)

}  // namespace epfem_gpu
