// Newton-loop linear algebra on the device:
// restricted_solve (linalg.cpp:69-115) as Jacobi-preconditioned conjugate
// gradients on K[free, free] — the reference's LinearSolver::conjugate_gradient
// (Eigen ConjugateGradient, DiagonalPreconditioner, tolerance rel_tol on
// |r| / |b|, at most 10 m iterations) — and energy_norm (linalg.cpp:117-121).
//
// The restriction is never formed: the masked SpMV y = M (K (M x)), M =
// diag(free), acts on the free block and leaves fixed dofs at zero, which is
// exactly the reference's restrict / solve / scatter.  Every reduction is a
// fixed two-stage tree (per-block partials, then one block over the partials
// in order), so a solve is bitwise reproducible run to run.  The scalars
// (alpha, beta, r.z) stay on the device; the host reads the residual every
// kCheck iterations.
#include <dlfcn.h>

#include <cmath>
#include <cub/cub.cuh>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace epfem_gpu {

namespace {

constexpr int kThreads = 256;
constexpr int kBlocks = 592;  // 4 x 148 SMs: partial-sum slots per reduction
constexpr int kCheck = 8;     // iterations between host residual checks

// warp per row: lanes stride the row's entries, fixed-order shuffle tree
__global__ void __launch_bounds__(kThreads) k_spmv_masked(int64_t n, const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ ci,
                                                          const double* __restrict__ v,
                                                          const uint8_t* __restrict__ mask,
                                                          const double* __restrict__ x, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  for (int64_t r = ((int64_t)blockIdx.x * kThreads + threadIdx.x) >> 5; r < n;
       r += ((int64_t)gridDim.x * kThreads) >> 5) {
    double s = 0.0;
    if (!mask || mask[r]) {
      for (int64_t k = rp[r] + lane; k < rp[r + 1]; k += 32) {
        const int32_t c = __ldg(ci + k);
        if (!mask || __ldg(mask + c)) s = __fma_rn(__ldg(v + k), __ldg(x + c), s);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
    }
    if (lane == 0) y[r] = s;
  }
}

__device__ __forceinline__ double block_sum(double s, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = s;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int k = 0; k < kThreads / 32; ++k) t = __dadd_rn(t, sh[k]);
  __syncthreads();
  return t;  // valid in thread 0
}

// partial[b] = sum over the block's grid-stride slice of a[i] * b[i] (two dots at once)
__global__ void __launch_bounds__(kThreads) k_dot2(int64_t n, const double* __restrict__ a0,
                                                   const double* __restrict__ b0, const double* __restrict__ a1,
                                                   const double* __restrict__ b1, double* partial) {
  __shared__ double sh[kThreads / 32];
  double s0 = 0.0, s1 = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    s0 = __fma_rn(a0[i], b0[i], s0);
    if (a1) s1 = __fma_rn(a1[i], b1[i], s1);
  }
  const double t0 = block_sum(s0, sh);
  const double t1 = block_sum(s1, sh);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = t0;
    partial[2 * blockIdx.x + 1] = t1;
  }
}

// scalar state: [0] r.z, [1] p.Ap, [2] r.r, [3] alpha, [4] beta, [5] b.b
enum { S_RZ = 0, S_PAP = 1, S_RR = 2, S_ALPHA = 3, S_BETA = 4, S_BB = 5 };

// sum the partials with a fixed-order tree (one 1024-thread block, partial b
// in slot b); mode 0: (r.z, r.r) -> beta; mode 1: p.Ap -> alpha; mode 2:
// initial (r.z, b.b)
constexpr int kFinish = 1024;
static_assert(kBlocks <= kFinish, "one finishing block");
__global__ void __launch_bounds__(kFinish) k_finish(const double* partial, int nb, double* sc, int mode) {
  __shared__ double s0[kFinish], s1[kFinish];
  const int t = threadIdx.x;
  s0[t] = t < nb ? partial[2 * t] : 0.0;
  s1[t] = t < nb ? partial[2 * t + 1] : 0.0;
  __syncthreads();
  for (int o = kFinish / 2; o > 0; o >>= 1) {
    if (t < o) {
      s0[t] = __dadd_rn(s0[t], s0[t + o]);
      s1[t] = __dadd_rn(s1[t], s1[t + o]);
    }
    __syncthreads();
  }
  if (t != 0) return;
  const double t0 = s0[0], t1 = s1[0];
  if (mode == 1) {
    sc[S_PAP] = t0;
    sc[S_ALPHA] = t0 != 0.0 ? sc[S_RZ] / t0 : 0.0;
  } else if (mode == 0) {
    sc[S_BETA] = sc[S_RZ] != 0.0 ? t0 / sc[S_RZ] : 0.0;
    sc[S_RZ] = t0;
    sc[S_RR] = t1;
  } else {
    sc[S_RZ] = t0;
    sc[S_BB] = t1;
    sc[S_RR] = t1;
  }
}

// x = 0, r = M b, z = M r / d, p = z; diag d from the CSR (fixed dofs: 1)
__global__ void k_cg_init(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                          const double* __restrict__ v, const uint8_t* __restrict__ mask,
                          const double* __restrict__ b, double* x, double* r, double* z, double* p, double* d) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    double di = 0.0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (ci[k] == i) di = v[k];
    const bool f = !mask || mask[i];
    // Eigen's DiagonalPreconditioner: 1 / diag, or 1 where the diagonal is 0
    const double inv = di != 0.0 ? 1.0 / di : 1.0;
    d[i] = inv;
    const double ri = f ? b[i] : 0.0;
    x[i] = 0.0;
    r[i] = ri;
    z[i] = f ? ri * inv : 0.0;
    p[i] = z[i];
  }
}

// x += alpha p; r -= alpha Ap; z = M r / d
__global__ void k_cg_update(int64_t n, const double* __restrict__ sc, const uint8_t* __restrict__ mask,
                            const double* __restrict__ d, const double* __restrict__ p,
                            const double* __restrict__ Ap, double* x, double* r, double* z) {
  const double alpha = sc[S_ALPHA];
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    x[i] = __fma_rn(alpha, p[i], x[i]);
    const double ri = __fma_rn(-alpha, Ap[i], r[i]);
    r[i] = ri;
    z[i] = (!mask || mask[i]) ? ri * d[i] : 0.0;
  }
}

// p = z + beta p
__global__ void k_cg_dir(int64_t n, const double* __restrict__ sc, const double* __restrict__ z, double* p) {
  const double beta = sc[S_BETA];
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    p[i] = __fma_rn(beta, p[i], z[i]);
}

// restart from the true residual: r = M (b - K x) (Ap holds K x), z = M r / d, p = z
__global__ void k_cg_restart(int64_t n, const uint8_t* __restrict__ mask, const double* __restrict__ b,
                             const double* __restrict__ Ap, const double* __restrict__ d, double* r, double* z,
                             double* p) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    const bool f = !mask || mask[i];
    const double ri = f ? b[i] - Ap[i] : 0.0;
    r[i] = ri;
    z[i] = f ? ri * d[i] : 0.0;
    p[i] = z[i];
  }
}

// rb = M (b - Ap)
__global__ void k_resid(int64_t n, const uint8_t* __restrict__ mask, const double* __restrict__ b,
                        const double* __restrict__ Ap, double* rb) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    rb[i] = (!mask || mask[i]) ? b[i] - Ap[i] : 0.0;
}

// Node-block Jacobi (block = dim, the `direct` method's preconditioner):
// per block of B consecutive dofs the inverse of K's B x B diagonal block of
// the restricted operator M K M + (I - M) (fixed dofs: identity rows and
// columns), explicit 2x2 / 3x3 cofactor inverse; a singular or non-finite
// block falls back to the scalar Jacobi of its diagonal.
template <int B>
__global__ void k_bj_setup(int64_t nb, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                           const double* __restrict__ v, const uint8_t* __restrict__ mask, double* binv) {
  for (int64_t blk = (int64_t)blockIdx.x * kThreads + threadIdx.x; blk < nb;
       blk += (int64_t)gridDim.x * kThreads) {
    const int64_t i0 = blk * B;
    double A[B][B];
    bool f[B];
    for (int r = 0; r < B; ++r) {
      f[r] = !mask || mask[i0 + r];
      for (int c = 0; c < B; ++c) A[r][c] = 0.0;
      for (int64_t k = rp[i0 + r]; k < rp[i0 + r + 1]; ++k) {
        const int64_t c = (int64_t)ci[k] - i0;
        if (c >= 0 && c < B) A[r][c] = v[k];
      }
    }
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < B; ++c)
        if (!f[r] || !f[c]) A[r][c] = r == c ? 1.0 : 0.0;
    double Ai[B][B];
    double det;
    if constexpr (B == 2) {
      det = A[0][0] * A[1][1] - A[0][1] * A[1][0];
      Ai[0][0] = A[1][1] / det;
      Ai[0][1] = -A[0][1] / det;
      Ai[1][0] = -A[1][0] / det;
      Ai[1][1] = A[0][0] / det;
    } else {
      const double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1];
      const double c01 = A[1][2] * A[2][0] - A[1][0] * A[2][2];
      const double c02 = A[1][0] * A[2][1] - A[1][1] * A[2][0];
      det = A[0][0] * c00 + A[0][1] * c01 + A[0][2] * c02;
      Ai[0][0] = c00 / det;
      Ai[1][0] = c01 / det;
      Ai[2][0] = c02 / det;
      Ai[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / det;
      Ai[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / det;
      Ai[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / det;
      Ai[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / det;
      Ai[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / det;
      Ai[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / det;
    }
    bool ok = det != 0.0 && isfinite(det);
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < B; ++c) ok = ok && isfinite(Ai[r][c]);
    for (int r = 0; r < B; ++r)
      for (int c = 0; c < B; ++c)
        binv[blk * B * B + r * B + c] =
            ok ? Ai[r][c] : (r == c ? (A[r][r] != 0.0 ? 1.0 / A[r][r] : 1.0) : 0.0);
  }
}

// z = M Binv r per block (fixed dofs: 0)
template <int B>
__global__ void k_bj_apply(int64_t nb, const uint8_t* __restrict__ mask, const double* __restrict__ binv,
                           const double* __restrict__ r, double* z) {
  for (int64_t blk = (int64_t)blockIdx.x * kThreads + threadIdx.x; blk < nb;
       blk += (int64_t)gridDim.x * kThreads) {
    const int64_t i0 = blk * B;
    double rr[B];
    for (int c = 0; c < B; ++c) rr[c] = r[i0 + c];
    for (int a = 0; a < B; ++a) {
      double acc = 0.0;
      for (int c = 0; c < B; ++c) acc = __fma_rn(binv[blk * B * B + a * B + c], rr[c], acc);
      z[i0 + a] = (!mask || mask[i0 + a]) ? acc : 0.0;
    }
  }
}

// one warp per row (the row loop of a warp is a chain of dependent loads:
// enough warps in flight is what hides it)
unsigned grid_rows(int64_t n) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + kThreads / 32 - 1) / (kThreads / 32), 1 << 22));
}

// Device scratch of one solve / norm: stream-ordered allocations
// (cudaMallocAsync / cudaFreeAsync on the solve's stream: no device-wide
// synchronisation per call, and freed on every return path).
struct Work {
  cudaStream_t st = nullptr;
  double *x = nullptr, *r = nullptr, *z = nullptr, *p = nullptr, *Ap = nullptr, *d = nullptr;
  double *partial = nullptr, *sc = nullptr, *binv = nullptr, *y = nullptr;
  explicit Work(cudaStream_t s) : st(s) {}
  cudaError_t alloc(double** q, size_t n) { return cudaMallocAsync(reinterpret_cast<void**>(q), sizeof(double) * n, st); }
  ~Work() {
    for (double* q : {x, r, z, p, Ap, d, partial, sc, binv, y})
      if (q) cudaFreeAsync(q, st);
  }
};

}  // namespace

int cg_solve(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, const uint8_t* mask,
             const double* b, double* x_out, double rel_tol, int64_t max_iters, cudaStream_t caller,
             int64_t* iters_out, double* residual_out, int block) {
  *iters_out = 0;
  *residual_out = 0.0;
  if (n == 0) return 0;
  if (block != 1 && block != 2 && block != 3) return fail(EPFEM_ERR_INVALID, "restricted_solve: block must be 1, 2 or 3");
  if (n % block) return fail(EPFEM_ERR_INVALID, "restricted_solve: dimension mismatch");
  const int64_t nb = n / block;
  // the solve runs on a private stream ordered after the caller's work (the
  // iteration chunks are captured into a graph, which the legacy default
  // stream does not allow); it is host-synchronous on return
  struct Stream {
    cudaStream_t s = nullptr;
    cudaEvent_t e = nullptr;
    ~Stream() {
      if (s) cudaStreamDestroy(s);
      if (e) cudaEventDestroy(e);
    }
  } ps;
  EPFEM_CUDA_TRY(cudaStreamCreateWithFlags(&ps.s, cudaStreamNonBlocking));
  EPFEM_CUDA_TRY(cudaEventCreateWithFlags(&ps.e, cudaEventDisableTiming));
  EPFEM_CUDA_TRY(cudaEventRecord(ps.e, caller));
  EPFEM_CUDA_TRY(cudaStreamWaitEvent(ps.s, ps.e, 0));
  cudaStream_t st = ps.s;
  Work w(st);
  for (double** q : {&w.x, &w.r, &w.z, &w.p, &w.Ap, &w.d}) EPFEM_CUDA_TRY(w.alloc(q, n));
  EPFEM_CUDA_TRY(w.alloc(&w.partial, 2 * kBlocks));
  EPFEM_CUDA_TRY(w.alloc(&w.sc, 8));
  const unsigned gb = (unsigned)std::min<int64_t>(kBlocks, (n + kThreads - 1) / kThreads);
  const unsigned gbb = (unsigned)std::min<int64_t>(kBlocks, (nb + kThreads - 1) / kThreads);
  // block > 1: z = M Binv r replaces the scalar z = M r / d after every
  // kernel that forms r (the scalar kernels' z is overwritten)
  auto apply_block = [&](bool set_p) -> int {
    if (block == 1) return 0;
    if (block == 2) k_bj_apply<2><<<gbb, kThreads, 0, st>>>(nb, mask, w.binv, w.r, w.z);
    else k_bj_apply<3><<<gbb, kThreads, 0, st>>>(nb, mask, w.binv, w.r, w.z);
    if (set_p) EPFEM_CUDA_TRY(cudaMemcpyAsync(w.p, w.z, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    return 0;
  };
  if (block > 1) {
    EPFEM_CUDA_TRY(w.alloc(&w.binv, nb * block * block));
    if (block == 2) k_bj_setup<2><<<gbb, kThreads, 0, st>>>(nb, rp, ci, v, mask, w.binv);
    else k_bj_setup<3><<<gbb, kThreads, 0, st>>>(nb, rp, ci, v, mask, w.binv);
  }
  k_cg_init<<<gb, kThreads, 0, st>>>(n, rp, ci, v, mask, b, w.x, w.r, w.z, w.p, w.d);
  if (int rc = apply_block(true)) return rc;
  k_dot2<<<gb, kThreads, 0, st>>>(n, w.r, w.z, w.r, w.r, w.partial);
  k_finish<<<1, kFinish, 0, st>>>(w.partial, gb, w.sc, 2);
  double h[8];
  EPFEM_CUDA_TRY(cudaMemcpyAsync(h, w.sc, sizeof(h), cudaMemcpyDeviceToHost, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  const double bnorm = std::sqrt(h[S_BB]);
  auto iteration = [&] {
    k_spmv_masked<<<grid_rows(n), kThreads, 0, st>>>(n, rp, ci, v, mask, w.p, w.Ap);
    k_dot2<<<gb, kThreads, 0, st>>>(n, w.p, w.Ap, nullptr, nullptr, w.partial);
    k_finish<<<1, kFinish, 0, st>>>(w.partial, gb, w.sc, 1);
    k_cg_update<<<gb, kThreads, 0, st>>>(n, w.sc, mask, w.d, w.p, w.Ap, w.x, w.r, w.z);
    apply_block(false);
    k_dot2<<<gb, kThreads, 0, st>>>(n, w.r, w.z, w.r, w.r, w.partial);
    k_finish<<<1, kFinish, 0, st>>>(w.partial, gb, w.sc, 0);
    k_cg_dir<<<gb, kThreads, 0, st>>>(n, w.sc, w.z, w.p);
  };
  struct GraphExec {
    cudaGraphExec_t e = nullptr;
    ~GraphExec() { if (e) cudaGraphExecDestroy(e); }
  } chunk_holder;
  cudaGraphExec_t& chunk = chunk_holder.e;
  int64_t it = 0;
  double res = 0.0;
  // CG on the recurrence residual, then the true residual |M (b - K x)|; on
  // recurrence drift (true residual above the tolerance although the
  // recurrence met it) restart from the true residual, at most 3 times (the
  // reference's direct solve refines likewise, linalg.cpp:92-96)
  for (int restart = 0;; ++restart) {
    if (bnorm > 0.0) {
      while (it < max_iters) {
        if (!chunk && max_iters - it >= kCheck) {
          // kCheck iterations as one CUDA graph (seven launches each): the
          // small systems of a Newton step are launch-bound otherwise
          cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
          cudaStreamIsCapturing(st, &cs);
          if (cs == cudaStreamCaptureStatusNone) {
            EPFEM_CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
            for (int k = 0; k < kCheck; ++k) iteration();
            cudaGraph_t g = nullptr;
            EPFEM_CUDA_TRY(cudaStreamEndCapture(st, &g));
            EPFEM_CUDA_TRY(cudaGraphInstantiate(&chunk, g, 0));
            cudaGraphDestroy(g);
          }
        }
        if (chunk && max_iters - it >= kCheck) {
          EPFEM_CUDA_TRY(cudaGraphLaunch(chunk, st));
          it += kCheck;
        } else {
          for (int k = 0; k < kCheck && it < max_iters; ++k, ++it) iteration();
        }
        EPFEM_CUDA_TRY(cudaGetLastError());
        EPFEM_CUDA_TRY(cudaMemcpyAsync(h, w.sc, sizeof(h), cudaMemcpyDeviceToHost, st));
        EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
        const double rn = std::sqrt(std::max(h[S_RR], 0.0));
        if (!(rn > rel_tol * bnorm)) break;  // also stops on NaN
      }
    }
    // true residual |M (b - K x)| / |M b| (linalg.cpp:105-109)
    k_spmv_masked<<<grid_rows(n), kThreads, 0, st>>>(n, rp, ci, v, mask, w.x, w.Ap);
    k_resid<<<gb, kThreads, 0, st>>>(n, mask, b, w.Ap, w.z);
    k_dot2<<<gb, kThreads, 0, st>>>(n, w.z, w.z, nullptr, nullptr, w.partial);
    k_finish<<<1, kFinish, 0, st>>>(w.partial, gb, w.sc, 1);
    EPFEM_CUDA_TRY(cudaMemcpyAsync(h, w.sc, sizeof(h), cudaMemcpyDeviceToHost, st));
    EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
    EPFEM_CUDA_TRY(cudaGetLastError());
    res = bnorm > 0.0 ? std::sqrt(std::max(h[S_PAP], 0.0)) / bnorm : 0.0;
    if (!(res > rel_tol) || restart == 3 || it >= max_iters || !std::isfinite(res)) break;
    k_cg_restart<<<gb, kThreads, 0, st>>>(n, mask, b, w.Ap, w.d, w.r, w.z, w.p);
    if (int rc = apply_block(true)) return rc;
    k_dot2<<<gb, kThreads, 0, st>>>(n, w.r, w.z, w.r, w.r, w.partial);
    k_finish<<<1, kFinish, 0, st>>>(w.partial, gb, w.sc, 2);  // r.z, r.r (the b.b slot is not read again)
  }
  EPFEM_CUDA_TRY(cudaMemcpyAsync(x_out, w.x, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  *iters_out = it;
  *residual_out = res;
  return 0;
}

int energy_norm(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, const double* x,
                cudaStream_t st, double* out) {
  *out = 0.0;
  if (n == 0) return 0;
  Work w(st);
  EPFEM_CUDA_TRY(w.alloc(&w.y, n));
  EPFEM_CUDA_TRY(w.alloc(&w.partial, 2 * kBlocks));
  EPFEM_CUDA_TRY(w.alloc(&w.sc, 8));
  double *y = w.y, *partial = w.partial, *sc = w.sc;
  const unsigned gb = (unsigned)std::min<int64_t>(kBlocks, (n + kThreads - 1) / kThreads);
  k_spmv_masked<<<grid_rows(n), kThreads, 0, st>>>(n, rp, ci, v, nullptr, x, y);
  k_dot2<<<gb, kThreads, 0, st>>>(n, x, y, nullptr, nullptr, partial);
  double zero[8] = {1.0, 0, 0, 0, 0, 0, 0, 0};  // r.z = 1: alpha slot unused
  EPFEM_CUDA_TRY(cudaMemcpyAsync(sc, zero, sizeof(zero), cudaMemcpyHostToDevice, st));
  k_finish<<<1, kFinish, 0, st>>>(partial, gb, sc, 1);
  double h[8];
  EPFEM_CUDA_TRY(cudaMemcpyAsync(h, sc, sizeof(h), cudaMemcpyDeviceToHost, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  EPFEM_CUDA_TRY(cudaGetLastError());
  *out = std::sqrt(std::max(h[S_PAP], 0.0));  // linalg.cpp:117-121
  return 0;
}

// ---------------------------------------------------------------------------
// LinearSolver::direct (linalg.cpp:84-96): the reference factorises
// K[free, free] (SimplicialLDLT) and applies up to three refinement sweeps.
// Here: the restricted matrix is formed on the device (free-index map by a
// prefix sum, per-row counts, fill); cuSOLVER's sparse Cholesky factorises it
// on the device (cusolverSpXcsrcholAnalysis once per pattern and free mask,
// cached in the context, then cusolverSpDcsrcholFactor / Solve per call);
// when the factor meets a zero pivot (not positive definite) that call falls
// back to QR (cusolverSpDcsrlsvqr).  Then up to three refinement sweeps on the
// true residual |M (b - K x)| / |M b| with the deterministic masked SpMV
// above.  cuSOLVER / cuSPARSE are loaded at run time (dlopen), so the library
// has no link dependency on them.
namespace {

struct SpApi {
  using Create = int (*)(void**);
  using Destroy = int (*)(void*);
  using SetStream = int (*)(void*, cudaStream_t);
  using Lsv = int (*)(void*, int, int, const void*, const double*, const int*, const int*, const double*, double,
                      int, double*, int*);
  using Analysis = int (*)(void*, int, int, const void*, const int*, const int*, void*);
  using BufInfo = int (*)(void*, int, int, const void*, const double*, const int*, const int*, void*, size_t*,
                          size_t*);
  using Factor = int (*)(void*, int, int, const void*, const double*, const int*, const int*, void*, void*);
  using ZeroPivot = int (*)(void*, void*, double, int*);
  using CholSolve = int (*)(void*, int, const double*, double*, void*, void*);
  Create create = nullptr, info_create = nullptr, descr_create = nullptr;
  Destroy destroy = nullptr, info_destroy = nullptr, descr_destroy = nullptr;
  SetStream set_stream = nullptr;
  Lsv qr = nullptr;
  Analysis analysis = nullptr;
  BufInfo buf_info = nullptr;
  Factor factor = nullptr;
  ZeroPivot zero_pivot = nullptr;
  CholSolve solve = nullptr;
  using DescrSet = int (*)(void*, int);
  DescrSet set_type = nullptr, set_base = nullptr;
  // dense cuSOLVER (the restricted systems of the drivers are small)
  using DnBuf = int (*)(void*, int, int, double*, int, int*);      // potrf_bufferSize(h, uplo, n, A, lda, lwork)
  using DnPotrf = int (*)(void*, int, int, double*, int, double*, int, int*);
  using DnPotrs = int (*)(void*, int, int, int, const double*, int, double*, int, int*);
  using DnGetrfBuf = int (*)(void*, int, int, double*, int, int*);
  using DnGetrf = int (*)(void*, int, int, double*, int, double*, int*, int*);
  using DnGetrs = int (*)(void*, int, int, int, const double*, int, const int*, double*, int, int*);
  Create dn_create = nullptr;
  Destroy dn_destroy = nullptr;
  SetStream dn_set_stream = nullptr;
  DnBuf potrf_buf = nullptr;
  DnPotrf potrf = nullptr;
  DnPotrs potrs = nullptr;
  DnGetrfBuf getrf_buf = nullptr;
  DnGetrf getrf = nullptr;
  DnGetrs getrs = nullptr;
  bool dense_ok = false;
  bool ok = false;
};

const SpApi& sp_api() {
  static SpApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    auto open = [](const char* soname, const char* path) {
      void* h = dlopen(soname, RTLD_NOW | RTLD_GLOBAL);
      return h ? h : dlopen(path, RTLD_NOW | RTLD_GLOBAL);
    };
    void* hs = open("libcusparse.so.12", "/usr/local/cuda/lib64/libcusparse.so.12");
    void* hv = open("libcusolver.so.11", "/usr/local/cuda/lib64/libcusolver.so.11");
    if (!hs || !hv) return;
    auto sym = [](void* h, const char* n) { return dlsym(h, n); };
    api.create = reinterpret_cast<SpApi::Create>(sym(hv, "cusolverSpCreate"));
    api.destroy = reinterpret_cast<SpApi::Destroy>(sym(hv, "cusolverSpDestroy"));
    api.set_stream = reinterpret_cast<SpApi::SetStream>(sym(hv, "cusolverSpSetStream"));
    api.qr = reinterpret_cast<SpApi::Lsv>(sym(hv, "cusolverSpDcsrlsvqr"));
    api.info_create = reinterpret_cast<SpApi::Create>(sym(hv, "cusolverSpCreateCsrcholInfo"));
    api.info_destroy = reinterpret_cast<SpApi::Destroy>(sym(hv, "cusolverSpDestroyCsrcholInfo"));
    api.analysis = reinterpret_cast<SpApi::Analysis>(sym(hv, "cusolverSpXcsrcholAnalysis"));
    api.buf_info = reinterpret_cast<SpApi::BufInfo>(sym(hv, "cusolverSpDcsrcholBufferInfo"));
    api.factor = reinterpret_cast<SpApi::Factor>(sym(hv, "cusolverSpDcsrcholFactor"));
    api.zero_pivot = reinterpret_cast<SpApi::ZeroPivot>(sym(hv, "cusolverSpDcsrcholZeroPivot"));
    api.solve = reinterpret_cast<SpApi::CholSolve>(sym(hv, "cusolverSpDcsrcholSolve"));
    api.descr_create = reinterpret_cast<SpApi::Create>(sym(hs, "cusparseCreateMatDescr"));
    api.descr_destroy = reinterpret_cast<SpApi::Destroy>(sym(hs, "cusparseDestroyMatDescr"));
    api.set_type = reinterpret_cast<SpApi::DescrSet>(sym(hs, "cusparseSetMatType"));
    api.set_base = reinterpret_cast<SpApi::DescrSet>(sym(hs, "cusparseSetMatIndexBase"));
    api.dn_create = reinterpret_cast<SpApi::Create>(sym(hv, "cusolverDnCreate"));
    api.dn_destroy = reinterpret_cast<SpApi::Destroy>(sym(hv, "cusolverDnDestroy"));
    api.dn_set_stream = reinterpret_cast<SpApi::SetStream>(sym(hv, "cusolverDnSetStream"));
    api.potrf_buf = reinterpret_cast<SpApi::DnBuf>(sym(hv, "cusolverDnDpotrf_bufferSize"));
    api.potrf = reinterpret_cast<SpApi::DnPotrf>(sym(hv, "cusolverDnDpotrf"));
    api.potrs = reinterpret_cast<SpApi::DnPotrs>(sym(hv, "cusolverDnDpotrs"));
    api.getrf_buf = reinterpret_cast<SpApi::DnGetrfBuf>(sym(hv, "cusolverDnDgetrf_bufferSize"));
    api.getrf = reinterpret_cast<SpApi::DnGetrf>(sym(hv, "cusolverDnDgetrf"));
    api.getrs = reinterpret_cast<SpApi::DnGetrs>(sym(hv, "cusolverDnDgetrs"));
    api.dense_ok = api.dn_create && api.dn_destroy && api.dn_set_stream && api.potrf_buf && api.potrf && api.potrs &&
                   api.getrf_buf && api.getrf && api.getrs;
    api.ok = api.create && api.destroy && api.set_stream && api.qr && api.info_create && api.info_destroy &&
             api.analysis && api.buf_info && api.factor && api.zero_pivot && api.solve && api.descr_create &&
             api.descr_destroy && api.set_type && api.set_base;
  });
  return api;
}

// free[i] -> 1 / 0 (int) for the prefix sum of the free-index map
__global__ void k_free_flags(int64_t n, const uint8_t* __restrict__ mask, int* flag) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    flag[i] = (!mask || mask[i]) ? 1 : 0;
}
// number of positions where two masks differ (null = all free)
__global__ void k_mask_diff(int64_t n, const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, int* out) {
  int c = 0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    c += ((!a || a[i]) ? 1 : 0) != ((!b || b[i]) ? 1 : 0);
  if (c) atomicAdd(out, c);
}
// the cached pattern differs from (rp, ci)?  rp first, then (only when the
// row pointers agree, so ci has the cached length) the column indices
__global__ void k_rp_diff(int64_t n, const int64_t* __restrict__ rp, const int64_t* __restrict__ crp, int* out) {
  int c = 0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i <= n; i += (int64_t)gridDim.x * kThreads)
    c += rp[i] != crp[i];
  if (c) atomicAdd(out, c);
}
__global__ void k_ci_diff(int64_t nnz, const int32_t* __restrict__ ci, const int32_t* __restrict__ cci, int* out) {
  if (*(volatile int*)out) return;
  int c = 0;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * kThreads)
    c += ci[i] != cci[i];
  if (c) atomicAdd(out, c);
}
__global__ void k_copy_mask(int64_t n, const uint8_t* __restrict__ mask, uint8_t* out) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    out[i] = (!mask || mask[i]) ? 1 : 0;
}
// per free row: its free entries (counts indexed by the row's free index)
__global__ void k_free_row_count(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                 const uint8_t* __restrict__ mask, const int* __restrict__ fidx, int* cnt) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    if (mask && !mask[i]) continue;
    int c = 0;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) c += (!mask || mask[ci[k]]) ? 1 : 0;
    cnt[fidx[i]] = c;
  }
}
// fill K[free, free] (columns stay sorted: the free-index map is monotone);
// fci == nullptr: values only (the pattern is cached)
__global__ void k_free_fill(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ v, const uint8_t* __restrict__ mask,
                            const int* __restrict__ fidx, const int* __restrict__ frp, int* fci, double* fv) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    if (mask && !mask[i]) continue;
    int o = frp[fidx[i]];
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int32_t c = ci[k];
      if (!mask || mask[c]) {
        if (fci) fci[o] = fidx[c];
        fv[o] = v[k];
        ++o;
      }
    }
  }
}
// the restricted CSR into a dense column-major m x m matrix (zeroed before)
__global__ void k_dense_scatter(int m, const int* __restrict__ frp, const int* __restrict__ fci,
                                const double* __restrict__ fv, double* A) {
  for (int r = blockIdx.x * kThreads + threadIdx.x; r < m; r += gridDim.x * kThreads)
    for (int o = frp[r]; o < frp[r + 1]; ++o) A[(size_t)fci[o] * m + r] = fv[o];
}
__global__ void k_gather_free(int64_t n, const uint8_t* __restrict__ mask, const int* __restrict__ fidx,
                              const double* __restrict__ r, double* rf) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    if (!mask || mask[i]) rf[fidx[i]] = r[i];
}
// x += scatter(xf) on free dofs (fixed dofs stay zero)
__global__ void k_scatter_add_free(int64_t n, const uint8_t* __restrict__ mask, const int* __restrict__ fidx,
                                   const double* __restrict__ xf, double* x) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    if (!mask || mask[i]) x[i] = __dadd_rn(x[i], xf[fidx[i]]);
}

}  // namespace

// The restricted pattern and its symbolic Cholesky analysis, cached per
// context for the last (matrix pattern, free mask) seen: a Newton loop
// factorises the same pattern every iteration.
struct DirectCache {
  int64_t n = -1;
  int m = 0, nnz = 0;
  uint8_t* mask = nullptr;  // the cached free mask (1 byte per row)
  int64_t* crp = nullptr;   // copies of the analysed pattern: a caller may free (rp, ci) and reuse the
  int32_t* cci = nullptr;   // addresses for another pattern, so the key is the content, not the pointers
  int64_t full_nnz = 0;
  int *fidx = nullptr, *frp = nullptr, *fci = nullptr, *cnt = nullptr;
  double* fv = nullptr;
  void *handle = nullptr, *descr = nullptr, *info = nullptr, *buf = nullptr;
  bool analysed = false;
  // dense path (m <= kDenseMax): factor, workspace, pivots, status word
  void* dn = nullptr;
  double *A = nullptr, *work = nullptr;
  int *ipiv = nullptr, *dinfo = nullptr;
  int lwork = 0;
  void release() {
    const SpApi& api = sp_api();
    if (info) api.info_destroy(info);
    info = nullptr;
    for (void* p : {(void*)mask, (void*)crp, (void*)cci, (void*)fidx, (void*)frp, (void*)fci, (void*)cnt, (void*)fv, buf, (void*)A,
                    (void*)work, (void*)ipiv, (void*)dinfo})
      if (p) cudaFree(p);
    A = work = nullptr;
    ipiv = dinfo = nullptr;
    lwork = 0;
    mask = nullptr;
    crp = nullptr;
    cci = nullptr;
    full_nnz = 0;
    fidx = frp = fci = cnt = nullptr;
    fv = nullptr;
    buf = nullptr;
    analysed = false;
    n = -1;
  }
  ~DirectCache() {
    release();
    const SpApi& api = sp_api();
    if (descr) api.descr_destroy(descr);
    if (handle) api.destroy(handle);
    if (dn) api.dn_destroy(dn);
  }
};

// restricted systems up to this size are factorised dense (cusolverDn potrf,
// getrf when not positive definite): the drivers' systems are small, and the
// dense factorisation on the device is far faster than the sparse one there.
// EPFEM_DIRECT_DENSE_MAX overrides it (tests: 0 forces the sparse path).
constexpr int kDenseMax = 16384;
static int dense_max() {
  const char* v = getenv("EPFEM_DIRECT_DENSE_MAX");
  return v ? atoi(v) : kDenseMax;
}

void direct_cache_free(void* c) { delete static_cast<DirectCache*>(c); }

int direct_solve(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, const uint8_t* mask,
                 const double* b, double* x_out, double rel_tol, cudaStream_t st, void** cache_slot, int* sweeps_out,
                 double* residual_out) {
  *sweeps_out = 0;
  *residual_out = 0.0;
  EPFEM_CUDA_TRY(cudaMemsetAsync(x_out, 0, sizeof(double) * std::max<int64_t>(n, 1), st));
  if (n == 0) return 0;
  const SpApi& api = sp_api();
  if (!api.ok) return fail(EPFEM_ERR_UNSUPPORTED, "restricted_solve: cuSOLVER sparse is not available");
  if (n >= INT32_MAX) return fail(EPFEM_ERR_UNSUPPORTED, "restricted_solve: direct solve needs int32 sizes");
  if (!*cache_slot) *cache_slot = new DirectCache;
  DirectCache& dc = *static_cast<DirectCache*>(*cache_slot);
  if (!dc.handle) {
    if (api.create(&dc.handle) != 0 || api.descr_create(&dc.descr) != 0)
      return fail(EPFEM_ERR_SOLVER, "restricted_solve: cuSOLVER initialisation failed");
    api.set_type(dc.descr, 0);  // CUSPARSE_MATRIX_TYPE_GENERAL (both triangles stored)
    api.set_base(dc.descr, 0);  // CUSPARSE_INDEX_BASE_ZERO
  }
  api.set_stream(dc.handle, st);
  const unsigned gb = (unsigned)std::min<int64_t>(kBlocks * 4, (n + kThreads - 1) / kThreads);
  // same pattern and free mask as the cached analysis?
  bool same = dc.analysed && dc.n == n;
  if (same) {
    int* diff = nullptr;
    EPFEM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void**>(&diff), sizeof(int), st));
    EPFEM_CUDA_TRY(cudaMemsetAsync(diff, 0, sizeof(int), st));
    k_mask_diff<<<gb, kThreads, 0, st>>>(n, mask, dc.mask, diff);
    k_rp_diff<<<gb, kThreads, 0, st>>>(n, rp, dc.crp, diff);
    k_ci_diff<<<gb, kThreads, 0, st>>>(dc.full_nnz, ci, dc.cci, diff);
    int h = 0;
    EPFEM_CUDA_TRY(cudaMemcpyAsync(&h, diff, sizeof(int), cudaMemcpyDeviceToHost, st));
    EPFEM_CUDA_TRY(cudaFreeAsync(diff, st));
    EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
    same = h == 0;
  }
  if (!same) {
    EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
    dc.release();
    EPFEM_CUDA_TRY(cudaMalloc(&dc.mask, n));
    EPFEM_CUDA_TRY(cudaMemcpyAsync(&dc.full_nnz, rp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
    EPFEM_CUDA_TRY(cudaMalloc(&dc.crp, sizeof(int64_t) * (n + 1)));
    EPFEM_CUDA_TRY(cudaMalloc(&dc.cci, sizeof(int32_t) * std::max<int64_t>(dc.full_nnz, 1)));
    EPFEM_CUDA_TRY(cudaMemcpyAsync(dc.crp, rp, sizeof(int64_t) * (n + 1), cudaMemcpyDeviceToDevice, st));
    EPFEM_CUDA_TRY(cudaMemcpyAsync(dc.cci, ci, sizeof(int32_t) * dc.full_nnz, cudaMemcpyDeviceToDevice, st));
    EPFEM_CUDA_TRY(cudaMalloc(&dc.fidx, sizeof(int) * (n + 1)));
    EPFEM_CUDA_TRY(cudaMalloc(&dc.cnt, sizeof(int) * (n + 1)));
    k_copy_mask<<<gb, kThreads, 0, st>>>(n, mask, dc.mask);
    k_free_flags<<<gb, kThreads, 0, st>>>(n, mask, dc.cnt);
    EPFEM_CUDA_TRY(cudaMemsetAsync(dc.cnt + n, 0, sizeof(int), st));
    size_t tmp_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, dc.cnt, dc.fidx, (int)n + 1, st);
    void* tmp = nullptr;
    EPFEM_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
    cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, dc.cnt, dc.fidx, (int)n + 1, st);
    EPFEM_CUDA_TRY(cudaMemcpyAsync(&dc.m, dc.fidx + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
    if (dc.m > 0) {
      EPFEM_CUDA_TRY(cudaMalloc(&dc.frp, sizeof(int) * ((size_t)dc.m + 1)));
      EPFEM_CUDA_TRY(cudaMemsetAsync(dc.cnt, 0, sizeof(int) * ((size_t)dc.m + 1), st));
      k_free_row_count<<<gb, kThreads, 0, st>>>(n, rp, ci, mask, dc.fidx, dc.cnt);
      cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, dc.cnt, dc.frp, dc.m + 1, st);
      EPFEM_CUDA_TRY(cudaMemcpyAsync(&dc.nnz, dc.frp + dc.m, sizeof(int), cudaMemcpyDeviceToHost, st));
      EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
      EPFEM_CUDA_TRY(cudaMalloc(&dc.fci, sizeof(int) * std::max(dc.nnz, 1)));
      EPFEM_CUDA_TRY(cudaMalloc(&dc.fv, sizeof(double) * std::max(dc.nnz, 1)));
      k_free_fill<<<gb, kThreads, 0, st>>>(n, rp, ci, v, mask, dc.fidx, dc.frp, dc.fci, dc.fv);
      if (dc.m <= dense_max() && api.dense_ok) {
        if (!dc.dn && api.dn_create(&dc.dn) != 0)
          return fail(EPFEM_ERR_SOLVER, "restricted_solve: cuSOLVER initialisation failed");
        api.dn_set_stream(dc.dn, st);
        EPFEM_CUDA_TRY(cudaMalloc(&dc.A, sizeof(double) * (size_t)dc.m * dc.m));
        EPFEM_CUDA_TRY(cudaMalloc(&dc.ipiv, sizeof(int) * dc.m));
        EPFEM_CUDA_TRY(cudaMalloc(&dc.dinfo, sizeof(int)));
        int l1 = 0, l2 = 0;
        if (api.potrf_buf(dc.dn, 0, dc.m, dc.A, dc.m, &l1) != 0 || api.getrf_buf(dc.dn, dc.m, dc.m, dc.A, dc.m, &l2) != 0)
          return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
        dc.lwork = std::max(std::max(l1, l2), 1);
        EPFEM_CUDA_TRY(cudaMalloc(&dc.work, sizeof(double) * dc.lwork));
      } else {
      // symbolic analysis once per pattern and mask (natural order: the mesh
      // numbering is lexicographic, hence banded)
      if (api.info_create(&dc.info) != 0 ||
          api.analysis(dc.handle, dc.m, dc.nnz, dc.descr, dc.frp, dc.fci, dc.info) != 0)
        return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
      size_t internal = 0, work = 0;
      if (api.buf_info(dc.handle, dc.m, dc.nnz, dc.descr, dc.fv, dc.frp, dc.fci, dc.info, &internal, &work) != 0)
        return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
      EPFEM_CUDA_TRY(cudaMalloc(&dc.buf, std::max<size_t>(work, 16)));
      }
    }
    EPFEM_CUDA_TRY(cudaFreeAsync(tmp, st));
    dc.n = n;
    dc.analysed = true;
  } else if (dc.m > 0) {
    k_free_fill<<<gb, kThreads, 0, st>>>(n, rp, ci, v, mask, dc.fidx, dc.frp, nullptr, dc.fv);
  }
  if (dc.m == 0) return 0;
  const int m = dc.m;
  Work w(st);
  EPFEM_CUDA_TRY(w.alloc(&w.r, n));
  EPFEM_CUDA_TRY(w.alloc(&w.Ap, n));
  EPFEM_CUDA_TRY(w.alloc(&w.z, (size_t)m));  // restricted rhs
  EPFEM_CUDA_TRY(w.alloc(&w.p, (size_t)m));  // restricted solution
  EPFEM_CUDA_TRY(w.alloc(&w.partial, 2 * kBlocks));
  EPFEM_CUDA_TRY(w.alloc(&w.sc, 8));
  double *r = w.r, *Ax = w.Ap, *bf = w.z, *xf = w.p;
  auto residual = [&](double* rr) -> int {  // r = M (b - K x); rr = |r|^2
    k_spmv_masked<<<grid_rows(n), kThreads, 0, st>>>(n, rp, ci, v, mask, x_out, Ax);
    k_resid<<<gb, kThreads, 0, st>>>(n, mask, b, Ax, r);
    const unsigned gd = (unsigned)std::min<int64_t>(kBlocks, (n + kThreads - 1) / kThreads);
    k_dot2<<<gd, kThreads, 0, st>>>(n, r, r, nullptr, nullptr, w.partial);
    k_finish<<<1, kFinish, 0, st>>>(w.partial, gd, w.sc, 2);
    double h[8];
    EPFEM_CUDA_TRY(cudaMemcpyAsync(h, w.sc, sizeof(h), cudaMemcpyDeviceToHost, st));
    EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
    *rr = h[S_RZ];
    return 0;
  };
  // numeric factorisation; not positive definite -> LU (dense) / QR (sparse)
  const bool dense = dc.A != nullptr;
  bool qr = false, lu = false;
  auto dense_matrix = [&]() -> int {
    EPFEM_CUDA_TRY(cudaMemsetAsync(dc.A, 0, sizeof(double) * (size_t)m * m, st));
    k_dense_scatter<<<std::max(1, std::min(kBlocks * 4, (m + kThreads - 1) / kThreads)), kThreads, 0, st>>>(
        m, dc.frp, dc.fci, dc.fv, dc.A);
    return 0;
  };
  auto dense_info = [&]() -> int {
    int h = 0;
    EPFEM_CUDA_TRY(cudaMemcpyAsync(&h, dc.dinfo, sizeof(int), cudaMemcpyDeviceToHost, st));
    EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
    return h;
  };
  if (dense) {
    api.dn_set_stream(dc.dn, st);
    if (int rc = dense_matrix()) return rc;
    if (api.potrf(dc.dn, 0, m, dc.A, m, dc.work, dc.lwork, dc.dinfo) != 0)
      return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
    if (dense_info() != 0) {  // not positive definite: partial-pivoting LU on a fresh copy
      lu = true;
      if (int rc = dense_matrix()) return rc;
      if (api.getrf(dc.dn, m, m, dc.A, m, dc.work, dc.ipiv, dc.dinfo) != 0 || dense_info() != 0)
        return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
    }
  } else {
    if (api.factor(dc.handle, m, dc.nnz, dc.descr, dc.fv, dc.frp, dc.fci, dc.info, dc.buf) != 0)
      return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
    int pos = -1;
    if (api.zero_pivot(dc.handle, dc.info, 1e-14, &pos) != 0) pos = 0;
    if (pos >= 0) qr = true;
  }
  // the first solve has x = 0, so its residual norm is |M b|
  double rr = 0.0;
  if (int rc = residual(&rr)) return rc;
  const double bnorm = std::sqrt(rr);
  if (bnorm == 0.0) return 0;
  for (int sweep = 0; sweep < 4; ++sweep) {
    k_gather_free<<<gb, kThreads, 0, st>>>(n, mask, dc.fidx, r, bf);
    if (dense) {
      EPFEM_CUDA_TRY(cudaMemcpyAsync(xf, bf, sizeof(double) * m, cudaMemcpyDeviceToDevice, st));
      const int rc = lu ? api.getrs(dc.dn, 0, m, 1, dc.A, m, dc.ipiv, xf, m, dc.dinfo)
                        : api.potrs(dc.dn, 0, m, 1, dc.A, m, xf, m, dc.dinfo);
      if (rc != 0) return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
    } else if (qr) {
      int sing = -1;
      if (api.qr(dc.handle, m, dc.nnz, dc.descr, dc.fv, dc.frp, dc.fci, bf, 1e-14, 2, xf, &sing) != 0 || sing >= 0)
        return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
    } else if (api.solve(dc.handle, m, bf, xf, dc.info, dc.buf) != 0) {
      return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
    }
    k_scatter_add_free<<<gb, kThreads, 0, st>>>(n, mask, dc.fidx, xf, x_out);
    EPFEM_CUDA_TRY(cudaGetLastError());
    *sweeps_out = sweep + 1;
    if (int rc2 = residual(&rr)) return rc2;
    *residual_out = std::sqrt(rr) / bnorm;
    if (!(*residual_out > rel_tol)) break;  // refinement sweeps keep the residual contract
  }
  return 0;
}

}  // namespace epfem_gpu
