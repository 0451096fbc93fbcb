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
// prefix sum, per-row counts, fill), factorised and solved by cuSOLVER's
// sparse Cholesky (cusolverSpDcsrlsvchol, symamd reordering) -- QR
// (cusolverSpDcsrlsvqr) when the Cholesky finds the matrix not positive
// definite -- then up to three refinement sweeps on the true residual
// |M (b - K x)| / |M b| with the deterministic masked SpMV above.  cuSOLVER /
// cuSPARSE are loaded at run time (dlopen), so the library has no link
// dependency on them.
namespace {

struct SpApi {
  using Create = int (*)(void**);
  using Destroy = int (*)(void*);
  using SetStream = int (*)(void*, cudaStream_t);
  using Solve = int (*)(void*, int, int, const void*, const double*, const int*, const int*, const double*, double,
                        int, double*, int*);
  using DescrCreate = int (*)(void**);
  using DescrDestroy = int (*)(void*);
  using DescrSet = int (*)(void*, int);
  Create create = nullptr;
  Destroy destroy = nullptr;
  SetStream set_stream = nullptr;
  Solve chol = nullptr, qr = nullptr;
  DescrCreate descr_create = nullptr;
  DescrDestroy descr_destroy = nullptr;
  DescrSet set_type = nullptr, set_base = nullptr;
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
    api.create = reinterpret_cast<SpApi::Create>(dlsym(hv, "cusolverSpCreate"));
    api.destroy = reinterpret_cast<SpApi::Destroy>(dlsym(hv, "cusolverSpDestroy"));
    api.set_stream = reinterpret_cast<SpApi::SetStream>(dlsym(hv, "cusolverSpSetStream"));
    api.chol = reinterpret_cast<SpApi::Solve>(dlsym(hv, "cusolverSpDcsrlsvchol"));
    api.qr = reinterpret_cast<SpApi::Solve>(dlsym(hv, "cusolverSpDcsrlsvqr"));
    api.descr_create = reinterpret_cast<SpApi::DescrCreate>(dlsym(hs, "cusparseCreateMatDescr"));
    api.descr_destroy = reinterpret_cast<SpApi::DescrDestroy>(dlsym(hs, "cusparseDestroyMatDescr"));
    api.set_type = reinterpret_cast<SpApi::DescrSet>(dlsym(hs, "cusparseSetMatType"));
    api.set_base = reinterpret_cast<SpApi::DescrSet>(dlsym(hs, "cusparseSetMatIndexBase"));
    api.ok = api.create && api.destroy && api.set_stream && api.chol && api.qr && api.descr_create &&
             api.descr_destroy && api.set_type && api.set_base;
  });
  return api;
}

// free[i] -> 1 / 0 (int) for the prefix sum of the free-index map
__global__ void k_free_flags(int64_t n, const uint8_t* __restrict__ mask, int* flag) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads)
    flag[i] = (!mask || mask[i]) ? 1 : 0;
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
// fill K[free, free] (columns stay sorted: the free-index map is monotone)
__global__ void k_free_fill(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                            const double* __restrict__ v, const uint8_t* __restrict__ mask,
                            const int* __restrict__ fidx, const int* __restrict__ frp, int* fci, double* fv) {
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < n; i += (int64_t)gridDim.x * kThreads) {
    if (mask && !mask[i]) continue;
    int o = frp[fidx[i]];
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const int32_t c = ci[k];
      if (!mask || mask[c]) {
        fci[o] = fidx[c];
        fv[o] = v[k];
        ++o;
      }
    }
  }
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

int direct_solve(int64_t n, const int64_t* rp, const int32_t* ci, const double* v, const uint8_t* mask,
                 const double* b, double* x_out, double rel_tol, cudaStream_t caller, int* sweeps_out,
                 double* residual_out) {
  *sweeps_out = 0;
  *residual_out = 0.0;
  EPFEM_CUDA_TRY(cudaMemsetAsync(x_out, 0, sizeof(double) * std::max<int64_t>(n, 1), caller));
  if (n == 0) return 0;
  const SpApi& api = sp_api();
  if (!api.ok) return fail(EPFEM_ERR_UNSUPPORTED, "restricted_solve: cuSOLVER sparse is not available");
  if (n >= INT32_MAX) return fail(EPFEM_ERR_UNSUPPORTED, "restricted_solve: direct solve needs int32 sizes");
  cudaStream_t st = caller;
  Work w(st);
  int *fidx = nullptr, *cnt = nullptr, *frp = nullptr, *fci = nullptr;
  auto ialloc = [&](int** p, size_t k) { return cudaMallocAsync(reinterpret_cast<void**>(p), sizeof(int) * k, st); };
  struct IntBufs {
    cudaStream_t s;
    std::vector<int*> p;
    ~IntBufs() {
      for (int* q : p)
        if (q) cudaFreeAsync(q, s);
    }
  } ib{st, {}};
  const unsigned gb = (unsigned)std::min<int64_t>(kBlocks * 4, (n + kThreads - 1) / kThreads);
  EPFEM_CUDA_TRY(ialloc(&fidx, n + 1));
  ib.p.push_back(fidx);
  // free-index map: exclusive prefix sum of the free flags
  EPFEM_CUDA_TRY(ialloc(&cnt, n + 1));
  ib.p.push_back(cnt);
  k_free_flags<<<gb, kThreads, 0, st>>>(n, mask, cnt);
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, fidx, (int)n + 1, st);
  void* tmp = nullptr;
  EPFEM_CUDA_TRY(cudaMallocAsync(&tmp, tmp_bytes, st));
  EPFEM_CUDA_TRY(cudaMemsetAsync(cnt + n, 0, sizeof(int), st));
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, fidx, (int)n + 1, st);
  int m = 0;
  EPFEM_CUDA_TRY(cudaMemcpyAsync(&m, fidx + n, sizeof(int), cudaMemcpyDeviceToHost, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  if (m == 0) {
    cudaFreeAsync(tmp, st);
    return 0;
  }
  // restricted CSR (int32, cuSOLVER's index type)
  EPFEM_CUDA_TRY(ialloc(&frp, (size_t)m + 1));
  ib.p.push_back(frp);
  EPFEM_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(int) * ((size_t)m + 1), st));
  k_free_row_count<<<gb, kThreads, 0, st>>>(n, rp, ci, mask, fidx, cnt);
  cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, frp, m + 1, st);
  int nnz = 0;
  EPFEM_CUDA_TRY(cudaMemcpyAsync(&nnz, frp + m, sizeof(int), cudaMemcpyDeviceToHost, st));
  EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
  cudaFreeAsync(tmp, st);
  EPFEM_CUDA_TRY(ialloc(&fci, (size_t)std::max(nnz, 1)));
  ib.p.push_back(fci);
  double *fv = nullptr, *bf = nullptr, *xf = nullptr, *r = nullptr, *Ax = nullptr;
  EPFEM_CUDA_TRY(w.alloc(&w.binv, (size_t)std::max(nnz, 1)));  // restricted values
  fv = w.binv;
  EPFEM_CUDA_TRY(w.alloc(&w.r, n));
  EPFEM_CUDA_TRY(w.alloc(&w.Ap, n));
  EPFEM_CUDA_TRY(w.alloc(&w.z, (size_t)m));  // restricted rhs
  EPFEM_CUDA_TRY(w.alloc(&w.p, (size_t)m));  // restricted solution
  EPFEM_CUDA_TRY(w.alloc(&w.partial, 2 * kBlocks));
  EPFEM_CUDA_TRY(w.alloc(&w.sc, 8));
  r = w.r;
  Ax = w.Ap;
  bf = w.z;
  xf = w.p;
  k_free_fill<<<gb, kThreads, 0, st>>>(n, rp, ci, v, mask, fidx, frp, fci, fv);
  EPFEM_CUDA_TRY(cudaGetLastError());
  void* handle = nullptr;
  void* descr = nullptr;
  struct Handles {
    const SpApi& a;
    void** h;
    void** d;
    ~Handles() {
      if (*d) a.descr_destroy(*d);
      if (*h) a.destroy(*h);
    }
  } hs{api, &handle, &descr};
  if (api.create(&handle) != 0 || api.descr_create(&descr) != 0)
    return fail(EPFEM_ERR_SOLVER, "restricted_solve: cuSOLVER initialisation failed");
  api.set_stream(handle, st);
  api.set_type(descr, 0);  // CUSPARSE_MATRIX_TYPE_GENERAL (both triangles stored)
  api.set_base(descr, 0);  // CUSPARSE_INDEX_BASE_ZERO
  auto residual = [&](double* rr) -> int {  // r = M (b - K x); rr = |r| / |M b|
    k_spmv_masked<<<grid_rows(n), kThreads, 0, st>>>(n, rp, ci, v, mask, x_out, Ax);
    k_resid<<<gb, kThreads, 0, st>>>(n, mask, b, Ax, r);
    const unsigned gd = (unsigned)std::min<int64_t>(kBlocks, (n + kThreads - 1) / kThreads);
    k_dot2<<<gd, kThreads, 0, st>>>(n, r, r, b, b, w.partial);
    k_finish<<<1, kFinish, 0, st>>>(w.partial, gd, w.sc, 2);
    double h[8];
    EPFEM_CUDA_TRY(cudaMemcpyAsync(h, w.sc, sizeof(h), cudaMemcpyDeviceToHost, st));
    EPFEM_CUDA_TRY(cudaStreamSynchronize(st));
    // masked b.b (k_dot2's second dot is unmasked): |M b| from the first residual
    *rr = h[S_RZ];
    return 0;
  };
  // the first solve has x = 0, so its residual norm is |M b|
  double rr = 0.0;
  if (int rc = residual(&rr)) return rc;
  const double bnorm = std::sqrt(rr);
  if (bnorm == 0.0) return 0;
  bool qr = false;
  for (int sweep = 0; sweep < 4; ++sweep) {
    k_gather_free<<<gb, kThreads, 0, st>>>(n, mask, fidx, r, bf);
    int sing = -1;
    int rc = qr ? api.qr(handle, m, nnz, descr, fv, frp, fci, bf, 1e-14, 2, xf, &sing)
                : api.chol(handle, m, nnz, descr, fv, frp, fci, bf, 1e-14, 2, xf, &sing);
    if (rc != 0) return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
    if (sing >= 0 && !qr) {  // not positive definite: QR on the same system
      qr = true;
      --sweep;
      continue;
    }
    if (sing >= 0) return fail(EPFEM_ERR_SOLVER, "restricted_solve: factorization failed");
    k_scatter_add_free<<<gb, kThreads, 0, st>>>(n, mask, fidx, xf, x_out);
    EPFEM_CUDA_TRY(cudaGetLastError());
    *sweeps_out = sweep + 1;
    if (int rc2 = residual(&rr)) return rc2;
    *residual_out = std::sqrt(rr) / bnorm;
    if (!(*residual_out > rel_tol)) break;  // refinement sweeps keep the residual contract
  }
  return 0;
}

}  // namespace epfem_gpu
