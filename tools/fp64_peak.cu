// FP64 peak microbenchmark (B200, sm_100a): DFMA on the CUDA cores vs
// DMMA (mma.sync.aligned.m8n8k4.row.col.f64) on the tensor pipe.  Every
// warp runs independent accumulator chains (enough ILP to cover the
// pipeline latency); the grid is a multiple of the SM count.  Prints
// TFLOP/s (2 flops per FMA) for each.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
#include <cstdio>

__global__ void k_dfma(double* out, int iters) {
  double a[8], b = 1.0000001, c = 0.9999999;
#pragma unroll
  for (int k = 0; k < 8; ++k) a[k] = threadIdx.x + k;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) a[k] = fma(a[k], b, c);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a[k];
  if (s == 12345.0) out[threadIdx.x] = s;
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void k_dmma(double* out, int iters) {
  double d[8][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) d[k][0] = d[k][1] = 0.0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) dmma(d[k][0], d[k][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += d[k][0] + d[k][1];
  if (s == 12345.0) out[threadIdx.x] = s;
}

// both pipes at once: does DMMA run beside DFMA (separate datapaths)?
__global__ void k_mixed(double* out, int iters) {
  double d[4][2];
  double a2[8], b2 = 1.0000001, c2 = 0.9999999;
#pragma unroll
  for (int k = 0; k < 4; ++k) d[k][0] = d[k][1] = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) a2[k] = threadIdx.x + k;
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) dmma(d[k][0], d[k][1], a, b);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) a2[k] = fma(a2[k], b2, c2);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k) s += d[k][0] + d[k][1];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += a2[k];
  if (s == 12345.0) out[threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    const int blocks = sms * 4, threads = 32 * wpb;
    k_dfma<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    k_dfma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 8 * (double)iters * blocks * threads;
    printf("DFMA  warps/CTA %2d x %d CTAs: %.1f TFLOP/s\n", wpb, blocks, fl / (ms * 1e-3) / 1e12);
    k_dmma<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    k_dmma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    const double fm = 2.0 * 256 * 8 * (double)iters * blocks * wpb;
    printf("DMMA  warps/CTA %2d x %d CTAs: %.1f TFLOP/s\n", wpb, blocks, fm / (ms * 1e-3) / 1e12);
  }
  for (int wpb : {8, 16}) {
    const int blocks = sms * 4, threads = 32 * wpb;
    k_mixed<<<blocks, threads>>>(out, 100);
    cudaEventRecord(e0);
    k_mixed<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    // per iteration per warp: 4 DMMA (4 x 256 FMA) + 32 DFMA instructions (32 x 32 FMA)
    const double fl = 2.0 * (4.0 * 256 + 32.0 * 32) * (double)iters * blocks * wpb;
    printf("MIXED warps/CTA %2d x %d CTAs: %.1f TFLOP/s (half DMMA, half DFMA flops)\n", wpb, blocks,
           fl / (ms * 1e-3) / 1e12);
  }
  return 0;
}
