// Microbenchmark (not a product path): shared-memory wavefronts of LDS.64 / LDS.128 under
// broadcast patterns.  Every warp issues N dependent-free loads from per-lane offsets; the time
// ratio between patterns gives wavefronts per instruction.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/_build/lds_bench tools/lds_bench.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int W>  // W = 1: 64-bit loads, 2: 128-bit
__global__ void k(const int* __restrict__ offs, double* out, int iters) {
  __shared__ __align__(16) double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int o = offs[lane];
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int idx = (o + u * 64 + (it & 7) * 2) & 4095;
      if (W == 1) {
        double v;
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(s + idx)));
        if (u & 1) a1 += v; else a0 += v;
      } else {
        double v, w;
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v), "=d"(w) : "r"((unsigned)__cvta_generic_to_shared(s + (idx & ~1))));
        a2 += v; a3 += w;
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 + a1 + a2 + a3;
}
int main() {
  struct P { const char* name; int (*f)(int); };
  P pats[] = {
      {"all lanes one address", [](int l) { return 0; }},
      {"32 distinct consecutive", [](int l) { return l; }},
      {"pairs (l/2): aabb", [](int l) { return l / 2; }},
      {"trios (l/3)", [](int l) { return l / 3; }},
      {"abab, a/b adjacent doubles: (l/4)*2 + l%2", [](int l) { return (l / 4) * 2 + l % 2; }},
      {"abab, a/b far apart: (l/4) + 8*(l%2)", [](int l) { return (l / 4) + 8 * (l % 2); }},
      {"aaab: l%4==3 ? 8+l/4 : l/4", [](int l) { return l % 4 == 3 ? 8 + l / 4 : l / 4; }},
      {"abba: (l/4)*2 + ((l%4==1||l%4==2)?1:0)", [](int l) { return (l / 4) * 2 + ((l % 4 == 1 || l % 4 == 2) ? 1 : 0); }},
      {"abcd in 16B pairs: l%4", [](int l) { return l % 4; }},
      {"l%2 (abab, 2 distinct)", [](int l) { return l % 2; }},
      {"pairs in same 16B chunk, 16 chunks: l", [](int l) { return l; }},
      {"pairs in same 16B chunk, 8 chunks: (l/4)*2+l%2 (dup)", [](int l) { return (l / 4) * 2 + l % 2; }},
      {"8-groups aaaabbbb.. (l/4)", [](int l) { return l / 4; }},
      {"8-groups aaabaaab: l%8==3||l%8==7 ? 8+l/8 : l/8", [](int l) { return (l % 4 == 3) ? 8 + l / 8 : l / 8; }},
      {"lane l and l^2 same: (l/4)*2+(l%2) == abab", [](int l) { return (l / 4) * 2 + (l % 2); }},
      {"aabb with a,b same 16B chunk: l/2 (dup)", [](int l) { return l / 2; }},
      {"aabb, 3-stride: 3*(l/2) mod 16", [](int l) { return (3 * (l / 2)) % 16; }},
      {"trio+idle via same addr: aaaa (l/4)*3", [](int l) { return (l / 4) * 3 % 16; }},
  };
  int* d_offs; double* d_out;
  cudaMalloc(&d_offs, 32 * sizeof(int));
  const int blocks = 148 * 4, threads = 256, iters = 4000;
  cudaMalloc(&d_out, blocks * threads * sizeof(double));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 1; w <= 2; ++w) {
    printf("== %d-bit loads\n", w * 64);
    for (auto& p : pats) {
      int h[32];
      for (int l = 0; l < 32; ++l) h[l] = p.f(l) * (w == 2 ? 2 : 1);
      cudaMemcpy(d_offs, h, sizeof(h), cudaMemcpyHostToDevice);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        if (w == 1) k<1><<<blocks, threads>>>(d_offs, d_out, iters); else k<2><<<blocks, threads>>>(d_offs, d_out, iters);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
      }
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      // warp-instructions per SM = 4 blocks * 8 warps * iters * 16; clocks ~ ms * 1.965e6
      const double winst = 4.0 * 8 * iters * 16;
      printf("  %-52s %.3f ms  %.2f clk per warp-load per SM\n", p.name, ms, ms * 1.965e6 / winst);
    }
  }
  return 0;
}
