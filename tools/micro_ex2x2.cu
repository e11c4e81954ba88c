// Microbenchmark: MUFU.EX2 throughput per SM for fp32, packed f16x2 and packed bf16x2 operands
// (does a packed exponential deliver two results per MUFU issue?).  8 independent chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int OP>
__global__ void k(int iters, unsigned long long* out, float* sink) {
  uint32_t u[8];
  float x[8];
  for (int i = 0; i < 8; ++i) { x[i] = -1e-3f * (threadIdx.x + i); u[i] = 0xBC00BC00u ^ (threadIdx.x + i); }
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[i]));
      if (OP == 1) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[i]));
      if (OP == 2) asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u[i]));
      if (OP == 3) asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(x[i]), "f"(__uint_as_float(u[i])));
      if (OP == 4) { uint32_t r; asm volatile("{.reg .f16 a, b; mov.b32 {a, b}, %1; cvt.f32.f16 %0, a;}" : "=f"(x[i]) : "r"(u[i])); u[i] += 1; }
    }
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[threadIdx.x >> 5] = t1 - t0;
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i] + __uint_as_float(u[i]);
  sink[threadIdx.x] = s;
}

int main() {
  unsigned long long* d; float* sink;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&sink, 4096 * 4);
  const char* names[] = {"ex2.f32", "ex2.f16x2", "ex2.bf16x2", "cvt.f16x2.f32", "cvt.f32.f16"};
  const int iters = 4096;
  for (int warps : {8, 16}) {
    for (int op = 0; op < 5; ++op) {
      void (*f)(int, unsigned long long*, float*);
      switch (op) { case 0: f = k<0>; break; case 1: f = k<1>; break; case 2: f = k<2>; break; case 3: f = k<3>; break; default: f = k<4>; }
      f<<<1, warps * 32>>>(iters, d, sink);
      cudaDeviceSynchronize();
      unsigned long long h[64]; cudaMemcpy(h, d, warps * 8, cudaMemcpyDeviceToHost);
      double cyc = 0; for (int w = 0; w < warps; ++w) cyc = cyc > h[w] ? cyc : h[w];
      printf("warps=%2d %-14s warp-instr/clk/SM = %.3f  lane-ops/clk/SM = %.1f\n", warps, names[op],
             (double)iters * 8 * warps / cyc, (double)iters * 8 * warps * 32 / cyc);
    }
  }
  return 0;
}
