// Microbenchmark: per-SM throughput of FFMA (3-reg / imm), FFMA2, FADD2, MUFU.EX2, F2FP pack,
// FMNMX3, IMAD.  8 warps, 8 independent chains per thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2502_21079_b200/csrc/common.cuh"
using namespace adaspa;

template <int OP>
__global__ void pipe_kernel(int iters, unsigned long long* out, float* sink, float a, float b) {
  float x[8];
  float2 y[8];
  uint32_t u[8];
  for (int k = 0; k < 8; ++k) { x[k] = threadIdx.x * 1e-3f + k; y[k] = make_float2(x[k], x[k] + 1); u[k] = threadIdx.x + k; }
  const float2 av = make_float2(a, a), bv = make_float2(b, b);
  __syncthreads();
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) x[k] = fmaf(x[k], a, b);                    // FFMA 3-reg
      if (OP == 1) x[k] = fmaf(x[k], 1.0001f, 0.37f);          // FFMA imm
      if (OP == 2) y[k] = ffma2(y[k], av, bv);                 // FFMA2
      if (OP == 3) y[k] = fadd2(y[k], bv);                     // FADD2
      if (OP == 4) x[k] = ex2_approx(x[k]);                    // MUFU.EX2
      if (OP == 5) u[k] = pack_bf16x2(__uint_as_float(u[k]), x[k]);  // F2FP
      if (OP == 6) x[k] = fmax3(x[k], a, b);                   // FMNMX3
      if (OP == 7) u[k] = u[k] * 8388608u + (uint32_t)(a);     // IMAD
      if (OP == 8) x[k] = x[k] + a;                            // FADD
    }
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[threadIdx.x >> 5] = t1 - t0;
  float s = 0;
  for (int k = 0; k < 8; ++k) s += x[k] + y[k].x + y[k].y + __uint_as_float(u[k]);
  sink[threadIdx.x] = s;
}

int main() {
  unsigned long long* d; float* sink;
  cudaMalloc(&d, 64 * 8); cudaMalloc(&sink, 4096 * 4);
  const char* names[] = {"FFMA 3-reg", "FFMA imm", "FFMA2", "FADD2", "MUFU.EX2", "F2FP.BF16 pack", "FMNMX3", "IMAD", "FADD"};
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    for (int op = 0; op < 9; ++op) {
      void (*k)(int, unsigned long long*, float*, float, float);
      switch (op) { case 0: k = pipe_kernel<0>; break; case 1: k = pipe_kernel<1>; break; case 2: k = pipe_kernel<2>; break;
        case 3: k = pipe_kernel<3>; break; case 4: k = pipe_kernel<4>; break; case 5: k = pipe_kernel<5>; break;
        case 6: k = pipe_kernel<6>; break; case 7: k = pipe_kernel<7>; break; default: k = pipe_kernel<8>; }
      k<<<1, warps * 32>>>(iters, d, sink, 0.999f, 0.001f);
      cudaDeviceSynchronize();
      unsigned long long h[64]; cudaMemcpy(h, d, warps * 8, cudaMemcpyDeviceToHost);
      double cyc = 0; for (int w = 0; w < warps; ++w) cyc = cyc > h[w] ? cyc : h[w];
      printf("warps=%2d %-16s warp-instr/clk/SM = %.3f   (lane-ops/clk/SM = %.1f)\n", warps, names[op],
             (double)iters * 8 * warps / cyc, (double)iters * 8 * warps * 32 / cyc);
    }
  }
  return 0;
}
