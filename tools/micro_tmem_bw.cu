// Microbenchmarks on sm_100a: tcgen05.ld (TMEM -> registers) throughput and MUFU.EX2 throughput.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_bw tmem_bw.cu && ./tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

#define R8(a, o) "=r"(a[o+0]),"=r"(a[o+1]),"=r"(a[o+2]),"=r"(a[o+3]),"=r"(a[o+4]),"=r"(a[o+5]),"=r"(a[o+6]),"=r"(a[o+7])
__device__ __forceinline__ void ld32(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : R8(r,0), R8(r,8), R8(r,16), R8(r,24) : "r"(taddr));
}
__device__ __forceinline__ void ldwait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

template <int NLD>
__global__ void tmem_ld_kernel(int iters, unsigned long long* out, float* sink) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t t = base + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 128;
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    uint32_t r[NLD][32];
#pragma unroll
    for (int j = 0; j < NLD; ++j) ld32(t + j * 32, r[j]);
    ldwait();
#pragma unroll
    for (int j = 0; j < NLD; ++j) acc += r[j][0] ^ r[j][31];
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + warp] = t1 - t0;
  sink[threadIdx.x] = (float)acc;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

__global__ void ex2_kernel(int iters, unsigned long long* out, float* sink) {
  float x[32];
  for (int k = 0; k < 32; ++k) x[k] = -0.001f * (threadIdx.x + k);
  unsigned long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 32; ++k) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[k]));
      x[k] = y - 1.0f;
    }
  }
  unsigned long long t1 = clock64();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 32 + (threadIdx.x >> 5)] = t1 - t0;
  float s = 0;
  for (int k = 0; k < 32; ++k) s += x[k];
  sink[threadIdx.x] = s;
}

int main() {
  unsigned long long* d_out; float* sink;
  cudaMalloc(&d_out, 148 * 32 * 8); cudaMalloc(&sink, 1024 * 4);
  unsigned long long h[32];
  const int iters = 4096;
  for (int warps : {4, 8}) {
    for (int nld : {1, 4}) {
      if (nld == 1) tmem_ld_kernel<1><<<1, warps * 32>>>(iters, d_out, sink);
      else tmem_ld_kernel<4><<<1, warps * 32>>>(iters, d_out, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d_out, warps * 8, cudaMemcpyDeviceToHost);
      double bytes_per_warp = (double)iters * nld * 32 * 32 * 4;
      double cyc = 0; for (int w = 0; w < warps; ++w) cyc = cyc > h[w] ? cyc : h[w];
      printf("tcgen05.ld x32: warps=%d lds/iter=%d  cycles=%.0f  SM bytes/clk=%.1f  per-warp B/clk=%.1f\n",
             warps, nld, cyc, bytes_per_warp * warps / cyc, bytes_per_warp / cyc);
    }
  }
  for (int warps : {4, 8, 16}) {
    ex2_kernel<<<1, warps * 32>>>(iters, d_out, sink);
    cudaDeviceSynchronize();
    cudaMemcpy(h, d_out, warps * 8, cudaMemcpyDeviceToHost);
    double cyc = 0; for (int w = 0; w < warps; ++w) cyc = cyc > h[w] ? cyc : h[w];
    printf("ex2 (+FADD chain): warps=%d  ex2/clk/SM=%.2f\n", warps, (double)iters * 32 * 32 * warps / cyc);
  }
  return 0;
}
