// Microbenchmark: tcgen05.mma issue/execute rate for the attention shapes (one CTA, one SM).
//   SS  : D[128x128] += A[128x16] (smem) * B[16x128] (smem)      (QK^T step)
//   TS  : D[128x128] += A[128x16] (tmem) * B[16x128] (smem)      (PV step, P in TMEM)
// cycles per MMA with descriptors precomputed vs recomputed per MMA.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2502_21079_b200/csrc/common.cuh"
using namespace adaspa;

template <int MODE, int N>
__global__ void mma_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    constexpr uint32_t idesc = idesc_bf16(128, N, false, MODE == 1);
    const uint64_t ad = desc_sw128(a, 16, 1024), bd = desc_sw128(b, MODE == 1 ? 16384 : 16, 1024);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 0) mma_ss(tmem, ad + 2 * kk, bd + 2 * kk, idesc, 1u);
        else if (MODE == 1) mma_ts(tmem + 256, tmem + kk * 8, bd + 128 * kk, idesc, 1u);
        else {  // recomputed descriptors like the attention kernel
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tmem, desc_sw128(a + off, 16, 1024), desc_sw128(b + off, 16, 1024), idesc, 1u);
        }
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 64);
  const int iters = 2000;
  auto run = [&](auto kern, const char* name) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    kern<<<1, 128, 140000>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-32s %s  cycles/MMA = %.1f\n", name, cudaGetErrorString(e), (double)h / (iters * 8));
  };
  run(mma_kernel<0, 128>, "SS M128 N128 K16 (precomputed)");
  run(mma_kernel<2, 128>, "SS M128 N128 K16 (recomputed)");
  run(mma_kernel<1, 128>, "TS M128 N128 K16 (A in TMEM)");
  run(mma_kernel<0, 256>, "SS M128 N256 K16 (precomputed)");
  run(mma_kernel<1, 64>, "TS M128 N64 K16");
  return 0;
}
