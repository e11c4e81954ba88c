// tcgen05.mma issue pattern of the attention kernel: per "tile", 8 TS MMAs (PV: A = P read from TMEM
// columns [s, s+64), D = O) followed by 8 SS MMAs (QK: D = S at columns [s, s+128)).  ALIAS=1: P lives
// in S's columns (write-after-read inside the tensor pipe), ALIAS=0: P in separate columns.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2502_21079_b200/csrc/common.cuh"
using namespace adaspa;

template <int ALIAS, int TILES>
__global__ void kern(int iters, unsigned long long* out) {
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
    constexpr uint32_t idqk = idesc_bf16(128, 128, false, false);
    constexpr uint32_t idpv = idesc_bf16(128, 128, false, true);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int t = 0; t < TILES; ++t) {
        const uint32_t s_col = t * 128;                         // S_t
        const uint32_t o_col = 256 + t * 128;                   // O_t
        const uint32_t p_col = ALIAS ? s_col : (TILES == 1 ? 128 : s_col + 64);  // P_t
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tmem + o_col, tmem + p_col + kk * 8, desc_sw128(b + kk * 2048, 16384, 1024), idpv, 1u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tmem + s_col, desc_sw128(a + off, 16, 1024), desc_sw128(b + off, 16, 1024), idqk, kk > 0);
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
  const int iters = 1000;
  auto run = [&](auto k, const char* name, int tiles) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    k<<<1, 128, 140000>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h = 0; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %s  cycles/MMA = %.1f\n", name, cudaGetErrorString(e), (double)h / (iters * 16 * tiles));
  };
  run(kern<1, 2>, "2 tiles, P aliased into S (kernel)", 2);
  run(kern<0, 2>, "2 tiles, P in S's spare upper half", 2);
  run(kern<1, 1>, "1 tile, P aliased", 1);
  run(kern<0, 1>, "1 tile, P separate", 1);
  return 0;
}
