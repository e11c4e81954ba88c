// Does SMEM traffic from other warps slow tcgen05.mma?  MMA loop (SS or TS, M128 N128 K16) issued
// by thread 0 while warps 1..NW write shared memory (st.shared.v4) as fast as they can.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2502_21079_b200/csrc/common.cuh"
using namespace adaspa;

template <int MODE, int NW>
__global__ void kern(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); stop = 0; }
  if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    constexpr uint32_t idesc = idesc_bf16(128, 128, false, MODE == 1);
    const uint64_t ad = desc_sw128(a, 16, 1024), bd = desc_sw128(b, MODE == 1 ? 16384 : 16, 1024);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 0) mma_ss(tmem, ad + 2 * kk, bd + 2 * kk, idesc, 1u);
        else mma_ts(tmem + 256, tmem + kk * 8, bd + 128 * kk, idesc, 1u);
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[0] = t1 - t0;
    stop = 1;
  } else if (warp >= 1 && warp <= NW) {
    // each writer warp streams 16-B stores over its own 8 KB region (bytes counted per warp)
    uint8_t* base = smem + 131072 + (warp - 1) * 8192;
    unsigned long long n = 0;
    uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
    unsigned long long t0 = clock64();
    while (!stop) {
#pragma unroll
      for (int r = 0; r < 16; ++r) {
        asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(smem_u32(base + (((r * 32 + (threadIdx.x & 31)) * 16) & 8191))),
                     "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
      }
      n += 16 * 32 * 16;
    }
    unsigned long long t1 = clock64();
    if ((threadIdx.x & 31) == 0) { out[warp * 2] = n; out[warp * 2 + 1] = t1 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d; cudaMalloc(&d, 1024);
  const int iters = 2000;
  auto run = [&](auto k, const char* name, int nw) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    cudaMemset(d, 0, 1024);
    k<<<1, 32 * (1 + 8), 200000>>>(iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[64]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
    double bytes = 0, cyc = 1;
    for (int w = 1; w <= nw; ++w) { bytes += h[w * 2]; cyc = h[w * 2 + 1] > cyc ? h[w * 2 + 1] : cyc; }
    printf("%-28s %s  cycles/MMA = %.1f   concurrent st.shared = %.1f B/clk\n", name, cudaGetErrorString(e),
           (double)h[0] / (iters * 8), bytes / cyc);
  };
  run(kern<0, 0>, "SS, no smem traffic", 0);
  run(kern<0, 2>, "SS, 2 writer warps", 2);
  run(kern<0, 8>, "SS, 8 writer warps", 8);
  run(kern<1, 0>, "TS, no smem traffic", 0);
  run(kern<1, 2>, "TS, 2 writer warps", 2);
  run(kern<1, 8>, "TS, 8 writer warps", 8);
  return 0;
}
