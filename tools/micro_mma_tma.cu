// Do SS tcgen05.mma operand reads starve TMA writes into shared memory?  Thread 0 (warp 0) streams
// 32 KB TMA tiles through a 3-slot ring (warp 1 releases them); thread 64 (warp 2) issues MMAs from a
// separate smem region: MODE 0 none, 1 = SS M128N128K16 back to back, 2 = TS (A from TMEM).
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2502_21079_b200/csrc/common.cuh"
using namespace adaspa;

template <int MODE>
__global__ void __launch_bounds__(128, 1) kern(const __grid_constant__ CUtensorMap tk, int ntiles,
                                               unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[3], empty[3], mbar;
  __shared__ uint32_t tbase;
  __shared__ volatile int stop;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 3; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    mbar_init(&mbar, 1);
    fence_mbar_init();
    stop = 0;
  }
  if (warp == 3) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  const int h = blockIdx.x % 24;
  if (threadIdx.x == 0) {
    uint32_t ph = 0; int slot = 0;
    unsigned long long t0 = clock64();
    for (int j = 0; j < ntiles; ++j) {
      mbar_wait(&empty[slot], ph ^ 1);
      mbar_arrive_expect_tx(&full[slot], 32768);
      uint8_t* dst = smem + 65536 + slot * 32768;
      const int row = (j * 128) % 111744;
      for (int c = 0; c < 2; ++c) {
        tma_load_4d(&tk, &full[slot], dst + c * 16384, c * 64, row, h, 0);
        tma_load_4d(&tk, &full[slot], dst + c * 16384 + 8192, c * 64, row + 64, h, 0);
      }
      if (++slot == 3) { slot = 0; ph ^= 1; }
    }
    (void)t0;
  } else if (threadIdx.x == 32) {
    uint32_t ph = 0; int slot = 0;
    unsigned long long t0 = clock64();
    for (int j = 0; j < ntiles; ++j) {
      mbar_wait(&full[slot], ph);
      mbar_arrive(&empty[slot]);
      if (++slot == 3) { slot = 0; ph ^= 1; }
    }
    unsigned long long t1 = clock64();
    out[blockIdx.x * 2] = t1 - t0;
    stop = 1;
  } else if (threadIdx.x == 64 && MODE > 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
    constexpr uint32_t idesc = idesc_bf16(128, 128, false, MODE == 2);
    const uint64_t ad = desc_sw128(a, 16, 1024), bd = desc_sw128(b, MODE == 2 ? 16384 : 16, 1024);
    unsigned long long n = 0;
    unsigned long long t0 = clock64();
    uint32_t mph = 0;
    while (!stop) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 1) mma_ss(tmem, ad + 2 * kk, bd + 2 * kk, idesc, 1u);
        else mma_ts(tmem + 256, tmem + kk * 8, bd + 128 * kk, idesc, 1u);
      }
      n += 8;
      if ((n & 63) == 0) { tc_commit(&mbar); mbar_wait(&mbar, mph); mph ^= 1; }
    }
    tc_commit(&mbar); mbar_wait(&mbar, mph);
    unsigned long long t1 = clock64();
    out[blockIdx.x * 2 + 1] = (t1 - t0) / (n ? n : 1);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 3) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  const int H = 24, N = 111856, D = 128;
  __nv_bfloat16* k; cudaMalloc(&k, (size_t)H * N * D * 2);
  cudaMemset(k, 0, (size_t)H * N * D * 2);
  unsigned long long* d; cudaMalloc(&d, 1024 * 8);
  CUtensorMap tk;
  cuuint64_t dims[4] = {(cuuint64_t)D, (cuuint64_t)N, (cuuint64_t)H, 1};
  cuuint64_t str[3] = {(cuuint64_t)D * 2, (cuuint64_t)N * D * 2, (cuuint64_t)H * N * D * 2};
  cuuint32_t box[4] = {64, 64, 1, 1}, es[4] = {1, 1, 1, 1};
  cuTensorMapEncodeTiled(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, k, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int ntiles = 2000;
  auto run = [&](auto kern, const char* name) {
    const int smem = 65536 + 3 * 32768 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<148, 128, smem>>>(tk, ntiles, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long hst[300]; cudaMemcpy(hst, d, 296 * 8, cudaMemcpyDeviceToHost);
    double mx = 0, mma = 0; for (int i = 0; i < 148; ++i) { mx = mx > hst[2 * i] ? mx : hst[2 * i]; mma += hst[2 * i + 1]; }
    printf("%-26s %s  TMA fill %.1f B/clk/SM   MMA %.1f cycles/MMA\n", name, cudaGetErrorString(e),
           (double)ntiles * 32768 / mx, mma / 148);
  };
  run(kern<0>, "TMA alone");
  run(kern<1>, "TMA + SS MMA loop");
  run(kern<2>, "TMA + TS MMA loop");
  return 0;
}
