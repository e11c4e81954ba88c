// L2 -> SMEM bandwidth with TMA at full chip: every CTA (one per SM) streams the K rows of one head
// (the attention kernels' access pattern: 128-row x 128-col bf16 tiles = 32 KB, four 64x64 boxes with
// 128-byte swizzle) through an NS-slot ring; CTAs of the same head run concurrently (L2-resident K).
//   MULTI=2: clusters of 2 CTAs, each loads half of every tile and multicasts it to both CTAs.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include "../paper_2502_21079_b200/csrc/common.cuh"
using namespace adaspa;

template <int NS, int MULTI>
__global__ void __launch_bounds__(128, 1) tma_kernel(const __grid_constant__ CUtensorMap tk, int ntiles, int heads,
                                                     unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t full[NS], empty[NS];
  uint32_t rank = 0;
  if (MULTI > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], MULTI); }
    fence_mbar_init();
  }
  if (MULTI > 1) { asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
  else __syncthreads();
  const int cl = MULTI > 1 ? blockIdx.x / MULTI : blockIdx.x;
  const int h = cl % heads;
  unsigned long long t0 = clock64();
  if (threadIdx.x == 0) {  // producer
    uint32_t ph = 0;
    int slot = 0;
    for (int j = 0; j < ntiles; ++j) {
      mbar_wait(&empty[slot], ph ^ 1);
      mbar_arrive_expect_tx(&full[slot], 32768);
      uint8_t* dst = smem + slot * 32768;
      const int row = (j * 128) % 111744;
      if (MULTI == 1) {
        for (int c = 0; c < 2; ++c) {
          tma_load_4d(&tk, &full[slot], dst + c * 16384, c * 64, row, h, 0);
          tma_load_4d(&tk, &full[slot], dst + c * 16384 + 8192, c * 64, row + 64, h, 0);
        }
      } else {  // my half (column chunk = rank) to both CTAs of the pair
        for (int r = 0; r < 2; ++r) {
          const uint32_t d = smem_u32(dst + rank * 16384 + r * 8192);
          asm volatile(
              "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
              " [%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(d), "l"(reinterpret_cast<uint64_t>(&tk)),
              "r"(smem_u32(&full[slot])), "r"((int)rank * 64), "r"(row + r * 64), "r"(h), "r"(0), "h"((uint16_t)3)
              : "memory");
        }
      }
      if (++slot == NS) { slot = 0; ph ^= 1; }
    }
  } else if (threadIdx.x == 32) {  // consumer: wait full, release (in both CTAs for multicast)
    uint32_t ph = 0;
    int slot = 0;
    for (int j = 0; j < ntiles; ++j) {
      mbar_wait(&full[slot], ph);
      if (MULTI == 1) mbar_arrive(&empty[slot]);
      else {
        for (uint32_t c = 0; c < 2; ++c) {
          uint32_t remote;
          asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&empty[slot])), "r"(c));
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
        }
      }
      if (++slot == NS) { slot = 0; ph ^= 1; }
    }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
  if (MULTI > 1) { asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
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
  CUresult r = cuTensorMapEncodeTiled(&tk, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, k, dims, str, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("encode failed %d\n", r); return 1; }
  const int ntiles = 3000;
  auto run = [&](auto kern, int ns, int multi, int grid) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * 32768 + 1024);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(128); cfg.dynamicSmemBytes = ns * 32768 + 1024;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = multi; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaLaunchKernelEx(&cfg, kern, tk, ntiles, H, d);  // warm
    cudaEventRecord(e0);
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, tk, ntiles, H, d);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[256]; cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
    double mx = 0; for (int i = 0; i < grid; ++i) mx = mx > h[i] ? mx : h[i];
    double smem_bytes = (double)grid * ntiles * 32768;   // bytes landing in SMEM
    double l2_bytes = smem_bytes / multi;                 // bytes read from L2
    printf("NS=%d multicast x%d grid %d: %s  %.3f ms  SMEM fill %.2f TB/s (%.0f B/clk/SM)  L2 reads %.2f TB/s\n", ns, multi,
           grid, cudaGetErrorString(e), ms, smem_bytes / ms / 1e9, smem_bytes / grid / mx, l2_bytes / ms / 1e9);
  };
  run(tma_kernel<4, 1>, 4, 1, 148);
  run(tma_kernel<6, 1>, 6, 1, 148);
  run(tma_kernel<4, 2>, 4, 2, 148);
  run(tma_kernel<6, 2>, 6, 2, 148);
  run(tma_kernel<4, 1>, 4, 1, 74);
  return 0;
}
