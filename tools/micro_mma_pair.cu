// Microbenchmark: tcgen05.mma throughput of the attention shapes, one SM (cta_group::1, M=128)
// vs a CTA pair (cta_group::2, M=256, B split across the pair), no TMA traffic.
//   SS : S += Q K^T step (A, B from smem), TS : O += P V step (A from TMEM), ALT: 8 SS + 8 TS.
// Prints cycles per MMA instruction (each instruction = 128 rows x N x 16 per SM).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2502_21079_b200/csrc/common.cuh"
using namespace adaspa;

template <int MODE, bool PAIR>
__global__ void __launch_bounds__(128, 1) mma_kernel(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar, bar2[4];
  __shared__ uint32_t tbase;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = PAIR ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) mbar_init(&bar2[i], 1); fence_mbar_init(); }
  if (warp == 0) {
    if (PAIR) { tmem_alloc_pair(&tbase, 512); tmem_relinquish_pair(); }
    else { tmem_alloc(&tbase, 512); tmem_relinquish(); }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tbase;
  if (threadIdx.x == 0 && rank == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    constexpr int M = PAIR ? 256 : 128;
    constexpr uint32_t id_ss = idesc_bf16(M, 128, false, false);
    constexpr uint32_t id_ts = idesc_bf16(M, 128, false, true);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (MODE == 7 || MODE == 8) {  // one 128-row kv tile of attention at d=128, one q tile
        // 7: QK as 8 SS N=128 + PV as 8 TS N=128 (P aliased in S)
        // 8: two 64-row half steps, each 8 SS N=64 (QK) + 4 TS N=128 (PV, K=64)
        constexpr uint32_t id64 = idesc_bf16(128, 64, false, false);
#pragma unroll
        for (int hs = 0; hs < (MODE == 7 ? 1 : 2); ++hs) {
#pragma unroll
          for (int kk = 0; kk < 8; ++kk) {
            const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
            const uint64_t ad = desc_sw128(a + off, 16, 1024), bd = desc_sw128(b + off + hs * 8192, 16, 1024);
            if (MODE == 7) mma_ss(tmem, ad, bd, id_ss, 1u);
            else mma_ss(tmem + 64 * hs, ad, bd, id64, 1u);
          }
#pragma unroll
          for (int kk = 0; kk < (MODE == 7 ? 8 : 4); ++kk) {
            const uint64_t bv = desc_sw128(b + (hs * 4 + kk) * 2048, 16384, 1024);
            mma_ts(tmem + 384, tmem + 128 + (hs * 4 + kk) * 8, bv, id_ts, 1u);
          }
        }
        continue;
      }
      if (MODE == 6) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          const uint64_t ad = desc_sw128(a + off, 16, 1024), bd = desc_sw128(b + off, 16, 1024);
          const uint64_t bv = desc_sw128(b + kk * 2048, 16384, 1024);
          if (PAIR) { mma_ts_pair(tmem + 384, tmem + 128 + kk * 8, bv, id_ts, 1u); mma_ss_pair(tmem, ad, bd, id_ss, 1u); }
          else { mma_ts(tmem + 384, tmem + 128 + kk * 8, bv, id_ts, 1u); mma_ss(tmem, ad, bd, id_ss, 1u); }
        }
        if (PAIR) tc_commit_pair(&bar2[3]); else tc_commit(&bar2[3]);
        mbar_wait(&bar2[3], i & 1);  // drain every iteration, like the kernel's waits
        continue;
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
        if (MODE == 0 || MODE >= 2) {
          const uint64_t ad = desc_sw128(a + off, 16, 1024), bd = desc_sw128(b + off, 16, 1024);
          if (PAIR) mma_ss_pair(tmem, ad, bd, id_ss, 1u); else mma_ss(tmem, ad, bd, id_ss, 1u);
        }
      }
      if (MODE == 3) { if (PAIR) tc_commit_pair(&bar2[0]); else tc_commit(&bar2[0]); }  // commit between the groups
      if (MODE == 5) {  // drain between the groups: wait for every MMA issued so far
        if (PAIR) tc_commit_pair(&bar2[3]); else tc_commit(&bar2[3]);
        mbar_wait(&bar2[3], i & 1);
      }
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        if (MODE == 1 || MODE >= 2) {
          const uint64_t bd = desc_sw128(b + kk * 2048, 16384, 1024);
          if (PAIR) mma_ts_pair(tmem + 384, tmem + 128 + kk * 8, bd, id_ts, 1u);
          else mma_ts(tmem + 384, tmem + 128 + kk * 8, bd, id_ts, 1u);
        }
      }
      if (MODE == 4) { if (PAIR) { tc_commit_pair(&bar2[1]); tc_commit_pair(&bar2[2]); } else { tc_commit(&bar2[1]); tc_commit(&bar2[2]); } }
    }
    if (PAIR) tc_commit_pair(&bar); else tc_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  if (PAIR && threadIdx.x == 0 && rank == 1) mbar_wait(&bar, 0);
  tc_fence_before();
  if (PAIR) cluster_sync_all(); else __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    if (PAIR) tmem_dealloc_pair(tmem, 512); else tmem_dealloc(tmem, 512);
  }
}

template <int MODE, bool PAIR>
void run(const char* name, int grid, unsigned long long* d) {
  const int iters = 2000;
  auto kern = mma_kernel<MODE, PAIR>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 140000;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = PAIR ? 2 : 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, iters, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[148] = {0};
  cudaMemcpy(h, d, 8 * grid, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const int per_iter = MODE >= 2 ? 16 : 8;  // modes 7/8: per 16 N=128-equivalent MMAs
  printf("%-34s grid %3d %s  cycles/MMA = %.1f\n", name, grid, cudaGetErrorString(e), (double)mx / (iters * per_iter));
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8 * 148);
  for (int grid : {2, 148}) {
    run<0, false>("1SM SS M128 N128 (QK)", grid, d);
    run<1, false>("1SM TS M128 N128 (PV)", grid, d);
    run<2, false>("1SM 8 SS + 8 TS", grid, d);
    run<0, true>("pair SS M256 N128 (QK)", grid, d);
    run<1, true>("pair TS M256 N128 (PV)", grid, d);
    run<2, true>("pair 8 SS + 8 TS", grid, d);
    run<3, true>("pair 8 SS, commit, 8 TS", grid, d);
    run<4, true>("pair 8 SS + 8 TS, 2 commits", grid, d);
    run<3, false>("1SM 8 SS, commit, 8 TS", grid, d);
    run<5, true>("pair 8 SS, drain, 8 TS", grid, d);
    run<6, true>("pair (TS,SS) x8 interleaved, drain", grid, d);
    run<5, false>("1SM 8 SS, drain, 8 TS", grid, d);
    run<7, false>("1SM kv tile: 8 SS128 + 8 TS", grid, d);
    run<8, false>("1SM kv tile: 2x(8 SS64 + 4 TS)", grid, d);
  }
  return 0;
}
