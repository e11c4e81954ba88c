// Does TMEM traffic (tcgen05.ld / tcgen05.st by other warps) slow tcgen05.mma?  Thread 0 runs the
// attention MMA pattern (8 TS into O, 8 SS into S, two tiles); warps 4..11 (two warpgroups, all lane
// quarters) loop LDTM.x32 (MODE 1), STTM.x16 (MODE 2) or FFMA/MUFU work only (MODE 3) on the S columns.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2502_21079_b200/csrc/common.cuh"
using namespace adaspa;

template <int MODE, int FILL = 0>
__global__ void kern(int iters, unsigned long long* out, float* sink) {
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
  if (FILL) {  // random-looking bf16 operands (power depends on the data)
    for (int i = threadIdx.x; i < 131072 / 4; i += blockDim.x) {
      uint32_t x = (i * 2654435761u) ^ (blockIdx.x * 97u);
      x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
      reinterpret_cast<uint32_t*>(smem)[i] = (x & 0x3fff3fffu) | 0x3c003c00u;  // |v| in [1, 2)-ish bf16 pairs
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 65536);
    constexpr uint32_t idqk = idesc_bf16(128, 128, false, false);
    constexpr uint32_t idpv = idesc_bf16(128, 128, false, true);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          mma_ts(tmem + 256 + t * 128, tmem + t * 128 + kk * 8, desc_sw128(b + kk * 2048, 16384, 1024), idpv, 1u);
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t off = (kk >> 2) * 16384 + (kk & 3) * 32;
          mma_ss(tmem + t * 128, desc_sw128(a + off, 16, 1024), desc_sw128(b + off, 16, 1024), idqk, kk > 0);
        }
      }
    }
    tc_commit(&bar);
    mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
    stop = 1;
  } else if (warp >= 4 && warp < 12) {
    const uint32_t lb = static_cast<uint32_t>((warp & 3) * 32) << 16;
    const uint32_t col = ((warp - 4) >> 2) * 128 + 64;   // upper half of S_t (not read by PV)
    float acc = 0.f;
    unsigned long long n = 0;
    unsigned long long t0 = clock64();
    while (!stop) {
      if (MODE == 1) {
        uint32_t r[32];
        tmem_ld32(tmem + lb + col, r);
        tmem_ld_wait32(r);
        acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
        n += 4096;
      } else if (MODE == 2) {
        uint32_t r[16];
        for (int k = 0; k < 16; ++k) r[k] = k + threadIdx.x;
        tmem_st16(tmem + lb + col, r);
        tmem_st_wait();
        n += 2048;
      } else if (MODE == 3) {
#pragma unroll
        for (int k = 0; k < 32; ++k) acc = ex2_approx(fmaf(acc, 0.999f, -0.001f * k));
        n += 1;
      }
    }
    unsigned long long t1 = clock64();
    if (blockIdx.x == 0 && (threadIdx.x & 31) == 0) { out[warp * 2] = n; out[warp * 2 + 1] = t1 - t0; }
    sink[threadIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  unsigned long long* d; float* sink;
  cudaMalloc(&d, 1024); cudaMalloc(&sink, 4096 * 4);
  const int iters = 1000;
  auto run = [&](auto k, const char* name, int grid = 1) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    cudaMemset(d, 0, 1024);
    k<<<grid, 384, 140000>>>(iters, d, sink);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[64]; cudaMemcpy(h, d, 512, cudaMemcpyDeviceToHost);
    double bytes = 0, cyc = 1;
    for (int w = 4; w < 12; ++w) { bytes += h[w * 2]; cyc = h[w * 2 + 1] > cyc ? h[w * 2 + 1] : cyc; }
    printf("%-36s %s  cycles/MMA = %.1f   side traffic = %.1f B/clk (or ops/clk)\n", name, cudaGetErrorString(e),
           (double)h[0] / (iters * 32), bytes / cyc);
  };
  run(kern<0>, "MMA only");
  run(kern<1>, "MMA + LDTM x32 loop (8 warps)");
  run(kern<2>, "MMA + STTM x16 loop (8 warps)");
  run(kern<3>, "MMA + FFMA/MUFU loop (8 warps)");
  run(kern<0, 1>, "MMA only, random data, 1 SM");
  run(kern<0, 1>, "MMA only, random data, 148 SMs", 148);
  run(kern<3, 1>, "MMA+MUFU, random data, 148 SMs", 148);
  run(kern<0, 0>, "MMA only, zero data, 148 SMs", 148);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    kern<0, 1><<<148, 384, 140000>>>(20000, d, sink);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h; cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("148 SMs random data 20000 iters: %.2f ms, cycles/MMA %.1f, implied clock %.0f MHz, %.0f TFLOP/s\n", ms,
           (double)h / (20000 * 32), (double)h / (ms * 1e3), 148.0 * 20000 * 32 * 2.0 * 128 * 128 * 16 / (ms * 1e9));
  }
  return 0;
}
