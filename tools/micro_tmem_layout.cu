// Probe: fragment layout of tcgen05.ld shapes 16x64b / 16x128b / 16x256b / 32x32b (which TMEM lane
// and column each (thread, register) receives).  TMEM is filled with lane*1000 + column through
// 32x32b stores first.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2502_21079_b200/csrc/common.cuh"
using namespace adaspa;

__global__ void probe(uint32_t* out) {
  __shared__ uint32_t base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) { tmem_alloc(&base, 512); tmem_relinquish(); }
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t t = base;
  // fill: warp w -> lanes 32w..32w+31, columns 0..63
  for (int c = 0; c < 64; c += 32) {
    uint32_t r[32];
    for (int i = 0; i < 32; ++i) r[i] = (32 * warp + lane) * 1000 + c + i;
    tmem_st32(t + ((32u * warp) << 16) + c, r);
  }
  tmem_st_wait();
  tc_fence_before(); __syncthreads(); tc_fence_after();
  if (warp == 1) {  // lane quarter 1 (lanes 32..63), lane offset +16 to see the half
    uint32_t a[4], b[2], c1[1], d[4], e[8];
    const uint32_t ta = t + ((32u + 16u) << 16);
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x1.b32 {%0}, [%1];" : "=r"(c1[0]) : "r"(ta));
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];" : "=r"(b[0]), "=r"(b[1]) : "r"(ta));
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x1.b32 {%0,%1}, [%2];" : "=r"(a[0]), "=r"(a[1]) : "r"(ta));
    asm volatile("tcgen05.ld.sync.aligned.16x128b.x2.b32 {%0,%1,%2,%3}, [%4];" : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]) : "r"(ta));
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x1.b32 {%0,%1,%2,%3}, [%4];" : "=r"(a[0]), "=r"(a[1]), "=r"(a[2]), "=r"(a[3]) : "r"(ta));
    asm volatile("tcgen05.ld.sync.aligned.16x256b.x2.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(e[0]), "=r"(e[1]), "=r"(e[2]), "=r"(e[3]), "=r"(e[4]), "=r"(e[5]), "=r"(e[6]), "=r"(e[7]) : "r"(ta));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    uint32_t* o = out + lane * 32;
    o[0] = c1[0]; o[1] = b[0]; o[2] = b[1];
    for (int i = 0; i < 4; ++i) o[3 + i] = d[i];
    for (int i = 0; i < 4; ++i) o[7 + i] = a[i];
    for (int i = 0; i < 8; ++i) o[11 + i] = e[i];
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(t, 512); }
}

int main() {
  uint32_t* d; cudaMalloc(&d, 32 * 32 * 4); cudaMemset(d, 0xff, 32 * 32 * 4);
  probe<<<1, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  uint32_t h[32 * 32]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  const char* names[] = {"16x64b.x1", "16x64b.x2", "16x128b.x2", "16x256b.x1", "16x256b.x2"};
  const int off[] = {0, 1, 3, 7, 11}, cnt[] = {1, 2, 4, 4, 8};
  for (int s = 0; s < 5; ++s) {
    printf("%s (value = lane*1000 + col; base lane 48):\n", names[s]);
    for (int th = 0; th < 32; ++th) {
      printf("  t%02d:", th);
      for (int r = 0; r < cnt[s]; ++r) { uint32_t v = h[th * 32 + off[s] + r]; printf(" L%d/c%d", v / 1000, v % 1000); }
      printf("\n");
    }
  }
  return 0;
}
