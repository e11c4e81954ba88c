// blockmass.cu -- the second half of the fused search step t_w (Alg. 1):
// block masses from the per-(row, kv block) log-sum-exps that the dense pass wrote (attn_fwd.cu,
// kModeBlse), with the fresh LSE of the same pass:
//
//   block_mass[b,h,qb,kb] = sum_{i in qb} sum_{j in kb} exp(s_ij - lse_i)
//                         = sum_{i in qb} 2^(blse[b,h,kb,i] - lrel[b,h,i])
//
// (W_sum_attn, reading R4.)  Both operands are relative to the same per-row
// reference (the row's first running max), so their difference is formed from small numbers and
// keeps fp32 precision.  No QK^T recompute and no second pass of exponentials over S: the dense
// pass already computed every exp(s_ij - m_i); this kernel reads N*nb floats per head (HBM-bound)
// and does one exponential per (row, kv block).
#include "attn.cuh"
#include "common.cuh"
#include "select_row.cuh"

namespace adaspa {

namespace {

constexpr int kWarps = 8;

// One CTA per (b, h, q-block): warp w takes kv blocks w, w+8, ...; lane l holds rows l + 32r of the
// q-block (coalesced 128-byte loads along the token axis of blse[b,h,kb,:]); the q-block's mass row
// is staged in shared memory and written contiguously.
// 5 CTAs per SM (48 registers) keep enough loads in flight for HBM; the selection epilogue spills a
// few words at that size (one warp, once per CTA).
// KPL > 0: the RECALL selection epilogue of the fused search (f1) -- warp 0 selects the row from the
// shared-memory masses with K3's routine (select_row.cuh), so the mass row never makes a round trip
// through HBM for the selection; KPL = ceil(nb/32) rounded up to an instantiated size.
template <int R, int KPL>
__global__ void __launch_bounds__(kWarps * 32, 5) block_mass_kernel(BlockMassParams p) {
  extern __shared__ float mrow[];
  const int nb = p.grid.nb;
  const int qb = blockIdx.x % nb;
  const int bhl = blockIdx.x / nb;
  const int b = bhl / p.nh;
  const int h = p.h0 + (bhl - b * p.nh);
  const int start = p.grid.start(qb);
  const int len = p.grid.len(qb);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float lr[R];
  bool ok[R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int i = lane + 32 * r;
    ok[r] = i < len;
    lr[r] = ok[r] ? __ldg(p.lrel + static_cast<int64_t>(bhl) * p.N + start + i) : 0.0f;
    if (!(lr[r] > -INFINITY)) ok[r] = false;  // an empty row (cannot occur in a dense pass) adds nothing
  }
  const float* base = p.blse + static_cast<int64_t>(bhl) * nb * p.N + start;
  constexpr int U = 4;  // kv blocks in flight per warp (the reduction below assumes 4)
  const int64_t Nl = p.N;
  for (int kb0 = warp * U; kb0 < nb; kb0 += kWarps * U) {
    float x[U][R];
    const float* src = base + kb0 * Nl + lane;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int r = 0; r < R; ++r)
        x[u][r] = (kb0 + u < nb && ok[r]) ? __ldcs(src + u * Nl + 32 * r) : -INFINITY;
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = 0.0f;
#pragma unroll
      for (int r = 0; r < R; ++r) v[u] += ex2_approx(x[u][r] - lr[r]);  // invalid rows: -inf -> 0
    }
    // transpose-reduce of the 4 per-lane sums over the warp: 6 shuffles instead of 4 x 5; lane
    // 8*i ends with the sum of kv block kb0 + i
    const bool hi16 = lane & 16, hi8 = lane & 8;
    const float a0 = (hi16 ? v[2] : v[0]) + __shfl_xor_sync(0xffffffffu, hi16 ? v[0] : v[2], 16);
    const float a1 = (hi16 ? v[3] : v[1]) + __shfl_xor_sync(0xffffffffu, hi16 ? v[1] : v[3], 16);
    float c = (hi8 ? a1 : a0) + __shfl_xor_sync(0xffffffffu, hi8 ? a0 : a1, 8);
    c += __shfl_xor_sync(0xffffffffu, c, 4);
    c += __shfl_xor_sync(0xffffffffu, c, 2);
    c += __shfl_xor_sync(0xffffffffu, c, 1);
    const int kb = kb0 + (lane >> 3);
    if ((lane & 7) == 0 && kb < nb) mrow[kb] = c;
  }
  __syncthreads();
  const int64_t row = (static_cast<int64_t>(b) * p.H + h) * nb + qb;
  if (p.mass) {
    float* out = p.mass + row * nb;
    for (int j = threadIdx.x; j < nb; j += kWarps * 32) out[j] = mrow[j];
  }
  if constexpr (KPL > 0) {
    __syncthreads();  // the row is rewritten in place below (non-candidates -> 0, padding to 32*KPL)
    if (warp == 0) {
      __shared__ selrow::Bracket br;
      selrow::SmemRow<KPL> mr(mrow);
      selrow::select_row<KPL>(p.sel, static_cast<int>(row), lane, mr, br, [&](int j) { return mrow[j]; });
    }
  }
}

template <int R, int KPL>
cudaError_t launch_bm(const BlockMassParams& p, int64_t ctas, size_t smem, cudaStream_t st) {
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(block_mass_kernel<R, KPL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
    return e;
  block_mass_kernel<R, KPL><<<static_cast<unsigned>(ctas), kWarps * 32, smem, st>>>(p);
  return cudaGetLastError();
}

template <int R>
cudaError_t launch_bm_r(const BlockMassParams& p, int64_t ctas, size_t smem, cudaStream_t st) {
  switch (p.select ? block_mass_select_kpl(p.grid.nb) : 0) {
    case 4: return launch_bm<R, 4>(p, ctas, smem, st);
    case 8: return launch_bm<R, 8>(p, ctas, smem, st);
    case 16: return launch_bm<R, 16>(p, ctas, smem, st);
    case 24: return launch_bm<R, 24>(p, ctas, smem, st);
    case 28: return launch_bm<R, 28>(p, ctas, smem, st);
    case 32: return launch_bm<R, 32>(p, ctas, smem, st);
    case 64: return launch_bm<R, 64>(p, ctas, smem, st);
    default: return launch_bm<R, 0>(p, ctas, smem, st);
  }
}

}  // namespace

int block_mass_select_kpl(int nb) {
  const int k = (nb + 31) / 32;
  if (k <= 4) return 4;
  if (k <= 8) return 8;
  if (k <= 16) return 16;
  if (k <= 24) return 24;
  if (k <= 28) return 28;
  if (k <= 32) return 32;
  if (k <= 64) return 64;
  return 0;  // nb > 2048: the selection runs as K3's select_rows kernel after the passes
}

cudaError_t launch_block_mass(const BlockMassParams& p, cudaStream_t st) {
  const int64_t ctas = static_cast<int64_t>(p.B) * p.nh * p.grid.nb;
  if (ctas <= 0) return cudaSuccess;
  if (ctas > 0x7fffffffLL) return cudaErrorInvalidValue;
  const int kpl = p.select ? block_mass_select_kpl(p.grid.nb) : 0;
  const size_t smem = sizeof(float) * (kpl > 0 ? 32 * kpl : p.grid.nb);
  return p.grid.bs == 64 ? launch_bm_r<2>(p, ctas, smem, st) : launch_bm_r<4>(p, ctas, smem, st);
}

}  // namespace adaspa
