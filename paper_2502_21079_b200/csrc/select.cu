// select.cu -- K3: head-adaptive hierarchical block selection -> CSR.
//
// PAPER.md:228-232 (Recall), 436-448 (S* = top-k of W_sum_attn), 527-533 (head tiers),
// 549-550 (Text Sink, Row Wise); readings R7-R13, R16, R17, R25 of DESIGN.md.
//
// One warp per q-block row (b,h,p).  The row's nb masses sit in registers (lane l holds
// kv-blocks l, l+32, ...).  Instead of sorting, the kernel finds the selection cut by a
// bisection over the fp32 bit pattern of the masses (non-negative floats order like their
// bits): the cut v* is the largest value such that the forced mass plus every candidate
// with mass >= v* reaches the target (RECALL, fp64 sums) or such that at least k
// candidates have mass >= v* (SPARSITY).  Candidates above v* are kept; candidates equal
// to v* are kept in ascending id order until the target is met -- exactly the greedy over
// the (mass desc, id asc) order that defines the selection.
//
// RECALL mode runs the bisection with fp32 sums (cheap) and then walks to the exact cut with
// fp64 sums over neighbouring distinct values, so the result is the fp64 definition's.
//
// Kernels: select_rows (per row: kept bitmask, count, kept/total mass), select_tiers
// (per batch element: head recalls -> tiered k), select_head (per head: local row offsets,
// nnz / recall, row-count histogram), select_scan (head offsets, LPT slots), select_write
// (row_ptr, bitmask -> ascending col_idx, LPT row order).
#include "common.cuh"
#include "select.cuh"
#include "select_row.cuh"

namespace adaspa {

using selrow::warp_sum_f64;

// k = max(1, floor((1 - s) * n + 0.5 + 1e-9)), capped at n -- evaluated with explicit
// round-to-nearest ops so that no FMA contraction changes the result (reading R11).
__host__ __device__ int k_from_sparsity(double s, int n) {
  if (n <= 0) return 0;
#ifdef __CUDA_ARCH__
  double x = __dadd_rn(__dadd_rn(__dmul_rn(__dadd_rn(1.0, -s), (double)n), 0.5), 1e-9);
#else
  volatile double a = 1.0 - s;
  volatile double b = a * (double)n;
  volatile double c = b + 0.5;
  double x = c + 1e-9;
#endif
  int k = (int)floor(x);
  if (k < 1) k = 1;
  if (k > n) k = n;
  return k;
}

template <int KPL>
__global__ void __launch_bounds__(256, KPL <= 28 ? 4 : (KPL <= 32 ? 3 : 1)) select_rows_kernel(SelectRowsParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= p.rows) return;
  const float* mrow = p.mass + static_cast<int64_t>(warp) * p.grid.nb;
  __shared__ selrow::Bracket br[8];
  selrow::RegRow<KPL> mr;
  selrow::select_row<KPL>(p, warp, lane, mr, br[threadIdx.x >> 5], [&](int j) { return __ldg(mrow + j); });
}

// Per batch element: head Recall from the base selection, tiers, new k per (b,h).  One warp per head
// sums the head's rows (lane-strided, then a fixed-order shuffle tree: deterministic).
__global__ void __launch_bounds__(1024) select_tiers_kernel(SelectTierParams p) {
  __shared__ double rec[kMaxHeads];
  const int b = blockIdx.x;
  const int H = p.heads;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int h = wid; h < H; h += nw) {
    const int64_t r0 = static_cast<int64_t>(b * H + h) * p.nb;
    double num = 0.0, den = 0.0;
#pragma unroll 8
    for (int q = lane; q < p.nb; q += 32) {
      num += p.row_kept[r0 + q];
      den += p.row_total[r0 + q];
    }
    num = warp_sum_f64(num);
    den = warp_sum_f64(den);
    if (lane == 0) rec[h] = den > 0.0 ? num / den : 0.0;
  }
  __syncthreads();
  int nabove = 0;
  for (int h = 0; h < H; ++h) nabove += rec[h] > p.tau ? 1 : 0;
  int n = nabove < H / 2 ? nabove : H / 2;
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    // rank in (recall desc, head asc) order
    int rank = 0;
    for (int g = 0; g < H; ++g) rank += (rec[g] > rec[h] || (rec[g] == rec[h] && g < h)) ? 1 : 0;
    double s = p.s_base[h];
    if (rank < n) s = __dmul_rn(__dadd_rn(1.0, s), 0.5);
    else if (rank >= H - n) s = __dmul_rn(__dadd_rn(__dmul_rn(3.0, s), -1.0), 0.5);
    p.k_per_bh[b * H + h] = k_from_sparsity(s, p.ncand);
  }
}

// Per (b,h) CTA: exclusive scan of the head's row counts (local offsets), head nnz / Recall
// (fixed-order fp64 sums: deterministic), and the histogram of row counts for the LPT order.
__global__ void __launch_bounds__(1024) select_head_kernel(SelectFinalParams p) {
  __shared__ int wsum[32];
  __shared__ double wk[32], wt[32];
  __shared__ int carry;
  const int bh = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t r0 = static_cast<int64_t>(bh) * p.nb;
  if (tid == 0) carry = 0;
  __syncthreads();
  double kept = 0.0, tot = 0.0;
  for (int base = 0; base < p.nb; base += 1024) {
    const int q = base + tid;
    const int v = q < p.nb ? p.row_nnz[r0 + q] : 0;
    if (q < p.nb) {
      kept += p.row_kept[r0 + q];
      tot += p.row_total[r0 + q];
      if (p.row_order) atomicAdd(p.hist + v, 1);
    }
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[wid] = x;
    __syncthreads();
    int before = carry;
    for (int w = 0; w < wid; ++w) before += wsum[w];
    if (q < p.nb) p.local_off[r0 + q] = before + x - v;
    __syncthreads();
    if (tid == 0) {
      int t = 0;
      for (int w = 0; w < 32; ++w) t += wsum[w];
      carry += t;
    }
    __syncthreads();
  }
  kept = warp_sum_f64(kept);
  tot = warp_sum_f64(tot);
  if (lane == 0) {
    wk[wid] = kept;
    wt[wid] = tot;
  }
  __syncthreads();
  if (tid == 0) {
    double k = 0.0, t = 0.0;
    for (int w = 0; w < 32; ++w) {
      k += wk[w];
      t += wt[w];
    }
    p.head_cnt[bh] = carry;
    if (p.head_recall) p.head_recall[bh] = t > 0.0 ? static_cast<float>(k / t) : 0.0f;
    if (p.head_nnz) p.head_nnz[bh] = carry;
  }
}

// One CTA: head offsets (exclusive scan over B*H heads), row_ptr[rows], and the descending
// exclusive offsets of the row-count histogram (LPT: longest rows first).
__global__ void __launch_bounds__(1024) select_scan_kernel(SelectFinalParams p) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1 && !p.row_order) break;
    const int n = pass == 0 ? p.bh : p.nb + 1;
    if (tid == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < n; base += 1024) {
      const int i = base + tid;
      // pass 0: heads in order; pass 1: histogram bins from the largest count down
      int* src = pass == 0 ? p.head_cnt : p.hist;
      const int idx = pass == 0 ? i : n - 1 - i;
      const int v = i < n ? src[idx] : 0;
      int x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (lane == 31) wsum[wid] = x;
      __syncthreads();
      int before = carry;
      for (int w = 0; w < wid; ++w) before += wsum[w];
      if (i < n) {
        if (pass == 0) p.head_base[idx] = before + x - v;
        else p.hist[idx] = before + x - v;
      }
      __syncthreads();
      if (tid == 0) {
        int t = 0;
        for (int w = 0; w < 32; ++w) t += wsum[w];
        carry += t;
      }
      __syncthreads();
    }
    if (pass == 0 && tid == 0) p.row_ptr[p.rows] = carry;
    __syncthreads();
  }
}

// One warp per row: row_ptr, LPT slot, and the row's ascending col_idx.  Per 32 keep words (1024
// kv-blocks): lane i loads word i, an exclusive scan of the word counts gives each lane its place in
// the row, the lane expands its set bits (lowest first) into a per-warp shared-memory run there, and
// the warp copies the run out with coalesced stores.
__global__ void __launch_bounds__(256) select_write_kernel(SelectWriteParams p) {
  __shared__ int stage[8][1024];
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= p.rows) return;
  int* buf = stage[threadIdx.x >> 5];
  const uint32_t* bits = p.bits + static_cast<int64_t>(row) * p.nwords;
  const int start = p.head_base[row / p.nb] + p.local_off[row];
  if (lane == 0) {
    p.row_ptr[row] = start;
    if (p.row_order) p.row_order[atomicAdd(p.hist + p.row_nnz[row], 1)] = row;
  }
  int off = start;
  for (int i0 = 0; i0 < p.nwords; i0 += 32) {
    const int i = i0 + lane;
    uint32_t w = i < p.nwords ? __ldg(bits + i) : 0u;
    const int c = __popc(w);
    int incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    int pos = incl - c;
    while (w) {
      buf[pos++] = i * 32 + __ffs(w) - 1;
      w &= w - 1u;
    }
    __syncwarp();
    for (int k = lane; k < total; k += 32) p.col_idx[off + k] = buf[k];
    __syncwarp();
    off += total;
  }
}

// ------------------------------------------------------------------ launchers
static cudaError_t launch_rows(const SelectRowsParams& p, cudaStream_t st) {
  const int threads = 256;
  const int blocks = (p.rows * 32 + threads - 1) / threads;
  const int kpl = (p.grid.nb + 31) / 32;
  if (kpl <= 4) select_rows_kernel<4><<<blocks, threads, 0, st>>>(p);
  else if (kpl <= 8) select_rows_kernel<8><<<blocks, threads, 0, st>>>(p);
  else if (kpl <= 16) select_rows_kernel<16><<<blocks, threads, 0, st>>>(p);
  else if (kpl <= 24) select_rows_kernel<24><<<blocks, threads, 0, st>>>(p);
  else if (kpl <= 28) select_rows_kernel<28><<<blocks, threads, 0, st>>>(p);
  else if (kpl <= 32) select_rows_kernel<32><<<blocks, threads, 0, st>>>(p);
  else if (kpl <= 64) select_rows_kernel<64><<<blocks, threads, 0, st>>>(p);
  else if (kpl <= 128) select_rows_kernel<128><<<blocks, threads, 0, st>>>(p);
  else select_rows_kernel<kMaxSelectBlocks / 32><<<blocks, threads, 0, st>>>(p);  // spills; K3 is <0.1% of a step
  return cudaGetLastError();
}

cudaError_t launch_select_final(const SelectLaunch& L, cudaStream_t st) {
  cudaError_t e;
  if (L.fin.row_order && (e = cudaMemsetAsync(L.fin.hist, 0, sizeof(int) * (L.fin.nb + 1), st)) != cudaSuccess)
    return e;
  select_head_kernel<<<L.fin.bh, 1024, 0, st>>>(L.fin);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  select_scan_kernel<<<1, 1024, 0, st>>>(L.fin);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int wblocks = (L.wr.rows * 32 + 255) / 256;
  select_write_kernel<<<wblocks, 256, 0, st>>>(L.wr);
  return cudaGetLastError();
}

cudaError_t launch_select_rows(const SelectRowsParams& p, cudaStream_t st) { return launch_rows(p, st); }

cudaError_t launch_select(const SelectLaunch& L, cudaStream_t st) {
  SelectRowsParams rp = L.rows;
  cudaError_t e;
  if (L.tiers) {
    rp.k_per_bh = nullptr;
    if ((e = launch_rows(rp, st)) != cudaSuccess) return e;
    select_tiers_kernel<<<L.batch, 1024, 0, st>>>(L.tier);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    rp.k_per_bh = L.tier.k_per_bh;
  }
  if ((e = launch_rows(rp, st)) != cudaSuccess) return e;
  return launch_select_final(L, st);
}

}  // namespace adaspa
