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

namespace adaspa {

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
// fp32 -> fp64 as a volatile asm: keeps the compiler from hoisting a double copy of a whole row
// of masses out of the selection loops (that would double the register footprint).
__device__ __forceinline__ double f2d_volatile(float x) {
  double d;
  asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(x));
  return d;
}
__device__ __forceinline__ float warp_sum_f32(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t warp_min_u32(uint32_t v) { return __reduce_min_sync(0xffffffffu, v); }
__device__ __forceinline__ uint32_t warp_max_u32(uint32_t v) { return __reduce_max_sync(0xffffffffu, v); }
__device__ __forceinline__ int warp_sum_i32(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

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
__global__ void __launch_bounds__(256, KPL <= 32 ? 3 : 1) select_rows_kernel(SelectRowsParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= p.rows) return;
  const int row = warp;
  const int nb = p.grid.nb;
  const int bh = row / nb;
  const int qb = row - bh * nb;
  const int h = bh % p.heads;
  const float* mrow = p.mass + static_cast<int64_t>(row) * nb;
  // text kv-blocks are ids [t0, t1)
  const int t0 = p.text_first ? 0 : p.grid.nb_first;
  const int t1 = p.text_first ? p.grid.nb_first : nb;

  // element i of this lane is kv-block j = 32 i + lane; candidate / forced bits per element in
  // ceil(KPL/32) words (KPL reaches 192 elements per lane; a single 32-bit mask overflowed)
  constexpr int KW = (KPL + 31) / 32;
  uint32_t cmask[KW], fmask[KW];
#pragma unroll
  for (int w = 0; w < KW; ++w) cmask[w] = fmask[w] = 0u;
  auto is_cand = [&](int i) -> bool { return (cmask[i >> 5] >> (i & 31)) & 1u; };
  auto is_forced = [&](int i) -> bool { return (fmask[i >> 5] >> (i & 31)) & 1u; };
  float m[KPL];
  int ncand_l = 0, nforced_l = 0;
  double tsum = 0.0, fsum = 0.0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int j = i * 32 + lane;
    const bool valid = j < nb;
    const float x = valid ? __ldg(mrow + j) : 0.0f;
    const bool forced = valid && p.text_sink && j >= t0 && j < t1;
    const bool cand = valid && !forced;
    tsum += f2d_volatile(x);
    if (forced) fsum += f2d_volatile(x);
    cmask[i >> 5] |= cand ? (1u << (i & 31)) : 0u;
    fmask[i >> 5] |= forced ? (1u << (i & 31)) : 0u;
    ncand_l += cand ? 1 : 0;
    nforced_l += forced ? 1 : 0;
    m[i] = cand ? x : 0.0f;  // candidate masses only (forced mass is F)
  }
  const double T = warp_sum_f64(tsum);
  const double F = warp_sum_f64(fsum);
  const int ncand = warp_sum_i32(ncand_l);

  // decision: 0 = keep all, 1 = forced only (+top-1 if none forced), 2 = cut at v*
  int decision;
  double R = 0.0;
  int kk = 0;
  const bool text_row = p.text_sink && qb >= t0 && qb < t1;
  if (text_row || ncand == 0) {
    decision = 0;
  } else if (p.mode == 0) {  // RECALL
    const double r = p.target[h];
    R = __dmul_rn(r, T);
    if (r >= 1.0) decision = 0;
    else if (F >= R || r <= 0.0) decision = 1;
    else decision = 2;
  } else {                   // SPARSITY
    kk = p.k_per_bh ? p.k_per_bh[bh] : p.k_head[h];
    if (kk > ncand) kk = ncand;
    decision = (kk >= ncand) ? 0 : 2;
  }

  // sum of the candidate masses >= thr (bit patterns of non-negative floats order like values;
  // non-candidates hold 0 and never change a sum)
  auto sum_ge = [&](uint32_t thr) -> double {
    double a = 0.0;
#pragma unroll
    for (int i = 0; i < KPL; ++i) a += f2d_volatile(__float_as_uint(m[i]) >= thr ? m[i] : 0.0f);
    return warp_sum_f64(a);
  };

  uint32_t vstar = 0;
  int ties_take = 0;
  if (decision == 2) {
    if (p.mode == 0) {
      // RECALL: v* = the largest candidate value v with F + sum_{cand, m >= v} m >= R (fp64).
      // Bisection over the bit patterns with fp32 sums (cheap) finds it approximately; an exact
      // fp64 walk over neighbouring distinct values then fixes it up.
      uint32_t bmin = 0xFFFFFFFFu, bmax = 0u;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const uint32_t b = __float_as_uint(m[i]);
        const bool c = is_cand(i);
        bmin = c && b < bmin ? b : bmin;
        bmax = c && b > bmax ? b : bmax;
      }
      bmin = warp_min_u32(bmin);
      bmax = warp_max_u32(bmax);
      const double s_all = sum_ge(0u);
      if (F + s_all < R) {
        decision = 0;  // rounding made the full candidate set fall short: keep everything
      } else {
        // predicate on the TAIL: sum_{m < mid} m <= budget = F + s_all - R.  The tail is small
        // next to the kept mass, so fp32 resolves it at the scale of the masses near the cut
        // (a head sum would blur cuts among masses ~1e-7 of the row total).
        const float budget = static_cast<float>((F + s_all) - R);
        uint32_t lo = bmin, hi = bmax + 1u;
        while (hi - lo > 1u) {
          const uint32_t mid = lo + ((hi - lo) >> 1);
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
          for (int i = 0; i < KPL; i += 4) {
            a0 += __float_as_uint(m[i]) < mid ? m[i] : 0.0f;
            if (i + 1 < KPL) a1 += __float_as_uint(m[i + 1]) < mid ? m[i + 1] : 0.0f;
            if (i + 2 < KPL) a2 += __float_as_uint(m[i + 2]) < mid ? m[i + 2] : 0.0f;
            if (i + 3 < KPL) a3 += __float_as_uint(m[i + 3]) < mid ? m[i + 3] : 0.0f;
          }
          if (warp_sum_f32((a0 + a1) + (a2 + a3)) <= budget) lo = mid; else hi = mid;
        }
        // snap to a value present in the row (the sum only changes at present values), then walk
        uint32_t v = 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < KPL; ++i) {
          const uint32_t b = __float_as_uint(m[i]);
          v = b >= lo && b < v ? b : v;
        }
        v = warp_min_u32(v);
        if (F + sum_ge(v) >= R) {
          for (;;) {  // up while the next larger present value still reaches R
            uint32_t u = 0xFFFFFFFFu;
#pragma unroll
            for (int i = 0; i < KPL; ++i) {
              const uint32_t b = __float_as_uint(m[i]);
              u = b > v && b < u ? b : u;
            }
            u = warp_min_u32(u);
            if (u == 0xFFFFFFFFu || F + sum_ge(u) < R) break;
            v = u;
          }
        } else {
          for (;;) {  // down to the next smaller present value until R is reached
            uint32_t u = 0u;
#pragma unroll
            for (int i = 0; i < KPL; ++i) {
              const uint32_t b = __float_as_uint(m[i]);
              u = b < v && b > u ? b : u;
            }
            u = warp_max_u32(u);
            v = u;
            if (u == 0u || F + sum_ge(v) >= R) break;
          }
        }
        vstar = v;
      }
    } else {
      // SPARSITY: the largest v with at least k candidates >= v (integer counts; non-candidate
      // zeros only pass at mid = 0, which the bisection never tests)
      uint32_t lo = 0u, hi = 0x7F800001u;
      while (hi - lo > 1u) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        int c = 0;
#pragma unroll
        for (int i = 0; i < KPL; ++i) c += __float_as_uint(m[i]) >= mid ? 1 : 0;
        if (warp_sum_i32(c) >= kk) lo = mid; else hi = mid;
      }
      vstar = lo;
    }
    if (decision == 2) {
      // mass / count strictly above the cut, ties at the cut (candidates only)
      double sgt = 0.0;
      int cgt = 0, ctie = 0;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const uint32_t b = __float_as_uint(m[i]);
        const bool c = is_cand(i);
        if (c && b > vstar) {
          sgt += f2d_volatile(m[i]);
          ++cgt;
        } else if (c && b == vstar) {
          ++ctie;
        }
      }
      sgt = warp_sum_f64(sgt);
      cgt = warp_sum_i32(cgt);
      ctie = warp_sum_i32(ctie);
      if (p.mode == 0) {
        double acc = F + sgt;
        const double vv = (double)__uint_as_float(vstar);
        ties_take = 0;
        while (acc < R && ties_take < ctie) {
          acc += vv;
          ++ties_take;
        }
        if (ties_take == 0) ties_take = 1;  // v* itself belongs to the minimal prefix
      } else {
        ties_take = kk - cgt;
      }
    }
  }

  // top-1 candidate for decision 1 with an empty forced set (reading R25)
  int top1 = -1;
  if (decision == 1 && warp_sum_i32(nforced_l) == 0) {
    uint32_t best = 0u;
    int bj = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int j = i * 32 + lane;
      const uint32_t b = __float_as_uint(m[i]);
      if (is_cand(i) && (b > best || (b == best && j < bj))) {
        best = b;
        bj = j;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint32_t ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
      if (ob > best || (ob == best && oj < bj)) {
        best = ob;
        bj = oj;
      }
    }
    top1 = bj;
  }

  // keep flags -> bitmask words (word i = ballot over kv-blocks 32i..32i+31)
  uint32_t* bits_out = p.bits + static_cast<int64_t>(row) * p.nwords;
  double kept = 0.0;
  int nnz = 0;
  int tie_seen = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int j = i * 32 + lane;
    const bool cand = is_cand(i);
    const bool forced = is_forced(i);
    bool keep;
    if (decision == 0) {
      keep = j < nb;
    } else if (decision == 1) {
      keep = forced || (cand && j == top1);
    } else {
      const uint32_t b = __float_as_uint(m[i]);
      const bool tie = cand && b == vstar;
      const uint32_t tb = __ballot_sync(0xffffffffu, tie);
      const int rank = tie_seen + __popc(tb & ((1u << lane) - 1u));
      tie_seen += __popc(tb);
      keep = forced || (cand && (b > vstar || (tie && rank < ties_take)));
    }
    const uint32_t word = __ballot_sync(0xffffffffu, keep);
    if (i * 32 < nb) {
      if (lane == 0) bits_out[i] = word;
      nnz += __popc(word);
    }
    if (keep && cand) kept += f2d_volatile(m[i]);  // forced blocks are always kept (mass F)
  }
  kept = warp_sum_f64(kept) + F;
  if (lane == 0) {
    p.row_nnz[row] = nnz;
    p.row_kept[row] = kept;
    p.row_total[row] = T;
  }
}

// Per batch element: head Recall from the base selection, tiers, new k per (b,h).
__global__ void select_tiers_kernel(SelectTierParams p) {
  __shared__ double rec[kMaxHeads];
  const int b = blockIdx.x;
  const int H = p.heads;
  for (int h = threadIdx.x; h < H; h += blockDim.x) {
    const int bh = b * H + h;
    double num = 0.0, den = 0.0;
    for (int q = 0; q < p.nb; ++q) {
      num += p.row_kept[(int64_t)bh * p.nb + q];
      den += p.row_total[(int64_t)bh * p.nb + q];
    }
    rec[h] = den > 0.0 ? num / den : 0.0;
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
__global__ void __launch_bounds__(256) select_head_kernel(SelectFinalParams p) {
  __shared__ int wsum[8];
  __shared__ double wk[8], wt[8];
  __shared__ int carry;
  const int bh = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t r0 = static_cast<int64_t>(bh) * p.nb;
  if (tid == 0) carry = 0;
  __syncthreads();
  double kept = 0.0, tot = 0.0;
  for (int base = 0; base < p.nb; base += 256) {
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
      for (int w = 0; w < 8; ++w) t += wsum[w];
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
    for (int w = 0; w < 8; ++w) {
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

// One warp per row: row_ptr, ascending col_idx from the kept bitmask, LPT slot.
__global__ void __launch_bounds__(256) select_write_kernel(SelectWriteParams p) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= p.rows) return;
  const uint32_t* bits = p.bits + static_cast<int64_t>(row) * p.nwords;
  const int start = p.head_base[row / p.nb] + p.local_off[row];
  if (lane == 0) {
    p.row_ptr[row] = start;
    if (p.row_order) p.row_order[atomicAdd(p.hist + p.row_nnz[row], 1)] = row;
  }
  int off = start;
  for (int i = 0; i < p.nwords; ++i) {
    const uint32_t w = bits[i];
    if ((w >> lane) & 1u) p.col_idx[off + __popc(w & ((1u << lane) - 1u))] = i * 32 + lane;
    off += __popc(w);
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

cudaError_t launch_select(const SelectLaunch& L, cudaStream_t st) {
  SelectRowsParams rp = L.rows;
  cudaError_t e;
  if (L.tiers) {
    rp.k_per_bh = nullptr;
    if ((e = launch_rows(rp, st)) != cudaSuccess) return e;
    select_tiers_kernel<<<L.batch, 256, 0, st>>>(L.tier);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    rp.k_per_bh = L.tier.k_per_bh;
  }
  if ((e = launch_rows(rp, st)) != cudaSuccess) return e;
  if (L.fin.row_order && (e = cudaMemsetAsync(L.fin.hist, 0, sizeof(int) * (L.fin.nb + 1), st)) != cudaSuccess)
    return e;
  select_head_kernel<<<L.fin.bh, 256, 0, st>>>(L.fin);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  select_scan_kernel<<<1, 1024, 0, st>>>(L.fin);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int wblocks = (L.wr.rows * 32 + 255) / 256;
  select_write_kernel<<<wblocks, 256, 0, st>>>(L.wr);
  return cudaGetLastError();
}

}  // namespace adaspa
