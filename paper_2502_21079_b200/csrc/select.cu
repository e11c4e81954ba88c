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
// Kernels: select_rows (per row: kept bitmask, count, kept/total mass), select_tiers
// (per batch element: head recalls -> tiered k), select_finalize (row_ptr scan, per-head
// nnz / recall, LPT row order), select_write (bitmask -> ascending col_idx).
#include "common.cuh"
#include "select.cuh"

namespace adaspa {

__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
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
__global__ void __launch_bounds__(256) select_rows_kernel(SelectRowsParams p) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= p.rows) return;
  const int row = warp;
  const int nb = p.grid.nb;
  const int bh = row / nb;
  const int qb = row - bh * nb;
  const int h = bh % p.heads;
  const float* mrow = p.mass + static_cast<int64_t>(row) * nb;

  float m[KPL];
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    int j = i * 32 + lane;
    m[i] = (j < nb) ? __ldg(mrow + j) : 0.0f;
  }
  auto is_text = [&](int j) -> bool { return p.text_first ? (j < p.grid.nb_first) : (j >= p.grid.nb_first); };

  double tsum = 0.0, fsum = 0.0;
  int ncand = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    int j = i * 32 + lane;
    if (j < nb) {
      tsum += (double)m[i];
      bool forced = p.text_sink && is_text(j);
      if (forced) fsum += (double)m[i]; else ++ncand;
    }
  }
  const double T = warp_sum_f64(tsum);
  const double F = warp_sum_f64(fsum);
  ncand = warp_sum_i32(ncand);

  // decision: 0 = keep all, 1 = forced only (+top-1 if none forced), 2 = cut at v*
  int decision;
  double R = 0.0;
  int kk = 0;
  const bool text_row = p.text_sink && is_text(qb);
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

  uint32_t vstar = 0;
  int ties_take = 0;
  if (decision == 2) {
    // bisection: lo satisfies the predicate, hi does not
    uint32_t lo = 0u, hi = 0x7F800001u;
    bool lo_ok;
    if (p.mode == 0) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        int j = i * 32 + lane;
        if (j < nb && !(p.text_sink && is_text(j))) s += (double)m[i];
      }
      lo_ok = (F + warp_sum_f64(s)) >= R;
    } else {
      lo_ok = true;
    }
    if (!lo_ok) {
      decision = 0;  // rounding made the full candidate set fall short: keep everything
    } else {
      while (hi - lo > 1u) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        bool ok;
        if (p.mode == 0) {
          double s = 0.0;
#pragma unroll
          for (int i = 0; i < KPL; ++i) {
            int j = i * 32 + lane;
            if (j < nb && !(p.text_sink && is_text(j)) && __float_as_uint(m[i]) >= mid) s += (double)m[i];
          }
          ok = (F + warp_sum_f64(s)) >= R;
        } else {
          int c = 0;
#pragma unroll
          for (int i = 0; i < KPL; ++i) {
            int j = i * 32 + lane;
            c += (j < nb && !(p.text_sink && is_text(j)) && __float_as_uint(m[i]) >= mid) ? 1 : 0;
          }
          ok = warp_sum_i32(c) >= kk;
        }
        if (ok) lo = mid; else hi = mid;
      }
      vstar = lo;
      // mass / count strictly above the cut
      double sgt = 0.0;
      int cgt = 0, ctie = 0;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        int j = i * 32 + lane;
        if (j < nb && !(p.text_sink && is_text(j))) {
          uint32_t bits = __float_as_uint(m[i]);
          if (bits > vstar) { sgt += (double)m[i]; ++cgt; }
          else if (bits == vstar) ++ctie;
        }
      }
      sgt = warp_sum_f64(sgt);
      cgt = warp_sum_i32(cgt);
      ctie = warp_sum_i32(ctie);
      if (p.mode == 0) {
        double acc = F + sgt;
        const double vv = (double)__uint_as_float(vstar);
        ties_take = 0;
        while (acc < R && ties_take < ctie) { acc += vv; ++ties_take; }
        if (ties_take == 0) ties_take = 1;  // v* itself belongs to the minimal prefix
      } else {
        ties_take = kk - cgt;
      }
    }
  }

  // top-1 candidate for decision 1 with an empty forced set (reading R25)
  int top1 = -1;
  if (decision == 1) {
    const int n_text_blocks = p.text_first ? p.grid.nb_first : nb - p.grid.nb_first;
    const bool any_forced = p.text_sink && n_text_blocks > 0;
    if (!any_forced) {
      uint32_t best = 0u; int bj = 0x7fffffff;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        int j = i * 32 + lane;
        if (j < nb) {
          uint32_t bits = __float_as_uint(m[i]);
          if (bits > best || (bits == best && j < bj)) { best = bits; bj = j; }
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        uint32_t ob = __shfl_xor_sync(0xffffffffu, best, o);
        int oj = __shfl_xor_sync(0xffffffffu, bj, o);
        if (ob > best || (ob == best && oj < bj)) { best = ob; bj = oj; }
      }
      top1 = bj;
    }
  }

  // keep flags -> bitmask words (word i = ballot over kv-blocks 32i..32i+31)
  uint32_t* bits_out = p.bits + static_cast<int64_t>(row) * p.nwords;
  double kept = 0.0;
  int nnz = 0;
  int tie_seen = 0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    int j = i * 32 + lane;
    bool valid = j < nb;
    bool forced = valid && p.text_sink && is_text(j);
    bool keep;
    if (decision == 0) keep = valid;
    else if (decision == 1) keep = forced || (valid && j == top1);
    else {
      uint32_t b = __float_as_uint(m[i]);
      bool cand = valid && !forced;
      bool tie = cand && b == vstar;
      uint32_t tb = __ballot_sync(0xffffffffu, tie);
      int rank = tie_seen + __popc(tb & ((1u << lane) - 1u));
      tie_seen += __popc(tb);
      keep = forced || (cand && (b > vstar || (tie && rank < ties_take)));
    }
    uint32_t word = __ballot_sync(0xffffffffu, keep);
    if (i * 32 < nb) {
      if (lane == 0) bits_out[i] = word;
      nnz += __popc(word);
    }
    if (keep) kept += (double)m[i];
  }
  kept = warp_sum_f64(kept);
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

// row_ptr scan, per-head nnz / recall, LPT row order.  One CTA of 1024 threads.
__global__ void __launch_bounds__(1024) select_finalize_kernel(SelectFinalParams p) {
  extern __shared__ int hist[];  // nb + 1 bins
  __shared__ int warp_tot[32];
  __shared__ int carry;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry = 0;
  for (int i = tid; i <= p.nb; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  for (int base = 0; base < p.rows; base += 1024) {
    const int r = base + tid;
    const int v = r < p.rows ? p.row_nnz[r] : 0;
    if (r < p.rows && p.row_order) atomicAdd(&hist[v], 1);
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      int t = warp_tot[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, t, o);
        if (lane >= o) t += y;
      }
      warp_tot[lane] = t;  // inclusive
    }
    __syncthreads();
    const int excl = carry + (wid ? warp_tot[wid - 1] : 0) + x - v;
    if (r < p.rows) p.row_ptr[r] = excl;
    __syncthreads();
    if (tid == 0) carry += warp_tot[31];
    __syncthreads();
  }
  if (tid == 0) p.row_ptr[p.rows] = carry;
  // per-(b,h) totals: one warp per head, fixed order -> deterministic
  for (int bh = wid; bh < p.bh; bh += 32) {
    double kept = 0.0, tot = 0.0;
    long long nnz = 0;
    for (int q = lane; q < p.nb; q += 32) {
      kept += p.row_kept[(int64_t)bh * p.nb + q];
      tot += p.row_total[(int64_t)bh * p.nb + q];
      nnz += p.row_nnz[(int64_t)bh * p.nb + q];
    }
    kept = warp_sum_f64(kept);
    tot = warp_sum_f64(tot);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nnz += __shfl_xor_sync(0xffffffffu, nnz, o);
    if (lane == 0) {
      if (p.head_recall) p.head_recall[bh] = tot > 0.0 ? (float)(kept / tot) : 0.0f;
      if (p.head_nnz) p.head_nnz[bh] = (int64_t)nnz;
    }
  }
  if (!p.row_order) return;
  __syncthreads();
  // descending-key exclusive offsets (serial over <= 4097 bins; tiny)
  if (tid == 0) {
    int acc = 0;
    for (int k = p.nb; k >= 0; --k) {
      int c = hist[k];
      hist[k] = acc;
      acc += c;
    }
  }
  __syncthreads();
  for (int r = tid; r < p.rows; r += blockDim.x) {
    int pos = atomicAdd(&hist[p.row_nnz[r]], 1);
    p.row_order[pos] = r;
  }
}

__global__ void __launch_bounds__(256) select_write_kernel(SelectWriteParams p) {
  const int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= p.rows) return;
  const uint32_t* bits = p.bits + static_cast<int64_t>(row) * p.nwords;
  int off = p.row_ptr[row];
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
  else if (kpl <= 32) select_rows_kernel<32><<<blocks, threads, 0, st>>>(p);
  else if (kpl <= 64) select_rows_kernel<64><<<blocks, threads, 0, st>>>(p);
  else select_rows_kernel<128><<<blocks, threads, 0, st>>>(p);
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
  const size_t shm = sizeof(int) * (size_t)(L.fin.nb + 1);
  select_finalize_kernel<<<1, 1024, shm, st>>>(L.fin);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  const int wblocks = (L.wr.rows * 32 + 255) / 256;
  select_write_kernel<<<wblocks, 256, 0, st>>>(L.wr);
  return cudaGetLastError();
}

}  // namespace adaspa
