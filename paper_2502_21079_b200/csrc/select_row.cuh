// select_row.cuh -- the per-row selection of K3 (one warp per q-block row), shared by
// select_rows_kernel (select.cu: masses read from HBM) and the fused search's block-mass kernel
// (blockmass.cu: the RECALL selection epilogue of the search step t_w, masses read from the
// shared-memory row the CTA has just reduced).
//
// PAPER.md:228-232 (Recall), 436-448 (S* = top-k of W_sum_attn), 549-550 (Text Sink, Row Wise);
// readings R7-R13, R25 of DESIGN.md.
//
// The row's nb masses sit in registers (lane l holds kv-blocks l, l+32, ...).  Instead of sorting,
// the cut is found by a bisection over the fp32 bit pattern of the masses (non-negative floats
// order like their bits): the cut v* is the largest value such that the forced mass plus every
// candidate with mass >= v* reaches the target (RECALL, fp64 sums) or such that at least k
// candidates have mass >= v* (SPARSITY).  Candidates above v* are kept; candidates equal to v* are
// kept in ascending id order until the target is met -- exactly the greedy over the (mass desc,
// id asc) order that defines the selection.
//
// Each bisection round tests one threshold t against every element with FMA-pipe arithmetic only:
// [m < t] = sat((t - m) * +inf) -- a positive difference (denormals included: no flush to zero)
// gives +inf -> 1, zero gives NaN -> 0, a negative one -inf -> 0 -- so a round costs a packed
// subtract, a saturating multiply and a packed FMA per element instead of an integer compare and a
// select on the (half-rate) ALU pipe (round 1: ALU 81% busy, ~30 rounds per row).  RECALL stops the
// bisection once the bracket is narrower than 2^-17 relative (kStopBits) and walks to the exact fp64
// cut over neighbouring distinct values, so the result is the fp64 definition's whatever the fp32
// rounding of the bisection; SPARSITY counts are exact (integers below 2^24 in fp32).
#pragma once
#include "select.cuh"

namespace adaspa {
namespace selrow {

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
__device__ __forceinline__ int warp_sum_i32(int v) { return __reduce_add_sync(0xffffffffu, v); }

// sat(d * +inf): 1 for d > 0 (any positive d, denormals included), 0 for d = 0 (NaN -> 0) or d < 0
__device__ __forceinline__ float pos_step(float d) {
  float s;
  asm("mul.rn.sat.f32 %0, %1, 0f7F800000;" : "=f"(s) : "f"(d));
  return s;
}
// packed (t - m) for a pair, one rounding (exact sign)
__device__ __forceinline__ float2 sub2(float2 t, float2 m) {
  uint64_t d;
  const float2 neg = make_float2(-1.0f, -1.0f);
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<const uint64_t*>(&m)), "l"(*reinterpret_cast<const uint64_t*>(&neg)),
        "l"(*reinterpret_cast<const uint64_t*>(&t)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)),
        "l"(*reinterpret_cast<const uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<const uint64_t*>(&a)), "l"(*reinterpret_cast<const uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}

constexpr uint32_t kStopBits = 64;  // RECALL bisection stops at a bracket of 64 ulps (2^-17 relative)

// Where the candidate masses of a row live while it is selected (element i of a lane is kv-block
// 32 i + lane; non-candidates read as 0, so they never change a sum):
//   RegRow  -- in registers (K3's select_rows_kernel: the row comes from HBM once);
//   SmemRow -- in a shared-memory row of 32*KPL floats (the fused search's block-mass CTA already
//              holds the row there; reading it per pass keeps that kernel at its streaming occupancy
//              instead of a register file sized for the row).
template <int KPL>
struct RegRow {
  static constexpr int KP = (KPL + 1) / 2;  // element pairs (an odd KPL pads one zero element)
  float2 m2[KP];
  __device__ __forceinline__ RegRow() {
#pragma unroll
    for (int q = 0; q < KP; ++q) m2[q] = make_float2(0.0f, 0.0f);
  }
  __device__ __forceinline__ void set(int i, int /*lane*/, float v) {
    if (i & 1) m2[i >> 1].y = v; else m2[i >> 1].x = v;
  }
  __device__ __forceinline__ float get(int i, int /*lane*/) const { return (i & 1) ? m2[i >> 1].y : m2[i >> 1].x; }
  __device__ __forceinline__ float2 get2(int q, int /*lane*/) const { return m2[q]; }
};
template <int KPL>
struct SmemRow {
  static constexpr int KP = (KPL + 1) / 2;
  volatile float* row;  // >= 32 * 2 * KP floats
  __device__ __forceinline__ explicit SmemRow(float* r) : row(r) {}
  __device__ __forceinline__ void set(int i, int lane, float v) { row[32 * i + lane] = v; }
  __device__ __forceinline__ float get(int i, int lane) const { return row[32 * i + lane]; }
  __device__ __forceinline__ float2 get2(int q, int lane) const {
    return make_float2(row[64 * q + lane], row[64 * q + 32 + lane]);
  }
};

// Selects row `row` (= (b*H + h)*nb + qb) of the masses that load(j) returns (j < nb) and writes
// its kept bitmask (p.bits), count (p.row_nnz), kept and total mass (p.row_kept, p.row_total).
// Called by a whole warp (all 32 lanes, warp-uniform row).  `mr` holds the candidate masses from the
// first pass on (RegRow or SmemRow; a SmemRow may alias the storage load() reads: element (i, lane)
// is read before it is written, by the same thread).
//
// Candidates are the valid non-forced blocks; the forced set (text sink) is the contiguous id range
// [t0, t1), so candidate-ness is recomputed from the id where it matters instead of being stored.
// Non-candidates hold mass 0 in `mr`; a candidate of mass 0 only matters when the cut is at 0
// (SPARSITY with k above the number of positive masses), which takes a separate path.
template <int KPL, class Row, class Load>
__device__ __forceinline__ void select_row(const SelectRowsParams& p, int row, int lane, Row& mr, Load load) {
  const int nb = p.grid.nb;
  const int bh = row / nb;
  const int qb = row - bh * nb;
  const int h = bh % p.heads;
  // text kv-blocks are ids [t0, t1); with the sink they are the forced set F
  const int t0 = p.text_first ? 0 : p.grid.nb_first;
  const int t1 = p.text_first ? p.grid.nb_first : nb;
  const int f0 = p.text_sink ? t0 : 0, f1 = p.text_sink ? t1 : 0;  // forced ids [f0, f1)
  const int ncand = nb - (f1 - f0);
  constexpr int KP = (KPL + 1) / 2;
  auto mval = [&](int i) -> float { return mr.get(i, lane); };
  auto is_forced = [&](int j) -> bool { return j >= f0 && j < f1; };
  double ssum = 0.0, fsum = 0.0;  // candidate mass, forced mass
#pragma unroll
  for (int i = 0; i < 2 * KP; ++i) {
    const int j = i * 32 + lane;
    const bool valid = i < KPL && j < nb;
    const float x = valid ? load(j) : 0.0f;
    const bool forced = is_forced(j);
    const double xd = f2d_volatile(x);
    if (forced) fsum += xd; else ssum += xd;
    mr.set(i, lane, forced ? 0.0f : x);  // candidate masses only (forced mass is F)
  }
  const double S = warp_sum_f64(ssum);  // sum of the candidate masses
  const double F = warp_sum_f64(fsum);
  const double T = S + F;

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
    else if (F + S < R) decision = 0;  // rounding made the full candidate set fall short: keep everything
    else decision = 2;
  } else {                   // SPARSITY
    kk = p.k_per_bh ? p.k_per_bh[bh] : p.k_head[h];
    if (kk > ncand) kk = ncand;
    decision = (kk >= ncand) ? 0 : 2;
  }

  // fp64 sum of the candidate masses >= thr (bit patterns of non-negative floats order like values;
  // non-candidates hold 0 and thr >= 1 here, so they never enter)
  auto sum_ge = [&](uint32_t thr) -> double {
    double a = 0.0;
#pragma unroll
    for (int i = 0; i < KPL; ++i) a += f2d_volatile(__float_as_uint(mval(i)) >= thr ? mval(i) : 0.0f);
    return warp_sum_f64(a);
  };

  uint32_t vstar = 0;
  int ties_take = 0;
  if (decision == 2) {
    float mx = 0.0f;
#pragma unroll
    for (int i = 0; i < KPL; ++i) mx = fmaxf(mx, mval(i));
    const uint32_t bmax = warp_max_u32(__float_as_uint(mx));
    if (p.mode == 0) {
      // RECALL: v* = the largest candidate value v with F + sum_{cand, m >= v} m >= R (fp64).  F + S >= R
      // here, so v* is a positive mass (zeros add nothing).  Predicate on the TAIL: sum_{m < t} m <=
      // budget = F + S - R.  The tail is small next to the kept mass, so fp32 resolves it at the scale
      // of the masses near the cut.  Invariant: tail(lo) <= budget < tail(hi).
      const float budget = static_cast<float>((F + S) - R);
      uint32_t lo = 0u, hi = bmax + 1u;
      while (hi - lo > kStopBits) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        const float tf = __uint_as_float(mid);
        const float2 t2 = make_float2(tf, tf);
        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          const float2 mq = mr.get2(q, lane);
          const float2 d = sub2(t2, mq);
          const float2 s = make_float2(pos_step(d.x), pos_step(d.y));
          if (q & 1) a1 = fma2(s, mq, a1); else a0 = fma2(s, mq, a0);
        }
        const float2 a = add2(a0, a1);
        if (warp_sum_f32(a.x + a.y) <= budget) lo = mid; else hi = mid;
      }
      // snap to a positive value present in the row (the sum only changes at present values), then walk
      const uint32_t lo1 = lo > 0u ? lo : 1u;
      uint32_t v = 0xFFFFFFFFu;
#pragma unroll
      for (int i = 0; i < KPL; ++i) {
        const uint32_t b = __float_as_uint(mval(i));
        v = b >= lo1 && b < v ? b : v;
      }
      v = warp_min_u32(v);
      if (F + sum_ge(v) >= R) {
        for (;;) {  // up while the next larger present value still reaches R
          uint32_t u = 0xFFFFFFFFu;
#pragma unroll
          for (int i = 0; i < KPL; ++i) {
            const uint32_t b = __float_as_uint(mval(i));
            u = b > v && b < u ? b : u;
          }
          u = warp_min_u32(u);
          if (u == 0xFFFFFFFFu || F + sum_ge(u) < R) break;
          v = u;
        }
      } else {
        for (;;) {  // down to the next smaller positive present value until R is reached
          uint32_t u = 0u;
#pragma unroll
          for (int i = 0; i < KPL; ++i) {
            const uint32_t b = __float_as_uint(mval(i));
            u = b < v && b > u ? b : u;
          }
          u = warp_max_u32(u);
          if (u == 0u) break;  // cannot happen (F + S >= R): v stays the smallest positive value
          v = u;
          if (F + sum_ge(v) >= R) break;
        }
      }
      vstar = v;
    } else {
      // SPARSITY: the largest v with at least k candidates >= v.  Invariant: count(>= lo) >= k >
      // count(>= hi); count(>= t) = #{m > pred(t)}, pred(t) the float just below t (t >= 1 here, so
      // the zeros of non-candidates never count; lo = 0 counts every candidate).
      uint32_t lo = 0u, hi = bmax + 1u;
      const float kf = static_cast<float>(kk);
      while (hi - lo > 1u) {
        const uint32_t mid = lo + ((hi - lo) >> 1);
        const float pf = __uint_as_float(mid - 1u);
        const float2 p2 = make_float2(pf, pf);
        float2 c0 = make_float2(0.f, 0.f), c1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          const float2 d = sub2(mr.get2(q, lane), p2);
          const float2 s = make_float2(pos_step(d.x), pos_step(d.y));
          if (q & 1) c1 = add2(c1, s); else c0 = add2(c0, s);
        }
        const float2 c = add2(c0, c1);
        if (warp_sum_f32(c.x + c.y) >= kf) lo = mid; else hi = mid;
      }
      vstar = lo;
    }
    // mass / count strictly above the cut, ties at the cut (candidates only; at a cut of 0 the ties
    // are the zero-mass candidates, told from non-candidates by id)
    double sgt = 0.0;
    int cgt = 0, ctie = 0;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int j = i * 32 + lane;
      const uint32_t b = __float_as_uint(mval(i));
      if (b > vstar) {
        sgt += f2d_volatile(mval(i));
        ++cgt;
      } else if (b == vstar && (vstar > 0u || (j < nb && !is_forced(j)))) {
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

  // top-1 candidate for decision 1 with an empty forced set (reading R25)
  int top1 = -1;
  if (decision == 1 && f1 == f0) {
    uint32_t best = 0u;
    int bj = 0x7fffffff;
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int j = i * 32 + lane;
      const uint32_t b = __float_as_uint(mval(i));
      if (j < nb && (b > best || (b == best && j < bj))) {
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
    const bool valid = j < nb;
    const bool forced = valid && is_forced(j);
    const uint32_t b = __float_as_uint(mval(i));
    bool keep;
    if (decision == 0) {
      keep = valid;
    } else if (decision == 1) {
      keep = forced || j == top1;
    } else {
      const bool tie = b == vstar && valid && !forced;
      const uint32_t tb = __ballot_sync(0xffffffffu, tie);
      const int rank = tie_seen + __popc(tb & ((1u << lane) - 1u));
      tie_seen += __popc(tb);
      keep = forced || b > vstar || (tie && rank < ties_take);
    }
    const uint32_t word = __ballot_sync(0xffffffffu, keep);
    if (i * 32 < nb) {
      if (lane == 0) bits_out[i] = word;
      nnz += __popc(word);
    }
    if (keep && !forced) kept += f2d_volatile(mval(i));  // forced blocks are always kept (mass F)
  }
  kept = warp_sum_f64(kept) + F;
  if (lane == 0) {
    p.row_nnz[row] = nnz;
    p.row_kept[row] = kept;
    p.row_total[row] = T;
  }
}

}  // namespace selrow
}  // namespace adaspa
