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
// subtract, a saturating multiply and two packed FMA-pipe accumulations (the tail sum and the count)
// per element pair instead of an integer compare and a select on the (half-rate) ALU pipe.  The
// count tells how many elements are still inside the bracket: once at most 32 are, the bisection
// stops (~6 rounds on the paper-shaped masses instead of ~25 to a 64-ulp bracket) and the cut is
// resolved exactly among those few (per-warp shared-memory slots, (mass desc, id asc) keys, fp64
// prefix sums).  RECALL checks that resolution in fp64 and, if the fp32 bisection's rounding put the
// cut outside the bracket (or ties keep more than 32 elements inside it), walks to the exact fp64
// cut over neighbouring distinct values, so the result is the fp64 definition's whatever the fp32
// rounding; SPARSITY counts are exact (integers below 2^24 in fp32).
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

__device__ __forceinline__ uint64_t warp_max_u64(uint64_t v) {
  const uint32_t h = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(v >> 32));
  const uint32_t l = __reduce_max_sync(0xffffffffu, static_cast<uint32_t>(v >> 32) == h ? static_cast<uint32_t>(v) : 0u);
  return (static_cast<uint64_t>(h) << 32) | l;
}

// The few candidates left inside the bisection bracket, one slot per lane (per-warp shared memory):
// key = mass bits << 32 | ~id orders them like the selection does -- (mass desc, id asc) is key desc.
struct Bracket {
  uint64_t key[32];
  double val[32];
};

// Writes the candidates with bit pattern in [lo, hi) (lo = 0: every candidate below hi, zero masses
// included, non-candidates told apart by id) into br in (i, lane) order; returns their number (<= 32
// whenever the caller's count of the bracket is).
template <int KPL, bool kSumAbove, class Row>
__device__ __forceinline__ int collect_bracket(const Row& mr, int lane, uint32_t lo, uint32_t hi, int nb, int f0,
                                               int f1, Bracket& br, double& above) {
  int n = 0;
  double g = 0.0;
#pragma unroll
  for (int i = 0; i < KPL; ++i) {
    const int j = i * 32 + lane;
    const float m = mr.get(i, lane);
    const uint32_t b = __float_as_uint(m);
    if (kSumAbove) g += f2d_volatile(b >= hi ? m : 0.0f);  // fp64 mass at or above the bracket
    const bool in = b >= lo && b < hi && (lo > 0u || (j < nb && !(j >= f0 && j < f1)));
    const uint32_t bal = __ballot_sync(0xffffffffu, in);
    const int slot = n + __popc(bal & ((1u << lane) - 1u));
    if (in && slot < 32) br.key[slot] = (static_cast<uint64_t>(b) << 32) | static_cast<uint32_t>(~j);
    n += __popc(bal);
  }
  if (kSumAbove) above = warp_sum_f64(g);
  n = n < 32 ? n : 32;
  __syncwarp();
  // one fp32 -> fp64 conversion per slot (lane s converts slot s), not one per element and pass
  if (lane < n) br.val[lane] = f2d_volatile(__uint_as_float(static_cast<uint32_t>(br.key[lane] >> 32)));
  __syncwarp();
  return n;
}

// Selects row `row` (= (b*H + h)*nb + qb) of the masses that load(j) returns (j < nb) and writes
// its kept bitmask (p.bits, unless null), count (p.row_nnz), kept and total mass (p.row_kept,
// p.row_total); returns the count.
// Called by a whole warp (all 32 lanes, warp-uniform row).  `mr` holds the candidate masses from the
// first pass on (RegRow or SmemRow; a SmemRow may alias the storage load() reads: element (i, lane)
// is read before it is written, by the same thread).
//
// Candidates are the valid non-forced blocks; the forced set (text sink) is the contiguous id range
// [t0, t1), so candidate-ness is recomputed from the id where it matters instead of being stored.
// Non-candidates hold mass 0 in `mr`; a candidate of mass 0 only matters when the cut is at 0
// (SPARSITY with k above the number of positive masses), which takes a separate path.
template <int KPL, class Row, class Load>
__device__ __forceinline__ int select_row(const SelectRowsParams& p, int row, int lane, Row& mr, Bracket& br,
                                          Load load) {
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
  double tsum = 0.0, fsum = 0.0;  // row mass, forced mass
  const unsigned nforced = static_cast<unsigned>(f1 - f0);
  // the forced (text) blocks first: a SmemRow aliasing load()'s storage zeroes them below
  for (int j = f0 + lane; j < f1; j += 32) fsum += f2d_volatile(load(j));
#pragma unroll
  for (int i = 0; i < 2 * KP; ++i) {
    const int j = i * 32 + lane;
    const bool valid = i < KPL && j < nb;
    const float x = valid ? load(j) : 0.0f;
    tsum += f2d_volatile(x);
    mr.set(i, lane, static_cast<unsigned>(j - f0) < nforced ? 0.0f : x);  // candidate masses only
  }
  const double T = warp_sum_f64(tsum);
  const double F = warp_sum_f64(fsum);

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
    else if (T < R) decision = 0;  // rounding made the full row fall short: keep everything
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
  int ties_take = 0, ties_all = 0;  // ties at the cut taken / present (all taken: no tie ranks needed)
  bool kept_known = false;          // kept_mass already known from the exact resolution (RECALL)
  double kept_mass = 0.0;
  if (decision == 2) {
    float mx = 0.0f;
#pragma unroll
    for (int i = 0; i < KPL; ++i) mx = fmaxf(mx, mval(i));
    const uint32_t bmax = warp_max_u32(__float_as_uint(mx));
    // Bracket [lo, hi) of bit patterns holding the cut.  Every round also counts the slots below its
    // threshold (all 64*KP slots, zeros of non-candidates included), so the number of slots inside
    // the bracket is known; once it is at most 32 the bisection stops and the cut is resolved
    // exactly among those few candidates (collect_bracket and the key order below).  On HYV-110K / CogX-45K
    // masses: ~6 rounds instead of ~25 (DESIGN.md §6 K3).
    uint32_t lo = 0u, hi = bmax + 1u;
    float nlo = 0.0f, nhi = static_cast<float>(64 * KP);  // slots below lo / below hi
    bool resolved = false;
    if (p.mode == 0) {
      // RECALL: v* = the largest candidate value v with F + sum_{cand, m >= v} m >= R (fp64).  T >= R
      // here, so v* is a positive mass (zeros add nothing).  Predicate on the TAIL: sum_{m < t} m <=
      // budget = T - R.  The tail is small next to the kept mass, so fp32 resolves it at the scale
      // of the masses near the cut.  Invariant: tail(lo) <= budget < tail(hi) (in fp32; the exact
      // resolution checks it in fp64 and falls back to the walk when rounding broke it).
      const float budget = static_cast<float>(T - R);
      // first probe: every candidate below budget / ncand sums to less than the budget, so that
      // threshold is almost always a valid lo and skips the rounds spent on the lower exponents
      uint32_t probe = __float_as_uint(budget * (0.999f / static_cast<float>(ncand)));
      while (hi - lo > kStopBits && nhi - nlo > 32.0f) {
        uint32_t mid = lo + ((hi - lo) >> 1);
        if (probe > lo && probe < hi) mid = probe;
        probe = 0u;
        const float tf = __uint_as_float(mid);
        const float2 t2 = make_float2(tf, tf);
        float2 a0 = make_float2(0.f, 0.f), a1 = make_float2(0.f, 0.f);
        float2 c0 = make_float2(0.f, 0.f), c1 = make_float2(0.f, 0.f);
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          const float2 mq = mr.get2(q, lane);
          const float2 d = sub2(t2, mq);
          const float2 s = make_float2(pos_step(d.x), pos_step(d.y));
          if (q & 1) { a1 = fma2(s, mq, a1); c1 = add2(c1, s); } else { a0 = fma2(s, mq, a0); c0 = add2(c0, s); }
        }
        const float2 a = add2(a0, a1), c = add2(c0, c1);
        const float tail = warp_sum_f32(a.x + a.y);
        const float cnt = warp_sum_f32(c.x + c.y);
        if (tail <= budget) { lo = mid; nlo = cnt; } else { hi = mid; nhi = cnt; }
      }
      if (nhi - nlo <= 32.0f) {
        // G = F + the candidate mass at or above hi (fp64); the bracket's candidates in (mass desc,
        // id asc) order extend it one by one: v* is the first whose prefix reaches R
        double above = 0.0;
        const int n = collect_bracket<KPL, true>(mr, lane, lo > 0u ? lo : 1u, hi, nb, f0, f1, br, above);
        const double G = F + above;
        if (G >= R) lo = hi;  // fp32 put the cut below hi, fp64 says at or above: walk up from hi
        if (G < R && n > 0) {
          uint64_t key = 0;
          double pre = 0.0;
          if (lane < n) {
            key = br.key[lane];
            for (int s = 0; s < n; ++s) pre += br.key[s] >= key ? br.val[s] : 0.0;  // precede-or-equal
          }
          const bool reached = lane < n && G + pre >= R;
          if (__any_sync(0xffffffffu, reached)) {
            const uint64_t first = warp_max_u64(reached ? key : 0ull);  // the earliest reached in order
            vstar = static_cast<uint32_t>(first >> 32);
            const bool tie = lane < n && static_cast<uint32_t>(key >> 32) == vstar;
            ties_take = __popc(__ballot_sync(0xffffffffu, tie && key >= first));
            ties_all = __popc(__ballot_sync(0xffffffffu, tie));
            // the kept mass is the prefix that reached R: G + pre of the first reached candidate
            const int fl = __ffs(__ballot_sync(0xffffffffu, lane < n && key == first)) - 1;
            kept_mass = G + __shfl_sync(0xffffffffu, pre, fl);
            kept_known = true;
            resolved = true;
          }
        }
      }
      if (!resolved) {
        // walk: snap to a positive value present in the row (the sum only changes at present
        // values), then step to the exact fp64 cut over neighbouring distinct values
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
            if (u == 0u) break;  // cannot happen (T >= R): v stays the smallest positive value
            v = u;
            if (F + sum_ge(v) >= R) break;
          }
        }
        vstar = v;
      }
    } else {
      // SPARSITY: the largest v with at least k candidates >= v.  Invariant: count(>= lo) >= k >
      // count(>= hi); count(>= t) = #{m > pred(t)}, pred(t) the float just below t (t >= 1 here, so
      // the zeros of non-candidates never count; lo = 0 counts every candidate).  Counts are exact
      // (integers below 2^24 in fp32), so the bracket always holds the cut.
      const float kf = static_cast<float>(kk);
      float clo = static_cast<float>(ncand), chi = 0.0f;  // candidates >= lo / >= hi
      while (hi - lo > 1u && clo - chi > 32.0f) {
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
        const float cnt = warp_sum_f32(c.x + c.y);
        if (cnt >= kf) { lo = mid; clo = cnt; } else { hi = mid; chi = cnt; }
      }
      if (clo - chi <= 32.0f) {
        // the (k - count(>= hi))-th candidate of the bracket in (mass desc, id asc) order is the last kept
        double unused = 0.0;
        const int n = collect_bracket<KPL, false>(mr, lane, lo, hi, nb, f0, f1, br, unused);
        const int need = kk - static_cast<int>(chi);  // 1 <= need <= n
        uint64_t key = 0;
        int rank = -1;
        if (lane < n) {
          key = br.key[lane];
          rank = 0;
          for (int s = 0; s < n; ++s) rank += br.key[s] > key ? 1 : 0;
        }
        const uint64_t last = warp_max_u64(rank == need - 1 ? key : 0ull);
        vstar = static_cast<uint32_t>(last >> 32);
        const bool tie = lane < n && static_cast<uint32_t>(key >> 32) == vstar;
        ties_take = __popc(__ballot_sync(0xffffffffu, tie && key >= last));
        ties_all = __popc(__ballot_sync(0xffffffffu, tie));
        resolved = true;
      } else {
        vstar = lo;
      }
    }
    if (!resolved) {
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
      ties_all = ctie;
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
  uint32_t* bits_out = p.bits ? p.bits + static_cast<int64_t>(row) * p.nwords : nullptr;
  double kept = 0.0;
  int nnz = 0;
  uint32_t lw = 0;
  // KPL <= 32: lane i keeps word i and the row's words go out in one coalesced store at the end
  constexpr bool kLaneWords = KPL <= 32;
  auto emit = [&](int i, uint32_t word) {
    if (i * 32 < nb) {
      if (!kLaneWords && bits_out && lane == 0) bits_out[i] = word;
      nnz += __popc(word);
    }
    if (kLaneWords && lane == i) lw = word;
  };
  if (decision == 2 && vstar > 0u && ties_take >= ties_all) {
    // every candidate at or above the cut is kept (no tie is split): keep = forced or m >= v*
    // (non-candidates hold 0 < v*)
#pragma unroll
    for (int i = 0; i < KPL; ++i) {
      const int j = i * 32 + lane;
      const bool forced = static_cast<unsigned>(j - f0) < static_cast<unsigned>(f1 - f0) && j < nb;
      const bool cand_keep = __float_as_uint(mval(i)) >= vstar;
      emit(i, __ballot_sync(0xffffffffu, forced || cand_keep));
      if (!kept_known) kept += f2d_volatile(cand_keep ? mval(i) : 0.0f);
    }
    if (!kept_known) kept = warp_sum_f64(kept) + F;
    else kept = kept_mass;
  } else {
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
      emit(i, __ballot_sync(0xffffffffu, keep));
      if (keep && !forced) kept += f2d_volatile(mval(i));  // forced blocks are always kept (mass F)
    }
    kept = warp_sum_f64(kept) + F;
  }
  if (lane == 0) {
    p.row_nnz[row] = nnz;
    p.row_kept[row] = kept;
    p.row_total[row] = T;
  }
  if (kLaneWords && bits_out && lane < p.nwords) bits_out[lane] = lw;
  return nnz;
}

}  // namespace selrow
}  // namespace adaspa
