// attn_one.cu -- K1 (dense attention + LSE) at d = 128 with ONE 128-row q tile per SM and two
// softmax warp groups that alternate kv steps.  Opt-in (ADASPA_ONE=1) until measured faster than
// attn_fwd.cu ("Next for d = 128").
//
// PAPER.md:194-202 (blockwise online softmax), 471-482 (Alg. 1 first pass: FA + LSE); readings
// R1-R3 of DESIGN.md (the standard recurrence).
//
// Why: attn_fwd.cu holds two q tiles per SM, each needing S (128 TMEM columns, P aliased into it)
// + O (128), so every tile runs the chain S ready -> softmax -> PV -> next QK and the tensor pipe
// idles while both softmaxes are in flight.  Here one tile has THREE S buffers + O (512 columns):
// QK(e+2) is issued interleaved with PV(e), into the buffer of step e-1 (whose PV was issued
// before), so S is always one to two kv steps ahead of the softmax, and the softmax only has to
// keep up in throughput.  One step's softmax (≈1800 cycles) is longer
// than its MMA work (1024 cycles), so two groups of 8 warps take alternate steps; the running max
// m of a row passes from one group to the other through shared memory once per step (published
// right after the row max, before the exponentials).
//
//   warp 0        TMA producer: Q tile, then K/V tiles in MMA consumption order
//                 K0 K1 V0 K2 V1 K3 ... into a ring of 6 slots.
//   warp 1        MMA issuer (one thread).
//   warp 2        TMEM allocator: S_0 | S_1 | S_2 | O.
//   warps 4-11    softmax group 0 (even global steps), warps 12-19 group 1 (odd); warp 4+i and
//                 warp 12+i own the same 16 rows (16-lane TMEM shapes as in attn_fwd.cu).
// Each group keeps its own row sum l relative to the last m it used; an O rescale (rare: only when
// m grows by more than 2^8) is done by the group that raises m, after PV of the previous step.
// Epilogue: the group without the item's last step hands (m, l) per row to the other, which stores O.
#include "attn.cuh"
#include "common.cuh"

#include <stdlib.h>

namespace adaspa {
namespace {

constexpr int kThreads1 = 640;
constexpr int kTile1 = 128 * 128 * 2;  // one 128-row tile of d = 128 bf16
constexpr int kChunk1 = 128 * 128;     // one 64-column (128-byte) chunk of a 128-row tile
constexpr int kNS1 = 6;
constexpr uint32_t kOCol = 384;
constexpr float kThr1 = 8.0f;  // rescale threshold, log2 units (as attn_fwd.cu)

struct OneBars {
  uint64_t kv_full[kNS1], kv_empty[kNS1];
  uint64_t q_full, q_empty;
  uint64_t s_full[3], p_half[3], p_full[3];
  uint64_t pv_done[2];  // committed after PV of every step, indexed by global step parity
  uint64_t o_full, o_empty;
  uint64_t pub[2][8];  // group g, warp i: running max of its rows for its latest step published
  uint64_t epi[8];     // warp i of the group without the item's last step: (m, l) published
  uint64_t rd[8];      // warp i of the other group: has read them
  uint32_t tmem_base;
};

struct OneShared {
  float mrow[2][128];           // running max per row, by global step parity
  float xl[8][16][2];           // [warp][row in warp]{m, l} at an item's end
};

constexpr int kQ1 = 0;
constexpr int kKV1 = kTile1;
constexpr int kBar1 = kKV1 + kNS1 * kTile1;
constexpr int kSh1 = kBar1 + 512;
// 6 K/V slots fill shared memory to the byte: no alignment slack, the dynamic base must already be
// 1024-aligned (checked at entry).
constexpr int kBytes1 = kSh1 + static_cast<int>(sizeof(OneShared));
static_assert(sizeof(OneBars) <= 512, "barrier block outgrew its reservation");
static_assert(kBytes1 <= 232448, "over 227 KB of shared memory");

struct OneItem {
  int b, h, q0, n;
};
__device__ __forceinline__ OneItem one_item(const AttnParams& p, int id) {
  OneItem it;
  const int bh = id / p.items_per_bh;
  it.b = bh / p.H;
  it.h = bh - it.b * p.H;
  it.q0 = (id - bh * p.items_per_bh) * 128;
  it.n = (p.N + 127) / 128;
  return it;
}

// ABL (diagnostic, ADASPA_ONE=2/3/4): 1 = no softmax (MMA + TMA pipeline alone), 2 = softmax without
// the exponentials (P = bf16 of the scaled argument), 3 = no softmax and no K/V loads after the
// first tiles (the MMA issue stream alone).
template <int ABL>
__global__ void __launch_bounds__(kThreads1, 1)
    attn_one_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023u) __trap();
  uint8_t* smem = smem_raw;
  uint8_t* sQ = smem + kQ1;
  uint8_t* sKV = smem + kKV1;
  OneBars* bars = reinterpret_cast<OneBars*>(smem + kBar1);
  OneShared* sh = reinterpret_cast<OneShared*>(smem + kSh1);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNS1; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int i = 0; i < 3; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_half[i], 8);
      mbar_init(&bars->p_full[i], 8);
    }
    mbar_init(&bars->pv_done[0], 1);
    mbar_init(&bars->pv_done[1], 1);
    mbar_init(&bars->o_full, 1);
    mbar_init(&bars->o_empty, 8);
    for (int g = 0; g < 2; ++g)
      for (int i = 0; i < 8; ++i) {
        mbar_init(&bars->pub[g][i], 1);
        if (g == 0) {
          mbar_init(&bars->epi[i], 1);
          mbar_init(&bars->rd[i], 1);
        }
      }
    fence_mbar_init();
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
  }
  if (warp == 2) {
    tmem_alloc(&bars->tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp < 4) {
    regs_dec<64>();
    if (warp == 0 && lane == 0) {
      // ============================================================ TMA producer
      int slot = 0;
      uint32_t ph = 0, qph = 0;
      const uint64_t pol_kv = l2_policy_evict_last();
      const uint64_t pol_q = l2_policy_evict_first();
      for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
        const OneItem it = one_item(p, item);
        mbar_wait(&bars->q_empty, qph ^ 1);
        qph ^= 1;
        mbar_arrive_expect_tx(&bars->q_full, kTile1);
        for (int c = 0; c < 2; ++c) tma_load_4d_hint(&tq, &bars->q_full, sQ + c * kChunk1, c * 64, it.q0, it.h, it.b, pol_q);
        auto load = [&](const CUtensorMap* m, int e) {
          mbar_wait(&bars->kv_empty[slot], ph ^ 1);
          if (ABL == 3 && (item != static_cast<int>(blockIdx.x) || e > 2)) {  // diagnostic: no K/V traffic
            mbar_arrive(&bars->kv_full[slot]);
            if (++slot == kNS1) { slot = 0; ph ^= 1; }
            return;
          }
          mbar_arrive_expect_tx(&bars->kv_full[slot], kTile1);
          for (int c = 0; c < 2; ++c)
            tma_load_4d_hint(m, &bars->kv_full[slot], sKV + slot * kTile1 + c * kChunk1, c * 64, 128 * e, it.h, it.b, pol_kv);
          if (++slot == kNS1) { slot = 0; ph ^= 1; }
        };
        const int k0 = it.n < 2 ? it.n : 2;
        for (int j = 0; j < k0; ++j) load(&tk, j);
        for (int e = 0; e < it.n; ++e) {
          load(&tv, e);
          if (e + 2 < it.n) load(&tk, e + 2);
        }
      }
    } else if (warp == 1 && lane == 0) {
      // ============================================================ MMA issuer
      constexpr uint32_t kIdescQK = idesc_bf16(128, 128, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, 128, false, true);
      const uint32_t sq_addr = smem_u32(sQ);
      const uint32_t skv_addr = smem_u32(sKV);
      int slot = 0;
      uint32_t ph = 0, qph = 0, oeph = 0;
      uint32_t gs = 0;  // global kv step of this CTA (buffers and phases follow it across items)
      bool o_dirty = false;
      auto next_slot = [&]() {
        const int s = slot;
        mbar_wait(&bars->kv_full[slot], ph);
        tc_fence_after();
        if (++slot == kNS1) { slot = 0; ph ^= 1; }
        return s;
      };
      // One k-step (K = 16) of QK into S buffer `qbuf` / of PV from P in buffer `pbuf` into O.  A chain
      // of MMAs on one accumulator runs at about half the tensor pipe's rate, so PV(e) and QK(e+2)
      // are issued interleaved, one k-step of each in turn (two independent accumulators).
      auto qk_step = [&](uint32_t qbuf, int ks, int kk) {
        const uint32_t off = (kk >> 2) * kChunk1 + (kk & 3) * 32;
        const uint64_t a = desc_sw128(sq_addr + off, 16, 1024);
        const uint64_t b = desc_sw128(skv_addr + ks * kTile1 + off, 16, 1024);
        mma_ss(tmem + qbuf * 128u, a, b, kIdescQK, kk > 0 ? 1u : 0u);
      };
      auto pv_step = [&](uint32_t pbuf, int vs, bool first, int kk) {
        const uint64_t b = desc_sw128(skv_addr + vs * kTile1 + kk * 2048, kChunk1, 1024);
        mma_ts(tmem + kOCol, tmem + pbuf * 128u + kk * 8, b, kIdescPV, (first && kk == 0) ? 0u : 1u);
      };
      for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
        const OneItem it = one_item(p, item);
        mbar_wait(&bars->q_full, qph);
        qph ^= 1;
        tc_fence_after();
        // prologue: QK(0), QK(1) interleaved
        {
          const int k0 = it.n < 2 ? it.n : 2;
          int ks[2];
          for (int j = 0; j < k0; ++j) ks[j] = next_slot();
#pragma unroll
          for (int kk = 0; kk < 8; ++kk)
            for (int j = 0; j < k0; ++j) qk_step((gs + j) % 3u, ks[j], kk);
          for (int j = 0; j < k0; ++j) {
            tc_commit(&bars->kv_empty[ks[j]]);
            tc_commit(&bars->s_full[(gs + j) % 3u]);
          }
          if (k0 == it.n) tc_commit(&bars->q_empty);
        }
        for (int e = 0; e < it.n; ++e) {
          const uint32_t g = gs + e;
          const uint32_t buf = g % 3u, par = (g / 3u) & 1u;
          const uint32_t qbuf = (g + 2) % 3u;  // held S(e-1) / P(e-1): PV(e-1) was issued before
          const bool qk = e + 2 < it.n;
          const int vs = next_slot();
          const int ks = qk ? next_slot() : 0;
          mbar_wait(&bars->p_half[buf], par);
          tc_fence_after();
          if (e == 0 && o_dirty) {  // the previous item's epilogue has drained O
            mbar_wait(&bars->o_empty, oeph);
            oeph ^= 1;
            o_dirty = false;
            tc_fence_after();
          }
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            pv_step(buf, vs, e == 0, kk);
            if (qk) qk_step(qbuf, ks, kk);
          }
          mbar_wait(&bars->p_full[buf], par);
          tc_fence_after();
#pragma unroll
          for (int kk = 4; kk < 8; ++kk) {
            pv_step(buf, vs, false, kk);
            if (qk) qk_step(qbuf, ks, kk);
          }
          tc_commit(&bars->kv_empty[vs]);
          tc_commit(&bars->pv_done[g & 1u]);
          if (e == it.n - 1) {
            tc_commit(&bars->o_full);
            o_dirty = true;
          }
          if (qk) {
            tc_commit(&bars->kv_empty[ks]);
            tc_commit(&bars->s_full[qbuf]);
            if (e + 2 == it.n - 1) tc_commit(&bars->q_empty);
          }
        }
        gs += it.n;
      }
    }
  } else {
    regs_inc<104>();
    // ============================================================ softmax groups
    const int sw = warp - 4;
    const int grp = sw >> 3;  // 0: even global steps, 1: odd
    const int wi = sw & 7;
    const int hh = (wi >> 2) & 1;
    const int wq = warp & 3;
    const int qd = lane & 3;
    const int row0 = wq * 32 + hh * 16 + (lane >> 2);  // tile rows of this thread: row0, row0 + 8
    const int row1 = row0 + 8;
    const int rloc = lane >> 2;  // row index within the warp's 16 rows (row0 -> rloc, row1 -> rloc + 8)
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32 + hh * 16) << 16;
    const uint32_t o_addr = tmem + lane_base + kOCol;
    const float sl2 = p.scale_log2;
    const Poly3x2 poly;
    uint32_t gs = 0, pubph = 0;
    int itc = 0;
    for (int item = blockIdx.x; item < p.num_items; item += gridDim.x, ++itc) {
      const OneItem it = one_item(p, item);
      float m_mine[2] = {-INFINITY, -INFINITY};
      float l_sum[2] = {0.0f, 0.0f};  // this thread's 32 columns, relative to m_mine
      const int lim_last = p.N - 128 * (it.n - 1);
      for (int e = ((gs & 1u) == static_cast<uint32_t>(grp)) ? 0 : 1; e < it.n; e += 2) {
        const uint32_t G = gs + e;
        const uint32_t buf = G % 3u, par = (G / 3u) & 1u;
        const uint32_t s_addr = tmem + lane_base + buf * 128u;
        mbar_wait(&bars->s_full[buf], par);
        tc_fence_after();
        if (ABL == 1 || ABL == 3) {
          if (G > 0) {
            mbar_wait(&bars->pub[grp ^ 1][wi], pubph);
            pubph ^= 1;
          }
          __syncwarp();
          if (lane == 0) {
            mbar_arrive(&bars->pub[grp][wi]);
            mbar_arrive(&bars->p_half[buf]);
            mbar_arrive(&bars->p_full[buf]);
          }
          continue;
        }
        uint32_t s[64];
        tmem_ld_16x256b_x8(s_addr, s);
        tmem_ld_16x256b_x8(s_addr + 64, s + 32);
        tmem_ld_wait32(s);
        reg_fence32(s + 32);
        float mxa[2], mxb[2];
        mxa[0] = fmaxf(__uint_as_float(s[0]), __uint_as_float(s[1]));
        mxb[0] = fmaxf(__uint_as_float(s[4]), __uint_as_float(s[5]));
        mxa[1] = fmaxf(__uint_as_float(s[2]), __uint_as_float(s[3]));
        mxb[1] = fmaxf(__uint_as_float(s[6]), __uint_as_float(s[7]));
#pragma unroll
        for (int k = 2; k < 16; k += 2) {
          mxa[0] = fmax3(mxa[0], __uint_as_float(s[4 * k]), __uint_as_float(s[4 * k + 1]));
          mxb[0] = fmax3(mxb[0], __uint_as_float(s[4 * k + 4]), __uint_as_float(s[4 * k + 5]));
          mxa[1] = fmax3(mxa[1], __uint_as_float(s[4 * k + 2]), __uint_as_float(s[4 * k + 3]));
          mxb[1] = fmax3(mxb[1], __uint_as_float(s[4 * k + 6]), __uint_as_float(s[4 * k + 7]));
        }
        const float lmx[2] = {fmaxf(mxa[0], mxb[0]) * sl2, fmaxf(mxa[1], mxb[1]) * sl2};
        // running max after the previous global step (the other group's), -inf at an item's start
        float m_prev[2] = {-INFINITY, -INFINITY};
        if (G > 0) {
          mbar_wait(&bars->pub[grp ^ 1][wi], pubph);
          pubph ^= 1;
          if (e > 0) {
            m_prev[0] = sh->mrow[(G - 1) & 1u][row0];
            m_prev[1] = sh->mrow[(G - 1) & 1u][row1];
          }
        }
        float m_new[2] = {m_prev[0], m_prev[1]};
        if (__any_sync(0xffffffffu, lmx[0] > m_prev[0] + kThr1 || lmx[1] > m_prev[1] + kThr1)) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            float mx = lmx[j];
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            if (mx > m_prev[j] + kThr1) m_new[j] = mx;  // also when m_prev == -inf
          }
        }
        if (qd == 0) {
          sh->mrow[G & 1u][row0] = m_new[0];
          sh->mrow[G & 1u][row1] = m_new[1];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->pub[grp][wi]);
        float alpha[2] = {1.0f, 1.0f};
        bool rescale = false;
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          if (m_new[j] != m_mine[j]) {
            l_sum[j] = (m_mine[j] == -INFINITY) ? 0.0f : l_sum[j] * exp2f(m_mine[j] - m_new[j]);
            m_mine[j] = m_new[j];
          }
          if (m_new[j] != m_prev[j] && m_prev[j] != -INFINITY) {
            alpha[j] = exp2f(m_prev[j] - m_new[j]);
            rescale = true;
          }
        }
        const float mb[2] = {m_new[0] == -INFINITY ? 0.0f : m_new[0], m_new[1] == -INFINITY ? 0.0f : m_new[1]};
        if (e == it.n - 1 && lim_last < 128) {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const int col = 8 * (i >> 2) + 2 * qd + (i & 1);
            s[i] = col < lim_last ? s[i] : __float_as_uint(-INFINITY);
          }
        }
        if (__any_sync(0xffffffffu, rescale)) {  // rare: O holds PV up to step G-1 at m_prev
          const uint32_t gp = G - 1;
          mbar_wait(&bars->pv_done[gp & 1u], (gp >> 1) & 1u);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < 4; ++c) {
            uint32_t r[16];
            tmem_ld_16x256b_x4(o_addr + c * 32, r);
            tmem_ld_wait16(r);
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha[(i >> 1) & 1]);
            tmem_st_16x256b_x4(o_addr + c * 32, r);
          }
        }
        const float2 sl2v = make_float2(sl2, sl2);
        const float2 nm0 = make_float2(-mb[0], -mb[0]);
        const float2 nm1 = make_float2(-mb[1], -mb[1]);
        float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const int i = 32 * c + 4 * k;
            const float2 x0 = ffma2(make_float2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sl2v, nm0);
            const float2 x1 = ffma2(make_float2(__uint_as_float(s[i + 2]), __uint_as_float(s[i + 3])), sl2v, nm1);
            float2 p0, p1;
            if (ABL == 2) {
              p0 = x0;
              p1 = x1;
            } else if (k == 7) {  // one group in eight on the FMA-pipe polynomial (as attn_fwd.cu)
              p0 = exp2_poly3x2(x0, poly);
              p1 = exp2_poly3x2(x1, poly);
            } else {
              p0.x = ex2_approx(x0.x);
              p0.y = ex2_approx(x0.y);
              p1.x = ex2_approx(x1.x);
              p1.y = ex2_approx(x1.y);
            }
            acc[(k & 1) * 2 + 0] = fadd2(acc[(k & 1) * 2 + 0], p0);
            acc[(k & 1) * 2 + 1] = fadd2(acc[(k & 1) * 2 + 1], p1);
            pk[2 * k] = pack_bf16x2(p0.x, p0.y);
            pk[2 * k + 1] = pack_bf16x2(p1.x, p1.y);
          }
          tmem_st_16x128b_x8(s_addr + c * 32, pk);
          if (c == 0) {
            tmem_st_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bars->p_half[buf]);
          }
        }
        const float2 a0 = fadd2(acc[0], acc[2]), a1 = fadd2(acc[1], acc[3]);
        l_sum[0] += a0.x + a0.y;
        l_sum[1] += a1.x + a1.y;
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->p_full[buf]);
      }
      // ---- epilogue: the group that ran the item's last step (X) stores O and LSE; the other (Y)
      // hands it (m, l) of its rows through shared memory.  The next global step is Y's, so Y moves
      // on to the next item while X drains O.
      float lq[2];
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        float l = l_sum[j];
        l += __shfl_xor_sync(0xffffffffu, l, 1);
        l += __shfl_xor_sync(0xffffffffu, l, 2);
        lq[j] = l;
      }
      const uint32_t iph = static_cast<uint32_t>(itc) & 1u;
      if (static_cast<int>((gs + it.n - 1) & 1u) != grp) {
        if (itc > 0) mbar_wait(&bars->rd[wi], iph ^ 1u);  // X has read the previous item's
        if (qd == 0) {
          sh->xl[wi][rloc][0] = m_mine[0];
          sh->xl[wi][rloc][1] = lq[0];
          sh->xl[wi][rloc + 8][0] = m_mine[1];
          sh->xl[wi][rloc + 8][1] = lq[1];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->epi[wi]);
      } else {
        mbar_wait(&bars->epi[wi], iph);
        float mo[2], lo[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          mo[j] = sh->xl[wi][rloc + 8 * j][0];
          lo[j] = sh->xl[wi][rloc + 8 * j][1];
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->rd[wi]);
        float m_fin[2], l_tot[2], inv[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          m_fin[j] = fmaxf(m_mine[j], mo[j]);
          float l = 0.0f;
          if (m_mine[j] != -INFINITY) l += lq[j] * exp2f(m_mine[j] - m_fin[j]);
          if (mo[j] != -INFINITY) l += lo[j] * exp2f(mo[j] - m_fin[j]);
          l_tot[j] = l;
          inv[j] = l > 0.0f ? 1.0f / l : 0.0f;
        }
        mbar_wait(&bars->o_full, iph);
        tc_fence_after();
        const int tok[2] = {it.q0 + row0, it.q0 + row1};
        const bool valid[2] = {tok[0] < p.N, tok[1] < p.N};
        __nv_bfloat16* optr[2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
          optr[j] = p.o + it.b * p.sb + it.h * p.sh + static_cast<int64_t>(valid[j] ? tok[j] : 0) * p.sn + 2 * qd;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[16];
          tmem_ld_16x256b_x4(o_addr + c * 32, r);
          tmem_ld_wait16(r);
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const int col = 32 * c + 8 * k;
            if (valid[0])
              *reinterpret_cast<uint32_t*>(optr[0] + col) =
                  pack_bf16x2(__uint_as_float(r[4 * k]) * inv[0], __uint_as_float(r[4 * k + 1]) * inv[0]);
            if (valid[1])
              *reinterpret_cast<uint32_t*>(optr[1] + col) =
                  pack_bf16x2(__uint_as_float(r[4 * k + 2]) * inv[1], __uint_as_float(r[4 * k + 3]) * inv[1]);
          }
        }
        if (qd == 0 && p.lse) {
#pragma unroll
          for (int j = 0; j < 2; ++j)
            if (valid[j])
              p.lse[(static_cast<int64_t>(it.b) * p.H + it.h) * p.N + tok[j]] =
                  l_tot[j] > 0.0f ? (m_fin[j] + __log2f(l_tot[j])) * kLn2 : -INFINITY;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->o_empty);
      }
      gs += it.n;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

}  // namespace

cudaError_t launch_attn_one(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                            const AttnParams& p0, int num_sms, cudaStream_t st) {
  AttnParams p = p0;
  p.items_per_bh = (p.N + 127) / 128;
  p.num_items = p.B * p.H * p.items_per_bh;
  static const int abl = [] {
    const char* v = getenv("ADASPA_ONE");
    return v && v[0] >= '2' && v[0] <= '4' ? v[0] - '1' : 0;
  }();
  auto kern = abl == 1   ? attn_one_kernel<1>
              : abl == 2 ? attn_one_kernel<2>
              : abl == 3 ? attn_one_kernel<3>
                         : attn_one_kernel<0>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kBytes1);
  if (e != cudaSuccess) return e;
  const int grid = p.num_items < num_sms ? p.num_items : num_sms;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, kThreads1, kBytes1, st>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace adaspa
