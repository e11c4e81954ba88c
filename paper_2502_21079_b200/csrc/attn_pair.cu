// attn_pair.cu -- K1 (dense attention + LSE) and K4 (block-sparse attention, block 128) for
// d = 128 on a CTA PAIR (cluster of 2 SMs, tcgen05 cta_group::2), three S buffers.
//
// Same method as attn_fwd.cu (PAPER.md:194-202 online softmax; 471-482 Alg. 1 pass 1 with
// readings R1-R3; 415-427 and 446-448 for the sparse pass); different schedule.  Why
// (clock64 traces of attn_fwd.cu): with two q tiles ping-ponging over ONE S
// buffer each, every tile runs the chain  QK -> softmax -> PV -> next QK  serially, and the
// tensor pipe waits for each softmax (3600 cycles per kv step for 2048 of MMA work).  Here each
// SM owns ONE 128-row q tile and TMEM holds THREE S buffers (3 x 128 columns) plus O
// (128 columns): the MMA thread runs two kv steps ahead, so the softmax only has to keep up in
// throughput, not in latency.  One q tile per SM would double the K/V traffic per FLOP; the
// CTA pair restores it: an M = 256 MMA spans the two SMs' q tiles and each SM holds HALF of
// every K/V tile (QK^T: B = K, N = 128 kv rows split 64/64; PV: B = V, N = d split 64/64).
//
// Work item (per pair) = two 128-row q tiles of one (b,h), tile r on CTA r (dense rows
// [256p + 128r, +128); sparse: q-block 2p + r), exactly the items and kv streams of attn_fwd.cu.
// Roles, in BOTH CTAs unless noted:
//   warp 0   TMA producer: own Q tile, own halves of K and V in consumption order
//            K0 K1 | V0 K2 | V1 K3 | ...; completion bytes counted on the LEADER's barriers.
//   warp 1   (leader only) MMA issuer: QK(0..1), then per step e: wait P(e), PV(e), QK(e+2).
//            Commits are multicast to both CTAs; per-step info is written into both CTAs.
//   warp 2   TMEM allocator (cta_group::2, 512 columns: S0 | S1 | S2 | O).
//   warps 4-11  softmax, each owning 16 whole rows (16-lane TMEM shapes, quad shuffles), every
//            step in order: m / l stay in registers.  P-ready / O-free arrivals go to the
//            leader (remote arrive from CTA 1).  A rare O rescale waits for PV(e-1) through two
//            alternating pv_done barriers.  A kv block this CTA's q-block does not keep (sparse
//            union) is skipped: P = 0 without exponentials.
#include "attn.cuh"
#include "common.cuh"

namespace adaspa {

#ifdef ADASPA_TRACE
// Diagnostic build only: clock64 stamps of cluster 0 -- role 0: MMA thread per step
// [P(e) seen, PV(e) issued, K(e+3) full seen, QK(e+3) issued + signalled]; role 1/2: softmax
// warp 4 of CTA 0/1 per step [S seen, S loaded, P stored, arrived]; read by adaspa_debug_trace_pair.
__device__ unsigned long long g_ptrace[3][4096];
#define PTR(role, k, step)                                                         \
  do {                                                                             \
    if (cluster_id_x() == 0 && (step) < 1000) g_ptrace[role][(step) * 4 + (k)] = clock64(); \
  } while (0)
#else
#define PTR(role, k, step) \
  do {                     \
  } while (0)
#endif

namespace {

#ifndef ADASPA_ABLATE
#define ADASPA_ABLATE 0  // diagnostic builds only: 4 = no softmax, 6 = softmax TMEM traffic only
#endif
constexpr int kThreads = 384;
constexpr int kD = 128;
constexpr int kTileQ = 128 * kD * 2;  // 32 KB: two 64-column chunks of 16 KB
constexpr int kChunkQ = 128 * 128;
constexpr int kSlot = 64 * kD * 2;    // 16 KB: half a K tile (64 rows x 128) or half a V tile (128 x 64)
constexpr int kNS = 10;
constexpr int kNB = 3;                // S buffers
// QK(e + kLook) is issued right after PV(e).  It writes the S buffer PV(e - 1) read, not the one
// PV(e) reads: a cta_group::2 MMA chain on one accumulator runs at 128 cycles per instruction
// (tools/micro_mma_pair.cu), two independent chains (O and S) interleave to the full 64.
constexpr int kLook = 2;
constexpr int kNI = 16;               // per-step info ring (written by each CTA's own producer)
constexpr int kOffQ = 0;
constexpr int kOffKV = kTileQ;
constexpr int kOffBar = kOffKV + kNS * kSlot;
constexpr int kSmemBytes = kOffBar + 2048 + 1024;
constexpr uint32_t kOCol = 384;
constexpr float kRescaleThreshold = 8.0f;  // log2 units
#ifndef ADASPA_PAIR_POLY_MASK
#define ADASPA_PAIR_POLY_MASK 0x22
#endif
// bit k: the k-th group of four exponentials per 32 columns goes to the FMA-pipe polynomial
// (exp2_poly3x2) instead of MUFU.EX2 -- the softmax of this kernel is MUFU-throughput bound.
constexpr uint32_t kPolyMask = ADASPA_PAIR_POLY_MASK;

enum : int { kNormal = 0, kAllEnd = 2 };

struct Info3 {
  int kind, lim0, lim1, skip, last;
  int b, h, start, len, pad;
};
constexpr int kInfoWords = sizeof(Info3) / 4;

struct Item3 {
  int kind, id, b, h, n_ent;
  int start[2], len[2];
};

struct Bars3 {
  uint64_t kv_full[kNS], kv_empty[kNS];
  uint64_t q_full, q_empty;
  uint64_t s_full[kNB], p_full[kNB];
  uint64_t pv_done[2];
  uint64_t o_full, o_empty;
  uint64_t item_full;
  int item_box, pad0;
  Info3 info[kNI];
  Item3 qitem;
  uint32_t tmem_base;
};

template <bool SPARSE>
__device__ __forceinline__ void decode_item3(const AttnParams& p, int id, Item3& it) {
  const int bh = id / p.items_per_bh;
  const int pi = id - bh * p.items_per_bh;
  it.kind = kNormal;
  it.id = id;
  it.b = bh / p.H;
  it.h = bh - it.b * p.H;
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    if (!SPARSE) {
      const int st = 256 * pi + 128 * r;
      int l = p.N - st;
      l = l < 0 ? 0 : (l > 128 ? 128 : l);
      it.start[r] = st;
      it.len[r] = l;
    } else {
      const int qb = 2 * pi + r;
      const bool ex = qb < p.grid.nb;
      it.start[r] = ex ? p.grid.start(qb) : p.N;  // absent tile: fully out of bounds (TMA zero fill)
      it.len[r] = ex ? p.grid.len(qb) : 0;
    }
  }
  it.n_ent = SPARSE ? __ldg(p.stream_len + id) : (p.N + 127) / 128;
}

// kv rows of step e: start and valid length; membership mask (bits 0-3: tile 0, 4-7: tile 1)
template <bool SPARSE>
__device__ __forceinline__ void step_kv(const AttnParams& p, const uint64_t* ent_ptr, int e, int& s0, int& l0,
                                        uint32_t& mask) {
  if (SPARSE) {
    const uint64_t ent = __ldg(reinterpret_cast<const unsigned long long*>(ent_ptr) + e);
    const int j = entry_id0(ent);
    s0 = p.grid.start(j);
    l0 = p.grid.len(j);
    mask = entry_mask(ent);
  } else {
    s0 = 128 * e;
    l0 = p.N - s0 < 128 ? p.N - s0 : 128;
    mask = 0xFFu;
  }
}

__device__ __forceinline__ void put_info3(Bars3* bars, int slot, uint32_t rank, const Info3& v, bool full) {
  Info3* dst = &bars->info[slot];
  const int n = full ? kInfoWords : 5;
  if (rank == 0) {
    int* d = reinterpret_cast<int*>(dst);
    const int* w = reinterpret_cast<const int*>(&v);
    for (int i = 0; i < n; ++i) d[i] = w[i];
    return;
  }
  const uint32_t base = mapa_shared(smem_u32(dst), rank);
  const int* w = reinterpret_cast<const int*>(&v);
  for (int i = 0; i < n; ++i) st_cluster_u32(base + 4u * i, static_cast<uint32_t>(w[i]));
}

template <bool SPARSE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn_pair_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + kOffQ;
  uint8_t* sKV = smem + kOffKV;
  Bars3* bars = reinterpret_cast<Bars3*>(smem + kOffBar);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < kNS; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int b = 0; b < kNB; ++b) {
      mbar_init(&bars->s_full[b], 1);   // MMA commit (multicast)
      mbar_init(&bars->p_full[b], 16);  // leader: 8 softmax warps in each CTA
    }
    mbar_init(&bars->pv_done[0], 1);
    mbar_init(&bars->pv_done[1], 1);
    mbar_init(&bars->o_full, 1);
    mbar_init(&bars->o_empty, 16);      // leader
    mbar_init(&bars->item_full, 1);
    fence_mbar_init();
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
  }
  if (warp == 2) {
    tmem_alloc_pair(&bars->tmem_base, 512);
    tmem_relinquish_pair();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp == 0 && lane == 0) {
    // ============================================================ TMA producer (both CTAs)
    const uint64_t pol_kv = l2_policy_evict_last();
    const uint64_t pol_q = l2_policy_evict_first();
    const uint32_t q_full_l = mapa_shared(smem_u32(&bars->q_full), 0);
    const int rr = static_cast<int>(rank);
    int slot = 0;
    uint32_t ph = 0, qph = 0, iph = 0;
    int g0 = 0;  // global step index of the item's step 0
    for (int it_n = 0;; ++it_n) {
      int item = 0;
      if (SPARSE && !leader) {
        mbar_wait_cluster(&bars->item_full, iph);
        iph ^= 1;
        item = *reinterpret_cast<volatile int*>(&bars->item_box);
      }
      mbar_wait(&bars->q_empty, qph ^ 1);
      qph ^= 1;
      if (SPARSE && leader) {
        // q_empty: the previous item's QKs completed, so the peer has read the previous item id
        item = atomicAdd(p.queue, 1);
        st_cluster_u32(mapa_shared(smem_u32(&bars->item_box), 1), static_cast<uint32_t>(item));
        mbar_arrive_remote_release(mapa_shared(smem_u32(&bars->item_full), 1));
      }
      if (!SPARSE) item = static_cast<int>(cluster_id_x() + it_n * cluster_num_x());
      if (item >= p.num_items) {
        if (leader) {
          bars->qitem.kind = kAllEnd;
          mbar_arrive(&bars->q_full);
        }
        break;
      }
      const int id = SPARSE ? __ldg(p.item_order + item) : item;
      Item3 it;
      decode_item3<SPARSE>(p, id, it);
      if (leader) {
        bars->qitem = it;
        mbar_arrive_expect_tx(&bars->q_full, 2 * kTileQ);
      }
      const int qs = rr ? it.start[1] : it.start[0];
#pragma unroll
      for (int c = 0; c < 2; ++c) tma_load_4d_pair(&tq, q_full_l, sQ + c * kChunkQ, c * 64, qs, it.h, it.b, pol_q);
      const uint64_t* ent_ptr = SPARSE ? p.stream + static_cast<int64_t>(id) * p.stream_stride : nullptr;
      const int n = it.n_ent;
      auto load_k = [&](int e) {
        int s0, l0;
        uint32_t mk;
        step_kv<SPARSE>(p, ent_ptr, e, s0, l0, mk);
        // this CTA's info for step g0 + e, read by its softmax after S(e) is ready (well after the
        // K bytes below have been consumed); the ring is deeper than the producer's lead
        Info3& v = bars->info[(g0 + e) % kNI];
        v.kind = kNormal;
        v.skip = ((mk >> (4 * rr)) & 0xFu) ? 0 : 1;
        v.lim0 = l0 < 64 ? l0 : 64;
        v.lim1 = l0;
        v.last = e == n - 1 ? 1 : 0;
        v.b = it.b;
        v.h = it.h;
        v.start = rr ? it.start[1] : it.start[0];
        v.len = rr ? it.len[1] : it.len[0];
        __threadfence_block();
        mbar_wait(&bars->kv_empty[slot], ph ^ 1);
        if (leader) mbar_arrive_expect_tx(&bars->kv_full[slot], 2 * kSlot);
        const uint32_t fb = mapa_shared(smem_u32(&bars->kv_full[slot]), 0);
        uint8_t* dst = sKV + slot * kSlot;
        tma_load_4d_pair(&tk, fb, dst, 0, s0 + 64 * rr, it.h, it.b, pol_kv);
        tma_load_4d_pair(&tk, fb, dst + kSlot / 2, 64, s0 + 64 * rr, it.h, it.b, pol_kv);
        if (++slot == kNS) { slot = 0; ph ^= 1; }
      };
      auto load_v = [&](int e) {
        int s0, l0;
        uint32_t mk;
        step_kv<SPARSE>(p, ent_ptr, e, s0, l0, mk);
        mbar_wait(&bars->kv_empty[slot], ph ^ 1);
        if (leader) mbar_arrive_expect_tx(&bars->kv_full[slot], 2 * kSlot);
        const uint32_t fb = mapa_shared(smem_u32(&bars->kv_full[slot]), 0);
        tma_load_4d_pair(&tv, fb, sKV + slot * kSlot, 64 * rr, s0, it.h, it.b, pol_kv);
        if (++slot == kNS) { slot = 0; ph ^= 1; }
      };
      for (int e = 0; e < n && e < kLook; ++e) load_k(e);
      for (int e = 0; e < n; ++e) {
        load_v(e);
        if (e + kLook < n) load_k(e + kLook);
      }
      g0 += n;
    }
    for (int i = 0; i < kNS; ++i) {  // drain: every multicast commit to this CTA's kv_empty landed
      mbar_wait(&bars->kv_empty[slot], ph ^ 1);
      if (++slot == kNS) { slot = 0; ph ^= 1; }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ============================================================ MMA issuer (leader)
    constexpr uint32_t kIdescQK = idesc_bf16(256, 128, false, false);
    constexpr uint32_t kIdescPV = idesc_bf16(256, kD, false, true);
    const uint32_t sq_addr = smem_u32(sQ);
    const uint32_t skv_addr = smem_u32(sKV);
    uint32_t s_full_peer[kNB];
    for (int b = 0; b < kNB; ++b) s_full_peer[b] = mapa_shared(smem_u32(&bars->s_full[b]), 1);
    int slot = 0;
    uint32_t ph = 0, qph = 0, oeph = 0;
    bool o_dirty = false;
    int g0 = 0;  // global step index of this item's step 0 (steps run through S buffers g % 3)
    for (;;) {
      mbar_wait(&bars->q_full, qph);
      qph ^= 1;
      tc_fence_after();
      const Item3 it = bars->qitem;
      if (it.kind == kAllEnd) {
        // every P has been consumed, so the softmax warps wait on exactly this phase
        const int b = g0 % kNB;
        Info3 v{};
        v.kind = kAllEnd;
        put_info3(bars, g0 % kNI, 0, v, false);
        put_info3(bars, g0 % kNI, 1, v, false);
        mbar_arrive(&bars->s_full[b]);
        mbar_arrive_remote_release(s_full_peer[b]);
        break;
      }
      const int n = it.n_ent;
      int pend_v = -1, pend_pv = -1, pend_k = -1, pend_s = -1;
      bool pend_q = false;
      auto issue_qk = [&](int e) {
        const int b = (g0 + e) % kNB;
        mbar_wait(&bars->kv_full[slot], ph);
        if (e >= kLook) PTR(0, 2, g0 + e - kLook);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint64_t a = desc_sw128(sq_addr + (kk >> 2) * kChunkQ + (kk & 3) * 32, 16, 1024);
          const uint64_t bd = desc_sw128(skv_addr + slot * kSlot + (kk >> 2) * (kSlot / 2) + (kk & 3) * 32, 16, 1024);
          mma_ss_pair(tmem + 128u * b, a, bd, kIdescQK, kk > 0 ? 1u : 0u);
        }
        // commits after both MMA groups of the step (see below)
        pend_k = slot;
        if (++slot == kNS) { slot = 0; ph ^= 1; }
        pend_s = b;
        pend_q = e == n - 1;
      };
      // A commit between the PV and the QK group would keep the two accumulation chains from
      // overlapping, so every step issues PV(e), QK(e+2) and only then its commits.
      auto flush = [&]() {
        if (pend_v >= 0) tc_commit_pair(&bars->kv_empty[pend_v]);
        if (pend_pv >= 0) tc_commit_pair(&bars->pv_done[pend_pv & 1]);
        if (pend_k >= 0) tc_commit_pair(&bars->kv_empty[pend_k]);
        if (pend_q) tc_commit_pair(&bars->q_empty);  // last reader of Q
        if (pend_s >= 0) tc_commit_pair(&bars->s_full[pend_s]);
        pend_v = pend_pv = pend_k = pend_s = -1;
        pend_q = false;
      };
      for (int e = 0; e < n && e < kLook; ++e) {
        issue_qk(e);
        flush();
      }
      for (int e = 0; e < n; ++e) {
        const int g = g0 + e;
        const int b = g % kNB;
        mbar_wait_cluster(&bars->p_full[b], (g / kNB) & 1);
        PTR(0, 0, g);
        tc_fence_after();
        if (e == 0 && o_dirty) {  // the epilogue of the previous item has read O
          mbar_wait_cluster(&bars->o_empty, oeph);
          oeph ^= 1;
          tc_fence_after();
        }
        mbar_wait(&bars->kv_full[slot], ph);
        tc_fence_after();
        const int vslot = slot;
        if (++slot == kNS) { slot = 0; ph ^= 1; }
        PTR(0, 1, g);
        const bool qk = e + kLook < n;
        const int kslot = slot;
        const int bq = (g + kLook) % kNB;
        if (qk) {
          mbar_wait(&bars->kv_full[kslot], ph);
          tc_fence_after();
          if (++slot == kNS) { slot = 0; ph ^= 1; }
        }
        PTR(0, 2, g);
        // PV(e) and QK(e+2) instruction by instruction: adjacent MMAs never share an accumulator
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t bd = desc_sw128(skv_addr + vslot * kSlot + kk * 2048, kSlot, 1024);
          mma_ts_pair(tmem + kOCol, tmem + 128u * b + kk * 8, bd, kIdescPV, (e == 0 && kk == 0) ? 0u : 1u);
          if (qk) {
            const uint64_t a = desc_sw128(sq_addr + (kk >> 2) * kChunkQ + (kk & 3) * 32, 16, 1024);
            const uint64_t bk = desc_sw128(skv_addr + kslot * kSlot + (kk >> 2) * (kSlot / 2) + (kk & 3) * 32, 16, 1024);
            mma_ss_pair(tmem + 128u * bq, a, bk, kIdescQK, kk > 0 ? 1u : 0u);
          }
        }
        tc_commit_pair(&bars->kv_empty[vslot]);
        tc_commit_pair(&bars->pv_done[g & 1]);
        if (qk) {
          tc_commit_pair(&bars->kv_empty[kslot]);
          if (e + kLook == n - 1) tc_commit_pair(&bars->q_empty);  // last reader of Q
          tc_commit_pair(&bars->s_full[bq]);
        }
        PTR(0, 3, g);
      }
      if (n > 0) {
        tc_commit_pair(&bars->o_full);
        o_dirty = true;
      }
      g0 += n;
    }
  } else if (warp >= 4) {
    // ============================================================ softmax (both CTAs)
    const int sw = warp - 4;
    const int wq = warp & 3;
    const int hh = sw >> 2;
    const int qd = lane & 3;
    const int row0 = wq * 32 + hh * 16 + (lane >> 2);
    const int row1 = row0 + 8;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32 + hh * 16) << 16;
    const uint32_t o_addr = tmem + lane_base + kOCol;
    const float sl2 = p.scale_log2;
    uint32_t p_full_l[kNB];
    for (int b = 0; b < kNB; ++b) p_full_l[b] = mapa_shared(smem_u32(&bars->p_full[b]), 0);
    const uint32_t o_empty_l = mapa_shared(smem_u32(&bars->o_empty), 0);
    uint32_t oph = 0;
    float m_used[2] = {-INFINITY, -INFINITY};
    float l_sum[2] = {0.0f, 0.0f};
    int ntile = 0;
    const Poly3x2 poly;
    for (int g = 0;; ++g) {
      const int b = g % kNB;
      mbar_wait_cluster(&bars->s_full[b], (g / kNB) & 1);
      if (warp == 4 && lane == 0) PTR(1 + rank, 0, g);
      tc_fence_after();
      const Info3* inf = &bars->info[g % kNI];
      const int kind = inf->kind;
      if (kind == kAllEnd) break;
      const volatile Info3* vinf = inf;  // issued before the TMEM load (see attn_fwd.cu)
      const int skip = vinf->skip, last = vinf->last;
      const int limA = vinf->lim0, limB = vinf->lim1;
      const uint32_t s_addr = tmem + lane_base + 128u * b;
      if (ADASPA_ABLATE == 4) {  // diagnostic: no softmax (MMA / TMA pipeline alone)
      } else if (ADASPA_ABLATE == 6) {  // diagnostic: the softmax's TMEM traffic only (P = 0)
        uint32_t s[64];
        tmem_ld_16x256b_x8(s_addr, s);
        tmem_ld_16x256b_x8(s_addr + 64, s + 32);
        tmem_ld_wait32(s);
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = s[i] & s[32 + i] & 0u;
        tmem_st_16x128b_x8(s_addr, z);
        tmem_st_16x128b_x8(s_addr + 32, z);
      } else if (!skip) {
        uint32_t s[64];
        tmem_ld_16x256b_x8(s_addr, s);
        tmem_ld_16x256b_x8(s_addr + 64, s + 32);
        tmem_ld_wait32(s);
        reg_fence32(s + 32);
        if (warp == 4 && lane == 0) PTR(1 + rank, 1, g);
        if (limA < 64 || limB < 128) {
#pragma unroll
          for (int i = 0; i < 64; ++i) {
            const int col = 8 * (i >> 2) + 2 * qd + (i & 1);
            const int lim = col < 64 ? limA : limB;
            s[i] = col < lim ? s[i] : __float_as_uint(-INFINITY);
          }
        }
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
        float mb[2];
        float alpha[2] = {1.0f, 1.0f};
        bool rescale = false;
        float lmx[2] = {fmaxf(mxa[0], mxb[0]) * sl2, fmaxf(mxa[1], mxb[1]) * sl2};
        // m_used only moves when the row max grows past it by more than 2^8, so the quad's row max is
        // needed only then: one warp vote instead of four shuffles (which queue behind MUFU in MIO).
        if (__any_sync(0xffffffffu, lmx[0] > m_used[0] + kRescaleThreshold || lmx[1] > m_used[1] + kRescaleThreshold)) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            float mx = lmx[j];
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
            mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
            const float m_new = fmaxf(m_used[j], mx);
            if (m_new > m_used[j] + kRescaleThreshold) {  // also true when m_used == -inf
              alpha[j] = (m_used[j] == -INFINITY) ? 0.0f : exp2f(m_used[j] - m_new);
              l_sum[j] *= alpha[j];
              m_used[j] = m_new;
              rescale |= alpha[j] != 0.0f && ntile > 0;
            }
          }
        }
        mb[0] = (m_used[0] == -INFINITY) ? 0.0f : m_used[0];
        mb[1] = (m_used[1] == -INFINITY) ? 0.0f : m_used[1];
        if (__any_sync(0xffffffffu, rescale)) {
          // rare: O must absorb PV(g-1) first (PV(g-3) is complete: the commit that signalled
          // S(g) covers every MMA issued before QK(g), PV(g-2) included)
          mbar_wait_cluster(&bars->pv_done[(g - 1) & 1], ((g - 1) >> 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int c = 0; c < kD / 32; ++c) {
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
            if ((kPolyMask >> k) & 1u) {
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
        }
        const float2 a0 = fadd2(acc[0], acc[2]), a1 = fadd2(acc[1], acc[3]);
        l_sum[0] += a0.x + a0.y;
        l_sum[1] += a1.x + a1.y;
      } else {
        // this CTA's q-block does not keep this kv block (the pair's other one does): P = 0
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
        tmem_st_16x128b_x8(s_addr, z);
        tmem_st_16x128b_x8(s_addr + 32, z);
      }
      tmem_st_wait();
      if (warp == 4 && lane == 0) PTR(1 + rank, 2, g);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&bars->p_full[b]);
        else mbar_arrive_remote(p_full_l[b]);
      }
      if (warp == 4 && lane == 0) PTR(1 + rank, 3, g);
      ++ntile;
      if (last) {
        // ---- epilogue of the item: O / l, LSE
        const int bb = inf->b, h = inf->h, start = inf->start, len = inf->len;
        float l_tot[2], inv[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          float l = l_sum[j];
          l += __shfl_xor_sync(0xffffffffu, l, 1);
          l += __shfl_xor_sync(0xffffffffu, l, 2);
          l_tot[j] = l;
          inv[j] = l > 0.0f ? 1.0f / l : 0.0f;
        }
        const bool valid[2] = {row0 < len, row1 < len};
        const int tok[2] = {start + row0, start + row1};
        mbar_wait_cluster(&bars->o_full, oph);
        oph ^= 1;
        tc_fence_after();
        __nv_bfloat16* optr[2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
          optr[j] = p.o + bb * p.sb + h * p.sh + static_cast<int64_t>(valid[j] ? tok[j] : 0) * p.sn + 2 * qd;
#pragma unroll
        for (int c = 0; c < kD / 32; ++c) {
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
              p.lse[(static_cast<int64_t>(bb) * p.H + h) * p.N + tok[j]] =
                  l_tot[j] > 0.0f ? (m_used[j] + __log2f(l_tot[j])) * kLn2 : -INFINITY;
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&bars->o_empty);
          else mbar_arrive_remote(o_empty_l);
        }
        m_used[0] = m_used[1] = -INFINITY;
        l_sum[0] = l_sum[1] = 0.0f;
        ntile = 0;
      }
    }
  }

  tc_fence_before();
  cluster_sync_all();  // no MMA of the pair reads this CTA's smem / TMEM any more
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair(tmem, 512);
  }
}

template <bool SPARSE>
cudaError_t launch_pair(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const AttnParams& p,
                        int num_sms, cudaStream_t st) {
  auto kern = attn_pair_kernel<SPARSE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (e != cudaSuccess) return e;
  const int pairs = num_sms / 2;
  const int grid = 2 * (p.num_items < pairs ? p.num_items : pairs);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, kThreads, kSmemBytes, st>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace

#ifdef ADASPA_TRACE
extern "C" int adaspa_debug_trace_pair(unsigned long long* host, int n) {
  if (cudaMemcpyFromSymbol(host, g_ptrace, sizeof(unsigned long long) * (n < 3 * 4096 ? n : 3 * 4096)) != cudaSuccess)
    return -1;
  return 0;
}
#endif

cudaError_t launch_attn_pair(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                             const AttnParams& p, bool sparse, int num_sms, cudaStream_t st) {
  return sparse ? launch_pair<true>(tq, tk, tv, p, num_sms, st) : launch_pair<false>(tq, tk, tv, p, num_sms, st);
}

}  // namespace adaspa
