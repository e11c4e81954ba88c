// attn2_fwd.cu -- K1 (dense attention + LSE) and K4 (block-sparse attention) for d = 128 on a CTA
// PAIR (cluster of 2 SMs of one TPC, tcgen05 cta_group::2).
//
// Same method as attn_fwd.cu (PAPER.md:194-202 online softmax; 471-482 Alg. 1 pass 1 with readings
// R1-R3; 415-427 and 446-448 for the sparse pass), different hardware mapping.  Why a pair
// (measured): on one SM an M=128 SS QK^T MMA reads A and B from shared memory at
// 128 B/clk and TMA writes of the K/V stream compete with it (64 -> ~83 cycles per MMA).  With
// M = 256 across two SMs each SM supplies its own 128 Q rows but only HALF of every K/V tile:
//   QK^T:  B = K tile (N = 128 kv rows): CTA r holds kv rows [64r, 64r+64) of the tile;
//   PV:    B = V tile (N = d = 128 columns): CTA r holds columns [64r, 64r+64) of all 128 rows;
// so each SM's TMA fill and MMA operand reads per kv step drop by a third, and the ring of K/V
// slots (16 KB each) is twice as deep in the same shared memory.
//
// Work item (per pair) = four 128-row q tiles of one (b,h): tile t of CTA r is q index s = 2t + r
// (dense: rows [512p + 128s, +128); sparse B=128: q-block 4p + s).  The kv stream is the same for
// the pair (sparse: union of the four CSR rows, each entry tagged with the 4-bit membership of
// the item's q-blocks).  Roles, in BOTH CTAs unless noted:
//   warp 0   TMA producer: its own Q tiles, its own halves of K and V; completion bytes are counted
//            on the LEADER's (rank 0) barriers, which expect both halves.
//   warp 1   (leader only) MMA issuer, one thread: S_t = Q_t K^T (M=256, N=128, SS),
//            O_t += P_t V (M=256, N=128, TS: P from each CTA's TMEM); commits are multicast to
//            both CTAs; per-tile TileInfo is written into both CTAs' shared memory.
//   warp 2   TMEM allocator (cta_group::2, 512 columns: S_0 | S_1 | O_0 | O_1 in each CTA).
//   warps 4-19  softmax of this CTA's two tiles, exactly as in attn_fwd.cu (two warps per TMEM lane
//            quarter and tile, one per 64-column half); P-ready and O-free arrivals go to the
//            leader's barriers (remote arrive from CTA 1).  A tile this CTA's q-block does not need
//            (sparse union) is skipped: P = 0 without exponentials.
#include "attn.cuh"
#include "common.cuh"

namespace adaspa {
namespace {

constexpr int kThreads = 640;
constexpr int kD = 128;
constexpr int kTileQ = 128 * kD * 2;  // one 128-row q tile: 32 KB (two 64-column chunks of 16 KB)
constexpr int kChunkQ = 128 * 128;    // 16 KB
constexpr int kSlot = 64 * kD * 2;    // 16 KB: half a K tile (64 rows x 128 cols) or half a V tile (128 x 64)
constexpr int kNS = 8;
constexpr int kOffQ = 0;
constexpr int kOffKV = 2 * kTileQ;
constexpr int kOffBar = kOffKV + kNS * kSlot;
constexpr int kSmemBytes = kOffBar + 6144 + 1024;
constexpr float kRescaleThreshold = 8.0f;  // log2 units

__device__ __forceinline__ uint32_t s_col(int t) { return static_cast<uint32_t>(t) * 128u; }
__device__ __forceinline__ uint32_t o_col(int t) { return 256u + static_cast<uint32_t>(t) * 128u; }

enum : int { kNormal = 0, kEnd = 1, kAllEnd = 2 };

// Per (CTA, q tile) event written by the MMA thread: a normal S tile (column limits of the two
// 64-column halves, or skip), the end of an item (store O) or the end of the work.
struct Info2 {
  int kind, lim0, lim1, skip;
  int has, b, h, start, len, pad;
};
constexpr int kInfoWords = sizeof(Info2) / 4;

struct Item2 {
  int kind;  // kNormal or kAllEnd
  int id, b, h, n_ent;
  int start[4], len[4];  // q index s = 2t + r
};

struct Bars2 {
  uint64_t kv_full[kNS], kv_empty[kNS];
  uint64_t q_full, q_empty;
  uint64_t s_full[2], p_full[2], o_full[2], o_empty[2];
  uint64_t item_full;
  int item_box;
  int pad0;
  Info2 info[2][2];
  Item2 qitem;
  uint32_t tmem_base;
  float xm[2][2 * 128];
  float xl[2][2 * 128];
};

template <bool SPARSE>
__device__ __forceinline__ void decode_item2(const AttnParams& p, int id, Item2& it) {
  const int bh = id / p.items_per_bh;
  const int pi = id - bh * p.items_per_bh;
  it.kind = kNormal;
  it.id = id;
  it.b = bh / p.H;
  it.h = bh - it.b * p.H;
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    if (!SPARSE) {
      const int st = 512 * pi + 128 * s;
      int l = p.N - st;
      l = l < 0 ? 0 : (l > 128 ? 128 : l);
      it.start[s] = st;
      it.len[s] = l;
    } else {
      const int qb = 4 * pi + s;
      const bool ex = qb < p.grid.nb;
      it.start[s] = ex ? p.grid.start(qb) : p.N;  // absent tile: fully out of bounds (TMA zero fill)
      it.len[s] = ex ? p.grid.len(qb) : 0;
    }
  }
  it.n_ent = SPARSE ? __ldg(p.stream_len + id) : (p.N + 127) / 128;
}

// Write an Info2 into CTA `rank`'s copy of bars->info[t][slot] (plain stores for the own CTA).
__device__ __forceinline__ void put_info(Bars2* bars, int t, int slot, uint32_t rank, uint32_t my_rank,
                                         const Info2& v, bool end_fields) {
  Info2* dst = &bars->info[t][slot];
  if (rank == my_rank) {
    if (end_fields) {
      *dst = v;
    } else {
      dst->kind = v.kind;
      dst->lim0 = v.lim0;
      dst->lim1 = v.lim1;
      dst->skip = v.skip;
    }
    return;
  }
  const uint32_t base = mapa_shared(smem_u32(dst), rank);
  const int* w = reinterpret_cast<const int*>(&v);
  const int n = end_fields ? kInfoWords : 4;
  for (int i = 0; i < n; ++i) st_cluster_u32(base + 4u * i, static_cast<uint32_t>(w[i]));
}

template <bool SPARSE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    attn2_fwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                     const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem + kOffQ;
  uint8_t* sKV = smem + kOffKV;
  Bars2* bars = reinterpret_cast<Bars2*>(smem + kOffBar);

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
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bars->s_full[t], 2);    // MMA commit + the MMA thread's info arrival
      mbar_init(&bars->p_full[t], 16);   // leader only: 8 softmax warps in each CTA
      mbar_init(&bars->o_full[t], 1);
      mbar_init(&bars->o_empty[t], 16);  // leader only
    }
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
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated in both
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;

  if (warp < 4) {
    regs_dec<64>();
    if (warp == 0 && lane == 0) {
      // ============================================================ TMA producer (both CTAs)
      const uint64_t pol_kv = l2_policy_evict_last();
      const uint64_t pol_q = l2_policy_evict_first();
      const uint32_t q_full_l = mapa_shared(smem_u32(&bars->q_full), 0);
      int slot = 0;
      uint32_t ph = 0, qph = 0, iph = 0;
      for (int it_n = 0;; ++it_n) {
        int item;
        if (SPARSE && !leader) {
          mbar_wait_cluster(&bars->item_full, iph);
          iph ^= 1;
          item = *reinterpret_cast<volatile int*>(&bars->item_box);
        }
        mbar_wait(&bars->q_empty, qph ^ 1);
        qph ^= 1;
        if (SPARSE && leader) {
          // Hand the item to the peer's producer.  It has read the previous one: q_empty means the
          // MMAs of the previous item completed, and they needed the peer's Q bytes of that item,
          // loaded after the peer read it.
          item = atomicAdd(p.queue, 1);
          st_cluster_u32(mapa_shared(smem_u32(&bars->item_box), 1), static_cast<uint32_t>(item));
          mbar_arrive_remote(mapa_shared(smem_u32(&bars->item_full), 1));
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
        Item2 it;
        decode_item2<SPARSE>(p, id, it);
        if (leader) {
          bars->qitem = it;
          mbar_arrive_expect_tx(&bars->q_full, 4 * kTileQ);
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          const int s = 2 * t + static_cast<int>(rank);
#pragma unroll
          for (int c = 0; c < 2; ++c)
            tma_load_4d_pair(&tq, q_full_l, sQ + t * kTileQ + c * kChunkQ, c * 64, it.start[s], it.h, it.b, pol_q);
        }
        const uint32_t* ent_ptr = SPARSE ? p.stream + static_cast<int64_t>(id) * p.stream_stride : nullptr;
        for (int e = 0; e < it.n_ent; ++e) {
          const int s0 = SPARSE ? p.grid.start(static_cast<int>(__ldg(ent_ptr + e) & 0xFFFu)) : 128 * e;
          // K: kv rows [s0 + 64 r, +64), both 64-column chunks
          mbar_wait(&bars->kv_empty[slot], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&bars->kv_full[slot], 2 * kSlot);
          {
            const uint32_t fb = mapa_shared(smem_u32(&bars->kv_full[slot]), 0);
            uint8_t* dst = sKV + slot * kSlot;
            tma_load_4d_pair(&tk, fb, dst, 0, s0 + 64 * static_cast<int>(rank), it.h, it.b, pol_kv);
            tma_load_4d_pair(&tk, fb, dst + kSlot / 2, 64, s0 + 64 * static_cast<int>(rank), it.h, it.b, pol_kv);
          }
          if (++slot == kNS) { slot = 0; ph ^= 1; }
          // V: columns [64 r, +64) of kv rows [s0, s0 + 128)
          mbar_wait(&bars->kv_empty[slot], ph ^ 1);
          if (leader) mbar_arrive_expect_tx(&bars->kv_full[slot], 2 * kSlot);
          {
            const uint32_t fb = mapa_shared(smem_u32(&bars->kv_full[slot]), 0);
            tma_load_4d_pair(&tv, fb, sKV + slot * kSlot, 64 * static_cast<int>(rank), s0, it.h, it.b, pol_kv);
          }
          if (++slot == kNS) { slot = 0; ph ^= 1; }
        }
      }
      // drain: every multicast commit aimed at this CTA's kv_empty / q_empty has landed
      for (int i = 0; i < kNS; ++i) {
        mbar_wait(&bars->kv_empty[slot], ph ^ 1);
        if (++slot == kNS) { slot = 0; ph ^= 1; }
      }
    } else if (warp == 1 && lane == 0 && leader) {
      // ============================================================ MMA issuer (leader)
      constexpr uint32_t kIdescQK = idesc_bf16(256, 128, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(256, kD, false, true);
      const uint32_t sq_addr = smem_u32(sQ);
      const uint32_t skv_addr = smem_u32(sKV);
      int slot = 0;
      uint32_t ph = 0, qph = 0;
      uint32_t pph[2] = {0u, 0u}, oeph[2] = {0u, 0u};
      int icnt[2] = {0, 0};
      bool o_dirty[2] = {false, false};
      const uint32_t s_full_peer[2] = {mapa_shared(smem_u32(&bars->s_full[0]), 1),
                                       mapa_shared(smem_u32(&bars->s_full[1]), 1)};

      auto issue_qk = [&](int t, int kslot) {
#pragma unroll
        for (int kk = 0; kk < kD / 16; ++kk) {
          const uint64_t a = desc_sw128(sq_addr + t * kTileQ + (kk >> 2) * kChunkQ + (kk & 3) * 32, 16, 1024);
          const uint64_t b = desc_sw128(skv_addr + kslot * kSlot + (kk >> 2) * (kSlot / 2) + (kk & 3) * 32, 16, 1024);
          mma_ss_pair(tmem + s_col(t), a, b, kIdescQK, kk > 0 ? 1u : 0u);
        }
      };
      auto issue_pv = [&](int t, int vslot, bool first) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t b = desc_sw128(skv_addr + vslot * kSlot + kk * 2048, kSlot, 1024);
          mma_ts_pair(tmem + o_col(t), tmem + s_col(t) + kk * 8, b, kIdescPV, (first && kk == 0) ? 0u : 1u);
        }
      };
      auto wait_p = [&](int t, bool first) {
        mbar_wait_cluster(&bars->p_full[t], pph[t]);
        pph[t] ^= 1;
        tc_fence_after();
        if (first && o_dirty[t]) {
          mbar_wait_cluster(&bars->o_empty[t], oeph[t]);
          oeph[t] ^= 1;
          o_dirty[t] = false;
          tc_fence_after();
        }
      };

      for (;;) {
        mbar_wait(&bars->q_full, qph);
        qph ^= 1;
        tc_fence_after();
        const Item2 it = bars->qitem;
        if (it.kind == kAllEnd) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            Info2 v{};
            v.kind = kAllEnd;
            const int sl = icnt[t] & 1;
            ++icnt[t];
            put_info(bars, t, sl, 0, 0, v, true);
            put_info(bars, t, sl, 1, 0, v, true);
            mbar_arrive_n(&bars->s_full[t], 2);
            mbar_arrive_n_remote(s_full_peer[t], 2);
          }
          break;
        }
        const uint32_t* ent_ptr = SPARSE ? p.stream + static_cast<int64_t>(it.id) * p.stream_stride : nullptr;
        bool pend[2] = {false, false};
        bool had[2] = {false, false};
        bool first_pv[2] = {true, true};
        int pvslot = -1;
        uint32_t pvph = 0;
        for (int e = 0; e < it.n_ent; ++e) {
          int l0;
          uint32_t memb;
          if (SPARSE) {
            const uint32_t ent = __ldg(ent_ptr + e);
            const int j = ent & 0xFFF;
            l0 = p.grid.len(j);
            memb = ent >> 24;
          } else {
            l0 = p.N - 128 * e < 128 ? p.N - 128 * e : 128;
            memb = 0xFu;
          }
          const int kslot = slot;
          const uint32_t kph = ph;
          if (++slot == kNS) { slot = 0; ph ^= 1; }
          const int vslot = slot;
          const uint32_t vph = ph;
          if (++slot == kNS) { slot = 0; ph ^= 1; }
          if (pvslot >= 0) {
            mbar_wait(&bars->kv_full[pvslot], pvph);
            tc_fence_after();
          }
          mbar_wait(&bars->kv_full[kslot], kph);
          tc_fence_after();
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (pend[t]) {
              wait_p(t, first_pv[t]);
              issue_pv(t, pvslot, first_pv[t]);
              first_pv[t] = false;
              pend[t] = false;
            }
            const uint32_t need = (memb >> (2 * t)) & 3u;  // bit r: CTA r's q-block needs this kv block
            if (need) {
              issue_qk(t, kslot);
              const int sl = icnt[t] & 1;
              ++icnt[t];
#pragma unroll
              for (uint32_t r = 0; r < 2; ++r) {
                Info2 v{};
                v.kind = kNormal;
                v.skip = ((need >> r) & 1u) ? 0 : 1;
                v.lim0 = l0 < 64 ? l0 : 64;
                v.lim1 = l0 - 64;
                put_info(bars, t, sl, r, 0, v, false);
              }
              tc_commit_pair(&bars->s_full[t]);
              mbar_arrive(&bars->s_full[t]);
              mbar_arrive_remote(s_full_peer[t]);
              pend[t] = true;
              had[t] = true;
            }
          }
          if (pvslot >= 0) tc_commit_pair(&bars->kv_empty[pvslot]);
          tc_commit_pair(&bars->kv_empty[kslot]);
          pvslot = vslot;
          pvph = vph;
        }
        // ---- end of the item: last PVs, release Q, hand O to the epilogue
        if (pvslot >= 0) {
          mbar_wait(&bars->kv_full[pvslot], pvph);
          tc_fence_after();
        }
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (!pend[t]) continue;
          wait_p(t, first_pv[t]);
          issue_pv(t, pvslot, first_pv[t]);
          first_pv[t] = false;
        }
        if (pvslot >= 0) tc_commit_pair(&bars->kv_empty[pvslot]);
        tc_commit_pair(&bars->q_empty);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          if (had[t]) {
            tc_commit_pair(&bars->o_full[t]);
            o_dirty[t] = true;
          }
          const int sl = icnt[t] & 1;
          ++icnt[t];
#pragma unroll
          for (uint32_t r = 0; r < 2; ++r) {
            Info2 v{};
            v.kind = kEnd;
            v.has = had[t] ? 1 : 0;
            v.b = it.b;
            v.h = it.h;
            v.start = it.start[2 * t + r];
            v.len = it.len[2 * t + r];
            put_info(bars, t, sl, r, 0, v, true);
          }
          mbar_arrive_n(&bars->s_full[t], 2);
          mbar_arrive_n_remote(s_full_peer[t], 2);
        }
      }
    }
  } else {
    regs_inc<104>();
    // ============================================================ softmax warps (both CTAs)
    const int sw = warp - 4;
    const int t = sw >> 3;
    const int hc = (sw >> 2) & 1;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + s_col(t);
    const uint32_t o_addr = tmem + lane_base + o_col(t) + hc * (kD / 2);
    float* xm = bars->xm[t];
    float* xl = bars->xl[t];
    const float sl2 = p.scale_log2;
    const uint32_t p_full_l = mapa_shared(smem_u32(&bars->p_full[t]), 0);
    const uint32_t o_empty_l = mapa_shared(smem_u32(&bars->o_empty[t]), 0);
    uint32_t sph = 0, oph = 0;
    int icnt = 0;
    float m_used = -INFINITY, l_sum = 0.0f;
    int ntile = 0;
    for (;;) {
      mbar_wait_cluster(&bars->s_full[t], sph);
      sph ^= 1;
      tc_fence_after();
      const Info2& inf = bars->info[t][icnt & 1];
      ++icnt;
      const int kind = inf.kind;
      if (kind == kAllEnd) break;
      if (kind == kEnd) {
        if (inf.has) {
          const int b = inf.b, h = inf.h;
          const int tok = inf.start + row;
          const bool valid = row < inf.len;
          xl[hc * 128 + row] = l_sum;
          named_bar_sync(1 + t, 256);
          const float l_tot = l_sum + xl[(1 - hc) * 128 + row];
          mbar_wait(&bars->o_full[t], oph);
          oph ^= 1;
          tc_fence_after();
          const float inv = l_tot > 0.0f ? 1.0f / l_tot : 0.0f;
          __nv_bfloat16* optr = p.o + b * p.sb + h * p.sh + static_cast<int64_t>(tok) * p.sn + hc * (kD / 2);
#pragma unroll
          for (int c = 0; c < kD / 64; ++c) {
            uint32_t r[32];
            tmem_ld32(o_addr + c * 32, r);
            tmem_ld_wait32(r);
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i)
              pk[i] = pack_bf16x2(__uint_as_float(r[2 * i]) * inv, __uint_as_float(r[2 * i + 1]) * inv);
            if (valid) {
              uint4* dst = reinterpret_cast<uint4*>(optr + c * 32);
#pragma unroll
              for (int i = 0; i < 4; ++i) dst[i] = make_uint4(pk[4 * i], pk[4 * i + 1], pk[4 * i + 2], pk[4 * i + 3]);
            }
          }
          if (hc == 0 && valid && p.lse) {
            const float lv = l_tot > 0.0f ? (m_used + __log2f(l_tot)) * kLn2 : -INFINITY;
            p.lse[(static_cast<int64_t>(b) * p.H + h) * p.N + tok] = lv;
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive(&bars->o_empty[t]);
            else mbar_arrive_remote(o_empty_l);
          }
        }
        m_used = -INFINITY;
        l_sum = 0.0f;
        ntile = 0;
        continue;
      }
      if (inf.skip) {
        // this CTA's q-block does not keep this kv block (the pair's other q-block does): P = 0
        uint32_t z[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) z[i] = 0u;
        tmem_st16(s_addr + hc * 32, z);
        tmem_st16(s_addr + hc * 32 + 16, z);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          if (leader) mbar_arrive(&bars->p_full[t]);
          else mbar_arrive_remote(p_full_l);
        }
        ++ntile;
        continue;
      }
      const int lim = hc == 0 ? inf.lim0 : inf.lim1;
      uint32_t s[64];
      tmem_ld32(s_addr + hc * 64, s);
      tmem_ld32(s_addr + hc * 64 + 32, s + 32);
      tmem_ld_wait32(s);
      reg_fence32(s + 32);
      if (lim < 64) {
#pragma unroll
        for (int i = 0; i < 64; ++i) s[i] = i < lim ? s[i] : __float_as_uint(-INFINITY);
      }
      float mx4[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) mx4[a] = fmaxf(__uint_as_float(s[a]), __uint_as_float(s[4 + a]));
#pragma unroll
      for (int i = 8; i < 64; i += 8) {
#pragma unroll
        for (int a = 0; a < 4; ++a) mx4[a] = fmax3(mx4[a], __uint_as_float(s[i + a]), __uint_as_float(s[i + 4 + a]));
      }
      const float lmx = fmax3(mx4[0], mx4[1], fmaxf(mx4[2], mx4[3]));
      // the partner warp holds the other 64 columns of the same rows; the barrier also orders
      // both halves' TMEM loads of S before either overwrites S columns with P
      xm[hc * 128 + row] = lmx;
      named_bar_sync(1 + t, 256);
      const float mx = fmaxf(lmx, xm[(1 - hc) * 128 + row]);
      const float mx2 = mx * sl2;
      const float m_new = fmaxf(m_used, mx2);
      const bool grow = m_new > m_used + kRescaleThreshold;  // also true when m_used == -inf
      float alpha = 1.0f;
      if (grow) {
        alpha = (m_used == -INFINITY) ? 0.0f : exp2f(m_used - m_new);
        l_sum *= alpha;
        m_used = m_new;
      }
      const bool rescale_o = grow && alpha != 0.0f && ntile > 0;
      if (__any_sync(0xffffffffu, rescale_o)) {
        const float a = rescale_o ? alpha : 1.0f;
#pragma unroll 1
        for (int c = 0; c < kD / 64; ++c) {
          uint32_t r[32];
          tmem_ld32(o_addr + c * 32, r);
          tmem_ld_wait32(r);
#pragma unroll
          for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * a);
          tmem_st32(o_addr + c * 32, r);
        }
      }
      const float mb = (m_used == -INFINITY) ? 0.0f : m_used;
      const float2 sl2v = make_float2(sl2, sl2);
      const float2 nmb = make_float2(-mb, -mb);
      float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float s0 = __uint_as_float(s[32 * c + 2 * i]), s1 = __uint_as_float(s[32 * c + 2 * i + 1]);
          const float2 x = ffma2(make_float2(s0, s1), sl2v, nmb);
          float2 pv;
          pv.x = ex2_approx(x.x);
          pv.y = ex2_approx(x.y);
          acc[i & 3] = fadd2(acc[i & 3], pv);
          pk[i] = pack_bf16x2(pv.x, pv.y);
        }
        tmem_st16(s_addr + hc * 32 + c * 16, pk);
      }
      const float2 a01 = fadd2(acc[0], acc[1]), a23 = fadd2(acc[2], acc[3]);
      const float2 a = fadd2(a01, a23);
      l_sum += a.x + a.y;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if (leader) mbar_arrive(&bars->p_full[t]);
        else mbar_arrive_remote(p_full_l);
      }
      ++ntile;
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
  auto kern = attn2_fwd_kernel<SPARSE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  if (e != cudaSuccess) return e;
  const int pairs = num_sms / 2;
  const int grid = 2 * (p.num_items < pairs ? p.num_items : pairs);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, kThreads, kSmemBytes, st>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attn_pair(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                             const AttnParams& p, bool sparse, int num_sms, cudaStream_t st) {
  return sparse ? launch_pair<true>(tq, tk, tv, p, num_sms, st) : launch_pair<false>(tq, tk, tv, p, num_sms, st);
}

}  // namespace adaspa
