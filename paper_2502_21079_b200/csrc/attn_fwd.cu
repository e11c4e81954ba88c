// attn_fwd.cu -- K1 (dense attention + LSE) and K4 (head-adaptive block-sparse attention)
// on sm_100a: TMA-staged Q/K/V tiles, tcgen05.mma into TMEM, softmax in registers.
//
// PAPER.md:194-202 (blockwise online softmax), 471-482 (Alg. 1 first pass: FA + LSE),
// 415-427 (blockified sparse attention, -c(1-M) with c = +inf), 446-448 (visit only S*),
// readings R1-R3 of DESIGN.md (garbled Alg. 1 initialisation / missing rescale / missing
// normalisation -> the standard recurrence).
//
// Design (one CTA per SM, persistent):
//   work item   = two 128-row q tiles (t = 0, 1) of one (b, h); dense: rows [256p, 256p+256);
//                 sparse B=128: q-blocks 2p, 2p+1; sparse B=64: q-blocks 4p..4p+3.
//   kv stream   = dense: every 128-row kv tile; sparse: the UNION of the tiles' CSR rows, each
//                 entry tagged with which (q-tile, 64-row half) x (kv half) pairs need it, so
//                 each K/V tile is loaded once for both q tiles.
//   warp 0      TMA producer: Q tiles, then K,V tiles into a ring of NS slots.
//   warp 1      MMA issuer (one thread): S_t = Q_t K^T (SS, M=128 N=128), O_t += P_t V
//               (TS: P read from TMEM, V MN-major from smem, M=128 N=d).  Order per entry:
//               PV_0(prev), QK_0(e), PV_1(prev), QK_1(e) -- softmax of one tile overlaps the
//               MMAs of the other (ping-pong).
//   warp 2      TMEM allocator (512 columns: S_0 | S_1 | O_0 | O_1).
//   warps 4-11  softmax for q tile 0, warps 12-19 for q tile 1; each warp owns 16 whole rows
//               (16-lane TMEM shapes, a thread quad per row: max / sum by quad shuffles, no
//               exchange between warps).  exp2 domain, conditional rescaling of O (only when the
//               running max grows by more than kRescaleThreshold in log2 units -- exact, the final normalisation
//               uses the same max), P written back to TMEM as bf16 over the first 64 columns of S_t.
#include "attn.cuh"
#include "common.cuh"

namespace adaspa {

#ifndef ADASPA_K4_PF
#define ADASPA_K4_PF 0  // diagnostic: -DADASPA_K4_PF=n prefetches K/V n stream entries ahead into L2 (A/B r02aq: no gain)
#endif

#ifdef ADASPA_TRACE
// Diagnostic build only (-DADASPA_TRACE): per-tile clock64 stamps of CTA 0 -- softmax warp 4
// (q tile 0, column half 0) events 0..3 and the MMA issuer's events -- read back through
// adaspa_debug_trace().  The product library is built without it.
__device__ unsigned long long g_trace[4][4096];
__device__ int g_trace_n[2];
#ifndef ADASPA_TRACE_SKIP
#define ADASPA_TRACE_SKIP 0  // tiles skipped before the 1000 recorded ones (-DADASPA_TRACE_SKIP=n: mid-kernel)
#endif
#define ADASPA_TRACE_IN(i) ((i) >= ADASPA_TRACE_SKIP && (i) < ADASPA_TRACE_SKIP + 1000)
#define ADASPA_TRACE_EV(k)                                                                    \
  do {                                                                                        \
    if (blockIdx.x == 0 && warp == 4 && lane == 0 && ADASPA_TRACE_IN(tr_k))                   \
      g_trace[0][(tr_k - ADASPA_TRACE_SKIP) * 4 + (k)] = clock64();                           \
    if ((k) == 3) ++tr_k;                                                                     \
  } while (0)
#define ADASPA_TRACE_MMA(k)                                                                   \
  do {                                                                                        \
    if (blockIdx.x == 0 && ADASPA_TRACE_IN(tr_n))                                             \
      g_trace[1 + ((k) >> 2)][(tr_n - ADASPA_TRACE_SKIP) * 4 + ((k) & 3)] = clock64();        \
    if ((k) == 5) ++tr_n;                                                                     \
  } while (0)
#define ADASPA_TRACE_TMA(k)                                                                   \
  do {                                                                                        \
    if (blockIdx.x == 0 && ADASPA_TRACE_IN(tp_n))                                             \
      g_trace[3][(tp_n - ADASPA_TRACE_SKIP) * 4 + (k)] = clock64();                           \
    if ((k) == 3) ++tp_n;                                                                     \
  } while (0)
#else
#define ADASPA_TRACE_TMA(k) \
  do {                      \
  } while (0)
#define ADASPA_TRACE_EV(k) \
  do {                     \
  } while (0)
#define ADASPA_TRACE_MMA(k) \
  do {                      \
  } while (0)
#endif

namespace {

constexpr int kThreads = 640;  // d=64: 4 + 16 softmax warps (16 rows per warp)
#ifndef ADASPA_ROW_THREAD
#define ADASPA_ROW_THREAD 1
#endif
// One S row per softmax thread (4 + 8 warps, the kRowThread softmax below) everywhere except the
// dense d=64 pass: A/B on one box (profiles/r02v_*, r02w_*): d=128 K1 / K4 unchanged, the fused search
// pass -4% (its block sums need no shuffles); d=64 K4 +1.5% and fused search -4%, but dense d=64 K1
// 795 -> 715 TFLOP/s (MUFU-bound: two MUFU-issuing warps per SMSP instead of four; still -2.3% with
// the 2^24 rescale threshold, r02ak).  ADASPA_ROW_THREAD=0
// builds the 16-row softmax everywhere (A/B).
template <int D, int MODE>
constexpr bool row_thread() { return ADASPA_ROW_THREAD != 0 && !(D == 64 && MODE == kModeDense); }
template <int D, int MODE>
constexpr int threads_of() { return row_thread<D, MODE>() ? 384 : kThreads; }
__device__ __forceinline__ uint32_t s_col(int t) { return static_cast<uint32_t>(t) * 128u; }
__device__ __forceinline__ uint32_t o_col(int t) { return 256u + static_cast<uint32_t>(t) * 128u; }
// d=64: O_t uses 64 of its 128 columns, so P_t gets the other 64 instead of aliasing S_t.  The next
// QK_t then only waits for the softmax to have LOADED S_t, not for PV_t: no softmax -> PV -> QK
// chain, and the kernel is bound by exponential throughput (at d=64 MUFU work is twice the MMA
// work).  d=128 has no spare TMEM and keeps P in S (the chain stays).
template <int D>
__device__ __forceinline__ uint32_t p_col(int t) { return D == 64 ? o_col(t) + 64u : s_col(t); }
// The running max m moves only when a row's max passes it by more than T (log2 units); P = 2^(x - m)
// then stays <= 2^T (bf16 and the fp32 sums and O accumulation hold 2^24 x |V| x N with room to
// spare), and the final normalisation uses the same m, so the result is exact for any T.  Fewer moves
// mean fewer O rescales (a TMEM read-modify-write of the tile's O): A/B profiles/r02ai_ab*.txt,
// T = 8 -> 12 -> 24: K4 1018 -> 1052 -> 1070 TFLOP/s, K1 1153 -> 1158 -> 1187 (same box).
#ifndef ADASPA_RESCALE_LOG2
#define ADASPA_RESCALE_LOG2 24
#endif
constexpr float kRescaleThreshold = static_cast<float>(ADASPA_RESCALE_LOG2);  // log2 units
// One exp group in ADASPA_EXP_POLY_MOD on an FMA-pipe polynomial instead of MUFU.EX2 (0: none).
// Round 1 measured 1 in 8 best; after the round-1 softmax changes (16-row warps, vote-gated max) the
// MUFU is no longer the limit and the polynomial's ~6 instructions per element cost more than they
// relieve: A/B on one box (profiles/r02_ab_poly.txt) K1 1106 -> 1145 (d=128), 764 -> 805 (d=64),
// K4 1007 -> 1044 TFLOP/s with none.  (K2 keeps its 1 pair in 8: 83.6 vs 85.2 ms, 22.9 vs 26.2.)
#ifndef ADASPA_EXP_POLY_MOD
#define ADASPA_EXP_POLY_MOD 0
#endif
#ifndef ADASPA_ABLATE
#define ADASPA_ABLATE 0  // diagnostic builds only: 4 = no softmax (MMA / TMA pipeline alone)
#endif
constexpr int kExpPolyMod = ADASPA_EXP_POLY_MOD;
#ifndef ADASPA_SPEC_MAX
#define ADASPA_SPEC_MAX 1
#endif
#ifndef ADASPA_BLSE_ABL
#define ADASPA_BLSE_ABL 0  // diagnostic builds only: 1 = no per-tile block-LSE epilogue, 2 = no store
#endif

enum : int { kNormal = 0, kEnd = 1, kAllEnd = 2 };

struct SlotMeta {
  int kind, mask, len0, len1;
  int id0, id1;  // kv block ids of the entry's two 64-row halves (grid / sparse modes)
};

struct TileInfo {
  int kind;
  int lim[4];      // [hq*2 + 0] column limit of kv half 0, [hq*2+1] of half 1 (exclusive, in 0..128)
  int has;         // END: this tile had >= 1 entry in the item (O must be stored)
  int b, h;
  int start0, len0, start1, len1;
};

struct ItemInfo {
  int b, h;
  int exists[2];
  int start0[2], len0[2], start1[2], len1[2];
};

template <int D>
struct Smem {
  static constexpr int kTile = 128 * D * 2;  // one 128-row tile of d bf16 columns
  // d=128: Q (64 KB) + 5 K/V slots (160 KB) + barriers fill the 227 KB; 5 slots let the producer
  // run ~2.5 entries ahead (with 4, the MMA thread waited ~280 cycles per entry for the next K).
  static constexpr int kNS = (D == 128) ? 5 : 10;
  static constexpr int kQ = 0;
  static constexpr int kKV = 2 * kTile;
  static constexpr int kBar = kKV + kNS * kTile;
  static constexpr int kBytes = kBar + 2048 + 1024;  // barriers/meta + alignment slack
};

struct Bars {
  uint64_t kv_full[12], kv_empty[12];
  uint64_t q_full, q_empty;
  uint64_t s_full[2], p_half[2], p_full[2], o_full[2], o_empty[2];
  uint64_t s_loaded[2], p_free[2];  // d=64 only: S_t in registers / PV_t done (P_t may be overwritten)
  SlotMeta meta[12];
  TileInfo info[2][2];
  ItemInfo qitem;
  uint32_t tmem_base;
};

__device__ __forceinline__ void decode_item(const AttnParams& p, bool sparse, bool two, int id, ItemInfo& it) {
  const int bh = id / p.items_per_bh;
  const int pi = id - bh * p.items_per_bh;
  it.b = bh / p.nh;
  it.h = p.h0 + (bh - it.b * p.nh);
  if (!sparse) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int s = 256 * pi + 128 * t;
      int l = p.N - s;
      l = l < 0 ? 0 : (l > 128 ? 128 : l);
      it.exists[t] = l > 0;
      it.start0[t] = s;
      it.len0[t] = l;
      it.start1[t] = s + 64;
      it.len1[t] = 0;
    }
  } else if (!two) {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int qb = 2 * pi + t;
      const bool ex = qb < p.grid.nb;
      it.exists[t] = ex;
      it.start0[t] = ex ? p.grid.start(qb) : 0;
      it.len0[t] = ex ? p.grid.len(qb) : 0;
      it.start1[t] = it.start0[t] + 64;
      it.len1[t] = 0;
    }
  } else {
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int qa = 4 * pi + 2 * t, qc = qa + 1;
      const bool ea = qa < p.grid.nb, ec = qc < p.grid.nb;
      it.exists[t] = ea;
      it.start0[t] = ea ? p.grid.start(qa) : 0;
      it.len0[t] = ea ? p.grid.len(qa) : 0;
      it.start1[t] = ec ? p.grid.start(qc) : it.start0[t];
      it.len1[t] = ec ? p.grid.len(qc) : 0;
    }
  }
}

static_assert(sizeof(Bars) <= 2048, "barrier block outgrew its reservation");
static_assert(Smem<128>::kBytes <= 232448 && Smem<64>::kBytes <= 232448, "over 227 KB of shared memory");

// MODE: kDense (K1: 128-row kv tiles from token 0), kBlse (K1 + block LSEs: kv tiles follow the
// block grid -- one block per tile, or two 64-row blocks with KVTWO -- and every (row, kv block)
// log-sum-exp is written for the fused block-mass reduction), kSparse (K4: the merged CSR stream).
// QTWO: a q tile is two 64-row q-blocks (sparse B=64); KVTWO: a kv tile is two 64-row kv blocks.
template <int D, bool QTWO, bool KVTWO, int MODE>
__global__ void __launch_bounds__(threads_of<D, MODE>(), 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                    const __grid_constant__ CUtensorMap tv, const AttnParams p) {
  constexpr bool SPARSE = MODE == kModeSparse;
  constexpr bool GRID = MODE != kModeDense;  // kv tiles follow the block grid
  constexpr bool BLSE = MODE == kModeBlse;
  // skip the exponentials of fully masked 64-column halves: only where they are common (the B=64
  // pairs of the sparse stream); elsewhere the branch costs registers for nothing
  constexpr bool kSkipDead = SPARSE && KVTWO;
  constexpr int kK4Prefetch = ADASPA_K4_PF;  // K4: stream entries between an L2 prefetch and its load
  constexpr bool kRowThread = row_thread<D, MODE>();
  constexpr int kSoftWarps = kRowThread ? 4 : 8;  // softmax warps per q tile
  // speculative first-half exponentials: A/B profiles/r02z_ab_*: K1 +1.8%, fused search -1.9%, K4 +1.3%
  // at B=128; K4 at B=64 -2.4% with the rescale threshold at 2^8, +1.2% at 2^24 (r02ak); not at d=64
  // (its registers spill)
  constexpr bool kSpecMax = ADASPA_SPEC_MAX != 0 && D == 128;
  using S = Smem<D>;
  constexpr int NS = S::kNS;
  constexpr bool kSepP = D == 64;
  // d=64: one MMA issuer per q tile (warps 1 and 3), the two tiles' chains are independent (P has
  // its own TMEM columns).  d=128: one issuer for both, whose PV0, QK0, PV1, QK1 order interleaves
  // the two chains on the tensor pipe (measured: two issuers there cost 13%).
  constexpr int kIssuers = kSepP ? 2 : 1;
  constexpr int TILE = S::kTile;
  constexpr int CH = D / 64;            // 64-column (128-byte) chunks per row
  constexpr int CHUNK = 128 * 128;      // bytes per chunk of a 128-row tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays a shared pointer
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sKV = smem + S::kKV;
  Bars* bars = reinterpret_cast<Bars*>(smem + S::kBar);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], kIssuers);  // one release per MMA issuer
    }
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, kIssuers);
    for (int t = 0; t < 2; ++t) {
      mbar_init(&bars->s_full[t], 2);
      mbar_init(&bars->p_half[t], kSoftWarps);  // P columns [0, 32) (kv rows 0-63) of every row stored
      mbar_init(&bars->p_full[t], kSoftWarps);
      mbar_init(&bars->s_loaded[t], kSoftWarps);
      mbar_init(&bars->p_free[t], 1);
      mbar_init(&bars->o_full[t], 1);
      mbar_init(&bars->o_empty[t], kSoftWarps);
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
  // 640 threads x 96 registers at launch; the producer/MMA warpgroup hands registers to the four
  // softmax warpgroups, which hold a 64-column half S row each.  The pool is what the launch
  // allocated, 640 x 96: 64*128 + 104*512 = 61440 (setmaxnreg.inc beyond it never returns).
  if (warp < 4) {
  if constexpr (kRowThread) regs_dec<80>(); else regs_dec<64>();
  if (warp == 0) {
    // ============================================================ TMA producer
    if (lane == 0) {
      int slot = 0;
      uint32_t ph = 0, qph = 0;
      const uint64_t pol_kv = l2_policy_evict_last();
      int tp_n = 0;
      (void)tp_n;
      const uint64_t pol_q = l2_policy_evict_first();
      for (int it_n = 0;; ++it_n) {
        int item;
        if (SPARSE) item = atomicAdd(p.queue, 1);
        else item = blockIdx.x + it_n * gridDim.x;
        if (item >= p.num_items) break;
        const int id = SPARSE ? __ldg(p.item_order + item) : item;
        ItemInfo it;
        decode_item(p, SPARSE, QTWO, id, it);
        mbar_wait(&bars->q_empty, qph ^ 1);
        qph ^= 1;
        bars->qitem = it;
        const uint32_t qbytes = (it.exists[0] ? TILE : 0) + (it.exists[1] ? TILE : 0);
        mbar_arrive_expect_tx(&bars->q_full, qbytes);
        for (int t = 0; t < 2; ++t) {
          if (!it.exists[t]) continue;
          const int r1 = QTWO ? it.start1[t] : it.start0[t] + 64;
          for (int c = 0; c < CH; ++c) {
            uint8_t* dst = sQ + t * TILE + c * CHUNK;
            tma_load_4d_hint(&tq, &bars->q_full, dst, c * 64, it.start0[t], it.h, it.b, pol_q);
            if (QTWO) tma_load_4d_hint(&tq, &bars->q_full, dst + CHUNK / 2, c * 64, r1, it.h, it.b, pol_q);  // B=64: second block; else one 128-row box
          }
        }
        const int n_ent = SPARSE ? __ldg(p.stream_len + id)
                          : GRID ? (KVTWO ? (p.grid.nb + 1) / 2 : p.grid.nb) : (p.N + 127) / 128;
        const uint64_t* ent_ptr = SPARSE ? p.stream + static_cast<int64_t>(id) * p.stream_stride : nullptr;
        const uint32_t dense_mask = (it.exists[0] ? 0x0Fu : 0u) | (it.exists[1] ? 0xF0u : 0u);
        for (int e = 0; e < n_ent; ++e) {
          int s0, l0, s1, l1, id0 = -1, id1 = -1;
          uint32_t mask;
          if (SPARSE) {
            const uint64_t ent = __ldg(reinterpret_cast<const unsigned long long*>(ent_ptr) + e);
            id0 = entry_id0(ent);
            id1 = entry_id1(ent);
            mask = entry_mask(ent);
            s0 = p.grid.start(id0);
            l0 = p.grid.len(id0);
            if (KVTWO) {
              s1 = p.grid.start(id1);
              l1 = p.grid.len(id1);
            } else {
              s1 = s0 + 64;
              l1 = 0;
            }
          } else if (GRID) {  // every kv block of the head, in order (one per tile, or two 64-row blocks)
            id0 = KVTWO ? 2 * e : e;
            id1 = (KVTWO && id0 + 1 < p.grid.nb) ? id0 + 1 : -1;
            s0 = p.grid.start(id0);
            l0 = p.grid.len(id0);
            s1 = id1 >= 0 ? p.grid.start(id1) : s0 + 64;
            l1 = id1 >= 0 ? p.grid.len(id1) : 0;
            mask = dense_mask;
          } else {
            s0 = 128 * e;
            l0 = p.N - s0 < 128 ? p.N - s0 : 128;
            s1 = s0 + 64;
            l1 = 0;
            mask = dense_mask;
          }
          // K4: warm L2 with the K/V tiles of the entry kK4Prefetch ahead (the gathered tiles of a
          // head's stream miss L2 now and then; the ring itself holds only 2.5 entries at d=128)
          if constexpr (SPARSE && kK4Prefetch > 0) {
            if (e + kK4Prefetch < n_ent) {
              const uint64_t en = __ldg(reinterpret_cast<const unsigned long long*>(ent_ptr) + e + kK4Prefetch);
              const int ps0 = p.grid.start(entry_id0(en));
              const int ps1 = KVTWO ? p.grid.start(entry_id1(en)) : 0;
              for (int c = 0; c < CH; ++c) {
                tma_prefetch_l2_4d(&tk, c * 64, ps0, it.h, it.b, pol_kv);
                tma_prefetch_l2_4d(&tv, c * 64, ps0, it.h, it.b, pol_kv);
                if (KVTWO) {
                  tma_prefetch_l2_4d(&tk, c * 64, ps1, it.h, it.b, pol_kv);
                  tma_prefetch_l2_4d(&tv, c * 64, ps1, it.h, it.b, pol_kv);
                }
              }
            }
          }
          // K
          ADASPA_TRACE_TMA(0);
          mbar_wait(&bars->kv_empty[slot], ph ^ 1);
          ADASPA_TRACE_TMA(1);
          bars->meta[slot] = SlotMeta{kNormal, static_cast<int>(mask), l0, l1, id0, id1};
          mbar_arrive_expect_tx(&bars->kv_full[slot], TILE);
          for (int c = 0; c < CH; ++c) {
            uint8_t* dst = sKV + slot * TILE + c * CHUNK;
            tma_load_4d_hint(&tk, &bars->kv_full[slot], dst, c * 64, s0, it.h, it.b, pol_kv);
            if (KVTWO) tma_load_4d_hint(&tk, &bars->kv_full[slot], dst + CHUNK / 2, c * 64, s1, it.h, it.b, pol_kv);  // B=64: second block; else one 128-row box
          }
          if (++slot == NS) { slot = 0; ph ^= 1; }
          // V
          ADASPA_TRACE_TMA(2);
          mbar_wait(&bars->kv_empty[slot], ph ^ 1);
          ADASPA_TRACE_TMA(3);
          mbar_arrive_expect_tx(&bars->kv_full[slot], TILE);
          for (int c = 0; c < CH; ++c) {
            uint8_t* dst = sKV + slot * TILE + c * CHUNK;
            tma_load_4d_hint(&tv, &bars->kv_full[slot], dst, c * 64, s0, it.h, it.b, pol_kv);
            if (KVTWO) tma_load_4d_hint(&tv, &bars->kv_full[slot], dst + CHUNK / 2, c * 64, s1, it.h, it.b, pol_kv);  // B=64: second block; else one 128-row box
          }
          if (++slot == NS) { slot = 0; ph ^= 1; }
        }
        mbar_wait(&bars->kv_empty[slot], ph ^ 1);
        bars->meta[slot].kind = kEnd;
        mbar_arrive(&bars->kv_full[slot]);
        if (++slot == NS) { slot = 0; ph ^= 1; }
      }
      mbar_wait(&bars->kv_empty[slot], ph ^ 1);
      bars->meta[slot].kind = kAllEnd;
      mbar_arrive(&bars->kv_full[slot]);
    }
  } else if (warp == 1 || (kIssuers == 2 && warp == 3)) {
    // ============================================================ MMA issuer(s)
    // kIssuers == 2: one issuer thread per q tile (warp 1: tile 0, warp 3: tile 1), each following
    // the same K/V ring, so a wait for one tile's P never holds back the other tile's MMAs; K/V
    // slots and Q are released after both issuers' commits (count-2 barriers).  T = -1: both tiles.
    if (lane == 0) {
      const int T = kIssuers == 1 ? -1 : (warp == 1 ? 0 : 1);
      constexpr uint32_t kIdescQK = idesc_bf16(128, 128, false, false);
      constexpr uint32_t kIdescPV = idesc_bf16(128, D, false, true);
      const uint32_t sq_addr = smem_u32(sQ);
      const uint32_t skv_addr = smem_u32(sKV);
      int slot = 0;
      uint32_t ph = 0, qph = 0;
      uint32_t pph[2] = {0u, 0u}, oeph[2] = {0u, 0u}, slph[2] = {0u, 0u};
      bool slp[2] = {false, false};  // kSepP: an S_t whose s_loaded arrival is not consumed yet
      auto wait_loaded = [&](int t) {
        if (!kSepP || !slp[t]) return;
        mbar_wait(&bars->s_loaded[t], slph[t]);
        slph[t] ^= 1;
        slp[t] = false;
        tc_fence_after();
      };
      int icnt[2] = {0, 0};
      bool o_dirty[2] = {false, false};
      int tr_n = 0;
      (void)tr_n;

      auto issue_qk = [&](int t, int kslot) {
#pragma unroll
        for (int kk = 0; kk < D / 16; ++kk) {
          const uint32_t off = (kk >> 2) * CHUNK + (kk & 3) * 32;
          const uint64_t a = desc_sw128(sq_addr + t * TILE + off, 16, 1024);
          const uint64_t b = desc_sw128(skv_addr + kslot * TILE + off, 16, 1024);
          mma_ss(tmem + s_col(t), a, b, kIdescQK, kk > 0 ? 1u : 0u);
        }
      };
      // PV in two halves: kv rows 0-63 (P columns 0-31) as soon as the softmax has stored them,
      // so they run while it computes the second half; then kv rows 64-127.
      auto issue_pv_half = [&](int t, int vslot, bool first, int half) {
#pragma unroll
        for (int k4 = 0; k4 < 4; ++k4) {
          const int kk = 4 * half + k4;
          const uint64_t b = desc_sw128(skv_addr + vslot * TILE + kk * 2048, CHUNK, 1024);
          mma_ts(tmem + o_col(t), tmem + p_col<D>(t) + kk * 8, b, kIdescPV, (first && kk == 0) ? 0u : 1u);
        }
      };
      // wait for P_t (both halves) and issue PV_t; O must have been drained by the epilogue first
      auto wait_issue_pv = [&](int t, int vslot, bool first) {
        mbar_wait(&bars->p_half[t], pph[t]);
        tc_fence_after();
        if (first && o_dirty[t]) {
          mbar_wait(&bars->o_empty[t], oeph[t]);
          oeph[t] ^= 1;
          o_dirty[t] = false;
          tc_fence_after();
        }
        issue_pv_half(t, vslot, first, 0);
        mbar_wait(&bars->p_full[t], pph[t]);
        pph[t] ^= 1;
        tc_fence_after();
        issue_pv_half(t, vslot, false, 1);
        if (kSepP) tc_commit(&bars->p_free[t]);
      };

      for (;;) {
        mbar_wait(&bars->kv_full[slot], ph);
        tc_fence_after();
        SlotMeta mt = bars->meta[slot];
        if (mt.kind == kAllEnd) {
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (T >= 0 && t != T) continue;
            bars->info[t][icnt[t] & 1].kind = kAllEnd;
            ++icnt[t];
            mbar_arrive_n(&bars->s_full[t], 2);
          }
          break;
        }
        mbar_wait(&bars->q_full, qph);
        qph ^= 1;
        tc_fence_after();
        const ItemInfo it = bars->qitem;
        bool pend[2] = {false, false};
        bool had[2] = {false, false};
        bool first_pv[2] = {true, true};
        int pvslot = -1;
        uint32_t pvph = 0;
        for (;;) {
          if (mt.kind == kEnd) {
            if (pvslot >= 0) {
              mbar_wait(&bars->kv_full[pvslot], pvph);
              tc_fence_after();
            }
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              if (T >= 0 && t != T) continue;
              if (!pend[t]) continue;
              wait_loaded(t);
              wait_issue_pv(t, pvslot, first_pv[t]);
              first_pv[t] = false;
            }
            if (pvslot >= 0) tc_commit(&bars->kv_empty[pvslot]);
            tc_commit(&bars->q_empty);
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              if (T >= 0 && t != T) continue;
              if (had[t]) {
                tc_commit(&bars->o_full[t]);
                o_dirty[t] = true;
              }
              TileInfo& inf = bars->info[t][icnt[t] & 1];
              ++icnt[t];
              inf.kind = kEnd;
              inf.has = had[t];
              inf.b = it.b;
              inf.h = it.h;
              inf.start0 = it.start0[t];
              inf.len0 = it.len0[t];
              inf.start1 = it.start1[t];
              inf.len1 = it.len1[t];
              mbar_arrive_n(&bars->s_full[t], 2);
            }
            mbar_arrive(&bars->kv_empty[slot]);
            if (++slot == NS) { slot = 0; ph ^= 1; }
            break;
          }
          // ---- normal entry: K in `slot`, V in the next slot
          const int kslot = slot;
          if (++slot == NS) { slot = 0; ph ^= 1; }
          const int vslot = slot;
          const uint32_t vph = ph;
          if (++slot == NS) { slot = 0; ph ^= 1; }
          if (pvslot >= 0) {
            mbar_wait(&bars->kv_full[pvslot], pvph);
            if (T <= 0) ADASPA_TRACE_MMA(4);
            tc_fence_after();
          }
          // kSepP (d=64): this entry's QKs go first (they only need the previous S_t loaded), then
          // the previous entry's PVs.  Otherwise PV_t(prev) must precede QK_t (P_t aliases S_t).
          bool pv_pend[2] = {pend[0], pend[1]};
          if (kSepP) {
#pragma unroll
            for (int t = 0; t < 2; ++t) pend[t] = false;
          }
#pragma unroll
          for (int t = 0; t < 2; ++t) {
            if (T >= 0 && t != T) continue;
            if (!kSepP && pv_pend[t]) {
              wait_issue_pv(t, pvslot, first_pv[t]);
              if (T <= 0) ADASPA_TRACE_MMA(t * 2 + 0);
              first_pv[t] = false;
              pend[t] = false;
            }
            const uint32_t need = (static_cast<uint32_t>(mt.mask) >> (4 * t)) & 0xFu;
            if (need) {
              wait_loaded(t);
              issue_qk(t, kslot);
              if (kSepP) slp[t] = true;
              if (T <= 0) ADASPA_TRACE_MMA(t * 2 + 1);
              TileInfo& inf = bars->info[t][icnt[t] & 1];
              ++icnt[t];
              inf.kind = kNormal;
#pragma unroll
              for (int hq = 0; hq < 2; ++hq) {
                const uint32_t bits = (need >> (2 * hq)) & 3u;
                if (!KVTWO) {
                  inf.lim[hq * 2 + 0] = (bits & 1u) ? (mt.len0 < 64 ? mt.len0 : 64) : 0;
                  inf.lim[hq * 2 + 1] = (bits & 2u) ? mt.len0 : 64;
                } else {
                  inf.lim[hq * 2 + 0] = (bits & 1u) ? mt.len0 : 0;
                  inf.lim[hq * 2 + 1] = (bits & 2u) ? 64 + mt.len1 : 64;
                }
              }
              if (BLSE) {
                inf.b = it.b;
                inf.h = it.h;
                inf.start0 = it.start0[t];
                inf.len0 = it.len0[t];
              }
              tc_commit(&bars->s_full[t]);
              mbar_arrive(&bars->s_full[t]);
              pend[t] = true;
              had[t] = true;
            }
          }
          if (kSepP) {
#pragma unroll
            for (int t = 0; t < 2; ++t) {
              if (T >= 0 && t != T) continue;
              if (!pv_pend[t]) continue;
              // a tile that skipped this entry still has its S loaded-arrival outstanding
              if (!((static_cast<uint32_t>(mt.mask) >> (4 * t)) & 0xFu)) wait_loaded(t);
              wait_issue_pv(t, pvslot, first_pv[t]);
              if (T <= 0) ADASPA_TRACE_MMA(t * 2 + 0);
              first_pv[t] = false;
            }
          }
          if (pvslot >= 0) tc_commit(&bars->kv_empty[pvslot]);
          tc_commit(&bars->kv_empty[kslot]);
          pvslot = vslot;
          pvph = vph;
          mbar_wait(&bars->kv_full[slot], ph);
          if (T <= 0) ADASPA_TRACE_MMA(5);
          tc_fence_after();
          mt = bars->meta[slot];
        }
      }
    }
  }
  } else if constexpr (kRowThread) {
    // 384 threads x 168 registers at launch (64512); the producer/MMA warpgroup drops to 80 (its MMA
    // issuer spills at 64 here), so the two softmax warpgroups take (64512 - 4*32*80) / 256 = 212 ->
    // 208 each: a whole 128-column S row (128 registers) per thread
    regs_inc<208>();
    // ============================================================ softmax warps, one row per thread
    // warps 4..11: q tile t = (warp - 4) >> 2; warp lane quarter wq = warp & 3 owns TMEM lanes
    // [32 wq, 32 wq + 32); thread = one row of the tile with all 128 columns (32x32b TMEM shapes).
    // The row max, the row sum and the per-block sums of the fused search are thread-local: no
    // shuffles, no votes; four warps per q tile arrive on each hand-off.
    const int t = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int hq = wq >> 1;  // 64-row half of the q tile (column-limit index)
    const int row = wq * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const uint32_t s_addr = tmem + lane_base + s_col(t);
    const uint32_t o_addr = tmem + lane_base + o_col(t);
    const uint32_t p_addr = tmem + lane_base + p_col<D>(t);  // d=128: P over S columns [0, 64); d=64: O's spare 64
    const float sl2 = p.scale_log2;
    uint32_t sph = 0, oph = 0;
    int icnt = 0;
    float m_used = -INFINITY;  // running max (log2 units), moved only when the row max passes it by kRescaleThreshold
    float l_sum = 0.0f;
    float ref = 0.0f;          // BLSE: the row's first running max
    int ntile = 0;
    float* blse_row = nullptr;  // BLSE: this row of the block-LSE scratch (per item)
    bool blse_ok = false;
    uint32_t rt_pfph = 0;  // kSepP (d=64): p_free phase; the n-th normal tile (n >= 1) waits for PV n-1
    int rt_pcnt = 0;
    int tr_k = 0;
    (void)tr_k;
    for (;;) {
      mbar_wait(&bars->s_full[t], sph);
      sph ^= 1;
      ADASPA_TRACE_EV(0);
      tc_fence_after();
      const TileInfo& inf = bars->info[t][icnt & 1];
      ++icnt;
      const int kind = inf.kind;
      if (kind == kAllEnd) break;
      if (kind == kEnd) {
        const int b = inf.b, h = inf.h;
        int tok;
        bool valid;
        if (!QTWO || row < 64) {
          tok = inf.start0 + row;
          valid = row < inf.len0;
        } else {
          tok = inf.start1 + row - 64;
          valid = row - 64 < inf.len1;
        }
        __nv_bfloat16* optr = p.o + b * p.sb + h * p.sh + static_cast<int64_t>(valid ? tok : 0) * p.sn;
        if (inf.has) {
          // a row with at least one kept column has l >= 1 (the element that set m contributes 2^0)
          const float inv = l_sum >= 0.25f ? 1.0f / l_sum : 0.0f;
          mbar_wait(&bars->o_full[t], oph);
          oph ^= 1;
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(o_addr + c * 32, r);
            tmem_ld_wait32(r);
            uint4 w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              w[i] = make_uint4(pack_bf16x2(__uint_as_float(r[8 * i + 0]) * inv, __uint_as_float(r[8 * i + 1]) * inv),
                                pack_bf16x2(__uint_as_float(r[8 * i + 2]) * inv, __uint_as_float(r[8 * i + 3]) * inv),
                                pack_bf16x2(__uint_as_float(r[8 * i + 4]) * inv, __uint_as_float(r[8 * i + 5]) * inv),
                                pack_bf16x2(__uint_as_float(r[8 * i + 6]) * inv, __uint_as_float(r[8 * i + 7]) * inv));
            if (valid) {
              uint4* dst = reinterpret_cast<uint4*>(optr + 32 * c);
#pragma unroll
              for (int i = 0; i < 4; ++i) dst[i] = w[i];
            }
          }
          if (valid && p.lse)
            p.lse[(static_cast<int64_t>(b) * p.H + h) * p.N + tok] =
                l_sum >= 0.25f ? (m_used + __log2f(l_sum)) * kLn2 : -INFINITY;
          if (BLSE && valid)  // the row LSE relative to ref (log2 units), for the block-mass reduction
            p.lrel[(static_cast<int64_t>(b) * p.nh + (h - p.h0)) * p.N + tok] =
                l_sum >= 0.25f ? (m_used - ref) + __log2f(l_sum) : -INFINITY;
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars->o_empty[t]);
        } else {  // no kept kv block for any row of this tile (a caller CSR with empty rows)
          if (valid) {
            uint4* dst = reinterpret_cast<uint4*>(optr);
#pragma unroll
            for (int i = 0; i < D / 8; ++i) dst[i] = make_uint4(0u, 0u, 0u, 0u);
            if (p.lse) p.lse[(static_cast<int64_t>(b) * p.H + h) * p.N + tok] = -INFINITY;
          }
        }
        m_used = -INFINITY;
        l_sum = 0.0f;
        ref = 0.0f;
        ntile = 0;
        continue;
      }
      const int limA = *reinterpret_cast<const volatile int*>(&inf.lim[hq * 2 + 0]);
      const int limB = *reinterpret_cast<const volatile int*>(&inf.lim[hq * 2 + 1]);
      if (BLSE && ntile == 0) {  // per item: this row in blse[b,h][kb][.] and whether it stores
        const int64_t bhl = static_cast<int64_t>(inf.b) * p.nh + (inf.h - p.h0);
        blse_row = p.blse + bhl * p.grid.nb * p.N + inf.start0 + row;
        blse_ok = row < inf.len0;
      }
      uint32_t s[128];
      tmem_ld32(s_addr, s);
      tmem_ld32(s_addr + 32, s + 32);
      tmem_ld32(s_addr + 64, s + 64);
      tmem_ld32(s_addr + 96, s + 96);
      tmem_ld_wait();
      reg_fence32(s);
      reg_fence32(s + 32);
      reg_fence32(s + 64);
      reg_fence32(s + 96);
      ADASPA_TRACE_EV(1);
      if (kSepP) {  // S_t is in registers: the next QK_t may overwrite it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->s_loaded[t]);
      }
      // dead halves (kSkipDead: masked for every row of the warp) skip their exponentials and stay
      // out of the max; a partial block (or an unneeded half without kSkipDead) is masked to -inf
      const bool deadA = kSkipDead && limA == 0, deadB = kSkipDead && limB <= 64;
      if ((limA < 64 && !deadA) || (limB < 128 && !deadB)) {
#pragma unroll
        for (int i = 0; i < 128; ++i) {
          const int lim = i < 64 ? limA : limB;
          s[i] = i < lim ? s[i] : __float_as_uint(-INFINITY);
        }
      }
      const float2 sl2v = make_float2(sl2, sl2);
      float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      // P = 2^(S*scale*log2e - m) for one 64-column half: FFMA2 for the argument, MUFU.EX2, packed to
      // bf16 pairs (S columns 2j, 2j+1 -> P column j, the TS MMA's A layout); sums into acc
      auto exp_half = [&](int c, float mbase, uint32_t* pk) {
        const float2 nm = make_float2(-mbase, -mbase);
#pragma unroll
        for (int k = 0; k < 32; ++k) {
          const int i = 64 * c + 2 * k;
          const float2 x = ffma2(make_float2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sl2v, nm);
          float2 e;
          e.x = ex2_approx(x.x);
          e.y = ex2_approx(x.y);
          acc[k & 3] = fadd2(acc[k & 3], e);
          pk[k] = pack_bf16x2(e.x, e.y);
        }
      };
      uint32_t pk[32];
      // kSpecMax: once the row has a running max, the first half's exponentials go first with it and
      // the full row max is taken only if that was not safe -- the half's sum above 2^T (then some
      // P may exceed 2^T, T = kRescaleThreshold) or the second half's max passing m + T (checked before anything is handed
      // over, so both halves always share one m); otherwise the max waits in the MUFU's shadow
      bool spec = false;
      if (kSpecMax && __all_sync(0xffffffffu, m_used > -INFINITY)) {
        float h0 = fmaxf(__uint_as_float(s[64]), __uint_as_float(s[65]));
        float h1 = fmaxf(__uint_as_float(s[66]), __uint_as_float(s[67]));
#pragma unroll
        for (int i = 4; i < 64; i += 4) {
          h0 = fmax3(h0, __uint_as_float(s[64 + i]), __uint_as_float(s[65 + i]));
          h1 = fmax3(h1, __uint_as_float(s[66 + i]), __uint_as_float(s[67 + i]));
        }
        const float mh1 = deadB ? -INFINITY : fmaxf(h0, h1) * sl2;
        if (deadA) {
#pragma unroll
          for (int i = 0; i < 32; ++i) pk[i] = 0u;
        } else {
          exp_half(0, m_used, pk);
        }
        const float2 a = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        const bool ok = (a.x + a.y <= exp2f(kRescaleThreshold)) && !(mh1 > m_used + kRescaleThreshold);
        spec = __all_sync(0xffffffffu, ok);
        if (!spec) {
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
        }
      }
      if (kSepP) {  // PV of the previous tile has read P_t and accumulated into O_t
        if (rt_pcnt > 0) {
          mbar_wait(&bars->p_free[t], rt_pfph);
          rt_pfph ^= 1;
          tc_fence_after();
        }
        ++rt_pcnt;
      }
      if (!spec) {
        float mx0 = fmaxf(__uint_as_float(s[0]), __uint_as_float(s[1]));
        float mx1 = fmaxf(__uint_as_float(s[2]), __uint_as_float(s[3]));
        float mx2 = fmaxf(__uint_as_float(s[64]), __uint_as_float(s[65]));
        float mx3 = fmaxf(__uint_as_float(s[66]), __uint_as_float(s[67]));
#pragma unroll
        for (int i = 4; i < 64; i += 4) {
          mx0 = fmax3(mx0, __uint_as_float(s[i]), __uint_as_float(s[i + 1]));
          mx1 = fmax3(mx1, __uint_as_float(s[i + 2]), __uint_as_float(s[i + 3]));
          mx2 = fmax3(mx2, __uint_as_float(s[64 + i]), __uint_as_float(s[65 + i]));
          mx3 = fmax3(mx3, __uint_as_float(s[66 + i]), __uint_as_float(s[67 + i]));
        }
        const float mxa = deadA ? -INFINITY : fmaxf(mx0, mx1), mxb = deadB ? -INFINITY : fmaxf(mx2, mx3);
        const float mx = fmaxf(mxa, mxb) * sl2;
        float alpha = 1.0f;
        bool rescale = false;
        if (mx > m_used + kRescaleThreshold) {  // also true when m_used == -inf (and mx finite)
          alpha = (m_used == -INFINITY) ? 0.0f : exp2f(m_used - mx);
          l_sum *= alpha;
          if (BLSE && m_used == -INFINITY) ref = mx;
          m_used = mx;
          rescale = alpha != 0.0f && ntile > 0;
        }
        if (__any_sync(0xffffffffu, rescale)) {  // rare: some row's max grew by more than 2^T
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t r[32];
            tmem_ld32(o_addr + c * 32, r);
            tmem_ld_wait32(r);
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st32(o_addr + c * 32, r);
          }
        }
        if (deadA) {
#pragma unroll
          for (int i = 0; i < 32; ++i) pk[i] = 0u;
        } else {
          exp_half(0, (m_used == -INFINITY) ? 0.0f : m_used, pk);
        }
      }
      const float mb = (m_used == -INFINITY) ? 0.0f : m_used;
      ADASPA_TRACE_EV(2);
      // first half of P stored: the MMA thread may start PV on kv rows 0-63
      tmem_st32(p_addr, pk);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->p_half[t]);
      float half0;  // the row sum over columns 0-63 (BLSE with KVTWO: kv block id0)
      {
        const float2 h01 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        half0 = h01.x + h01.y;
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
      }
      if (deadB) {
#pragma unroll
        for (int i = 0; i < 32; ++i) pk[i] = 0u;
      } else {
        exp_half(1, mb, pk);
      }
      tmem_st32(p_addr + 32, pk);
      const float2 h23 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
      const float half1 = h23.x + h23.y;
      l_sum += half0 + half1;
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      ADASPA_TRACE_EV(3);
      if (lane == 0) mbar_arrive(&bars->p_full[t]);
      if (BLSE && blse_ok) {
        // this tile's per-block log-sum-exps relative to the row's first max (thread-local sums):
        // log2 sum_{j in kb} 2^(s_ij*scale*log2e) - ref = log2(t) + (m_used - ref); tile n is block n
        // (KVTWO: blocks 2n and 2n+1); tt = 0 gives -inf
        const float mref = m_used - ref;
        if (KVTWO) {
          __stcs(blse_row + static_cast<int64_t>(2 * ntile) * p.N, __log2f(half0) + mref);
          if (2 * ntile + 1 < p.grid.nb)
            __stcs(blse_row + static_cast<int64_t>(2 * ntile + 1) * p.N, __log2f(half1) + mref);
        } else {
          __stcs(blse_row + static_cast<int64_t>(ntile) * p.N, __log2f(half0 + half1) + mref);
        }
      }
      ++ntile;
    }
  } else {
    regs_inc<104>();
    // ============================================================ softmax warps
    // warps 4..19: sw = warp - 4, q tile t = sw >> 3; the warp owns 16 WHOLE rows of the tile: TMEM
    // lanes [32 wq + 16 hh, +16) with wq = warp & 3 (its lane quarter) and hh = (sw >> 2) & 1.
    // Through the 16-lane TMEM shapes a thread quad shares a row (thread i: rows r0 = base + i/4 and
    // r1 = r0 + 8, 32 of the 128 columns each), so the row max and row sum are two quad shuffles and
    // P overwrites only S columns of the warp's own rows: no shared-memory exchange, no barrier
    // between warps on the per-tile path.
    const int sw = warp - 4;
    const int t = sw >> 3;
    const int hh = (sw >> 2) & 1;
    const int wq = warp & 3;
    const int hq = wq >> 1;                        // 64-row half of the q tile
    const int qd = lane & 3;                       // position in the quad
    const int row0 = wq * 32 + hh * 16 + (lane >> 2);
    const int row1 = row0 + 8;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32 + hh * 16) << 16;
    const uint32_t s_addr = tmem + lane_base + s_col(t);
    const uint32_t o_addr = tmem + lane_base + o_col(t);
    const uint32_t p_addr = tmem + lane_base + p_col<D>(t);
    uint32_t pfph = 0;
    int pcnt = 0;  // kSepP: normal tiles processed; the n-th (n >= 1) waits for PV of the (n-1)-th
    auto wait_p_free = [&]() {
      if (!kSepP || pcnt == 0) return;
      mbar_wait(&bars->p_free[t], pfph);
      pfph ^= 1;
      tc_fence_after();
    };
    const float sl2 = p.scale_log2;
    uint32_t sph = 0, oph = 0;
    int icnt = 0;
    float m_used[2] = {-INFINITY, -INFINITY};
    float l_sum[2] = {0.0f, 0.0f};  // this thread's share (its 32 columns) of the row sums
    float ref[2] = {0.0f, 0.0f};    // BLSE: the row's first running max (log2 units)
    float mref = 0.0f;              // BLSE: m_used - ref of this lane's block-LSE row (qd & 1), kept with m
    int ntile = 0;
    float* blse_row = nullptr;  // BLSE: this lane's row of the block-LSE scratch (per item)
    bool blse_ok = false;
    int tr_k = 0;
    (void)tr_k;
    const Poly3x2 poly;
    // BLSE: the block sums feed the block masses, so the FMA-pipe exponentials use the degree-5
    // polynomial (rel. error 2.3e-7, ex2.approx class) instead of the degree-3 one (7.5e-5, enough
    // for P's bf16 rounding but not for a block mass to ~1e-6)
    const Poly5x2 poly5;
    // BLSE: a tile's per-(row, kv block) sums, quad-reduced, as log-sum-exps relative to the row's ref:
    // log2 sum_{j in kb} 2^(s_ij*scale*log2e) - ref_i = log2(t) + (m_used - ref).  Quad lane qd writes
    // (row qd&1, block half qd>>1), rows of a warp contiguous in blse[bh][kb][.].  The transpose-reduce
    // over the quad halves the values a lane keeps per exchange, so lane qd ends with value qd in 2
    // shuffles (one block per tile) or 3 (KVTWO).  (Deferring this to the next tile's first P hand-off
    // measured slower: profiles/r02k_ab_*.txt.)
    auto blse_store = [&](float t0v, float t1v, float h0v, float h1v, int tile) {
      const int j = qd & 1, hf = qd >> 1;
      float tt;
      if (KVTWO) {
        // values: (r0,h0) (r1,h0) (r0,h1) (r1,h1); xor 2 splits the halves, xor 1 the rows
        const float keep0 = hf ? t0v : h0v, send0 = hf ? h0v : t0v;
        const float keep1 = hf ? t1v : h1v, send1 = hf ? h1v : t1v;
        const float r0 = keep0 + __shfl_xor_sync(0xffffffffu, send0, 2);
        const float r1 = keep1 + __shfl_xor_sync(0xffffffffu, send1, 2);
        const float keep = j ? r1 : r0, send = j ? r0 : r1;
        tt = keep + __shfl_xor_sync(0xffffffffu, send, 1);
      } else {
        const float keep = j ? t1v : t0v, send = j ? t0v : t1v;
        tt = keep + __shfl_xor_sync(0xffffffffu, send, 1);
        tt += __shfl_xor_sync(0xffffffffu, tt, 2);
      }
      // kv tiles follow the block grid, every tile of the item in order: tile n is block n (KVTWO:
      // blocks 2n and 2n+1)
      const int kb = KVTWO ? 2 * tile + hf : tile;
      if (blse_ok && kb < p.grid.nb) {
        const float Lb = __log2f(tt) + mref;  // tt = 0 (or a denormal): -inf
        if (ADASPA_BLSE_ABL != 2 || p.N < 0) __stcs(blse_row + static_cast<int64_t>(kb) * p.N, Lb);  // streamed: K/V stay in L2
      }
    };
    for (;;) {
      mbar_wait(&bars->s_full[t], sph);
      sph ^= 1;
      ADASPA_TRACE_EV(0);
      tc_fence_after();
      const TileInfo& inf = bars->info[t][icnt & 1];
      ++icnt;
      const int kind = inf.kind;
      if (kind == kAllEnd) break;
      if (kind == kEnd) {
        const int b = inf.b, h = inf.h;
        int tok[2];
        bool valid[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int row = j ? row1 : row0;
          if (!QTWO) {
            tok[j] = inf.start0 + row;
            valid[j] = row < inf.len0;
          } else if (row < 64) {
            tok[j] = inf.start0 + row;
            valid[j] = row < inf.len0;
          } else {
            tok[j] = inf.start1 + row - 64;
            valid[j] = row - 64 < inf.len1;
          }
        }
        __nv_bfloat16* optr[2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
          optr[j] = p.o + b * p.sb + h * p.sh + static_cast<int64_t>(valid[j] ? tok[j] : 0) * p.sn + 2 * qd;
        if (inf.has) {
          float l_tot[2], inv[2];
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            float l = l_sum[j];
            l += __shfl_xor_sync(0xffffffffu, l, 1);
            l += __shfl_xor_sync(0xffffffffu, l, 2);
            l_tot[j] = l;
            // a row with at least one kept column has l >= 1 (the element that set m_used contributes
            // 2^0); below that only the 2^-126 floor of the polynomial exp on masked columns: empty row
            inv[j] = l >= 0.25f ? 1.0f / l : 0.0f;
          }
          mbar_wait(&bars->o_full[t], oph);
          oph ^= 1;
          tc_fence_after();
#pragma unroll
          for (int c = 0; c < D / 32; ++c) {
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
                p.lse[(static_cast<int64_t>(b) * p.H + h) * p.N + tok[j]] =
                    l_tot[j] >= 0.25f ? (m_used[j] + __log2f(l_tot[j])) * kLn2 : -INFINITY;
          }
          if (BLSE && qd == 1) {  // the row LSE relative to ref (log2 units), for the block-mass reduction
#pragma unroll
            for (int j = 0; j < 2; ++j)
              if (valid[j])
                p.lrel[(static_cast<int64_t>(b) * p.nh + (h - p.h0)) * p.N + tok[j]] =
                    l_tot[j] >= 0.25f ? (m_used[j] - ref[j]) + __log2f(l_tot[j]) : -INFINITY;
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars->o_empty[t]);
        } else {  // no kept kv block for any row of this tile (a caller CSR with empty rows): O = 0, LSE = -inf
#pragma unroll
          for (int c = 0; c < D / 32; ++c)
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
              for (int j = 0; j < 2; ++j)
                if (valid[j]) *reinterpret_cast<uint32_t*>(optr[j] + 32 * c + 8 * k) = 0u;
          if (qd == 0 && p.lse) {
#pragma unroll
            for (int j = 0; j < 2; ++j)
              if (valid[j]) p.lse[(static_cast<int64_t>(b) * p.H + h) * p.N + tok[j]] = -INFINITY;
          }
        }
        m_used[0] = m_used[1] = -INFINITY;
        l_sum[0] = l_sum[1] = 0.0f;
        ref[0] = ref[1] = 0.0f;
        mref = 0.0f;
        ntile = 0;
        continue;
      }
      if (ADASPA_ABLATE == 4) {  // diagnostic: no softmax (MMA/TMA pipeline alone)
        ADASPA_TRACE_EV(1);
        ADASPA_TRACE_EV(2);
        tc_fence_before();
        __syncwarp();
        ADASPA_TRACE_EV(3);
        if (lane == 0) {
          if (kSepP) mbar_arrive(&bars->s_loaded[t]);
          mbar_arrive(&bars->p_half[t]);
          mbar_arrive(&bars->p_full[t]);
        }
        ++ntile;
        continue;
      }
      // valid columns: [0, limA) of kv half 0 and [64, limB) of kv half 1 (absolute, 0..128); read
      // (volatile) before the TMEM load, used only before the exponentials
      const int limA = *reinterpret_cast<const volatile int*>(&inf.lim[hq * 2 + 0]);
      const int limB = *reinterpret_cast<const volatile int*>(&inf.lim[hq * 2 + 1]);
      if (BLSE && ntile == 0) {  // per item: this lane's row in blse[b,h][kb][.] and whether it stores
        const int row = (qd & 1) ? row1 : row0;
        const int64_t bhl = static_cast<int64_t>(inf.b) * p.nh + (inf.h - p.h0);
        blse_row = p.blse + bhl * p.grid.nb * p.N + inf.start0 + row;
        blse_ok = (KVTWO || (qd >> 1) == 0) && row < inf.len0;
      }
      uint32_t s[64];
      tmem_ld_16x256b_x8(s_addr, s);
      tmem_ld_16x256b_x8(s_addr + 64, s + 32);
      tmem_ld_wait32(s);
      reg_fence32(s + 32);
      if (kSepP) {  // S_t is in registers: the next QK_t may overwrite it
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->s_loaded[t]);
      }
      ADASPA_TRACE_EV(1);
      // Row max over the whole tile first: the column limits (a shared-memory load that queues
      // behind MUFU work in MIO) stay off the critical path of full tiles.  A partial tile or an
      // unneeded half (limits below 64 / 128, warp-uniform; rare) then masks those columns to -inf
      // and redoes the running-max update from the saved state with the max of the kept columns, so
      // masked columns -- TMA zero fill past the sequence end, the excluded half of a B=64 pair, the
      // neighbour block behind a partial block -- never set m.  (With them in m, a row whose kept
      // logits sit ~90 nats below them would underflow to l = 0.)
      float mxa[2], mxb[2];  // two partial maxima per row
      // two partial maxima per row (four independent chains).  kSkipDead: mxa[j] over columns 0-63
      // (s[i], i < 32) and mxb[j] over 64-127, so a dead half (its exponentials skipped) stays out of
      // the row max without the masking pass; otherwise split by column group parity (measured 0.5%
      // faster for K1)
      auto row_max = [&]() {
        if (kSkipDead) {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            mxa[j] = fmaxf(__uint_as_float(s[2 * j]), __uint_as_float(s[2 * j + 1]));
            mxb[j] = fmaxf(__uint_as_float(s[32 + 2 * j]), __uint_as_float(s[33 + 2 * j]));
          }
#pragma unroll
          for (int k = 1; k < 8; ++k) {
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              mxa[j] = fmax3(mxa[j], __uint_as_float(s[4 * k + 2 * j]), __uint_as_float(s[4 * k + 2 * j + 1]));
              mxb[j] = fmax3(mxb[j], __uint_as_float(s[32 + 4 * k + 2 * j]), __uint_as_float(s[33 + 4 * k + 2 * j]));
            }
          }
        } else {
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
        }
      };
      row_max();
      float mb[2];
      float alpha[2] = {1.0f, 1.0f};
      bool rescale = false;
      const float m_prev[2] = {m_used[0], m_used[1]};
      const float l_prev[2] = {l_sum[0], l_sum[1]};
      // m_used moves when the quad's row max exceeds it by more than 2^T (log2 units)
      auto update_max = [&](const float lmx0, const float lmx1) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          float mx = j ? lmx1 : lmx0;
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
          const float m_new = fmaxf(m_used[j], mx);
          if (m_new > m_used[j] + kRescaleThreshold) {  // also true when m_used == -inf
            alpha[j] = (m_used[j] == -INFINITY) ? 0.0f : exp2f(m_used[j] - m_new);
            l_sum[j] *= alpha[j];
            if (BLSE && m_used[j] == -INFINITY) ref[j] = m_new;
            m_used[j] = m_new;
            rescale |= alpha[j] != 0.0f && ntile > 0;
          }
        }
        if (BLSE) mref = (qd & 1) ? (m_used[1] - ref[1]) : (m_used[0] - ref[0]);
      };
      // dead halves (kSkipDead: a 64-column half masked for every row of the warp) skip their
      // exponentials, so leaving them out of the max needs no masking; a partial block (or, without
      // kSkipDead, an unneeded half) takes the masking pass below
      const bool deadA = kSkipDead && limA == 0, deadB = kSkipDead && limB <= 64;
      {
        const float ma0 = deadA ? -INFINITY : mxa[0], ma1 = deadA ? -INFINITY : mxa[1];
        const float mb0 = deadB ? -INFINITY : mxb[0], mb1 = deadB ? -INFINITY : mxb[1];
        const float lmx0 = fmaxf(ma0, mb0) * sl2, lmx1 = fmaxf(ma1, mb1) * sl2;
        // the quad's row max is needed only when some thread's max passes m_used + 8: one warp vote
        // instead of four shuffles (which queue behind MUFU in MIO)
        if (__any_sync(0xffffffffu, lmx0 > m_used[0] + kRescaleThreshold || lmx1 > m_used[1] + kRescaleThreshold))
          update_max(lmx0, lmx1);
      }
      if ((limA < 64 && !deadA) || (limB < 128 && !deadB)) {  // partial block / unneeded half: -> -inf (P = 0)
#pragma unroll
        for (int i = 0; i < 64; ++i) {
          const int col = 8 * (i >> 2) + 2 * qd + (i & 1);
          const int lim = col < 64 ? limA : limB;
          s[i] = col < lim ? s[i] : __float_as_uint(-INFINITY);
        }
        row_max();
        m_used[0] = m_prev[0];
        m_used[1] = m_prev[1];
        l_sum[0] = l_prev[0];
        l_sum[1] = l_prev[1];
        alpha[0] = alpha[1] = 1.0f;
        rescale = false;
        update_max(fmaxf(mxa[0], mxb[0]) * sl2, fmaxf(mxa[1], mxb[1]) * sl2);
      }
      mb[0] = (m_used[0] == -INFINITY) ? 0.0f : m_used[0];
      mb[1] = (m_used[1] == -INFINITY) ? 0.0f : m_used[1];
      ADASPA_TRACE_EV(2);
      wait_p_free();  // kSepP: PV of the previous tile has read P_t and accumulated into O_t
      ++pcnt;
      if (__any_sync(0xffffffffu, rescale)) {  // rare: the running max grew by more than 2^T
#pragma unroll 1
        for (int c = 0; c < D / 32; ++c) {
          uint32_t r[16];
          tmem_ld_16x256b_x4(o_addr + c * 32, r);
          tmem_ld_wait16(r);
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha[(i >> 1) & 1]);
          tmem_st_16x256b_x4(o_addr + c * 32, r);
        }
      }
      // P = 2^(S*scale*log2e - m): FFMA2 for the argument, MUFU.EX2 (one pair in kExpPolyMod on a
      // packed degree-3 polynomial on the FMA pipe, rel. error 1e-4 -- below P's bf16 rounding),
      // packed to bf16 pairs: S columns 8k + 2qd + {0,1} -> P column 4k + qd (16x128b layout).
      const float2 sl2v = make_float2(sl2, sl2);
      const float2 nm0 = make_float2(-mb[0], -mb[0]);
      const float2 nm1 = make_float2(-mb[1], -mb[1]);
      float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      float half0[2] = {0.0f, 0.0f};  // BLSE with KVTWO: the row sums of kv block id0 (columns 0-63)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t pk[16];
        // a 64-column half masked for every row of the warp (a dropped quadrant of a B=64 pair, the
        // empty half of an odd B=64 tail, a dense tail shorter than 64): P = 0 without exponentials
        // (at d = 64 the MUFU is the bound, and these are ~18% of the tile work at CogX-45K)
        const bool dead = c == 0 ? deadA : deadB;
        if (dead) {
#pragma unroll
          for (int i = 0; i < 16; ++i) pk[i] = 0u;
        } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int i = 32 * c + 4 * k;
          const float2 x0 = ffma2(make_float2(__uint_as_float(s[i]), __uint_as_float(s[i + 1])), sl2v, nm0);
          const float2 x1 = ffma2(make_float2(__uint_as_float(s[i + 2]), __uint_as_float(s[i + 3])), sl2v, nm1);
          float2 p0, p1;
          if (kExpPolyMod > 0 && (k % (kExpPolyMod > 0 ? kExpPolyMod : 1)) == kExpPolyMod - 1) {
            if (BLSE) {
              p0 = exp2_poly5x2(x0, poly5);
              p1 = exp2_poly5x2(x1, poly5);
            } else {
              p0 = exp2_poly3x2(x0, poly);
              p1 = exp2_poly3x2(x1, poly);
            }
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
        }
        tmem_st_16x128b_x8(p_addr + c * 32, pk);
        if (c == 0) {  // first half of P stored: the MMA thread may start PV on kv rows 0-63
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars->p_half[t]);
          if (BLSE && KVTWO) {  // kv block id0 ends here: keep its row sums apart from block id1's
            const float2 h0 = fadd2(acc[0], acc[2]), h1 = fadd2(acc[1], acc[3]);
            half0[0] = h0.x + h0.y;
            half0[1] = h1.x + h1.y;
#pragma unroll
            for (int i = 0; i < 4; ++i) acc[i] = make_float2(0.f, 0.f);
          }
        }
      }
      const float2 a0 = fadd2(acc[0], acc[2]), a1 = fadd2(acc[1], acc[3]);
      const float tsum[2] = {a0.x + a0.y, a1.x + a1.y};  // (KVTWO BLSE: kv block id1 only)
      l_sum[0] += tsum[0] + half0[0];
      l_sum[1] += tsum[1] + half0[1];
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      ADASPA_TRACE_EV(3);
      if (lane == 0) mbar_arrive(&bars->p_full[t]);
      // off the critical path (P is handed over): this tile's block log-sum-exps
      if (BLSE && ADASPA_BLSE_ABL != 1) blse_store(tsum[0], tsum[1], half0[0], half0[1], ntile);
      ++ntile;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ------------------------------------------------------------------ sparse schedule prep
// One warp per work item: union of the item's CSR rows (2 q-blocks at B=128, 4 at B=64) as a
// bitmap pass over kv-block words, emitted with membership masks.  B=128: one kv block per entry,
// ascending.  B=64: an entry pairs two kv blocks into one 128-row tile and a q tile computes the
// whole tile if either of its q-blocks keeps either block, so blocks are grouped by membership
// pattern (which of the 4 q-blocks keep them; ascending within a group) before pairing -- in id
// order 25% of the executed tile work was on dropped pairs (tools/sparse_efficiency.py).
__device__ __forceinline__ void stream_word(const SparsePrepParams& p, int w, int lane, int* cur, const int* rend,
                                            uint32_t* word) {
  for (int s = 0; s < 4; ++s) {
    uint32_t acc = 0;
    // lane-parallel: each lane checks one candidate element of list s in this word
    while (true) {
      const int idx = cur[s] + lane;
      int v = (idx < rend[s]) ? p.col_idx[idx] : 0x7fffffff;
      const bool in = v < (w + 1) * 32;
      if (in) acc |= 1u << (v - w * 32);
      const uint32_t bal = __ballot_sync(0xffffffffu, in);
      const int n_in = __popc(bal);
      cur[s] += n_in;
      if (n_in < 32) break;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc |= __shfl_xor_sync(0xffffffffu, acc, o);
    word[s] = acc;
  }
}

__global__ void __launch_bounds__(256) sparse_stream_kernel(SparsePrepParams p) {
  __shared__ int grp[8][2][16];  // per warp: pattern counts, then running positions
  const int item = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int wl = threadIdx.x >> 5;
  if (item >= p.num_items) return;
  const int bh = item / p.items_per_bh;
  const int pi = item - bh * p.items_per_bh;
  const int nb = p.grid.nb;
  const int nq = p.two ? 4 : 2;
  int rbeg[4], rend[4];
  for (int s = 0; s < 4; ++s) {
    const int qb = nq * pi + s;
    if (s < nq && qb < nb) {
      const int64_t row = static_cast<int64_t>(bh) * nb + qb;
      rbeg[s] = p.row_ptr[row];
      rend[s] = p.row_ptr[row + 1];
    } else {
      rbeg[s] = rend[s] = 0;
    }
  }
  uint64_t* out = p.stream + static_cast<int64_t>(item) * p.stream_stride;
  const int nwords = (nb + 31) / 32;
  int cur[4];
  if (p.two) {
    // pass 1: how many union blocks have each membership pattern (1..15)
    if (lane < 16) grp[wl][0][lane] = 0;
    __syncwarp();
    for (int s = 0; s < 4; ++s) cur[s] = rbeg[s];
    for (int w = 0; w < nwords; ++w) {
      uint32_t word[4];
      stream_word(p, w, lane, cur, rend, word);
      uint32_t memb = 0;
      for (int s = 0; s < 4; ++s) memb |= ((word[s] >> lane) & 1u) << s;
      const uint32_t same = __match_any_sync(0xffffffffu, memb);
      if (memb && lane == __ffs(same) - 1) grp[wl][0][memb] += __popc(same);
      __syncwarp();
    }
    // exclusive prefix over patterns -> running positions
    if (lane == 0) {
      int acc = 0;
      for (int m = 0; m < 16; ++m) {
        grp[wl][1][m] = acc;
        acc += grp[wl][0][m];
      }
    }
    __syncwarp();
  }
  // emit (B=128: ascending union; B=64: pattern groups, ascending within a group)
  for (int s = 0; s < 4; ++s) cur[s] = rbeg[s];
  int u_count = 0;  // union elements emitted so far
  for (int w = 0; w < nwords; ++w) {
    uint32_t word[4];
    stream_word(p, w, lane, cur, rend, word);
    const uint32_t uni = word[0] | word[1] | word[2] | word[3];
    const bool mine = (uni >> lane) & 1u;
    const uint32_t bal = __ballot_sync(0xffffffffu, mine);
    uint32_t memb = 0;
    for (int s = 0; s < 4; ++s) memb |= ((word[s] >> lane) & 1u) << s;
    const int j = w * 32 + lane;
    if (!p.two) {
      if (mine) {
        const int pos = u_count + __popc(bal & ((1u << lane) - 1u));
        const uint32_t mask = ((memb & 1u) ? 0x0Fu : 0u) | ((memb & 2u) ? 0xF0u : 0u);
        out[pos] = stream_entry(j, j, mask);
      }
    } else {
      const uint32_t same = __match_any_sync(0xffffffffu, memb);
      const int pos = grp[wl][1][memb] + __popc(same & ((1u << lane) - 1u));
      __syncwarp();
      if (mine) {
        const int hf = pos & 1;
        uint32_t mask = 0;
        for (int s = 0; s < 4; ++s)
          if ((memb >> s) & 1u) mask |= 1u << (2 * s + hf);  // bit 4t + 2hq + hf with s = 2t + hq
        const uint64_t part = (static_cast<uint64_t>(j) << (16 * hf)) | (static_cast<uint64_t>(mask) << 32);
        atomicOr(reinterpret_cast<unsigned long long*>(out + (pos >> 1)), static_cast<unsigned long long>(part));
        if (lane == __ffs(same) - 1) grp[wl][1][memb] += __popc(same);
      }
      __syncwarp();
    }
    u_count += __popc(bal);
  }
  __syncwarp();
  if (lane == 0) {
    int n = u_count;
    if (p.two) {
      n = (u_count + 1) / 2;
      if (u_count & 1) {  // odd union: duplicate id0 into the empty half (mask bits stay 0)
        const uint64_t e = out[n - 1];
        out[n - 1] = e | (static_cast<uint64_t>(entry_id0(e)) << 16);
      }
    }
    p.stream_len[item] = n;
  }
}

// One CTA per (b,h): order the head's items by stream length, longest first (LPT within a
// head; heads stay in order so concurrently running CTAs share one head's K/V in L2).
__global__ void __launch_bounds__(256) sparse_order_kernel(SparsePrepParams p) {
  const int bh = blockIdx.x;
  const int P = p.items_per_bh;
  const int base = bh * P;
  for (int i = threadIdx.x; i < P; i += blockDim.x) {
    const int ci = p.stream_len[base + i];
    int rank = 0;
    for (int j = 0; j < P; ++j) {
      const int cj = p.stream_len[base + j];
      rank += (cj > ci || (cj == ci && j < i)) ? 1 : 0;
    }
    p.item_order[base + rank] = base + i;
  }
}

}  // namespace

#ifdef ADASPA_TRACE
extern "C" int adaspa_debug_trace(unsigned long long* host, int n) {
  if (cudaMemcpyFromSymbol(host, g_trace, sizeof(unsigned long long) * (n < 16384 ? n : 16384)) != cudaSuccess) return -1;
  return 0;
}
#endif

cudaError_t launch_sparse_prep(const SparsePrepParams& p, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(p.stream, 0, sizeof(uint64_t) * static_cast<size_t>(p.num_items) * p.stream_stride, st);
  if (e != cudaSuccess) return e;
  const int blocks = (p.num_items * 32 + 255) / 256;
  sparse_stream_kernel<<<blocks, 256, 0, st>>>(p);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  sparse_order_kernel<<<p.B * p.H, 256, 0, st>>>(p);
  return cudaGetLastError();
}

template <int D, bool QTWO, bool KVTWO, int MODE>
static cudaError_t launch_one(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                              const AttnParams& p, int num_sms, cudaStream_t st) {
  auto kern = attn_fwd_kernel<D, QTWO, KVTWO, MODE>;
  const int smem = Smem<D>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int grid = p.num_items < num_sms ? p.num_items : num_sms;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, threads_of<D, MODE>(), smem, st>>>(tq, tk, tv, p);
  return cudaGetLastError();
}

template <int D>
static cudaError_t launch_d(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                            const AttnParams& p, bool two, int mode, int num_sms, cudaStream_t st) {
  if (mode == kModeDense) return launch_one<D, false, false, kModeDense>(tq, tk, tv, p, num_sms, st);
  if (mode == kModeBlse)
    return two ? launch_one<D, false, true, kModeBlse>(tq, tk, tv, p, num_sms, st)
               : launch_one<D, false, false, kModeBlse>(tq, tk, tv, p, num_sms, st);
  return two ? launch_one<D, true, true, kModeSparse>(tq, tk, tv, p, num_sms, st)
             : launch_one<D, false, false, kModeSparse>(tq, tk, tv, p, num_sms, st);
}

cudaError_t launch_attn(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                        const AttnParams& p, int head_dim, bool two, int mode, int num_sms,
                        cudaStream_t st) {
  return head_dim == 128 ? launch_d<128>(tq, tk, tv, p, two, mode, num_sms, st)
                         : launch_d<64>(tq, tk, tv, p, two, mode, num_sms, st);
}

}  // namespace adaspa
