// search.cu -- K2: LSE-cached online search (Alg. 2; Alg. 1 second pass,
// PAPER.md:484-493):  block_mass[b,h,p,j] = sum_{i in p, t in j} exp(scale*q_i.k_t - lse_i)
// (W_sum_attn; reading R4: "Log(qk - LSE)" is exp(qk*scale - LSE)).
//
// Same skeleton as attn_fwd.cu without the PV product: persistent CTAs, a work item is two
// 128-row q tiles of one head (q-blocks 2p,2p+1 at B=128; 4p..4p+3 at B=64), the kv stream is
// every kv tile of the head (one block at B=128, two at B=64).  S tiles are double-buffered
// per q tile in TMEM (4 x 128 columns), so the tensor core runs ahead of the exp work.
// Exp-role warps: two per TMEM lane quarter, each on one 64-column half of the S row (one kv block
// at B=64, one half block at B=128): x = fma(S, scale*log2e, -lse*log2e), p = 2^x (MUFU.EX2, one
// pair in 8 on the FMA pipe), fp32 partial sums, a warp-shuffle sum over the warp's 32 rows into
// shared memory, and every kChunk kv tiles one fixed-order fp64 sum over the warps of the q tile
// gives one fp32 mass per (q-block, kv-block) -- no per-tile barrier.  S never touches memory.
#include "attn.cuh"
#include "common.cuh"

namespace adaspa {

namespace {

constexpr int kThreads = 640;

constexpr int kChunk = 256;  // kv tiles per flush of the per-warp partial masses
#ifndef ADASPA_SEARCH_POLY_MASK
#define ADASPA_SEARCH_POLY_MASK 0x80
#endif
// bit (i % 8): pair i of a 64-column half goes to the FMA-pipe polynomial instead of MUFU.EX2
constexpr uint32_t kSearchPolyMask = ADASPA_SEARCH_POLY_MASK;

template <int D>
struct SSmem {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kNS = (D == 128) ? 4 : 8;
  static constexpr int kQ = 0;
  static constexpr int kK = 2 * kTile;
  static constexpr int kPart = kK + kNS * kTile;                  // float [2 tiles][2 halves][4 warps][kChunk]
  static constexpr int kBar = kPart + 2 * 4 * kChunk * 2 * 4;
  static constexpr int kBytes = kBar + 1024 + 1024;
};

struct SBars {
  uint64_t kv_full[8], kv_empty[8];
  uint64_t q_full, q_empty;
  uint64_t s_full[2][2], s_empty[2][2];
  uint32_t tmem_base;
};

struct QTiles {
  int b, h, bh;
  int exists[2];
  int qb0[2], qb1[2];            // q-block ids (qb1 = -1 if none / B=128)
  int start0[2], len0[2], start1[2], len1[2];
};

__device__ __forceinline__ void decode_search_item(const SearchParams& p, bool two, int id, QTiles& q) {
  const int bh = id / p.items_per_bh;
  const int pi = id - bh * p.items_per_bh;
  q.bh = bh;
  q.b = bh / p.H;
  q.h = bh - q.b * p.H;
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    if (!two) {
      const int qb = 2 * pi + t;
      const bool ex = qb < p.grid.nb;
      q.exists[t] = ex;
      q.qb0[t] = ex ? qb : -1;
      q.qb1[t] = -1;
      q.start0[t] = ex ? p.grid.start(qb) : 0;
      q.len0[t] = ex ? p.grid.len(qb) : 0;
      q.start1[t] = q.start0[t] + 64;
      q.len1[t] = 0;
    } else {
      const int qa = 4 * pi + 2 * t, qc = qa + 1;
      const bool ea = qa < p.grid.nb, ec = qc < p.grid.nb;
      q.exists[t] = ea;
      q.qb0[t] = ea ? qa : -1;
      q.qb1[t] = ec ? qc : -1;
      q.start0[t] = ea ? p.grid.start(qa) : 0;
      q.len0[t] = ea ? p.grid.len(qa) : 0;
      q.start1[t] = ec ? p.grid.start(qc) : q.start0[t];
      q.len1[t] = ec ? p.grid.len(qc) : 0;
    }
  }
}

// kv tile j -> (row start / valid length of each 64-row half) and the kv-block ids
__device__ __forceinline__ void kv_tile(const SearchParams& p, bool two, int j, int& s0, int& l0, int& s1,
                                        int& l1, int& kb0, int& kb1) {
  if (!two) {
    kb0 = j;
    kb1 = -1;
    s0 = p.grid.start(j);
    l0 = p.grid.len(j);
    s1 = s0 + 64;
    l1 = 0;
  } else {
    kb0 = 2 * j;
    kb1 = 2 * j + 1 < p.grid.nb ? 2 * j + 1 : -1;
    s0 = p.grid.start(kb0);
    l0 = p.grid.len(kb0);
    s1 = kb1 >= 0 ? p.grid.start(kb1) : s0;
    l1 = kb1 >= 0 ? p.grid.len(kb1) : 0;
  }
}

// Sum of 2^x over 64 consecutive columns held in s[0..63] (fp32 bits), x = S*scale*log2e - lse*log2e
// (reading R4); columns at or beyond `lim` are excluded.  The argument is one FFMA2 per pair; one
// pair in kSearchPolyMod goes through the degree-5 polynomial on the FMA pipe (relative error 2.3e-7,
// the same class as ex2.approx's 2^-22), the rest through MUFU.EX2; 4 packed partial sums, then a
// tree.  (Measured on HYV-110K / CogX-45K: 1 in 8 is best; 1 in 4 or 3 loses to the FMA pipe.)
template <bool FULL>
__device__ __forceinline__ float half_mass(const uint32_t* s, float2 sl2, float2 nl, int lim) {
  const Poly5x2 poly;
  float2 acc[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const float2 x = ffma2(make_float2(__uint_as_float(s[2 * i]), __uint_as_float(s[2 * i + 1])), sl2, nl);
    float2 e;
    if ((kSearchPolyMask >> (i & 7)) & 1u) {
      e = exp2_poly5x2(x, poly);
    } else {
      e.x = ex2_approx(x.x);
      e.y = ex2_approx(x.y);
    }
    if (!FULL) {
      e.x = (2 * i < lim) ? e.x : 0.0f;
      e.y = (2 * i + 1 < lim) ? e.y : 0.0f;
    }
    acc[i & 3] = fadd2(acc[i & 3], e);
  }
  const float2 a = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
  return a.x + a.y;
}

template <int D, bool TWO>
__global__ void __launch_bounds__(kThreads, 1)
    search_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                  const SearchParams p) {
  using S = SSmem<D>;
  constexpr int NS = S::kNS;
  constexpr int TILE = S::kTile;
  constexpr int CH = D / 64;
  constexpr int CHUNK = 128 * 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + S::kQ;
  uint8_t* sK = smem + S::kK;
  float* part = reinterpret_cast<float*>(smem + S::kPart);
  SBars* bars = reinterpret_cast<SBars*>(smem + S::kBar);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 2);  // one release per MMA issuer (one per q tile)
    }
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 2);
    for (int t = 0; t < 2; ++t)
      for (int b = 0; b < 2; ++b) {
        mbar_init(&bars->s_full[t][b], 1);
        mbar_init(&bars->s_empty[t][b], 8);
      }
    fence_mbar_init();
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
  }
  if (warp == 2) {
    tmem_alloc(&bars->tmem_base, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = bars->tmem_base;
  const int ntiles = p.kv_tiles;

  if (warp < 4) {
  regs_dec<64>();  // pool = 640 x 96 at launch: 64*128 + 104*512 = 61440
  if (warp == 0) {
    if (lane == 0) {
      int slot = 0;
      uint32_t ph = 0, qph = 0;
      const uint64_t pol_k = l2_policy_evict_last();
      const uint64_t pol_q = l2_policy_evict_first();
      for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
        QTiles q;
        decode_search_item(p, TWO, item, q);
        mbar_wait(&bars->q_empty, qph ^ 1);
        qph ^= 1;
        mbar_arrive_expect_tx(&bars->q_full, (q.exists[0] ? TILE : 0) + (q.exists[1] ? TILE : 0));
        for (int t = 0; t < 2; ++t) {
          if (!q.exists[t]) continue;
          const int r1 = TWO ? q.start1[t] : q.start0[t] + 64;
          for (int c = 0; c < CH; ++c) {
            uint8_t* dst = sQ + t * TILE + c * CHUNK;
            tma_load_4d_hint(&tq, &bars->q_full, dst, c * 64, q.start0[t], q.h, q.b, pol_q);
            if (TWO) tma_load_4d_hint(&tq, &bars->q_full, dst + CHUNK / 2, c * 64, r1, q.h, q.b, pol_q);  // B=64: second block; else one 128-row box
          }
        }
        for (int j = 0; j < ntiles; ++j) {
          int s0, l0, s1, l1, kb0, kb1;
          kv_tile(p, TWO, j, s0, l0, s1, l1, kb0, kb1);
          mbar_wait(&bars->kv_empty[slot], ph ^ 1);
          mbar_arrive_expect_tx(&bars->kv_full[slot], TILE);
          for (int c = 0; c < CH; ++c) {
            uint8_t* dst = sK + slot * TILE + c * CHUNK;
            tma_load_4d_hint(&tk, &bars->kv_full[slot], dst, c * 64, s0, q.h, q.b, pol_k);
            if (TWO) tma_load_4d_hint(&tk, &bars->kv_full[slot], dst + CHUNK / 2, c * 64, s1, q.h, q.b, pol_k);  // B=64: second block; else one 128-row box
          }
          if (++slot == NS) { slot = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1 || warp == 3) {
    // one MMA issuer per q tile (warp 1: tile 0, warp 3: tile 1): a tile whose exp warps lag
    // does not hold back the other tile's QK^T; K slots and Q are released by both (count 2)
    if (lane == 0) {
      const int T = warp == 1 ? 0 : 1;
      constexpr uint32_t kIdesc = idesc_bf16(128, 128, false, false);
      const uint32_t sq_addr = smem_u32(sQ);
      const uint32_t sk_addr = smem_u32(sK);
      int slot = 0;
      uint32_t ph = 0, qph = 0;
      uint32_t seph[2][2] = {{0u, 0u}, {0u, 0u}};
      for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
        QTiles q;
        decode_search_item(p, TWO, item, q);
        mbar_wait(&bars->q_full, qph);
        qph ^= 1;
        tc_fence_after();
        for (int j = 0; j < ntiles; ++j) {
          mbar_wait(&bars->kv_full[slot], ph);
          tc_fence_after();
          const int buf = j & 1;
          for (int t = 0; t < 2; ++t) {
            if (t != T || !q.exists[t]) continue;
            mbar_wait(&bars->s_empty[t][buf], seph[t][buf] ^ 1);
            seph[t][buf] ^= 1;
            tc_fence_after();
#pragma unroll
            for (int kk = 0; kk < D / 16; ++kk) {
              const uint32_t off = (kk >> 2) * CHUNK + (kk & 3) * 32;
              mma_ss(tmem + t * 256 + buf * 128, desc_sw128(sq_addr + t * TILE + off, 16, 1024),
                     desc_sw128(sk_addr + slot * TILE + off, 16, 1024), kIdesc, kk > 0 ? 1u : 0u);
            }
            tc_commit(&bars->s_full[t][buf]);
          }
          tc_commit(&bars->kv_empty[slot]);
          if (++slot == NS) { slot = 0; ph ^= 1; }
        }
        tc_commit(&bars->q_empty);
      }
    }
  }
  } else {
    regs_inc<104>();
    // ============================================================ exp / block-sum warps
    // warps 4..19: sw = warp - 4, q tile t = sw >> 3, column half hc = (sw >> 2) & 1 (= kv half:
    // kv block kb0 / kb1 at B=64, the two halves of one block at B=128), TMEM lane quarter wq.
    // Two warps per row, each on its own 64 columns: 2 warps per SMSP per q tile, no exchange.
    const int sw = warp - 4;
    const int t = sw >> 3;
    const int hc = (sw >> 2) & 1;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const float2 sl2v = make_float2(p.scale_log2, p.scale_log2);
    uint32_t sfph[2] = {0u, 0u};
    const int nb = p.grid.nb;
    float* my_part = part + ((t * 2 + hc) * 4 + wq) * kChunk;   // this warp's [kChunk] partial masses
    const float* grp_part = part + t * 8 * kChunk;             // [hc][wq][kChunk] of this q tile
    for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
      QTiles q;
      decode_search_item(p, TWO, item, q);
      if (!q.exists[t]) continue;
      int tok;
      bool rvalid;
      if (!TWO || row < 64) {
        tok = q.start0[t] + row;
        rvalid = row < q.len0[t];
      } else {
        tok = q.start1[t] + row - 64;
        rvalid = (row - 64) < q.len1[t];
      }
      const float nl = rvalid ? -__ldg(p.lse + static_cast<int64_t>(q.bh) * p.N + tok) * kLog2e : 0.0f;
      const float2 nlv = make_float2(nl, nl);
      float* mout = p.mass + static_cast<int64_t>(q.bh) * nb * nb;
      for (int j0 = 0; j0 < ntiles; j0 += kChunk) {
        const int j1 = j0 + kChunk < ntiles ? j0 + kChunk : ntiles;
        for (int j = j0; j < j1; ++j) {
          const int buf = j & 1;
          int s0, l0, s1, l1, kb0, kb1;
          kv_tile(p, TWO, j, s0, l0, s1, l1, kb0, kb1);
          mbar_wait(&bars->s_full[t][buf], sfph[buf]);
          sfph[buf] ^= 1;
          tc_fence_after();
          uint32_t s[64];
          const uint32_t sa = tmem + lane_base + t * 256 + buf * 128 + hc * 64;
          tmem_ld32(sa + 0, s);
          tmem_ld32(sa + 32, s + 32);
          tmem_ld_wait32(s);
          reg_fence32(s + 32);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars->s_empty[t][buf]);
          // valid columns of my half (kv block kb0 / kb1 at B=64; the two halves of kb0 at B=128)
          const int lim = TWO ? (hc == 0 ? l0 : l1) : (hc == 0 ? (l0 < 64 ? l0 : 64) : l0 - 64);
          float mh;
          if (lim >= 64) mh = half_mass<true>(s, sl2v, nlv, 64);
          else mh = lim > 0 ? half_mass<false>(s, sl2v, nlv, lim) : 0.0f;
          if (!rvalid) mh = 0.0f;
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) mh += __shfl_xor_sync(0xffffffffu, mh, o);
          if (lane == 0) my_part[j - j0] = mh;
        }
        // flush the chunk: one fixed-order fp64 sum per (q-block, kv-block)
        named_bar_sync(1 + t, 256);
        for (int jj = sw * 32 + lane - t * 256; jj < j1 - j0; jj += 256) {
          const int j = j0 + jj;
          if (!TWO) {
            double m = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) m += (double)grp_part[w * kChunk + jj];
            mout[static_cast<int64_t>(q.qb0[t]) * nb + j] = static_cast<float>(m);
          } else {
#pragma unroll
            for (int qh = 0; qh < 2; ++qh) {
              const int qb = qh == 0 ? q.qb0[t] : q.qb1[t];
              if (qb < 0) continue;
#pragma unroll
              for (int hf = 0; hf < 2; ++hf) {
                const int kb = 2 * j + hf;
                if (kb >= nb) continue;
                const double m = (double)grp_part[(hf * 4 + 2 * qh) * kChunk + jj] +
                                 (double)grp_part[(hf * 4 + 2 * qh + 1) * kChunk + jj];
                mout[static_cast<int64_t>(qb) * nb + kb] = static_cast<float>(m);
              }
            }
          }
        }
        named_bar_sync(1 + t, 256);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int D, bool TWO>
cudaError_t launch_search_t(const CUtensorMap& tq, const CUtensorMap& tk, const SearchParams& p, int num_sms,
                            cudaStream_t st) {
  auto kern = search_kernel<D, TWO>;
  const int smem = SSmem<D>::kBytes;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int grid = p.num_items < num_sms ? p.num_items : num_sms;
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, kThreads, smem, st>>>(tq, tk, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_search(const CUtensorMap& tq, const CUtensorMap& tk, const SearchParams& p, int head_dim,
                          bool two, int num_sms, cudaStream_t st) {
  if (head_dim == 128) return two ? launch_search_t<128, true>(tq, tk, p, num_sms, st)
                                  : launch_search_t<128, false>(tq, tk, p, num_sms, st);
  return two ? launch_search_t<64, true>(tq, tk, p, num_sms, st) : launch_search_t<64, false>(tq, tk, p, num_sms, st);
}

}  // namespace adaspa
