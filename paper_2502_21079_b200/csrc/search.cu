// search.cu -- K2: LSE-cached online search (Alg. 2; Alg. 1 second pass,
// PAPER.md:484-493):  block_mass[b,h,p,j] = sum_{i in p, t in j} exp(scale*q_i.k_t - lse_i)
// (W_sum_attn; reading R4: "Log(qk - LSE)" is exp(qk*scale - LSE)).
//
// Same skeleton as attn_fwd.cu without the PV product: persistent CTAs, a work item is two
// 128-row q tiles of one head (q-blocks 2p,2p+1 at B=128; 4p..4p+3 at B=64), the kv stream is
// every kv tile of the head (one block at B=128, two at B=64).  S tiles are double-buffered
// per q tile in TMEM (4 x 128 columns), so the tensor core runs ahead of the exp work.
// Softmax-role threads own one row: x = fma(S, scale*log2e, -lse*log2e), p = 2^x, a pairwise
// (tree) fp32 sum per kv block, then an fp64 cross-row reduction (warp shuffle + shared
// memory) gives one fp32 mass per (q-block, kv-block).  S is never written to memory.
#include "attn.cuh"
#include "common.cuh"

namespace adaspa {

namespace {

constexpr int kThreads = 384;

template <int D>
struct SSmem {
  static constexpr int kTile = 128 * D * 2;
  static constexpr int kNS = (D == 128) ? 5 : 11;
  static constexpr int kQ = 0;
  static constexpr int kK = 2 * kTile;
  static constexpr int kBar = kK + kNS * kTile;
  static constexpr int kBytes = kBar + 2048 + 1024;
};

struct SBars {
  uint64_t kv_full[12], kv_empty[12];
  uint64_t q_full, q_empty;
  uint64_t s_full[2][2], s_empty[2][2];
  double red[2][2][4][2];   // [tile][buf][warp quarter][kv half]
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

// Pairwise sum of 2^x over 64 consecutive columns held in s[0..63] (fp32 bits); columns
// at or beyond `lim` are excluded.
template <bool FULL>
__device__ __forceinline__ float half_mass(const uint32_t* s, float sl2, float nl, int lim) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    float a = ex2_approx(fmaf(__uint_as_float(s[2 * i]), sl2, nl));
    float b = ex2_approx(fmaf(__uint_as_float(s[2 * i + 1]), sl2, nl));
    if (!FULL) {
      a = (2 * i < lim) ? a : 0.0f;
      b = (2 * i + 1 < lim) ? b : 0.0f;
    }
    v[i] = a + b;
  }
#pragma unroll
  for (int w = 16; w >= 1; w >>= 1) {
#pragma unroll
    for (int i = 0; i < w; ++i) v[i] += v[i + w];
  }
  return v[0];
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
  SBars* bars = reinterpret_cast<SBars*>(smem + S::kBar);
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&bars->kv_full[i], 1);
      mbar_init(&bars->kv_empty[i], 1);
    }
    mbar_init(&bars->q_full, 1);
    mbar_init(&bars->q_empty, 1);
    for (int t = 0; t < 2; ++t)
      for (int b = 0; b < 2; ++b) {
        mbar_init(&bars->s_full[t][b], 1);
        mbar_init(&bars->s_empty[t][b], 4);
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
            tma_load_4d_hint(&tq, &bars->q_full, dst + CHUNK / 2, c * 64, r1, q.h, q.b, pol_q);
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
            tma_load_4d_hint(&tk, &bars->kv_full[slot], dst + CHUNK / 2, c * 64, s1, q.h, q.b, pol_k);
          }
          if (++slot == NS) { slot = 0; ph ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
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
            if (!q.exists[t]) continue;
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
  } else if (warp >= 4) {
    const int t = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const int hq = wq >> 1;
    const uint32_t lane_base = static_cast<uint32_t>(wq * 32) << 16;
    const float sl2 = p.scale_log2;
    uint32_t sfph[2] = {0u, 0u};
    const int nb = p.grid.nb;
    for (int item = blockIdx.x; item < p.num_items; item += gridDim.x) {
      QTiles q;
      decode_search_item(p, TWO, item, q);
      if (!q.exists[t]) continue;
      int tok;
      bool rvalid;
      int my_qb;
      if (!TWO) {
        tok = q.start0[t] + row;
        rvalid = row < q.len0[t];
        my_qb = q.qb0[t];
      } else if (row < 64) {
        tok = q.start0[t] + row;
        rvalid = row < q.len0[t];
        my_qb = q.qb0[t];
      } else {
        tok = q.start1[t] + row - 64;
        rvalid = (row - 64) < q.len1[t];
        my_qb = q.qb1[t];
      }
      const float nl = rvalid ? -__ldg(p.lse + static_cast<int64_t>(q.bh) * p.N + tok) * kLog2e : 0.0f;
      float* mout = p.mass + static_cast<int64_t>(q.bh) * nb * nb;
      for (int j = 0; j < ntiles; ++j) {
        const int buf = j & 1;
        int s0, l0, s1, l1, kb0, kb1;
        kv_tile(p, TWO, j, s0, l0, s1, l1, kb0, kb1);
        mbar_wait(&bars->s_full[t][buf], sfph[buf]);
        sfph[buf] ^= 1;
        tc_fence_after();
        uint32_t s[128];
        const uint32_t sa = tmem + lane_base + t * 256 + buf * 128;
        tmem_ld32(sa + 0, s);
        tmem_ld32(sa + 32, s + 32);
        tmem_ld32(sa + 64, s + 64);
        tmem_ld32(sa + 96, s + 96);
        tmem_ld_wait32(s);
        reg_fence32(s + 32);
        reg_fence32(s + 64);
        reg_fence32(s + 96);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->s_empty[t][buf]);
        // column limits of the two 64-column halves
        int lim_a, lim_b;
        if (!TWO) {
          lim_a = l0 < 64 ? l0 : 64;
          lim_b = l0 - 64;
        } else {
          lim_a = l0;
          lim_b = l1;
        }
        float ma = (lim_a >= 64) ? half_mass<true>(s, sl2, nl, 64) : half_mass<false>(s, sl2, nl, lim_a);
        float mb = (lim_b >= 64) ? half_mass<true>(s + 64, sl2, nl, 64)
                                 : (lim_b > 0 ? half_mass<false>(s + 64, sl2, nl, lim_b) : 0.0f);
        if (!rvalid) {
          ma = 0.0f;
          mb = 0.0f;
        }
        double da = ma, db = mb;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          da += __shfl_xor_sync(0xffffffffu, da, o);
          db += __shfl_xor_sync(0xffffffffu, db, o);
        }
        if (lane == 0) {
          bars->red[t][buf][wq][0] = da;
          bars->red[t][buf][wq][1] = db;
        }
        named_bar_sync(1 + t, 128);
        if (wq == 0 && lane < 4) {
          const double(*r)[2] = bars->red[t][buf];
          if (!TWO) {
            if (lane == 0) {
              const double m = ((r[0][0] + r[0][1]) + (r[1][0] + r[1][1])) + ((r[2][0] + r[2][1]) + (r[3][0] + r[3][1]));
              mout[static_cast<int64_t>(my_qb) * nb + kb0] = static_cast<float>(m);
            }
          } else {
            const int qh = lane >> 1, hf = lane & 1;
            const int qb = qh == 0 ? q.qb0[t] : q.qb1[t];
            const int kb = hf == 0 ? kb0 : kb1;
            if (qb >= 0 && kb >= 0)
              mout[static_cast<int64_t>(qb) * nb + kb] = static_cast<float>(r[2 * qh][hf] + r[2 * qh + 1][hf]);
          }
        }
      }
      (void)my_qb;
      (void)hq;
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
