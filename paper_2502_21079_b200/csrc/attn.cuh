// attn.cuh -- parameter blocks for the attention kernels (attn_fwd.cu: K1/K4, search.cu: K2).
#pragma once
#include <stdint.h>

#include "common.cuh"
#include "select.cuh"

namespace adaspa {

// A stream entry of the block-sparse kernel: one 128-row kv tile made of one B=128 block
// (id0) or two B=64 blocks (id0, id1; 16 bits each), plus an 8-bit membership mask in bits 32-39.
// Mask bit (4*t + 2*hq + hf) says that the 64-row half hq of q-tile t needs kv half hf.
__host__ __device__ __forceinline__ uint64_t stream_entry(int id0, int id1, uint32_t mask) {
  return static_cast<uint64_t>(id0) | (static_cast<uint64_t>(id1) << 16) | (static_cast<uint64_t>(mask) << 32);
}
__host__ __device__ __forceinline__ int entry_id0(uint64_t e) { return static_cast<int>(e & 0xFFFFu); }
__host__ __device__ __forceinline__ int entry_id1(uint64_t e) { return static_cast<int>((e >> 16) & 0xFFFFu); }
__host__ __device__ __forceinline__ uint32_t entry_mask(uint64_t e) { return static_cast<uint32_t>(e >> 32); }
constexpr int kMaxSparseBlocks = 65535;

enum : int { kModeDense = 0, kModeBlse = 1, kModeSparse = 2 };

struct AttnParams {
  int B, H, N;
  int h0, nh;                // heads [h0, h0 + nh) of the H in the tensors (items cover B * nh heads)
  BlockGrid grid;
  float scale_log2;          // softmax_scale * log2(e)
  __nv_bfloat16* o;          // output, same strides as Q/K/V
  int64_t sb, sh, sn;        // element strides
  float* lse;                // [B,H,N] or null
  int num_items;             // work items (pairs of 128-row q tiles)
  int items_per_bh;
  // block-sparse only
  const int* item_order;     // [num_items]: processing order (head-major, longest first in a head)
  const uint64_t* stream;    // [num_items, stream_stride]
  const int* stream_len;     // [num_items]
  int stream_stride;
  int* queue;                // atomic work counter
  // kModeBlse only (fused search at t_w): per (row, kv block) log-sum-exps and per-row LSEs, both in
  // log2 units relative to the row's first running max ref_i (small magnitudes keep them exact):
  //   blse[((b*nh + h-h0)*nb + kb)*N + i] = log2 sum_{j in kb} 2^(s_ij*scale*log2e) - ref_i
  //   lrel[(b*nh + h-h0)*N + i]           = log2 sum_j     2^(s_ij*scale*log2e) - ref_i
  float* blse;
  float* lrel;
};

// Fused search, second half: block_mass[b,h,qb,kb] = sum_{i in qb} 2^(blse[.., kb, i] - lrel[.., i])
struct BlockMassParams {
  int B, H, N;
  int h0, nh;
  BlockGrid grid;
  const float* blse;
  const float* lrel;
  float* mass;               // [B, H, nb, nb], or null (not written: the selection epilogue consumes the row)
  // RECALL selection epilogue (f1): with select != 0, warp 0 of each CTA selects its q-block row from the
  // shared-memory mass row (select_row.cuh, the same routine as K3's select_rows_kernel) into the K3
  // workspace arrays of `sel` (row = (b*H + h)*nb + qb); `sel.mass` is unused.
  int select;
  SelectRowsParams sel;
};

struct SparsePrepParams {
  int B, H;
  BlockGrid grid;
  int two;                   // block 64 (two blocks per 128-row tile)
  int items_per_bh, num_items;
  const int32_t* row_ptr;
  const int32_t* col_idx;
  uint64_t* stream;
  int* stream_len;
  int* item_order;
  int stream_stride;
};

struct SearchParams {
  int B, H, N;
  BlockGrid grid;
  float scale_log2;
  const float* lse;          // [B,H,N]
  float* mass;               // [B,H,nb,nb]
  int num_items;
  int items_per_bh;
  int kv_tiles;              // kv tiles per head
};

cudaError_t launch_attn(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                        const AttnParams& p, int head_dim, bool two, int mode, int num_sms,
                        cudaStream_t st);
cudaError_t launch_block_mass(const BlockMassParams& p, cudaStream_t st);
// rows per lane of the fused selection epilogue: 0 (nb too large: run K3's select_rows after the passes)
int block_mass_select_kpl(int nb);
cudaError_t launch_sparse_prep(const SparsePrepParams& p, cudaStream_t st);
cudaError_t launch_search(const CUtensorMap& tq, const CUtensorMap& tk, const SearchParams& p, int head_dim,
                          bool two, int num_sms, cudaStream_t st);

}  // namespace adaspa
