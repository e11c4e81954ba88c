// api.cu -- the C ABI of include/adaspa.h: argument validation, TMA tensor maps, workspace
// layout and kernel launches.  No host synchronisation anywhere on this path.
#include <cuda.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>

#include "../../include/adaspa.h"
#include "attn.cuh"
#include "common.cuh"
#include "select.cuh"

#include <nvtx3/nvToolsExt.h>

using namespace adaspa;

namespace {

thread_local std::string g_last_error = "no error";

adaspa_status fail(adaspa_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return s;
}

adaspa_status cuda_fail(cudaError_t e, const char* where) {
  return fail(ADASPA_ERR_CUDA, "%s: %s", where, cudaGetErrorString(e));
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  return n;
}

BlockGrid make_grid(const adaspa_attn_desc* d) {
  BlockGrid g;
  g.n = d->seq_len;
  g.bs = d->block_size;
  const int n_video = d->seq_len - d->n_text;
  g.n_first = d->text_first ? d->n_text : n_video;
  g.nb_first = (g.n_first + g.bs - 1) / g.bs;
  g.nb = g.nb_first + (d->seq_len - g.n_first + g.bs - 1) / g.bs;
  return g;
}

adaspa_status check_desc(const adaspa_attn_desc* d) {
  if (!d) return fail(ADASPA_ERR_INVALID_ARG, "desc is NULL");
  if (d->batch < 1 || d->heads < 1 || d->seq_len < 1)
    return fail(ADASPA_ERR_INVALID_ARG, "batch, heads and seq_len must be >= 1 (got %d, %d, %d)", d->batch,
                d->heads, d->seq_len);
  if (d->head_dim != 64 && d->head_dim != 128)
    return fail(ADASPA_ERR_UNSUPPORTED, "head_dim %d unsupported (64 or 128)", d->head_dim);
  if (d->block_size != 64 && d->block_size != 128)
    return fail(ADASPA_ERR_UNSUPPORTED, "block_size %d unsupported (64 or 128)", d->block_size);
  if (d->n_text < 0 || d->n_text > d->seq_len)
    return fail(ADASPA_ERR_INVALID_ARG, "n_text %d outside [0, seq_len=%d]", d->n_text, d->seq_len);
  if (d->text_first != 0 && d->text_first != 1) return fail(ADASPA_ERR_INVALID_ARG, "text_first must be 0 or 1");
  if (!(d->softmax_scale == d->softmax_scale) || isinf(d->softmax_scale))
    return fail(ADASPA_ERR_INVALID_ARG, "softmax_scale is not finite");
  if (d->stride_n < 1 || d->stride_h < 1 || d->stride_b < 1)
    return fail(ADASPA_ERR_INVALID_ARG, "strides must be >= 1");
  if ((d->stride_n * 2) % 16 || (d->stride_h * 2) % 16 || (d->stride_b * 2) % 16)
    return fail(ADASPA_ERR_INVALID_ARG, "strides must be multiples of 8 elements (16 bytes)");
  if (d->stride_n < d->head_dim) return fail(ADASPA_ERR_INVALID_ARG, "stride_n < head_dim: rows overlap");
  return ADASPA_OK;
}

float scale_of(const adaspa_attn_desc* d) {
  return d->softmax_scale > 0.0f ? d->softmax_scale : 1.0f / sqrtf(static_cast<float>(d->head_dim));
}

adaspa_status check_ptr16(const void* p, const char* name) {
  if (!p) return fail(ADASPA_ERR_INVALID_ARG, "%s is NULL", name);
  if (reinterpret_cast<uintptr_t>(p) % 16) return fail(ADASPA_ERR_INVALID_ARG, "%s is not 16-byte aligned", name);
  return ADASPA_OK;
}

// Box = 64 columns (128 B, the swizzle span) x box_rows rows: 128-row boxes fetch a whole 128-row tile
// chunk with one TMA instruction (B = 128, dense); B = 64 tiles are two independent 64-row blocks.
adaspa_status make_map(CUtensorMap* map, const void* base, const adaspa_attn_desc* d, const char* name,
                       int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return fail(ADASPA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t dims[4] = {(cuuint64_t)d->head_dim, (cuuint64_t)d->seq_len, (cuuint64_t)d->heads,
                        (cuuint64_t)d->batch};
  cuuint64_t strides[3] = {(cuuint64_t)d->stride_n * 2, (cuuint64_t)d->stride_h * 2, (cuuint64_t)d->stride_b * 2};
  cuuint32_t box[4] = {64, (cuuint32_t)box_rows, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(ADASPA_ERR_INVALID_ARG, "cuTensorMapEncodeTiled(%s) failed: %d", name, (int)r);
  return ADASPA_OK;
}

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

// fused search workspace per (batch element, head): block LSEs [nb][N] + row LSEs [N], fp32
size_t fused_head_bytes(const adaspa_attn_desc* d) {
  return sizeof(float) * (static_cast<size_t>(make_grid(d).nb) + 1) * static_cast<size_t>(d->seq_len);
}

struct SelectWs {
  size_t bits, nnz, kept, total, kbh, loff, hcnt, hbase, hist, bytes;
};
SelectWs select_ws_layout(const adaspa_attn_desc* d) {
  const BlockGrid g = make_grid(d);
  const size_t rows = (size_t)d->batch * d->heads * g.nb;
  const size_t nwords = (g.nb + 31) / 32;
  SelectWs w;
  size_t off = 0;
  w.bits = off; off = align256(off + rows * nwords * 4);
  w.nnz = off; off = align256(off + rows * 4);
  w.kept = off; off = align256(off + rows * 8);
  w.total = off; off = align256(off + rows * 8);
  w.kbh = off; off = align256(off + (size_t)d->batch * d->heads * 4);
  w.loff = off; off = align256(off + rows * 4);
  w.hcnt = off; off = align256(off + (size_t)d->batch * d->heads * 4);
  w.hbase = off; off = align256(off + (size_t)d->batch * d->heads * 4);
  w.hist = off; off = align256(off + (size_t)(g.nb + 1) * 4);
  w.bytes = off;
  return w;
}

struct SparseWs {
  int items_per_bh, num_items, stride;
  size_t queue, len, order, stream, bytes;
};
SparseWs sparse_ws_layout(const adaspa_attn_desc* d) {
  const BlockGrid g = make_grid(d);
  const bool two = d->block_size == 64;
  SparseWs w;
  w.items_per_bh = two ? (g.nb + 3) / 4 : (g.nb + 1) / 2;
  w.num_items = d->batch * d->heads * w.items_per_bh;
  w.stride = two ? (g.nb + 1) / 2 : g.nb;
  size_t off = 0;
  w.queue = off; off = align256(off + 4);
  w.len = off; off = align256(off + (size_t)w.num_items * 4);
  w.order = off; off = align256(off + (size_t)w.num_items * 4);
  w.stream = off; off = align256(off + (size_t)w.num_items * w.stride * 8);
  w.bytes = off;
  return w;
}

}  // namespace

// An NVTX range around each compute entry of the C ABI (header-only NVTX3: a no-op unless a tool
// such as nsys or ncu --nvtx is attached), so profiles group the kernels of one call under its name.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

extern "C" {

int32_t adaspa_abi_version(void) { return ADASPA_ABI_VERSION; }

int32_t adaspa_num_blocks(const adaspa_attn_desc* desc) {
  if (check_desc(desc) != ADASPA_OK) return -1;
  return make_grid(desc).nb;
}

const char* adaspa_status_string(adaspa_status s) {
  switch (s) {
    case ADASPA_OK: return "ADASPA_OK";
    case ADASPA_ERR_INVALID_ARG: return "ADASPA_ERR_INVALID_ARG";
    case ADASPA_ERR_UNSUPPORTED: return "ADASPA_ERR_UNSUPPORTED";
    case ADASPA_ERR_CUDA: return "ADASPA_ERR_CUDA";
    case ADASPA_ERR_WORKSPACE_TOO_SMALL: return "ADASPA_ERR_WORKSPACE_TOO_SMALL";
  }
  return "ADASPA_ERR_UNKNOWN";
}

const char* adaspa_last_error(void) { return g_last_error.c_str(); }

adaspa_status adaspa_dense_attn_lse(const adaspa_attn_desc* desc, const void* q, const void* k, const void* v,
                                    void* o, float* lse, adaspa_stream_t stream) {
  NvtxRange nvtx_range("adaspa_dense_attn_lse");
  adaspa_status s;
  if ((s = check_desc(desc)) != ADASPA_OK) return s;
  if ((s = check_ptr16(q, "q")) || (s = check_ptr16(k, "k")) || (s = check_ptr16(v, "v")) ||
      (s = check_ptr16(o, "o")))
    return s;
  CUtensorMap tq, tk, tv;
  if ((s = make_map(&tq, q, desc, "q", 128)) || (s = make_map(&tk, k, desc, "k", 128)) ||
      (s = make_map(&tv, v, desc, "v", 128)))
    return s;
  AttnParams p{};
  p.B = desc->batch;
  p.H = desc->heads;
  p.N = desc->seq_len;
  p.grid = make_grid(desc);
  p.scale_log2 = scale_of(desc) * kLog2e;
  p.o = static_cast<__nv_bfloat16*>(o);
  p.sb = desc->stride_b;
  p.sh = desc->stride_h;
  p.sn = desc->stride_n;
  p.lse = lse;
  p.h0 = 0;
  p.nh = desc->heads;
  p.items_per_bh = (desc->seq_len + 255) / 256;
  p.num_items = desc->batch * desc->heads * p.items_per_bh;
  cudaError_t e = launch_attn(tq, tk, tv, p, desc->head_dim, false, kModeDense, num_sms(), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "dense_attn_lse launch");
  return ADASPA_OK;
}

size_t adaspa_fused_search_workspace_bytes(const adaspa_attn_desc* desc, int32_t heads_per_pass) {
  if (check_desc(desc) != ADASPA_OK) return 0;
  const int hp = (heads_per_pass <= 0 || heads_per_pass > desc->heads) ? desc->heads : heads_per_pass;
  return fused_head_bytes(desc) * static_cast<size_t>(desc->batch) * hp;
}

namespace {

// The passes of the fused search step over `ws` (>= one head of every batch element): per pass of hc
// heads, the dense pass with block LSEs, then the block-mass reduction (with the RECALL selection
// epilogue when sel != null and nb allows it).  Arguments validated by the caller.
adaspa_status fused_search_passes(const adaspa_attn_desc* desc, const void* q, const void* k, const void* v,
                                  void* o, float* lse, float* block_mass, const SelectRowsParams* sel, void* ws,
                                  size_t ws_bytes, cudaStream_t st) {
  adaspa_status s;
  const size_t per_head = fused_head_bytes(desc) * static_cast<size_t>(desc->batch);
  const int hc = static_cast<int>(ws_bytes / per_head < (size_t)desc->heads ? ws_bytes / per_head
                                                                              : (size_t)desc->heads);
  CUtensorMap tq, tk, tv;
  const int rows_kv = desc->block_size == 64 ? 64 : 128;
  if ((s = make_map(&tq, q, desc, "q", 128)) || (s = make_map(&tk, k, desc, "k", rows_kv)) ||
      (s = make_map(&tv, v, desc, "v", rows_kv)))
    return s;
  const BlockGrid g = make_grid(desc);
  for (int h0 = 0; h0 < desc->heads; h0 += hc) {
    const int nh = desc->heads - h0 < hc ? desc->heads - h0 : hc;
    float* blse = static_cast<float*>(ws);
    float* lrel = blse + static_cast<size_t>(desc->batch) * nh * g.nb * desc->seq_len;
    AttnParams p{};
    p.B = desc->batch;
    p.H = desc->heads;
    p.N = desc->seq_len;
    p.grid = g;
    p.scale_log2 = scale_of(desc) * kLog2e;
    p.o = static_cast<__nv_bfloat16*>(o);
    p.sb = desc->stride_b;
    p.sh = desc->stride_h;
    p.sn = desc->stride_n;
    p.lse = lse;
    p.h0 = h0;
    p.nh = nh;
    p.items_per_bh = (desc->seq_len + 255) / 256;
    p.num_items = desc->batch * nh * p.items_per_bh;
    p.blse = blse;
    p.lrel = lrel;
    cudaError_t e = launch_attn(tq, tk, tv, p, desc->head_dim, desc->block_size == 64, kModeBlse, num_sms(), st);
    if (e != cudaSuccess) return cuda_fail(e, "fused search launch (dense pass)");
    BlockMassParams m{};
    m.B = desc->batch;
    m.H = desc->heads;
    m.N = desc->seq_len;
    m.h0 = h0;
    m.nh = nh;
    m.grid = g;
    m.blse = blse;
    m.lrel = lrel;
    m.mass = block_mass;
    m.select = sel != nullptr && block_mass_select_kpl(g.nb) > 0;
    if (m.select) m.sel = *sel;
    if ((e = launch_block_mass(m, st)) != cudaSuccess) return cuda_fail(e, "fused search launch (block mass)");
  }
  return ADASPA_OK;
}

}  // namespace

adaspa_status adaspa_dense_attn_lse_search(const adaspa_attn_desc* desc, const void* q, const void* k, const void* v,
                                           void* o, float* lse, float* block_mass, void* workspace,
                                           size_t workspace_bytes, adaspa_stream_t stream) {
  NvtxRange nvtx_range("adaspa_dense_attn_lse_search");
  adaspa_status s;
  if ((s = check_desc(desc)) != ADASPA_OK) return s;
  if ((s = check_ptr16(q, "q")) || (s = check_ptr16(k, "k")) || (s = check_ptr16(v, "v")) ||
      (s = check_ptr16(o, "o")))
    return s;
  if (!block_mass) return fail(ADASPA_ERR_INVALID_ARG, "block_mass must not be NULL");
  if (reinterpret_cast<uintptr_t>(block_mass) % 4 || reinterpret_cast<uintptr_t>(lse) % 4)
    return fail(ADASPA_ERR_INVALID_ARG, "lse / block_mass misaligned");
  const size_t per_head = fused_head_bytes(desc) * static_cast<size_t>(desc->batch);
  if (!workspace || workspace_bytes < per_head)
    return fail(ADASPA_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes (one head of every batch element)",
                workspace_bytes, per_head);
  return fused_search_passes(desc, q, k, v, o, lse, block_mass, nullptr, workspace, workspace_bytes,
                             (cudaStream_t)stream);
}

adaspa_status adaspa_lse_cached_search(const adaspa_attn_desc* desc, const void* q, const void* k,
                                       const float* lse, float* block_mass, adaspa_stream_t stream) {
  NvtxRange nvtx_range("adaspa_lse_cached_search");
  adaspa_status s;
  if ((s = check_desc(desc)) != ADASPA_OK) return s;
  if ((s = check_ptr16(q, "q")) || (s = check_ptr16(k, "k"))) return s;
  if (!lse || !block_mass) return fail(ADASPA_ERR_INVALID_ARG, "lse and block_mass must not be NULL");
  if (reinterpret_cast<uintptr_t>(lse) % 4 || reinterpret_cast<uintptr_t>(block_mass) % 4)
    return fail(ADASPA_ERR_INVALID_ARG, "lse / block_mass misaligned");
  CUtensorMap tq, tk;
  const int rows_s = desc->block_size == 64 ? 64 : 128;
  if ((s = make_map(&tq, q, desc, "q", rows_s)) || (s = make_map(&tk, k, desc, "k", rows_s))) return s;
  SearchParams p{};
  p.B = desc->batch;
  p.H = desc->heads;
  p.N = desc->seq_len;
  p.grid = make_grid(desc);
  p.scale_log2 = scale_of(desc) * kLog2e;
  p.lse = lse;
  p.mass = block_mass;
  const bool two = desc->block_size == 64;
  p.items_per_bh = two ? (p.grid.nb + 3) / 4 : (p.grid.nb + 1) / 2;
  p.num_items = desc->batch * desc->heads * p.items_per_bh;
  p.kv_tiles = two ? (p.grid.nb + 1) / 2 : p.grid.nb;
  cudaError_t e = launch_search(tq, tk, p, desc->head_dim, two, num_sms(), (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "lse_cached_search launch");
  return ADASPA_OK;
}

size_t adaspa_select_workspace_bytes(const adaspa_attn_desc* desc) {
  if (check_desc(desc) != ADASPA_OK) return 0;
  return select_ws_layout(desc).bytes;
}

namespace {

// Validation of the selection arguments shared by adaspa_select_blocks and adaspa_search_select.
adaspa_status check_select(const adaspa_attn_desc* desc, adaspa_select_mode mode, const double* target,
                           uint32_t flags, double tier_tau, const int32_t* row_ptr, const int32_t* col_idx,
                           int64_t col_capacity) {
  if (!row_ptr || !col_idx || !target)
    return fail(ADASPA_ERR_INVALID_ARG, "target, row_ptr and col_idx must not be NULL");
  if (mode != ADASPA_SELECT_RECALL && mode != ADASPA_SELECT_SPARSITY)
    return fail(ADASPA_ERR_INVALID_ARG, "unknown selection mode %d", (int)mode);
  if (flags & ~3u) return fail(ADASPA_ERR_INVALID_ARG, "unknown flag bits 0x%x", flags);
  if (desc->heads > kMaxHeads) return fail(ADASPA_ERR_UNSUPPORTED, "heads > %d", kMaxHeads);
  const BlockGrid g = make_grid(desc);
  if (g.nb > kMaxSelectBlocks) return fail(ADASPA_ERR_UNSUPPORTED, "nb = %d > %d blocks", g.nb, kMaxSelectBlocks);
  const int64_t rows = (int64_t)desc->batch * desc->heads * g.nb;
  const int64_t need_cap = rows * g.nb;
  if (need_cap > INT32_MAX) return fail(ADASPA_ERR_UNSUPPORTED, "B*H*nb*nb exceeds int32 CSR indexing");
  if (col_capacity < need_cap)
    return fail(ADASPA_ERR_INVALID_ARG, "col_capacity %lld < B*H*nb*nb = %lld", (long long)col_capacity,
                (long long)need_cap);
  const bool tiers = (flags & ADASPA_FLAG_HEAD_TIERS) != 0;
  if (tiers && mode != ADASPA_SELECT_SPARSITY)
    return fail(ADASPA_ERR_INVALID_ARG, "ADASPA_FLAG_HEAD_TIERS applies to SPARSITY mode only");
  for (int h = 0; h < desc->heads; ++h) {
    const double t = target[h];
    if (!(t == t) || isinf(t)) return fail(ADASPA_ERR_INVALID_ARG, "target[%d] is not finite", h);
    if (mode == ADASPA_SELECT_SPARSITY && (t < 0.0 || t >= 1.0))
      return fail(ADASPA_ERR_INVALID_ARG, "sparsity target[%d] = %g outside [0,1)", h, t);
    if (tiers && t < 1.0 / 3.0)
      return fail(ADASPA_ERR_INVALID_ARG, "head tiers need sparsity >= 1/3 (target[%d] = %g)", h, t);
  }
  if (tiers && !(tier_tau == tier_tau)) return fail(ADASPA_ERR_INVALID_ARG, "tier_tau is NaN");
  return ADASPA_OK;
}

// Launch parameters of the selection over a K3 workspace `ws` (select_ws_layout).
void build_select(const adaspa_attn_desc* desc, const float* block_mass, adaspa_select_mode mode,
                  const double* target, uint32_t flags, double tier_tau, int32_t* row_ptr, int32_t* col_idx,
                  int32_t* row_order, float* head_recall, int64_t* head_nnz, uint8_t* ws, SelectLaunch& L) {
  const BlockGrid g = make_grid(desc);
  const SelectWs w = select_ws_layout(desc);
  const int64_t rows = (int64_t)desc->batch * desc->heads * g.nb;
  const bool sink = (flags & ADASPA_FLAG_TEXT_SINK) != 0;
  const int n_text_blocks = desc->text_first ? g.nb_first : g.nb - g.nb_first;
  const int ncand = sink ? g.nb - n_text_blocks : g.nb;
  L = SelectLaunch{};
  L.batch = desc->batch;
  L.tiers = (flags & ADASPA_FLAG_HEAD_TIERS) != 0;
  SelectRowsParams& rp = L.rows;
  rp.mass = block_mass;
  rp.rows = static_cast<int>(rows);
  rp.heads = desc->heads;
  rp.grid = g;
  rp.text_first = desc->text_first;
  rp.text_sink = sink ? 1 : 0;
  rp.mode = mode == ADASPA_SELECT_RECALL ? 0 : 1;
  for (int h = 0; h < desc->heads; ++h) {
    rp.target[h] = target[h];
    rp.k_head[h] = mode == ADASPA_SELECT_SPARSITY ? k_from_sparsity(target[h], ncand) : 0;
  }
  rp.k_per_bh = nullptr;
  rp.nwords = (g.nb + 31) / 32;
  rp.bits = reinterpret_cast<uint32_t*>(ws + w.bits);
  rp.row_nnz = reinterpret_cast<int*>(ws + w.nnz);
  rp.row_kept = reinterpret_cast<double*>(ws + w.kept);
  rp.row_total = reinterpret_cast<double*>(ws + w.total);
  SelectTierParams& tp = L.tier;
  tp.heads = desc->heads;
  tp.nb = g.nb;
  tp.ncand = ncand;
  tp.tau = tier_tau;
  for (int h = 0; h < desc->heads; ++h) tp.s_base[h] = target[h];
  tp.row_kept = rp.row_kept;
  tp.row_total = rp.row_total;
  tp.k_per_bh = reinterpret_cast<int*>(ws + w.kbh);
  SelectFinalParams& fp = L.fin;
  fp.rows = rp.rows;
  fp.nb = g.nb;
  fp.bh = desc->batch * desc->heads;
  fp.row_nnz = rp.row_nnz;
  fp.row_kept = rp.row_kept;
  fp.row_total = rp.row_total;
  fp.local_off = reinterpret_cast<int*>(ws + w.loff);
  fp.head_cnt = reinterpret_cast<int*>(ws + w.hcnt);
  fp.head_base = reinterpret_cast<int*>(ws + w.hbase);
  fp.hist = reinterpret_cast<int*>(ws + w.hist);
  fp.row_ptr = row_ptr;
  fp.row_order = row_order;
  fp.head_recall = head_recall;
  fp.head_nnz = head_nnz;
  SelectWriteParams& wp = L.wr;
  wp.rows = rp.rows;
  wp.nwords = rp.nwords;
  wp.nb = g.nb;
  wp.bits = rp.bits;
  wp.row_nnz = rp.row_nnz;
  wp.local_off = fp.local_off;
  wp.head_base = fp.head_base;
  wp.hist = fp.hist;
  wp.row_ptr = row_ptr;
  wp.row_order = row_order;
  wp.col_idx = col_idx;
}

}  // namespace

adaspa_status adaspa_select_blocks(const adaspa_attn_desc* desc, const float* block_mass, adaspa_select_mode mode,
                                   const double* target, uint32_t flags, double tier_tau, int32_t* row_ptr,
                                   int32_t* col_idx, int64_t col_capacity, int32_t* row_order, float* head_recall,
                                   int64_t* head_nnz, void* workspace, size_t workspace_bytes,
                                   adaspa_stream_t stream) {
  NvtxRange nvtx_range("adaspa_select_blocks");
  adaspa_status s;
  if ((s = check_desc(desc)) != ADASPA_OK) return s;
  if (!block_mass) return fail(ADASPA_ERR_INVALID_ARG, "block_mass must not be NULL");
  if ((s = check_select(desc, mode, target, flags, tier_tau, row_ptr, col_idx, col_capacity)) != ADASPA_OK) return s;
  const SelectWs w = select_ws_layout(desc);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ADASPA_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes", workspace_bytes, w.bytes);
  SelectLaunch L;
  build_select(desc, block_mass, mode, target, flags, tier_tau, row_ptr, col_idx, row_order, head_recall, head_nnz,
               static_cast<uint8_t*>(workspace), L);
  cudaError_t e = launch_select(L, (cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_fail(e, "select_blocks launch");
  return ADASPA_OK;
}

size_t adaspa_search_select_workspace_bytes(const adaspa_attn_desc* desc, int32_t heads_per_pass) {
  if (check_desc(desc) != ADASPA_OK) return 0;
  const int hp = (heads_per_pass <= 0 || heads_per_pass > desc->heads) ? desc->heads : heads_per_pass;
  return align256(select_ws_layout(desc).bytes) + fused_head_bytes(desc) * static_cast<size_t>(desc->batch) * hp;
}

adaspa_status adaspa_search_select(const adaspa_attn_desc* desc, const void* q, const void* k, const void* v, void* o,
                                   float* lse, float* block_mass, const double* recall, uint32_t flags,
                                   int32_t* row_ptr, int32_t* col_idx, int64_t col_capacity, int32_t* row_order,
                                   float* head_recall, int64_t* head_nnz, void* workspace, size_t workspace_bytes,
                                   adaspa_stream_t stream) {
  NvtxRange nvtx_range("adaspa_search_select");
  adaspa_status s;
  if ((s = check_desc(desc)) != ADASPA_OK) return s;
  if ((s = check_ptr16(q, "q")) || (s = check_ptr16(k, "k")) || (s = check_ptr16(v, "v")) ||
      (s = check_ptr16(o, "o")))
    return s;
  if (flags & ADASPA_FLAG_HEAD_TIERS)
    return fail(ADASPA_ERR_INVALID_ARG, "adaspa_search_select is RECALL mode: ADASPA_FLAG_HEAD_TIERS not allowed");
  if ((s = check_select(desc, ADASPA_SELECT_RECALL, recall, flags, 0.0, row_ptr, col_idx, col_capacity)) != ADASPA_OK)
    return s;
  const BlockGrid g = make_grid(desc);
  const bool fused_select = block_mass_select_kpl(g.nb) > 0;
  if (!block_mass && !fused_select)
    return fail(ADASPA_ERR_INVALID_ARG, "block_mass may be NULL only for nb <= 2048 (nb = %d)", g.nb);
  if (reinterpret_cast<uintptr_t>(block_mass) % 4 || reinterpret_cast<uintptr_t>(lse) % 4)
    return fail(ADASPA_ERR_INVALID_ARG, "lse / block_mass misaligned");
  const size_t sel_bytes = align256(select_ws_layout(desc).bytes);
  const size_t per_head = fused_head_bytes(desc) * static_cast<size_t>(desc->batch);
  if (!workspace || workspace_bytes < sel_bytes + per_head)
    return fail(ADASPA_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes (selection + one head of every batch element)",
                workspace_bytes, sel_bytes + per_head);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  SelectLaunch L;
  build_select(desc, block_mass, ADASPA_SELECT_RECALL, recall, flags, 0.0, row_ptr, col_idx, row_order, head_recall,
               head_nnz, ws, L);
  cudaStream_t st = (cudaStream_t)stream;
  if ((s = fused_search_passes(desc, q, k, v, o, lse, block_mass, &L.rows, ws + sel_bytes, workspace_bytes - sel_bytes,
                               st)) != ADASPA_OK)
    return s;
  cudaError_t e;
  if (!fused_select && (e = launch_select_rows(L.rows, st)) != cudaSuccess) return cuda_fail(e, "search_select launch (rows)");
  if ((e = launch_select_final(L, st)) != cudaSuccess) return cuda_fail(e, "search_select launch (CSR)");
  return ADASPA_OK;
}

size_t adaspa_sparse_workspace_bytes(const adaspa_attn_desc* desc) {
  if (check_desc(desc) != ADASPA_OK) return 0;
  return sparse_ws_layout(desc).bytes;
}

adaspa_status adaspa_block_sparse_attn(const adaspa_attn_desc* desc, const void* q, const void* k, const void* v,
                                       const int32_t* row_ptr, const int32_t* col_idx, void* o, float* lse,
                                       void* workspace, size_t workspace_bytes, adaspa_stream_t stream) {
  NvtxRange nvtx_range("adaspa_block_sparse_attn");
  adaspa_status s;
  if ((s = check_desc(desc)) != ADASPA_OK) return s;
  if ((s = check_ptr16(q, "q")) || (s = check_ptr16(k, "k")) || (s = check_ptr16(v, "v")) ||
      (s = check_ptr16(o, "o")))
    return s;
  if (!row_ptr || !col_idx) return fail(ADASPA_ERR_INVALID_ARG, "row_ptr / col_idx must not be NULL");
  const BlockGrid g = make_grid(desc);
  if (g.nb > kMaxSparseBlocks) return fail(ADASPA_ERR_UNSUPPORTED, "nb = %d > %d blocks", g.nb, kMaxSparseBlocks);
  const SparseWs w = sparse_ws_layout(desc);
  if (!workspace || workspace_bytes < w.bytes)
    return fail(ADASPA_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu bytes", workspace_bytes, w.bytes);
  CUtensorMap tq, tk, tv;
  const int rows_s = desc->block_size == 64 ? 64 : 128;
  if ((s = make_map(&tq, q, desc, "q", rows_s)) || (s = make_map(&tk, k, desc, "k", rows_s)) ||
      (s = make_map(&tv, v, desc, "v", rows_s)))
    return s;
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const bool two = desc->block_size == 64;
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(ws + w.queue, 0, 4, st);
  if (e != cudaSuccess) return cuda_fail(e, "block_sparse_attn memset");
  SparsePrepParams pp{};
  pp.B = desc->batch;
  pp.H = desc->heads;
  pp.grid = g;
  pp.two = two ? 1 : 0;
  pp.items_per_bh = w.items_per_bh;
  pp.num_items = w.num_items;
  pp.row_ptr = row_ptr;
  pp.col_idx = col_idx;
  pp.stream = reinterpret_cast<uint64_t*>(ws + w.stream);
  pp.stream_len = reinterpret_cast<int*>(ws + w.len);
  pp.item_order = reinterpret_cast<int*>(ws + w.order);
  pp.stream_stride = w.stride;
  if ((e = launch_sparse_prep(pp, st)) != cudaSuccess) return cuda_fail(e, "block_sparse_attn prep");
  AttnParams p{};
  p.B = desc->batch;
  p.H = desc->heads;
  p.N = desc->seq_len;
  p.grid = g;
  p.scale_log2 = scale_of(desc) * kLog2e;
  p.o = static_cast<__nv_bfloat16*>(o);
  p.sb = desc->stride_b;
  p.sh = desc->stride_h;
  p.sn = desc->stride_n;
  p.lse = lse;
  p.h0 = 0;
  p.nh = desc->heads;
  p.items_per_bh = w.items_per_bh;
  p.num_items = w.num_items;
  p.item_order = pp.item_order;
  p.stream = pp.stream;
  p.stream_len = pp.stream_len;
  p.stream_stride = w.stride;
  p.queue = reinterpret_cast<int*>(ws + w.queue);
  e = launch_attn(tq, tk, tv, p, desc->head_dim, two, kModeSparse, num_sms(), st);
  if (e != cudaSuccess) return cuda_fail(e, "block_sparse_attn launch");
  return ADASPA_OK;
}

}  // extern "C"
