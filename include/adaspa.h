/*
 * adaspa.h -- C ABI of the B200-native AdaSpa hot path (arXiv 2502.21079).
 *
 * Four entry points, one per step of the data-parallel hot path
 * (BASELINE.json north_star):
 *
 *   adaspa_dense_attn_lse     K1  dense attention forward + per-row LSE
 *   adaspa_lse_cached_search  K2  block attention mass  sum exp(S - LSE)
 *   adaspa_select_blocks      K3  head-adaptive hierarchical selection -> CSR
 *   adaspa_block_sparse_attn  K4  block-sparse attention forward on the CSR
 *
 * plus the fused search step t_w, K1 and K2 with the
 * fresh LSE in one dense pass:
 *
 *   adaspa_dense_attn_lse_search  K1+K2  dense forward + LSE + block mass
 *
 * and the whole RECALL-mode search step t_w (f1 with its fused selection epilogue):
 *
 *   adaspa_search_select      K1+K2+K3  dense forward + LSE + block mass + CSR
 *
 * Conventions (all functions):
 *  - Plain pointers only.  Every tensor argument is a DEVICE pointer owned by
 *    the caller unless its comment says "host".  The library allocates no
 *    persistent device memory; scratch comes from a caller workspace whose size
 *    is given by the matching *_workspace_bytes() query.
 *  - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *    default stream) and never synchronises the host.
 *  - Argument errors (shape, stride, alignment, null pointer, target range,
 *    capacity, unsupported head_dim / block_size) return
 *    ADASPA_ERR_INVALID_ARG or ADASPA_ERR_UNSUPPORTED and launch nothing;
 *    adaspa_last_error() then holds a thread-local message.  A CUDA launch
 *    failure returns ADASPA_ERR_CUDA.
 *  - Data-dependent conditions are handled in-band (no host sync): K3 always
 *    keeps >= 1 block per row; K4 writes O = 0 and LSE' = -inf for a row with
 *    no kept block.
 *
 *  - No environment variable changes what the product library computes.
 *
 * Numbers: Q, K, V, O are bf16; accumulation, softmax, LSE and block mass are
 * fp32 (the block-mass cross-row reduction and every selection prefix sum are
 * fp64).  LSE is the natural-log log-sum-exp of the SCALED logits
 * softmax_scale * q.k, i.e. what Alg. 1 line 11 caches
 * (PAPER.md:481).
 */
#ifndef ADASPA_H_
#define ADASPA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADASPA_ABI_VERSION 1

/* Same object as cudaStream_t / CUstream; declared here so this header needs
 * no CUDA include. */
typedef struct CUstream_st* adaspa_stream_t;

typedef enum {
  ADASPA_OK = 0,
  ADASPA_ERR_INVALID_ARG = 1,
  ADASPA_ERR_UNSUPPORTED = 2,
  ADASPA_ERR_CUDA = 3,
  ADASPA_ERR_WORKSPACE_TOO_SMALL = 4
} adaspa_status;

typedef enum {
  ADASPA_SELECT_RECALL = 0,   /* per-head recall target r_h (north_star)        */
  ADASPA_SELECT_SPARSITY = 1  /* per-head sparsity s_h, row-wise top-k (S*)      */
} adaspa_select_mode;

enum {
  ADASPA_FLAG_TEXT_SINK = 1u,  /* always keep vt, tv, tt parts      */
  ADASPA_FLAG_HEAD_TIERS = 2u  /* hierarchical head tiers       */
};

/*
 * Problem description, following the paper's problem statement:
 *   Q, K, V in R^{H x L x D}, here with a batch dimension;
 *   L = f*h*w + t  (eq:seqlen): seq_len = n_video + n_text;
 *   block size B;
 *   the text/video split drives the modality-aware block grid: each modality
 *   segment is cut into blocks of `block_size` on its own, so no block straddles
 *   the boundary and each segment's last block may be partial.  Block ids run in
 *   sequence order; nb = ceil(n_video/B) + ceil(n_text/B).
 *
 * Q, K, V and O share one layout: element (b, h, n, c) lives at
 *   base + b*stride_b + h*stride_h + n*stride_n + c      (in bf16 elements),
 * so both head-major [B,H,N,d] and token-major [B,N,H,d] (Ulysses) work.
 * Requirements: stride_d == 1 (implicit), stride_n*2, stride_h*2, stride_b*2 and
 * every base pointer multiples of 16 bytes.
 * LSE tensors are dense fp32 [B,H,N]; block_mass is dense fp32 [B,H,nb,nb].
 */
typedef struct {
  int32_t batch;        /* B  >= 1                                              */
  int32_t heads;        /* H  >= 1 (a head shard on multi-GPU)                  */
  int32_t seq_len;      /* N  >= 1                                              */
  int32_t head_dim;     /* d  in {64, 128}                                      */
  int32_t block_size;   /* 64 or 128 (paper default 64)           */
  int32_t n_text;       /* text tokens, 0 <= n_text <= N                        */
  int32_t text_first;   /* 0: [video|text] (HunyuanVideo), 1: [text|video]      */
  float softmax_scale;  /* <= 0 selects 1/sqrt(head_dim)         */
  int64_t stride_b, stride_h, stride_n;  /* in elements; see above              */
} adaspa_attn_desc;

/* ABI version compiled into the library (== ADASPA_ABI_VERSION). */
int32_t adaspa_abi_version(void);

/* nb = ceil(n_video/B) + ceil(n_text/B), or -1 if the descriptor is invalid. */
int32_t adaspa_num_blocks(const adaspa_attn_desc* desc);

/*
 * K1 -- dense attention forward with LSE (Alg. 1 first pass, PAPER.md:471-482;
 * online softmax of PAPER.md:194-202, readings R1-R3 of DESIGN.md):
 *   S = scale * Q K^T,  lse_i = log sum_j exp(S_ij),  O_i = sum_j exp(S_ij - lse_i) V_j.
 * q, k, v: bf16 (layout above).  o: bf16 output, same layout.
 * lse: fp32 [B,H,N] output, may be NULL (warm-up steps do not need it).
 */
adaspa_status adaspa_dense_attn_lse(const adaspa_attn_desc* desc, const void* q, const void* k,
                                    const void* v, void* o, float* lse, adaspa_stream_t stream);

/*
 * K1+K2 fused -- the search step t_w (Alg. 1 whole; W_sum_attn,
 * PAPER.md:428-434, reading R4), with the outputs of K1 followed by K2 on the
 * fresh LSE:
 *   o, lse      as adaspa_dense_attn_lse (lse may be NULL),
 *   block_mass  fp32 [B,H,nb,nb]: sum_{i in p} sum_{t in j} exp(scale*q_i.k_t - lse_i).
 * Algorithm: ONE dense pass over the kv blocks of the grid; besides O and the
 * row LSE it writes every per-(row, kv block) log-sum-exp
 *   log2 sum_{t in j} 2^(scale*log2e*q_i.k_t)  (relative to a per-row reference)
 * to the workspace, from the exponentials the pass computes anyway; a second,
 * HBM-bound kernel forms block_mass = sum_i 2^(blockLSE_ij - LSE_i).  Exact up
 * to rounding (no second QK^T, no second pass of exponentials over S).  Alg. 2
 * (later key steps, cached LSE) stays adaspa_lse_cached_search.
 * workspace: device scratch of >= adaspa_fused_search_workspace_bytes(desc, 1)
 * bytes (4*(nb+1)*N bytes per head and batch element: 0.39 GB per head at
 * HunyuanVideo-110K); heads are processed in passes of as many heads as fit
 * (a workspace of adaspa_fused_search_workspace_bytes(desc, 0) runs all heads
 * in one pass).  Too small: ADASPA_ERR_WORKSPACE_TOO_SMALL, nothing launched.
 */
adaspa_status adaspa_dense_attn_lse_search(const adaspa_attn_desc* desc, const void* q, const void* k,
                                           const void* v, void* o, float* lse, float* block_mass,
                                           void* workspace, size_t workspace_bytes, adaspa_stream_t stream);

/* Workspace bytes of adaspa_dense_attn_lse_search for passes of `heads_per_pass`
 * heads (<= 0 or > H: all heads in one pass). */
size_t adaspa_fused_search_workspace_bytes(const adaspa_attn_desc* desc, int32_t heads_per_pass);

/*
 * K1+K2+K3 fused -- the whole search step t_w in RECALL mode (Alg. 1, PAPER.md:459-497,
 * with the selection of PAPER.md:228-232 per q-block row; the fused RECALL epilogue of
 * SURVEY.md 8(f) f1): the dense pass of adaspa_dense_attn_lse_search, then per q-block
 * row the block masses with the fresh LSE AND that row's selection in the same CTA (the
 * mass row is selected from shared memory; it is not re-read from HBM), then the CSR.
 *   o, lse      as adaspa_dense_attn_lse (lse may be NULL);
 *   block_mass  fp32 [B,H,nb,nb] output, or NULL (not written) when nb <= 2048; for
 *               nb > 2048 it is required (the selection then runs as K3's row kernel on it);
 *   recall      HOST double[H]: r_h, as adaspa_select_blocks in ADASPA_SELECT_RECALL mode;
 *   flags       ADASPA_FLAG_TEXT_SINK or 0 (head tiers are a SPARSITY-mode rule: rejected);
 *   row_ptr, col_idx, col_capacity, row_order, head_recall, head_nnz: as
 *               adaspa_select_blocks -- bit-identical to adaspa_select_blocks on block_mass.
 * workspace: >= adaspa_search_select_workspace_bytes(desc, 1) bytes (the K3 workspace
 * followed by the fused-search scratch; heads are processed in passes as in
 * adaspa_dense_attn_lse_search).  Argument errors as adaspa_dense_attn_lse_search and
 * adaspa_select_blocks; nothing is launched on an error.
 */
adaspa_status adaspa_search_select(const adaspa_attn_desc* desc, const void* q, const void* k, const void* v,
                                   void* o, float* lse, float* block_mass, const double* recall, uint32_t flags,
                                   int32_t* row_ptr, int32_t* col_idx, int64_t col_capacity, int32_t* row_order,
                                   float* head_recall, int64_t* head_nnz, void* workspace,
                                   size_t workspace_bytes, adaspa_stream_t stream);

/* Workspace bytes of adaspa_search_select for passes of `heads_per_pass` heads
 * (<= 0 or > H: all heads in one pass). */
size_t adaspa_search_select_workspace_bytes(const adaspa_attn_desc* desc, int32_t heads_per_pass);

/*
 * K2 -- LSE-cached online search (Alg. 2; Alg. 1 second
 * pass; W_sum_attn; reading R4):
 *   block_mass[b,h,p,j] = sum_{i in block p} sum_{t in block j} exp(scale * q_i.k_t - lse_i).
 * With lse = the exact LSE of the same (Q,K) (from K1 at step t_w) every row of
 * block_mass sums to the q-block's token count; at later key steps lse is the
 * cached t_w LSE.  q, k: bf16; lse: fp32 [B,H,N] (finite);
 * block_mass: fp32 [B,H,nb,nb] output (every entry written).
 */
adaspa_status adaspa_lse_cached_search(const adaspa_attn_desc* desc, const void* q, const void* k,
                                       const float* lse, float* block_mass, adaspa_stream_t stream);

/* Workspace bytes adaspa_select_blocks needs for this descriptor. */
size_t adaspa_select_workspace_bytes(const adaspa_attn_desc* desc);

/*
 * K3 -- head-adaptive hierarchical block selection into CSR.
 * Rows are (b, h, p) in that order, row = (b*H + h)*nb + p.  Per row,
 * T = sum_j block_mass[row, j]; with ADASPA_FLAG_TEXT_SINK the forced set F is
 * every text kv-block, and a text q-block row keeps every block (PAPER.md:549,
 * reading R13); without it F is empty and every block is a candidate.
 *   RECALL   (target[h] = r_h): keep F, then candidates by (mass desc, id asc)
 *            until the kept mass >= r_h * T (fp64); r_h >= 1 keeps all
 *            (PAPER.md:228-232 per row; readings R7-R9, R12, R25).
 *   SPARSITY (target[h] = s_h in [0,1)): keep F plus the top
 *            k_h = max(1, floor((1 - s_h) * |candidates| + 0.5 + 1e-9)) candidates
 *            (S*, PAPER.md:436-448 with Row Wise; reading R11).
 *   ADASPA_FLAG_HEAD_TIERS (SPARSITY only): select at s_h, compute each head's
 *            Recall R = kept mass / total mass over all rows, n = min(#{R > tier_tau},
 *            floor(H/2)); the n highest-R heads use (1+s_h)/2, the n lowest
 *            (3*s_h-1)/2 (readings R16-R17); select again.
 *            Requires every s_h >= 1/3.  Tiers are formed per batch element.
 * Ties are broken by kv-block id ascending (reading R10).
 *
 * block_mass : fp32 [B,H,nb,nb] (device, finite, >= 0).
 * target     : HOST double[H] (copied into the launch; may be freed on return).
 * tier_tau   : Recall threshold of the tiers (paper: 0.8).
 * row_ptr    : int32 [B*H*nb + 1] output (exclusive prefix of per-row counts).
 * col_idx    : int32 [col_capacity] output; ascending within a row.
 *              col_capacity must be >= B*H*nb*nb (no host round-trip for nnz).
 * row_order  : int32 [B*H*nb] output or NULL: rows sorted by kept count,
 *              descending (longest-processing-time order; order among equal
 *              counts unspecified).
 * head_recall: fp32 [B,H] output or NULL: achieved Recall per head.
 * head_nnz   : int64 [B,H] output or NULL: kept blocks per head.
 * Limits: nb <= 6144 (one warp holds a row) and B*H*nb*nb < 2^31, else
 * ADASPA_ERR_UNSUPPORTED.
 */
adaspa_status adaspa_select_blocks(const adaspa_attn_desc* desc, const float* block_mass,
                                   adaspa_select_mode mode, const double* target, uint32_t flags,
                                   double tier_tau, int32_t* row_ptr, int32_t* col_idx,
                                   int64_t col_capacity, int32_t* row_order, float* head_recall,
                                   int64_t* head_nnz, void* workspace, size_t workspace_bytes,
                                   adaspa_stream_t stream);

/* Workspace bytes adaspa_block_sparse_attn needs for this descriptor. */
size_t adaspa_sparse_workspace_bytes(const adaspa_attn_desc* desc);

/*
 * K4 -- head-adaptive hierarchical block-sparse attention forward
 * (PAPER.md:415-427 with c = +inf, visiting only kept blocks):
 * for query i of q-block p, J = tokens of the kv-blocks in CSR row p,
 *   lse'_i = log sum_{t in J} exp(S_it),  O_i = sum_{t in J} exp(S_it - lse'_i) V_t.
 * row_ptr / col_idx: the CSR of adaspa_select_blocks (ids ascending, < nb);
 *            nb <= 65535 (16-bit block ids in the kv stream), else ADASPA_ERR_UNSUPPORTED.
 * o: bf16 output.  lse: fp32 [B,H,N] output ("sparse LSE") or NULL.
 * workspace: device scratch of >= adaspa_sparse_workspace_bytes(desc) bytes
 * (the per-launch work schedule is built there).
 */
adaspa_status adaspa_block_sparse_attn(const adaspa_attn_desc* desc, const void* q, const void* k,
                                       const void* v, const int32_t* row_ptr, const int32_t* col_idx,
                                       void* o, float* lse, void* workspace, size_t workspace_bytes,
                                       adaspa_stream_t stream);

const char* adaspa_status_string(adaspa_status status);

/* Thread-local message describing the last non-OK status on this thread. */
const char* adaspa_last_error(void);

/*
 * Multi-GPU plumbing -- the Ulysses exchange over peer memory (
 * the method is orthogonal to sequence parallelism).  No arithmetic of the method:
 * a rank maps every peer's receive buffers into its address space (CUDA IPC), pushes its
 * head slices into them with copy-engine 2-D copies (NVLink, no SMs), raises one 32-bit flag per
 * destination, and a consumer's compute stream waits until its flags reach the exchange's epoch.
 * All calls are asynchronous on `stream` except export / import / close (host calls).  Errors:
 * ADASPA_ERR_INVALID_ARG (NULL / sizes) or ADASPA_ERR_CUDA; message in adaspa_peer_last_error().
 */
typedef struct {
  uint8_t handle[64];   /* cudaIpcMemHandle_t of the allocation holding the pointer */
  int64_t offset;       /* byte offset of the pointer inside that allocation        */
} adaspa_peer_handle;

/* Host: an IPC handle for a device pointer (any pointer inside a cudaMalloc allocation). */
adaspa_status adaspa_peer_export(const void* dev_ptr, adaspa_peer_handle* out);
/* Host: map a peer process's pointer; *dev_ptr = mapped pointer, *base = what to pass to close.
 * Not for a handle exported by the calling process itself (use the local pointer). */
adaspa_status adaspa_peer_import(const adaspa_peer_handle* in, void** dev_ptr, void** base);
adaspa_status adaspa_peer_close(void* base);
/* Stream-ordered 2-D copy between any device pointers the caller can address (local or mapped
 * peer memory): `rows` rows of `width_bytes`, pitches in bytes (cudaMemcpy2DAsync). */
adaspa_status adaspa_peer_copy2d(void* dst, int64_t dst_pitch, const void* src, int64_t src_pitch,
                                 int64_t width_bytes, int64_t rows, adaspa_stream_t stream);
/* Stream-ordered write of `value` to a (local or peer) 32-bit flag, after prior work on `stream`. */
adaspa_status adaspa_peer_signal(uint32_t* flag, uint32_t value, adaspa_stream_t stream);
/* Later work on `stream` waits until every flags[i] >= value (i < n).  Flags must be device memory
 * of this process (the peers write them). */
adaspa_status adaspa_peer_wait(const uint32_t* flags, int32_t n, uint32_t value, adaspa_stream_t stream);
const char* adaspa_peer_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* ADASPA_H_ */
