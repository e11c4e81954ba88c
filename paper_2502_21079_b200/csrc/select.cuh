// select.cuh -- parameter blocks of the K3 selection kernels (select.cu).
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace adaspa {

constexpr int kMaxHeads = 256;

struct SelectRowsParams {
  const float* mass;      // [rows, nb]
  int rows;               // B*H*nb
  int heads;
  BlockGrid grid;
  int text_first;
  int text_sink;
  int mode;               // 0 recall, 1 sparsity
  double target[kMaxHeads];  // recall targets (mode 0)
  int k_head[kMaxHeads];     // sparsity budgets per head (mode 1, no tiers)
  const int* k_per_bh;       // sparsity budgets per (b,h) (tiers pass 2) or null
  int nwords;             // ceil(nb/32)
  uint32_t* bits;         // [rows, nwords]
  int* row_nnz;           // [rows]
  double* row_kept;       // [rows]
  double* row_total;      // [rows]
};

struct SelectTierParams {
  int heads, nb, ncand;
  double tau;
  double s_base[kMaxHeads];
  const double* row_kept;
  const double* row_total;
  int* k_per_bh;          // [B*H] output
};

struct SelectFinalParams {
  int rows, nb, bh;
  const int* row_nnz;
  const double* row_kept;
  const double* row_total;
  int* local_off;         // [rows]   exclusive offset of a row within its head
  int* head_cnt;          // [B*H]    kept blocks per head
  int* head_base;         // [B*H]    exclusive offset of a head in col_idx
  int* hist;              // [nb+1]   row-count histogram -> LPT slots
  int32_t* row_ptr;
  int32_t* row_order;     // may be null
  float* head_recall;     // may be null
  int64_t* head_nnz;      // may be null
};

struct SelectWriteParams {
  int rows, nwords, nb;
  const uint32_t* bits;
  const int* row_nnz;
  const int* local_off;
  const int* head_base;
  int* hist;
  int32_t* row_ptr;
  int32_t* row_order;     // may be null
  int32_t* col_idx;
};

struct SelectLaunch {
  int batch;
  bool tiers;
  SelectRowsParams rows;
  SelectTierParams tier;
  SelectFinalParams fin;
  SelectWriteParams wr;
};

cudaError_t launch_select(const SelectLaunch& L, cudaStream_t st);
// the two halves of launch_select (no tiers): per-row selection, then CSR assembly from its arrays
cudaError_t launch_select_rows(const SelectRowsParams& p, cudaStream_t st);
cudaError_t launch_select_final(const SelectLaunch& L, cudaStream_t st);

__host__ __device__ int k_from_sparsity(double s, int n);
constexpr int kMaxSelectBlocks = 6144;  // one warp holds a row: 192 masses per lane at most

}  // namespace adaspa
