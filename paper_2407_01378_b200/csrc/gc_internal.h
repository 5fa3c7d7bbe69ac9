// Shared host-side helpers for the C-ABI translation units.
#pragma once
#include <string>

#include "gradcomp_b200.h"

#define GC_ABI_VERSION 1

void gc_set_error(const std::string &msg);

#define GC_REQUIRE(cond, msg)          \
  do {                                 \
    if (!(cond)) {                     \
      gc_set_error(std::string(msg));  \
      return GC_ERR_INVALID;           \
    }                                  \
  } while (0)

#ifdef __CUDACC__
#include <cuda_runtime.h>
// Check the launch that was just enqueued (never synchronises).
// tcgen05 P = M Q pass (gc_psgd_umma.cu): fp64 split-K partials; returns the split count.
int gc_psgd_mq_umma_launch(int32_t L, int32_t workers, const int64_t *row_offsets, int64_t ld, int64_t d,
                           int64_t rows, int64_t cols, int32_t rank, const float *grads, float *resid, const float *q,
                           double *partial, int a16, cudaStream_t st);
// TMA-fed tcgen05 P = M Q with ef_apply / deferred EF (gc_psgd_tma.cu).
int gc_psgd_mq_tma_supported_impl(int32_t tensors, int32_t workers, const int64_t *host_tensor_offsets, int64_t ld,
                                  int64_t d, int64_t rows, int64_t cols, int32_t rank, const void *grads,
                                  const void *resid);
int gc_psgd_mq_tma_launch(int32_t T, int32_t L, const int64_t *host_tensor_offsets, const int64_t *row_start,
                          int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                          float *resid, const float *q, const float *ef_ph, const float *ef_qw, double *partial,
                          int64_t max_splits, cudaStream_t st);
int gc_psgd_mtp_tma_launch(int32_t T, int32_t L, const int64_t *host_tensor_offsets, const int64_t *row_start,
                           int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
                           const float *p_hat, double *partial, int64_t max_splits, cudaStream_t st);
int gc_psgd_mtp_umma_launch(int32_t L, int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
                            const float *p_hat, double *partial, int64_t max_splits, cudaStream_t st);
int gc_psgd_mq_async_supported_impl(int32_t rank, const void *grads, const void *resid);
int gc_psgd_mq_async_launch(int32_t T, int32_t L, const int64_t *row_offsets, const int64_t *host_tensor_offsets,
                            int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                            float *resid, const float *q, const float *ef_ph, const float *ef_qw, double *partial,
                            int64_t max_splits, cudaStream_t st);
int gc_psgd_mtp_async_launch(int32_t V, int32_t L, const int64_t *row_offsets, int64_t ld, int64_t d, int64_t rows,
                             int64_t cols, int32_t rank, const float *c, const float *p_hat, double *partial,
                             int64_t max_splits, cudaStream_t st);
int gc_psgd_mq_pair_supported_impl(int32_t tensors, int32_t workers, const int64_t *host_tensor_offsets, int64_t ld,
                                   int64_t d, int64_t rows, int64_t cols, int32_t rank, const void *grads,
                                   const void *resid);
int gc_psgd_mq_pair_launch(int32_t T, int32_t L, const int64_t *host_tensor_offsets, const int64_t *row_start,
                           int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                           float *resid, const float *q, const float *ef_ph, const float *ef_qw, double *partial,
                           int64_t max_splits, cudaStream_t st);
int gc_psgd_mtp_pair_launch(int32_t T, int32_t L, const int64_t *host_tensor_offsets, const int64_t *row_start,
                            int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
                            const float *p_hat, double *partial, int64_t max_splits, cudaStream_t st);
// column splits the P = M Q passes may use (split-K partials in the workspace): >= 8 chunks each
inline int64_t gc_psgd_mq_max_splits(int64_t cols) { return cols >= 256 ? (cols + 255) / 256 : 1; }
#define GC_LAUNCH_CHECK(what)                                                     \
  do {                                                                            \
    cudaError_t e_ = cudaGetLastError();                                          \
    if (e_ != cudaSuccess) {                                                      \
      gc_set_error(std::string(what) + ": " + cudaGetErrorString(e_));            \
      return GC_ERR_CUDA;                                                         \
    }                                                                             \
  } while (0)
#endif
