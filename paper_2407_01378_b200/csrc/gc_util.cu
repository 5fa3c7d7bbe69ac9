// Round-level utilities: input validation and the nmse diagnostic.
//
//  * gc_check_finite   -- GradientPipeline._checked finite test (pipelines.py:184-197).
//  * gc_nmse_accumulate -- RoundResult.nmse (pipelines.py:172-179, metrics.py:22-37):
//    reference = fp64 mean over workers of the corrected inputs (sequential fp64 sum in
//    worker order, then / n), accumulating sum((est - ref)^2) and sum(ref^2).
#include <cuda_runtime.h>

#include "gc_device.cuh"
#include "gc_internal.h"

namespace {

constexpr int kNT = 256;

int grid_for(int64_t work) {
  int64_t g = (work + kNT - 1) / kNT;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

__global__ void __launch_bounds__(kNT) check_finite_kernel(int64_t rows, const float *data, int64_t ld, int64_t cols,
                                                           unsigned long long *count) {
  unsigned long long bad = 0;
  const int64_t total = rows * cols;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const int64_t r = e / cols, c = e - r * cols;
    bad += !isfinite(data[r * ld + c]);
  }
  for (int o = 16; o; o >>= 1) bad += __shfl_xor_sync(0xffffffffu, bad, o);
  if ((threadIdx.x & 31) == 0 && bad) atomicAdd(count, bad);
}

__global__ void __launch_bounds__(kNT) nmse_kernel(int n, int64_t d, const float *grads, const float *resid,
                                                   int64_t ld, const float *est, double *acc) {
  double num = 0.0, den = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; i < d;
       i += static_cast<int64_t>(gridDim.x) * kNT) {
    double s = 0.0;
    for (int w = 0; w < n; ++w) {
      float c = grads[w * ld + i];
      if (resid) c = c + resid[w * ld + i];
      s += static_cast<double>(c);
    }
    const double ref = s / static_cast<double>(n);
    const double err = static_cast<double>(est[i]) - ref;
    num += err * err;
    den += ref * ref;
  }
  for (int o = 16; o; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&acc[0], num);
    atomicAdd(&acc[1], den);
  }
}

}  // namespace

extern "C" {

int gc_check_finite(int64_t rows, const float *data, int64_t ld, int64_t cols, int64_t *count, void *stream) {
  GC_REQUIRE(rows >= 0 && cols >= 0 && ld >= cols && count, "invalid argument");
  if (rows * cols == 0) return GC_OK;
  GC_REQUIRE(data != nullptr, "null data");
  check_finite_kernel<<<grid_for(rows * cols), kNT, 0, static_cast<cudaStream_t>(stream)>>>(
      rows, data, ld, cols, reinterpret_cast<unsigned long long *>(count));
  GC_LAUNCH_CHECK("check_finite_kernel");
  return GC_OK;
}

int gc_nmse_accumulate(int32_t n, int64_t d, const float *grads, const float *resid, int64_t ld,
                       const float *estimate, double *acc, void *stream) {
  GC_REQUIRE(n >= 1 && d >= 1 && grads && estimate && acc && ld >= d, "invalid argument");
  nmse_kernel<<<grid_for(d), kNT, 0, static_cast<cudaStream_t>(stream)>>>(n, d, grads, resid, ld, estimate, acc);
  GC_LAUNCH_CHECK("nmse_kernel");
  return GC_OK;
}

int gc_copy_rows_async(void *dst, int64_t dst_pitch, const void *src, int64_t src_pitch, int64_t row_bytes,
                       int64_t rows, void *stream) {
  GC_REQUIRE(rows >= 0 && row_bytes >= 0 && dst_pitch >= row_bytes && src_pitch >= row_bytes &&
                 (rows * row_bytes == 0 || (dst && src)),
             "invalid argument");
  if (rows * row_bytes == 0) return GC_OK;
  if (cudaMemcpy2DAsync(dst, static_cast<size_t>(dst_pitch), src, static_cast<size_t>(src_pitch),
                        static_cast<size_t>(row_bytes), static_cast<size_t>(rows), cudaMemcpyDefault,
                        static_cast<cudaStream_t>(stream)) != cudaSuccess) {
    gc_set_error("cudaMemcpy2DAsync failed");
    return GC_ERR_CUDA;
  }
  return GC_OK;
}

}  // extern "C"
