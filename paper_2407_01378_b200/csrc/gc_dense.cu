// Float ring folds: the FloatSum ring_all_reduce semantics (collectives.py:112-120, 177-236)
// executed as an ordered fold per element, plus the elementwise helpers around them.
//
//  * element e (global index offset+e) of a length-`len` vector belongs to ring block
//    s = (offset+e) / ring_block and folds in worker order s, s+1, ..., s+n-1 (mod n);
//  * wire_fp16: every transmitted partial and the final value are rounded through binary16
//    with +-65504 saturation (fp16_round_trip, vectors.py:136-152); the accumulation is f32;
//  * round_inputs: inputs are first rounded to fp16 (the dense FP16 bar, pipelines.py:373);
//  * divisor > 0: the folded value is divided by it in f32 (estimate = summed / n).
// One thread per element reads the n worker rows coalesced: HBM traffic = 4n + 4 bytes per
// element, the bound for this op.
#include <cuda_runtime.h>

#include "gc_device.cuh"
#include "gc_internal.h"

namespace {

constexpr int kNT = 256;

template <bool WIRE16, bool ROUND_IN>
__global__ void __launch_bounds__(kNT) float_fold_kernel(int n, int64_t len, const float *in, int64_t ld,
                                                         int64_t offset, int64_t ring_block, int divisor,
                                                         float *out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const int s = static_cast<int>((offset + e) / ring_block);
    float acc = in[s * ld + e];
    if (ROUND_IN) acc = gc::fp16_round_trip(acc);
    int w = s;
    for (int k = 1; k < n; ++k) {
      w = (w + 1 == n) ? 0 : w + 1;
      float x = in[w * ld + e];
      if (ROUND_IN) x = gc::fp16_round_trip(x);
      const float sent = WIRE16 ? gc::fp16_round_trip(acc) : acc;
      acc = sent + x;
    }
    if (WIRE16 && n > 1) acc = gc::fp16_round_trip(acc);
    out[e] = divisor > 0 ? acc / static_cast<float>(divisor) : acc;
  }
}

__global__ void scale_div_kernel(int64_t len, const float *in, int divisor, float *out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * kNT)
    out[e] = in[e] / static_cast<float>(divisor);
}

__global__ void fp16_round_kernel(int64_t len, const float *in, float *out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * kNT)
    out[e] = gc::fp16_round_trip(in[e]);
}

int grid_for(int64_t work) {
  int64_t g = (work + kNT - 1) / kNT;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

int gc_float_fold(int32_t n, int64_t len, const float *inputs, int64_t ld, int64_t offset, int64_t ring_block,
                  int32_t wire_fp16, int32_t round_inputs, int32_t divisor, float *out, void *stream) {
  GC_REQUIRE(n >= 1 && len >= 0 && ld >= len && ring_block >= 1 && inputs && out, "invalid argument");
  if (len == 0) return GC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int g = grid_for(len);
  if (wire_fp16 && round_inputs)
    float_fold_kernel<true, true><<<g, kNT, 0, st>>>(n, len, inputs, ld, offset, ring_block, divisor, out);
  else if (wire_fp16)
    float_fold_kernel<true, false><<<g, kNT, 0, st>>>(n, len, inputs, ld, offset, ring_block, divisor, out);
  else if (round_inputs)
    float_fold_kernel<false, true><<<g, kNT, 0, st>>>(n, len, inputs, ld, offset, ring_block, divisor, out);
  else
    float_fold_kernel<false, false><<<g, kNT, 0, st>>>(n, len, inputs, ld, offset, ring_block, divisor, out);
  GC_LAUNCH_CHECK("float_fold_kernel");
  return GC_OK;
}

int gc_scale_div(int64_t len, const float *in, int32_t divisor, float *out, void *stream) {
  GC_REQUIRE(len >= 0 && divisor >= 1 && in && out, "invalid argument");
  if (len == 0) return GC_OK;
  scale_div_kernel<<<grid_for(len), kNT, 0, static_cast<cudaStream_t>(stream)>>>(len, in, divisor, out);
  GC_LAUNCH_CHECK("scale_div_kernel");
  return GC_OK;
}

int gc_fp16_round(int64_t len, const float *in, float *out, void *stream) {
  GC_REQUIRE(len >= 0 && in && out, "invalid argument");
  if (len == 0) return GC_OK;
  fp16_round_kernel<<<grid_for(len), kNT, 0, static_cast<cudaStream_t>(stream)>>>(len, in, out);
  GC_LAUNCH_CHECK("fp16_round_kernel");
  return GC_OK;
}

}  // extern "C"
