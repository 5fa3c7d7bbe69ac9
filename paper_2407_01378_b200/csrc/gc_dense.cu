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
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "gc_device.cuh"
#include "gc_internal.h"

namespace {

constexpr int kNT = 256;

// MAXN: workers whose loads are issued up front (8 or 16; larger n: rolled loop)

// One element's ordered fold over the n values x[0..n) already in registers, x[k] from worker
// (s + k) mod n.
template <bool WIRE16, bool ROUND_IN, int kMaxFold>
__device__ __forceinline__ float fold_values(const float (&x)[kMaxFold], int n) {
  float acc = ROUND_IN ? gc::fp16_round_trip(x[0]) : x[0];
#pragma unroll
  for (int k = 1; k < kMaxFold; ++k) {
    if (k < n) {
      const float v = ROUND_IN ? gc::fp16_round_trip(x[k]) : x[k];
      const float sent = WIRE16 ? gc::fp16_round_trip(acc) : acc;
      acc = sent + v;
    }
  }
  if (WIRE16 && n > 1) acc = gc::fp16_round_trip(acc);
  return acc;
}

template <bool WIRE16, bool ROUND_IN, int kMaxFold>
__global__ void __launch_bounds__(kNT) float_fold_kernel(int n, int64_t len, const float *in, int64_t ld,
                                                         int64_t offset, int64_t ring_block, int divisor,
                                                         float *out, int64_t in_stride, int64_t out_stride,
                                                         int vec) {
  in += blockIdx.y * in_stride;   // batch of independent folds
  out += blockIdx.y * out_stride;
  const gc::DivN dv(divisor > 0 ? divisor : 1);
  // vec: 4 elements per thread with float4 rows (ld, in, out 16-byte aligned); a group that
  // straddles a ring-block boundary folds its elements one by one.  All n row loads of a group
  // are issued before the fold (n <= kMaxFold), so each thread keeps n loads in flight.
  const int64_t groups = vec ? (len + 3) / 4 : len;
  for (int64_t gi = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; gi < groups;
       gi += static_cast<int64_t>(gridDim.x) * kNT) {
    const int64_t e0 = vec ? 4 * gi : gi;
    const int s = static_cast<int>((offset + e0) / ring_block);
    if (n <= kMaxFold && vec && e0 + 3 < len && (offset + e0 + 3) / ring_block == s) {
      float4 x4[kMaxFold];
      int w = s;
#pragma unroll
      for (int k = 0; k < kMaxFold; ++k) {
        if (k < n) {
          x4[k] = __ldcs(reinterpret_cast<const float4 *>(in + w * ld + e0));
          w = (w + 1 == n) ? 0 : w + 1;
        }
      }
      float r[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float x[kMaxFold];
#pragma unroll
        for (int k = 0; k < kMaxFold; ++k) x[k] = c == 0 ? x4[k].x : (c == 1 ? x4[k].y : (c == 2 ? x4[k].z : x4[k].w));
        const float acc = fold_values<WIRE16, ROUND_IN, kMaxFold>(x, n);
        r[c] = divisor > 0 ? dv(acc) : acc;
      }
      __stcs(reinterpret_cast<float4 *>(out + e0), make_float4(r[0], r[1], r[2], r[3]));
      continue;
    }
    const int64_t e1 = vec ? min(e0 + 4, len) : e0 + 1;
    for (int64_t e = e0; e < e1; ++e) {
      const int se = static_cast<int>((offset + e) / ring_block);
      float acc;
      if (n <= kMaxFold) {
        float x[kMaxFold];
        int w = se;
#pragma unroll
        for (int k = 0; k < kMaxFold; ++k) {
          if (k < n) {
            x[k] = in[w * ld + e];
            w = (w + 1 == n) ? 0 : w + 1;
          }
        }
        acc = fold_values<WIRE16, ROUND_IN, kMaxFold>(x, n);
      } else {
        acc = in[se * ld + e];
        if (ROUND_IN) acc = gc::fp16_round_trip(acc);
        int w = se;
        for (int k = 1; k < n; ++k) {
          w = (w + 1 == n) ? 0 : w + 1;
          float x = in[w * ld + e];
          if (ROUND_IN) x = gc::fp16_round_trip(x);
          const float sent = WIRE16 ? gc::fp16_round_trip(acc) : acc;
          acc = sent + x;
        }
        if (WIRE16 && n > 1) acc = gc::fp16_round_trip(acc);
      }
      out[e] = divisor > 0 ? dv(acc) : acc;
    }
  }
}

// Dense fp32 bypass of a batch of small tensors: segment blockIdx.y, ring block ceil(len/n).
// c holds the corrected values; zero (may alias c) receives the new residual 0.
__global__ void __launch_bounds__(kNT) segment_fold_kernel(int n, const int64_t *seg_off, const int64_t *seg_len,
                                                           const float *g, float *r, int64_t ld, float *est,
                                                           int apply_ef) {
  // g: corrected values (apply_ef: raw gradients, corrected = f32(g + r)), r: residual rows to
  // zero (nullable)
  const int64_t off = seg_off[blockIdx.y], len = seg_len[blockIdx.y];
  const int64_t blk = (len + n - 1) / n;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const int64_t i = off + e;
    const int s = static_cast<int>(e / blk);
    float acc = 0.0f;
    int w = s;
    for (int k = 0; k < n; ++k) {
      const float c = apply_ef ? g[w * ld + i] + r[w * ld + i] : g[w * ld + i];
      acc = (k == 0) ? c : acc + c;
      w = (w + 1 == n) ? 0 : w + 1;
    }
    est[i] = gc::DivN(n)(acc);
    if (r)
      for (int u = 0; u < n; ++u) r[u * ld + i] = 0.0f;   // corrected - own with own = corrected
  }
}

__global__ void scale_div_kernel(int64_t len, const float *in, int divisor, float *out) {
  const gc::DivN dv(divisor);
  int64_t head = 0;
  if (((reinterpret_cast<uintptr_t>(in) | reinterpret_cast<uintptr_t>(out)) & 15) == 0) {   // float4 body
    head = len & ~int64_t{3};
    for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; 4 * e < head;
         e += static_cast<int64_t>(gridDim.x) * kNT) {
      const float4 v = __ldcs(reinterpret_cast<const float4 *>(in) + e);
      __stcs(reinterpret_cast<float4 *>(out) + e, make_float4(dv(v.x), dv(v.y), dv(v.z), dv(v.w)));
    }
  }
  for (int64_t e = head + blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * kNT)
    out[e] = dv(in[e]);
}

__global__ void fp16_round_kernel(int64_t len, const float *in, float *out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * kNT)
    out[e] = gc::fp16_round_trip(in[e]);
}


// FP16 bar across ranks, the local half: fold this rank's L rows with fp16 inputs and wire
// (as float_fold_kernel<true, true>) and emit the binary16 bits the NCCL half all-reduce sends.
__global__ void __launch_bounds__(kNT) fold_to_half_kernel(int L, int64_t len, const float *in, int64_t ld,
                                                           __half *out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; 2 * e < len;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    float acc[2];
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const int64_t i = 2 * e + c;
      float a = 0.0f;
      if (i < len) {
        a = gc::fp16_round_trip(in[i]);
        for (int w = 1; w < L; ++w) a = gc::fp16_round_trip(gc::fp16_round_trip(a) + gc::fp16_round_trip(in[w * ld + i]));
      }
      acc[c] = a;
    }
    if (2 * e + 1 < len && (reinterpret_cast<uintptr_t>(out) & 3) == 0)
      *reinterpret_cast<__half2 *>(out + 2 * e) = __floats2half2_rn(acc[0], acc[1]);
    else {
      out[2 * e] = __float2half_rn(acc[0]);
      if (2 * e + 1 < len) out[2 * e + 1] = __float2half_rn(acc[1]);
    }
  }
}

// ... and the other half: the all-reduced binary16 sums -> f32 estimate = sum / n, with the
// fp16 wire's +-65504 saturation (vectors.py:136-152) applied to partial sums that overflowed
// to +-inf inside NCCL's half adds.
__global__ void __launch_bounds__(kNT) half_mean_kernel(int64_t len, const __half *in, int divisor, float *out) {
  const gc::DivN dv(divisor);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    float x = __half2float(in[e]);
    if (isinf(x)) x = copysignf(65504.0f, x);
    out[e] = dv(x);
  }
}

// Vectorised forms for 16-byte aligned buffers (the FP16 bar at full size): 8 coordinates per
// thread and iteration -- two float4 loads per worker row in, one 16-byte store of 8 halves out
// (and back: one 16-byte load of 8 halves, two float4 stores).  Same per-element arithmetic.
__global__ void __launch_bounds__(kNT) fold_to_half_vec_kernel(int L, int64_t n8, const float *in, int64_t ld,
                                                               __half *out) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < n8;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const float4 *p = reinterpret_cast<const float4 *>(in) + 2 * e;
    float4 a0 = __ldcs(p), a1 = __ldcs(p + 1);
    float a[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
    for (int c = 0; c < 8; ++c) a[c] = gc::fp16_round_trip(a[c]);
    for (int w = 1; w < L; ++w) {
      const float4 *pw = reinterpret_cast<const float4 *>(in + w * ld) + 2 * e;
      const float4 b0 = __ldcs(pw), b1 = __ldcs(pw + 1);
      const float b[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int c = 0; c < 8; ++c) a[c] = gc::fp16_round_trip(gc::fp16_round_trip(a[c]) + gc::fp16_round_trip(b[c]));
    }
    __half2 h[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) h[c] = __floats2half2_rn(a[2 * c], a[2 * c + 1]);
    __stcs(reinterpret_cast<uint4 *>(out) + e, *reinterpret_cast<const uint4 *>(h));
  }
}

__global__ void __launch_bounds__(kNT) half_mean_vec_kernel(int64_t n8, const __half *in, int divisor, float *out) {
  const gc::DivN dv(divisor);
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < n8;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const uint4 u = __ldcs(reinterpret_cast<const uint4 *>(in) + e);
    const __half2 *h = reinterpret_cast<const __half2 *>(&u);
    float x[8];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const float2 f = __half22float2(h[c]);
      x[2 * c] = f.x;
      x[2 * c + 1] = f.y;
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (isinf(x[c])) x[c] = copysignf(65504.0f, x[c]);
      x[c] = dv(x[c]);
    }
    float4 *o = reinterpret_cast<float4 *>(out) + 2 * e;
    __stcs(o, make_float4(x[0], x[1], x[2], x[3]));
    __stcs(o + 1, make_float4(x[4], x[5], x[6], x[7]));
  }
}

int grid_for(int64_t work) {
  int64_t g = (work + kNT - 1) / kNT;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

int fold_launch(int32_t batch, int32_t n, int64_t len, const float *inputs, int64_t ld, int64_t in_stride,
                int64_t offset, int64_t ring_block, int32_t wire_fp16, int32_t round_inputs, int32_t divisor,
                float *out, int64_t out_stride, cudaStream_t st) {
  const int vec = (ld % 4) == 0 && (in_stride % 4) == 0 && (out_stride % 4) == 0 &&
                  ((reinterpret_cast<uintptr_t>(inputs) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const dim3 g(grid_for(vec ? (len + 3) / 4 : len), batch);
#define GC_FOLD(W, R, M)                                                                                 \
  float_fold_kernel<W, R, M><<<g, kNT, 0, st>>>(n, len, inputs, ld, offset, ring_block, divisor, out, in_stride, \
                                                out_stride, vec)
#define GC_FOLD_N(W, R) \
  if (n <= 8)           \
    GC_FOLD(W, R, 8);   \
  else                  \
    GC_FOLD(W, R, 16);
  if (wire_fp16 && round_inputs) {
    GC_FOLD_N(true, true)
  } else if (wire_fp16) {
    GC_FOLD_N(true, false)
  } else if (round_inputs) {
    GC_FOLD_N(false, true)
  } else {
    GC_FOLD_N(false, false)
  }
#undef GC_FOLD_N
#undef GC_FOLD
  GC_LAUNCH_CHECK("float_fold_kernel");
  return GC_OK;
}

}  // namespace

extern "C" {

int gc_float_fold(int32_t n, int64_t len, const float *inputs, int64_t ld, int64_t offset, int64_t ring_block,
                  int32_t wire_fp16, int32_t round_inputs, int32_t divisor, float *out, void *stream) {
  GC_REQUIRE(n >= 1 && len >= 0 && ld >= len && ring_block >= 1 && inputs && out, "invalid argument");
  if (len == 0) return GC_OK;
  return fold_launch(1, n, len, inputs, ld, 0, offset, ring_block, wire_fp16, round_inputs, divisor, out, 0,
                     static_cast<cudaStream_t>(stream));
}

int gc_float_fold_batched(int32_t batch, int32_t n, int64_t len, const float *inputs, int64_t ld, int64_t in_stride,
                          int32_t wire_fp16, int32_t round_inputs, int32_t divisor, float *out, int64_t out_stride,
                          void *stream) {
  GC_REQUIRE(batch >= 1 && batch <= 65535 && n >= 1 && len >= 0 && ld >= len && inputs && out, "invalid argument");
  if (len == 0) return GC_OK;
  return fold_launch(batch, n, len, inputs, ld, in_stride, 0, (len + n - 1) / n, wire_fp16, round_inputs, divisor,
                     out, out_stride, static_cast<cudaStream_t>(stream));
}

int gc_float_fold_batched_slice(int32_t batch, int32_t n, int64_t len, const float *inputs, int64_t ld,
                                int64_t in_stride, int64_t offset, int64_t ring_block, int32_t wire_fp16,
                                int32_t round_inputs, int32_t divisor, float *out, int64_t out_stride, void *stream) {
  GC_REQUIRE(batch >= 1 && batch <= 65535 && n >= 1 && len >= 0 && ld >= len && offset >= 0 && ring_block >= 1 &&
                 inputs && out,
             "invalid argument");
  if (len == 0) return GC_OK;
  return fold_launch(batch, n, len, inputs, ld, in_stride, offset, ring_block, wire_fp16, round_inputs, divisor, out,
                     out_stride, static_cast<cudaStream_t>(stream));
}

int gc_segment_fold_ef(int32_t n, int32_t nseg, const int64_t *seg_off, const int64_t *seg_len, const float *grads,
                       float *resid, int64_t ld, float *estimate, void *stream) {
  GC_REQUIRE(n >= 1 && nseg >= 0 && nseg <= 65535 && (nseg == 0 || (seg_off && seg_len)) && grads && estimate,
             "invalid argument");
  if (nseg == 0) return GC_OK;
  segment_fold_kernel<<<dim3(4, nseg), kNT, 0, static_cast<cudaStream_t>(stream)>>>(n, seg_off, seg_len, grads, resid,
                                                                                  ld, estimate, 0);
  GC_LAUNCH_CHECK("segment_fold_kernel");
  return GC_OK;
}

int gc_segment_ef_fold(int32_t n, int32_t nseg, const int64_t *seg_off, const int64_t *seg_len, const float *grads,
                       float *resid, int64_t ld, float *estimate, void *stream) {
  GC_REQUIRE(n >= 1 && nseg >= 0 && nseg <= 65535 && (nseg == 0 || (seg_off && seg_len)) && grads && resid && estimate,
             "invalid argument");
  if (nseg == 0) return GC_OK;
  segment_fold_kernel<<<dim3(4, nseg), kNT, 0, static_cast<cudaStream_t>(stream)>>>(n, seg_off, seg_len, grads, resid,
                                                                                  ld, estimate, 1);
  GC_LAUNCH_CHECK("segment_fold_kernel");
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

int gc_fold_to_half(int32_t L, int64_t len, const float *inputs, int64_t ld, void *out_half, void *stream) {
  GC_REQUIRE(L >= 1 && len >= 0 && ld >= len && inputs && out_half, "invalid argument");
  if (len == 0) return GC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec = ((reinterpret_cast<uintptr_t>(inputs) | reinterpret_cast<uintptr_t>(out_half)) & 15) == 0 &&
                   (L == 1 || ld % 4 == 0);
  const int64_t n8 = vec ? len / 8 : 0;
  if (n8) {
    fold_to_half_vec_kernel<<<grid_for(n8), kNT, 0, st>>>(L, n8, inputs, ld, static_cast<__half *>(out_half));
    GC_LAUNCH_CHECK("fold_to_half_vec_kernel");
  }
  if (len > 8 * n8) {   // the tail (or everything, unaligned)
    fold_to_half_kernel<<<grid_for((len - 8 * n8 + 1) / 2), kNT, 0, st>>>(L, len - 8 * n8, inputs + 8 * n8, ld,
                                                                          static_cast<__half *>(out_half) + 8 * n8);
    GC_LAUNCH_CHECK("fold_to_half_kernel");
  }
  return GC_OK;
}

int gc_half_mean_sat(int64_t len, const void *in_half, int32_t divisor, float *out, void *stream) {
  GC_REQUIRE(len >= 0 && divisor >= 1 && in_half && out, "invalid argument");
  if (len == 0) return GC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const bool vec = ((reinterpret_cast<uintptr_t>(in_half) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  const int64_t n8 = vec ? len / 8 : 0;
  if (n8) {
    half_mean_vec_kernel<<<grid_for(n8), kNT, 0, st>>>(n8, static_cast<const __half *>(in_half), divisor, out);
    GC_LAUNCH_CHECK("half_mean_vec_kernel");
  }
  if (len > 8 * n8) {
    half_mean_kernel<<<grid_for(len - 8 * n8), kNT, 0, st>>>(len - 8 * n8, static_cast<const __half *>(in_half) + 8 * n8,
                                                             divisor, out + 8 * n8);
    GC_LAUNCH_CHECK("half_mean_kernel");
  }
  return GC_OK;
}

}  // extern "C"
