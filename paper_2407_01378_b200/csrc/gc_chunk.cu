// TopK-Chunked (consensus chunk selection) building blocks and ef_apply.
//
// Reference: _round_chunked (pipelines.py:213-258): chunk energies chunk_sq_norms
// (vectors.py:180-192) -> f32 -> fp16 -> fp16-wire ring sum (norm-consensus) ->
// select_chunks (compressors.py:412-414) -> chunk_values (compressors.py:417-430, fp16) ->
// fp16-wire ring sum (chunk-aggregate) -> chunkset_to_dense (compressors.py:433-438) / n;
// own = the worker's own chunk values; optional shared coordinate permutation
// (transforms.py:129-151) applied before chunking and undone after.
//
// Chunk energies must match numpy bit for bit (they drive the selection): the squares are
// exact in fp64 (f32 x f32), and the sum follows numpy's pairwise summation of a reduction
// row: 0 + pairwise(row) with 8 strided accumulators for n <= 128 combined as
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)), leftovers added sequentially, and halving (rounded
// down to a multiple of 8) above 128 elements.  C <= 128 with C % 8 == 0 (the paper's
// C = 64) uses 8 lanes per chunk (one accumulator each, coalesced loads, shuffle tree in the
// same order); other C run the recursion one thread per chunk.
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

__device__ __forceinline__ double sq_at(const float *row, const int64_t *perm, int64_t i, int64_t d) {
  if (i >= d) return 0.0;                       // zero-padded final chunk
  const float x = perm ? row[perm[i]] : row[i];
  const double v = static_cast<double>(x);
  return v * v;                                 // exact in fp64
}

// numpy pairwise_sum (loops_utils.h.src) over n squares starting at logical index i0.
__device__ double pairwise_sq(const float *row, const int64_t *perm, int64_t i0, int64_t n, int64_t d) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += sq_at(row, perm, i0 + i, d);
    return res;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = sq_at(row, perm, i0 + j, d);
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += sq_at(row, perm, i0 + i + j, d);
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += sq_at(row, perm, i0 + i, d);
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pairwise_sq(row, perm, i0, n2, d) + pairwise_sq(row, perm, i0 + n2, n - n2, d);
}

__global__ void __launch_bounds__(kNT) norms_generic_kernel(int64_t d, int64_t C, int64_t nc, const float *vals,
                                                            int64_t ld, const int64_t *perm, float *out) {
  const int w = blockIdx.y;
  const float *row = vals + w * ld;
  for (int64_t c = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; c < nc;
       c += static_cast<int64_t>(gridDim.x) * kNT) {
    const double e = 0.0 + pairwise_sq(row, perm, c * C, C, d);
    out[w * nc + c] = gc::fp16_round_trip(static_cast<float>(e));   // pipelines.py:221-223
  }
}

// C % 8 == 0 and C <= 128: lane group of 8 per chunk, lane j owns accumulator r[j].
// With grads != NULL (no permutation) ef_apply is fused: corrected = f32(g + r) is formed here and
// written over r (vals == r then, or the corrected copy when r is NULL).
__global__ void __launch_bounds__(kNT) norms_lanes_kernel(int64_t d, int C, int64_t nc, const float *vals,
                                                          int64_t ld, const int64_t *perm, float *out,
                                                          const float *grads, float *resid) {
  const int w = blockIdx.y;
  const float *row = vals + w * ld;
  const float *grow = grads ? grads + w * ld : nullptr;
  float *rrow = resid ? resid + w * ld : nullptr;
  const int j = threadIdx.x & 7;
  const int group = (threadIdx.x & 31) >> 3;   // 4 chunks per warp
  const int64_t stride = static_cast<int64_t>(gridDim.x) * (kNT / 8);
  for (int64_t cw = blockIdx.x * static_cast<int64_t>(kNT / 8) + (threadIdx.x >> 5) * 4; cw < nc; cw += stride) {
    const int64_t c = cw + group;   // warp-uniform loop, per-group chunk
    const bool live = c < nc;
    double r = 0.0;
    if (live) {
      const int64_t i0 = c * C;
      if (grow) {   // fused ef_apply (compressors.py:624-626): all loads issued before any store
        float gv[16], rv[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          const int64_t x = i0 + t * 8 + j;
          const bool ok = t * 8 < C && x < d;
          gv[t] = ok ? __ldcs(grow + x) : 0.0f;
          rv[t] = (ok && rrow) ? __ldcs(rrow + x) : 0.0f;
        }
#pragma unroll
        for (int t = 0; t < 16; ++t) {
          if (t * 8 < C) {
            const int64_t x = i0 + t * 8 + j;
            const float cv = rrow ? gv[t] + rv[t] : gv[t];
            if (rrow && x < d) rrow[x] = cv;
            const double v = static_cast<double>(cv);
            r = (t == 0) ? v * v : r + v * v;
          }
        }
      } else {
        r = sq_at(row, perm, i0 + j, d);
        for (int i = 8; i < C; i += 8) r += sq_at(row, perm, i0 + i + j, d);
      }
    }
    r += __shfl_xor_sync(0xffffffffu, r, 1);   // (r0+r1), (r2+r3), ...
    r += __shfl_xor_sync(0xffffffffu, r, 2);   // ((r0+r1)+(r2+r3)), ...
    r += __shfl_xor_sync(0xffffffffu, r, 4);   // (...) + ((r4+r5)+(r6+r7))
    if (live && j == 0) out[w * nc + c] = gc::fp16_round_trip(static_cast<float>(0.0 + r));
  }
}

// Fused ef_apply + chunk energies with float4 traffic (aligned rows, C % 8 == 0, C <= 128):
// two lanes per chunk, lane half h owning numpy's accumulators 4h..4h+3 (elements 8t + 4h + q),
// so one float4 of g and one of r per lane and 8-element step; corrected is written back over
// r as float4.  In-lane ((r0+r1)+(r2+r3)), then one shuffle adds the other half: the same
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree as numpy.  x*x is exact in fp64, so
// fma(x, x, r) == r + x*x bit for bit.  Chunks that cross d take the scalar path.
__global__ void __launch_bounds__(kNT, 2) norms_ef_vec_kernel(int64_t d, int C, int64_t nc, const float *grads,
                                                           float *resid, int64_t ld, float *out) {
  const int w = blockIdx.y;
  const float *grow = grads + w * ld;
  float *rrow = resid ? resid + w * ld : nullptr;
  const int half = threadIdx.x & 1;
  const int nt = C >> 3;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * (kNT / 2);
  for (int64_t c = blockIdx.x * static_cast<int64_t>(kNT / 2) + (threadIdx.x >> 1); c - (threadIdx.x & 31) / 2 < nc;
       c += stride) {
    const bool live = c < nc;
    const int64_t i0 = c * C + 4 * half;
    double r[4] = {0.0, 0.0, 0.0, 0.0};
    if (live && (c + 1) * C <= d) {
      for (int t0 = 0; t0 < nt; t0 += 8) {   // 8 steps of loads in flight per lane
        float4 gv[8], rv[8];
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (t0 + t < nt) {
            const int64_t x = i0 + 8 * (t0 + t);
            gv[t] = __ldcs(reinterpret_cast<const float4 *>(grow + x));
            rv[t] = rrow ? __ldcs(reinterpret_cast<const float4 *>(rrow + x)) : make_float4(0.f, 0.f, 0.f, 0.f);
          }
#pragma unroll
        for (int t = 0; t < 8; ++t)
          if (t0 + t < nt) {
            float4 cv = gv[t];
            if (rrow) {
              cv.x = cv.x + rv[t].x; cv.y = cv.y + rv[t].y; cv.z = cv.z + rv[t].z; cv.w = cv.w + rv[t].w;
              *reinterpret_cast<float4 *>(rrow + i0 + 8 * (t0 + t)) = cv;
            }
            const double a = cv.x, b = cv.y, e = cv.z, f = cv.w;
            r[0] = fma(a, a, r[0]);
            r[1] = fma(b, b, r[1]);
            r[2] = fma(e, e, r[2]);
            r[3] = fma(f, f, r[3]);
          }
      }
    } else if (live) {
      for (int t = 0; t < nt; ++t)
        for (int q = 0; q < 4; ++q) {
          const int64_t x = i0 + 8 * t + q;
          float cv = 0.0f;
          if (x < d) {
            cv = grow[x];
            if (rrow) {
              cv = cv + rrow[x];
              rrow[x] = cv;
            }
          }
          const double v = cv;
          r[q] = fma(v, v, r[q]);
        }
    }
    double sum = (r[0] + r[1]) + (r[2] + r[3]);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);   // half 0: (r0..r3) + (r4..r7); same on half 1
    if (live && half == 0) out[w * nc + c] = gc::fp16_round_trip(static_cast<float>(0.0 + sum));
  }
}

// payload[w][jj*C + t] = fp16(work_w[sel[jj]*C + t]) (0 past d)  -- chunk_values.
__global__ void __launch_bounds__(kNT) pack_kernel(int64_t d, int64_t C, int64_t J, const int32_t *sel,
                                                   const float *vals, int64_t ld, const int64_t *perm,
                                                   float *out) {
  const int w = blockIdx.y;
  const int64_t total = J * C;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const int64_t jj = e / C, t = e - jj * C;
    const int64_t i = static_cast<int64_t>(sel[jj]) * C + t;
    float x = 0.0f;
    if (i < d) x = perm ? vals[w * ld + perm[i]] : vals[w * ld + i];
    out[w * total + e] = gc::fp16_round_trip(x);
  }
}

// est[pos(sel[jj]*C + t)] = summed[jj*C + t] / divisor  -- chunkset_to_dense / n (est pre-zeroed).
__global__ void __launch_bounds__(kNT) scatter_kernel(int64_t d, int64_t C, int64_t J, const int32_t *sel,
                                                      const float *summed, int divisor, const int64_t *perm,
                                                      float *est) {
  const int64_t total = J * C;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const int64_t jj = e / C, t = e - jj * C;
    const int64_t i = static_cast<int64_t>(sel[jj]) * C + t;
    if (i < d) est[perm ? perm[i] : i] = gc::DivN(divisor)(summed[e]);
  }
}

// resid[w][pos] -= payload  (ef_update with own = the worker's chunk values; resid holds corrected).
__global__ void __launch_bounds__(kNT) chunk_ef_kernel(int64_t d, int64_t C, int64_t J, const int32_t *sel,
                                                       const float *packs, const int64_t *perm, float *resid,
                                                       int64_t ld) {
  const int w = blockIdx.y;
  const int64_t total = J * C;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const int64_t jj = e / C, t = e - jj * C;
    const int64_t i = static_cast<int64_t>(sel[jj]) * C + t;
    if (i < d) {
      const int64_t p = w * ld + (perm ? perm[i] : i);
      resid[p] = resid[p] - packs[w * total + e];
    }
  }
}

__global__ void __launch_bounds__(kNT) ef_apply_kernel(int64_t d, const float *g, const float *r, int64_t ld,
                                                       float *out, int64_t ldo, bool vec) {
  const int w = blockIdx.y;
  if (vec) {   // float4 path (ld, ldo multiples of 4 and 16-byte aligned rows)
    const int64_t d4 = d / 4;
    const float4 *g4 = reinterpret_cast<const float4 *>(g + w * ld);
    const float4 *r4 = r ? reinterpret_cast<const float4 *>(r + w * ld) : nullptr;
    float4 *o4 = reinterpret_cast<float4 *>(out + w * ldo);
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; i < d4;
         i += static_cast<int64_t>(gridDim.x) * kNT) {
      float4 c = __ldcs(g4 + i);
      if (r4) {
        const float4 rv = __ldcs(r4 + i);
        c.x = c.x + rv.x; c.y = c.y + rv.y; c.z = c.z + rv.z; c.w = c.w + rv.w;
      }
      __stcs(o4 + i, c);
    }
    for (int64_t i = d4 * 4 + blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; i < d;
         i += static_cast<int64_t>(gridDim.x) * kNT) {
      float c = g[w * ld + i];
      if (r) c = c + r[w * ld + i];
      out[w * ldo + i] = c;
    }
    return;
  }
  for (int64_t i = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; i < d;
       i += static_cast<int64_t>(gridDim.x) * kNT) {
    float c = g[w * ld + i];
    if (r) c = c + r[w * ld + i];
    out[w * ldo + i] = c;
  }
}

}  // namespace

extern "C" {

int gc_ef_apply(int32_t workers, int64_t d, const float *grads, const float *resid, int64_t ld, float *out,
                int64_t ld_out, void *stream) {
  GC_REQUIRE(workers >= 1 && workers <= 65535 && d >= 1 && grads && out && ld >= d && ld_out >= d,
             "invalid argument");
  const bool vec = ld % 4 == 0 && ld_out % 4 == 0 &&
                   ((reinterpret_cast<uintptr_t>(grads) | reinterpret_cast<uintptr_t>(resid) |
                     reinterpret_cast<uintptr_t>(out)) & 15) == 0;
  ef_apply_kernel<<<dim3(grid_for(vec ? d / 4 + 1 : d), workers), kNT, 0, static_cast<cudaStream_t>(stream)>>>(
      d, grads, resid, ld, out, ld_out, vec);
  GC_LAUNCH_CHECK("ef_apply_kernel");
  return GC_OK;
}

int gc_chunk_norms(int32_t workers, int64_t d, int64_t chunk, const float *vals, int64_t ld, const int64_t *perm,
                   float *norms, void *stream) {
  GC_REQUIRE(workers >= 1 && workers <= 65535 && d >= 1 && chunk >= 1 && vals && norms && ld >= d,
             "invalid argument");
  const int64_t nc = (d + chunk - 1) / chunk;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (chunk % 8 == 0 && chunk <= 128) {
    norms_lanes_kernel<<<dim3(grid_for(nc * 8), workers), kNT, 0, st>>>(d, static_cast<int>(chunk), nc, vals, ld,
                                                                       perm, norms, nullptr, nullptr);
  } else {
    norms_generic_kernel<<<dim3(grid_for(nc), workers), kNT, 0, st>>>(d, chunk, nc, vals, ld, perm, norms);
  }
  GC_LAUNCH_CHECK("chunk norms");
  return GC_OK;
}

int gc_chunk_norms_ef(int32_t workers, int64_t d, int64_t chunk, const float *grads, float *resid, int64_t ld,
                      float *norms, void *stream) {
  GC_REQUIRE(workers >= 1 && workers <= 65535 && d >= 1 && chunk >= 1 && grads && norms && ld >= d,
             "invalid argument");
  GC_REQUIRE(chunk % 8 == 0 && chunk <= 128, "fused ef_apply + norms needs chunk % 8 == 0 and chunk <= 128");
  const int64_t nc = (d + chunk - 1) / chunk;
  const bool vec = (ld % 4) == 0 && ((reinterpret_cast<uintptr_t>(grads) | reinterpret_cast<uintptr_t>(resid)) & 15) == 0;
  if (vec) {
    norms_ef_vec_kernel<<<dim3(grid_for(nc * 2), workers), kNT, 0, static_cast<cudaStream_t>(stream)>>>(
        d, static_cast<int>(chunk), nc, grads, resid, ld, norms);
  } else {
    norms_lanes_kernel<<<dim3(grid_for(nc * 8), workers), kNT, 0, static_cast<cudaStream_t>(stream)>>>(
        d, static_cast<int>(chunk), nc, resid ? resid : grads, ld, nullptr, norms, grads, resid);
  }
  GC_LAUNCH_CHECK("norms_lanes_kernel");
  return GC_OK;
}

int gc_chunk_pack(int32_t workers, int64_t d, int64_t chunk, int64_t selected, const int32_t *sel,
                  const float *vals, int64_t ld, const int64_t *perm, float *packs, void *stream) {
  GC_REQUIRE(workers >= 1 && workers <= 65535 && d >= 1 && chunk >= 1 && selected >= 1 && sel && vals && packs,
             "invalid argument");
  pack_kernel<<<dim3(grid_for(selected * chunk), workers), kNT, 0, static_cast<cudaStream_t>(stream)>>>(
      d, chunk, selected, sel, vals, ld, perm, packs);
  GC_LAUNCH_CHECK("pack_kernel");
  return GC_OK;
}

int gc_chunk_scatter(int64_t d, int64_t chunk, int64_t selected, const int32_t *sel, const float *summed,
                     int32_t divisor, const int64_t *perm, float *estimate, void *stream) {
  GC_REQUIRE(d >= 1 && chunk >= 1 && selected >= 1 && divisor >= 1 && sel && summed && estimate,
             "invalid argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(estimate, 0, sizeof(float) * d, st);
  scatter_kernel<<<grid_for(selected * chunk), kNT, 0, st>>>(d, chunk, selected, sel, summed, divisor, perm,
                                                             estimate);
  GC_LAUNCH_CHECK("scatter_kernel");
  return GC_OK;
}

int gc_chunk_ef_update(int32_t workers, int64_t d, int64_t chunk, int64_t selected, const int32_t *sel,
                       const float *packs, const int64_t *perm, float *resid, int64_t ld, void *stream) {
  GC_REQUIRE(workers >= 1 && workers <= 65535 && d >= 1 && chunk >= 1 && selected >= 1 && sel && packs && resid,
             "invalid argument");
  chunk_ef_kernel<<<dim3(grid_for(selected * chunk), workers), kNT, 0, static_cast<cudaStream_t>(stream)>>>(
      d, chunk, selected, sel, packs, perm, resid, ld);
  GC_LAUNCH_CHECK("chunk_ef_kernel");
  return GC_OK;
}

}  // extern "C"
