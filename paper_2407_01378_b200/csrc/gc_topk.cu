// Top-k selection by magnitude with the reference tie-break, and the sparse aggregation.
//
// topk_indices (compressors.py:387-396) = argsort(-|x|, stable)[:k] sorted ascending: the k
// largest |x|, lower index first among equal magnitudes, emitted in ascending index order.
// Used for TopK (pipelines.py:201-211) and for the chunk selection of TopK-Chunked
// (select_chunks, compressors.py:412-414).
//
// B200 design (HBM-bound integer work): keys are the f32 bit patterns with the sign
// cleared (order-preserving for |x|, +-0 equal).  A three-level radix select (11 + 10 + 10
// bits) finds the threshold key T and m = how many elements equal to T are taken.  Only
// three passes touch the whole row:
//   1. level-0 histogram (float4 loads; fused with ef_apply, writing corrected over r);
//   2. collect: per 4096-element tile the count of keys above the level-0 boundary bin, and
//      the boundary bin's elements appended (key, index) to a per-worker candidate list
//      (warp-aggregated atomics; typically < 1 % of the row) -- levels 1 and 2 and the tie
//      counts then run on the candidates only;
//   3. write: per tile, offsets from a scan of the (above, tie) counts.  The collect pass
//      also appends every key above the boundary bin, so the candidate list holds all
//      selected elements (raw f32 bits + index) in per-tile segments: the write pass reads
//      only those segments (~ k + boundary-bin entries, not the row) and ranks each entry by
//      index with two 4096-bit tile bitmaps (selected, ties), so no sort is needed.
// If the candidates overflow the capacity (k above ~len/16, or degenerate inputs such as a
// constant row) the select falls back to full-row passes for levels 1-2, the tile counts
// and the write (ascending emission with warp ballots over the row).  Every
// count is an integer sum, so the result does not depend on the atomic order.  All L rows
// (workers) run in the same launches (grid.y = worker).
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include "gc_device.cuh"
#include "gc_internal.h"

namespace {

constexpr int kNT = 256;
constexpr int kTileE = 4096;          // elements per tile (8 warps x 16 steps x 32 lanes)
constexpr int kSteps = kTileE / kNT;  // 16
// radix digits of the 31-bit magnitude key: 13 + 10 + 8 bits.  The wide level-0 digit (32 bins
// per octave) keeps the boundary bin -- and so the candidate list -- small even when EF piles
// many magnitudes up just below the threshold.
constexpr int kBins0 = 8192, kShift0 = 18, kShift1 = 8;
#ifndef GC_TOPK_H0_CTAS
#define GC_TOPK_H0_CTAS 16
#endif
constexpr int kH0Ctas = GC_TOPK_H0_CTAS * 148;   // persistent level-0 CTAs per worker

constexpr unsigned int kNoGuess = 0xFFFFFFFFu;

struct RowState {  // per worker, lives in the workspace
  unsigned int prefix;     // key bits fixed so far
  unsigned int hint;       // persists across calls: 1 + the previous call's level-0 boundary bin (0: none)
  long long k_rem;         // elements still to take at the current level
  long long gt;            // elements strictly above the current prefix
  unsigned int thresh;     // final threshold key T
  unsigned int guess;      // candidate floor bin of pass 1 (kNoGuess: pass 1 collects nothing)
  long long take_eq;       // m: number of T-keyed elements taken (lowest indices)
  unsigned long long cand_count;   // candidates appended (may exceed the capacity)
  int spec_ok;             // pass 1's candidates are complete: the collect pass is skipped
  unsigned int spec_fail;  // persists: consecutive calls whose speculation failed
  unsigned int calls;      // persists: calls on this workspace
  unsigned int hint2;      // persists: the hint of the call before (trend of the boundary bin)
};

struct Work {
  RowState *state;              // [L]
  unsigned int *hist;           // [L][kBins0]
  unsigned int *tile_gt;        // [L][tiles]
  unsigned int *tile_eq;        // [L][tiles]
  long long *tile_sel_off;      // [L][tiles]
  long long *tile_eq_off;       // [L][tiles]
  unsigned int *cand_key;       // [L][cap]  raw f32 bits of the candidate (sign kept for the value)
  unsigned int *cand_idx;       // [L][cap]
  unsigned long long *tile_cbase;   // [L][tiles] first candidate slot of the tile's segment
  unsigned int *tile_ccnt;      // [L][tiles] candidates the tile appended
  int64_t cap;
};

__host__ __device__ inline int64_t cand_cap_for(int64_t len) {
  const int64_t c = len / 16 > (int64_t{1} << 16) ? len / 16 : (int64_t{1} << 16);
  return c < len ? c : len;
}

__host__ __device__ inline int64_t align256(int64_t x) { return (x + 255) & ~int64_t{255}; }

__host__ __device__ inline Work carve(void *ws, int L, int64_t tiles, int64_t len) {
  char *p = static_cast<char *>(ws);
  Work w;
  w.state = reinterpret_cast<RowState *>(p);
  p += align256(sizeof(RowState) * L);
  w.hist = reinterpret_cast<unsigned int *>(p);
  p += align256(int64_t{4} * kBins0 * L);
  w.tile_gt = reinterpret_cast<unsigned int *>(p);
  p += align256(int64_t{4} * tiles * L);
  w.tile_eq = reinterpret_cast<unsigned int *>(p);
  p += align256(int64_t{4} * tiles * L);
  w.tile_sel_off = reinterpret_cast<long long *>(p);
  p += align256(int64_t{8} * tiles * L);
  w.tile_eq_off = reinterpret_cast<long long *>(p);
  p += align256(int64_t{8} * tiles * L);
  w.tile_cbase = reinterpret_cast<unsigned long long *>(p);
  p += align256(int64_t{8} * tiles * L);
  w.tile_ccnt = reinterpret_cast<unsigned int *>(p);
  p += align256(int64_t{4} * tiles * L);
  w.cap = cand_cap_for(len);
  w.cand_key = reinterpret_cast<unsigned int *>(p);
  p += align256(int64_t{4} * w.cap * L);
  w.cand_idx = reinterpret_cast<unsigned int *>(p);
  return w;
}

int64_t ws_bytes(int L, int64_t tiles, int64_t len) {
  return align256(sizeof(RowState) * L) + align256(int64_t{4} * kBins0 * L) + 3 * align256(int64_t{4} * tiles * L) +
         3 * align256(int64_t{8} * tiles * L) + 2 * align256(int64_t{4} * cand_cap_for(len) * L);
}

__device__ __forceinline__ unsigned int key_of(float x) { return __float_as_uint(x) & 0x7FFFFFFFu; }

// level 0: bits 30..18 (8192 bins); level 1: bits 17..8 for keys with the level-0 prefix;
// level 2: bits 7..0 for keys with the level-1 prefix.
__device__ __forceinline__ int bin_of(unsigned int key, int level, unsigned int prefix) {
  if (level == 0) return static_cast<int>(key >> kShift0);
  if (level == 1) return (key >> kShift0) == prefix ? static_cast<int>((key >> kShift1) & 1023u) : -1;
  return (key >> kShift1) == prefix ? static_cast<int>(key & 255u) : -1;
}

__global__ void __launch_bounds__(kNT) init_kernel(Work wk, int L, int64_t k, int speculate) {
  for (int i = blockIdx.x * kNT + threadIdx.x; i < kBins0 * L; i += gridDim.x * kNT) wk.hist[i] = 0;
  for (int r = blockIdx.x * kNT + threadIdx.x; r < L; r += gridDim.x * kNT) {
    RowState &s = wk.state[r];
    // pass 1 collects the bins >= guess = previous boundary bin - 2 (two 1/32-octave bins of
    // margin) + the bin's last upward step: when the new boundary bin is at or above the guess
    // the collect pass is skipped (verified on the device).  After a failed speculation
    // (threshold falling, or too many candidates) pass 1 stays plain except for a re-probe every
    // 8th call, so an unpredictable workload pays little for the attempt.
    const unsigned int h = s.hint;
    const bool probe = s.spec_fail == 0 || (s.calls & 7u) == 0;
    s.calls = s.calls + 1;
    // a boundary bin that moved up since the call before is expected to keep moving (gradient
    // scales drift over training; EF residuals grow): the guess follows the last step
    const unsigned int h2 = s.hint2;
    const int trend = (h2 >= 1 && h2 <= static_cast<unsigned int>(kBins0) && h > h2) ? static_cast<int>(h - h2) : 0;
    const int g0 = static_cast<int>(h) - 3 + trend;
    s.guess = !speculate || !probe || h == 0 || h > static_cast<unsigned int>(kBins0)
                  ? kNoGuess
                  : static_cast<unsigned int>(g0 > 0 ? (g0 < kBins0 ? g0 : kBins0 - 1) : 0);
    s.spec_ok = 0;
    s.prefix = 0;
    s.k_rem = k;
    s.gt = 0;
    s.thresh = 0;
    s.take_eq = 0;
    s.cand_count = 0;
  }
}

// Optional fused producer for level 0: corrected = f32(g + r) written over r (ef_apply,
// compressors.py:624-626) while building the level-0 histogram of |corrected|.
__global__ void __launch_bounds__(kNT) hist_kernel(Work wk, int level, int64_t len, const float *vals, int64_t ld,
                                                   const float *grads, float *resid) {
  __shared__ unsigned int h[kBins0];
  const int w = blockIdx.y;
  const int nb = level == 0 ? kBins0 : 1024;
  for (int i = threadIdx.x; i < nb; i += kNT) h[i] = 0;
  __syncthreads();
  const unsigned int prefix = wk.state[w].prefix;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTileE;
  const int64_t end = min(base + kTileE, len);
  for (int64_t i = base + threadIdx.x; i < end; i += kNT) {
    float x;
    if (grads) {   // fused ef_apply
      x = grads[w * ld + i];
      if (resid) {
        x = x + resid[w * ld + i];
        resid[w * ld + i] = x;
      }
    } else {
      x = vals[w * ld + i];
    }
    const int b = bin_of(key_of(x), level, prefix);
    if (b >= 0) atomicAdd(&h[b], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < nb; i += kNT)
    if (h[i]) atomicAdd(&wk.hist[w * kBins0 + i], h[i]);
}

// Reserve `mine` consecutive candidate slots per thread for a CTA (warp scans, one global atomic
// per CTA) and return the thread's first slot; the CTA's segment base / size go to the tile.
__device__ __forceinline__ unsigned long long reserve_slots(unsigned int mine, RowState &st, unsigned int *s_wcnt,
                                                            unsigned long long *s_base, unsigned int *s_tot,
                                                            unsigned long long *tile_cbase, unsigned int *tile_ccnt) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int incl = mine;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_wcnt[warp] = incl;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int tot = 0;
    for (int j = 0; j < kNT / 32; ++j) {
      const unsigned int c = s_wcnt[j];
      s_wcnt[j] = tot;
      tot += c;
    }
    const unsigned long long b = tot ? atomicAdd(&st.cand_count, static_cast<unsigned long long>(tot)) : 0ull;
    *s_base = b;
    *s_tot = tot;
    *tile_cbase = b;
    *tile_ccnt = tot;
  }
  __syncthreads();
  return *s_base + s_wcnt[warp] + (incl - mine);
}

// Level 0 with float4 loads (aligned rows): persistent CTAs walk the tiles of their worker and
// keep the 8192-bin histogram in shared memory (one flush per CTA).  Per tile a thread's 16
// elements are 4 float4 at stride 256 (element 4 * (tid + 256u) + q), all loads issued before
// the shared-memory atomics.  grads != NULL fuses ef_apply.  With a guess bin from the previous
// call, elements in bins >= guess are appended to the candidate list as the tile's segment
// (pass 2 then only runs if the guess turns out above the new boundary bin).
__global__ void __launch_bounds__(kNT) hist0_vec_kernel(Work wk, int64_t len, const float *vals, int64_t ld,
                                                        const float *grads, float *resid, int64_t tiles) {
  __shared__ unsigned int h[kBins0];
  __shared__ unsigned int s_wcnt[kNT / 32];
  __shared__ unsigned long long s_base;
  __shared__ unsigned int s_tot;
  const int w = blockIdx.y;
  RowState &st = wk.state[w];
  const unsigned int guess = st.guess;
  for (int i = threadIdx.x; i < kBins0; i += kNT) h[i] = 0;
  __syncthreads();
  const float *src = grads ? grads + w * ld : vals + w * ld;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t base = tile * kTileE;
    float4 x[4];
    unsigned int valid = 0xFFFFu;
    if (base + kTileE <= len) {
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = __ldcs(reinterpret_cast<const float4 *>(src + base) + threadIdx.x + kNT * u);
      if (grads && resid) {
        float4 *rr = reinterpret_cast<float4 *>(resid + w * ld + base);
        float4 r4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) r4[u] = __ldcs(rr + threadIdx.x + kNT * u);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          x[u].x = x[u].x + r4[u].x; x[u].y = x[u].y + r4[u].y; x[u].z = x[u].z + r4[u].z; x[u].w = x[u].w + r4[u].w;
          rr[threadIdx.x + kNT * u] = x[u];
        }
      }
    } else {
      valid = 0u;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        float t[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int64_t i = base + 4 * (threadIdx.x + kNT * u) + q;
          float v = 0.0f;
          if (i < len) {
            v = src[i];
            if (grads && resid) {
              v = v + resid[w * ld + i];
              resid[w * ld + i] = v;
            }
            valid |= 1u << (4 * u + q);
          }
          t[q] = v;
        }
        x[u] = make_float4(t[0], t[1], t[2], t[3]);
      }
    }
    unsigned int bits[16];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bits[4 * u] = __float_as_uint(x[u].x); bits[4 * u + 1] = __float_as_uint(x[u].y);
      bits[4 * u + 2] = __float_as_uint(x[u].z); bits[4 * u + 3] = __float_as_uint(x[u].w);
    }
    unsigned int cmask = 0;
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const unsigned int b0 = (bits[e] & 0x7FFFFFFFu) >> kShift0;
      if ((valid >> e) & 1u) {
        atomicAdd(&h[b0], 1u);
        cmask |= (b0 >= guess ? 1u : 0u) << e;
      }
    }
    if (guess != kNoGuess) {   // grid-uniform
      unsigned long long pos = reserve_slots(__popc(cmask), st, s_wcnt, &s_base, &s_tot,
                                             &wk.tile_cbase[w * tiles + tile], &wk.tile_ccnt[w * tiles + tile]);
      while (cmask) {
        const int e = __ffs(cmask) - 1;
        cmask &= cmask - 1u;
        if (pos < static_cast<unsigned long long>(wk.cap)) {
          wk.cand_key[w * wk.cap + pos] = bits[e];
          wk.cand_idx[w * wk.cap + pos] = static_cast<unsigned int>(base + 4 * (threadIdx.x + kNT * (e >> 2)) + (e & 3));
        }
        ++pos;
      }
      __syncthreads();   // s_wcnt / s_base are reused by the next tile
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins0; i += kNT)
    if (h[i]) atomicAdd(&wk.hist[w * kBins0 + i], h[i]);
}

// Pass 2 (skipped when pass 1's guess held): per tile, every element at or above the level-0
// boundary bin p0 (raw bits, index) is appended to the worker's candidate list as the tile's
// segment (tile_cbase / tile_ccnt).  Persistent CTAs walk the tiles.
__global__ void __launch_bounds__(kNT) collect_kernel(Work wk, int64_t len, const float *vals, int64_t ld,
                                                      int64_t tiles, int vec) {
  __shared__ unsigned int s_wcnt[kNT / 32];
  __shared__ unsigned int s_tot;
  __shared__ unsigned long long s_base;
  const int w = blockIdx.y;
  RowState &st = wk.state[w];
  if (st.spec_ok) return;
  const unsigned int p0 = st.prefix;
  const float *row = vals + w * ld;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t base = tile * kTileE;
    unsigned int keys[kSteps];   // raw f32 bits; element 4 * (tid + 256u) + q  <->  keys[4u + q]
    unsigned int cmask = 0;
    if (vec && base + kTileE <= len) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 x = __ldcs(reinterpret_cast<const float4 *>(row + base) + threadIdx.x + kNT * u);
        keys[4 * u + 0] = __float_as_uint(x.x);
        keys[4 * u + 1] = __float_as_uint(x.y);
        keys[4 * u + 2] = __float_as_uint(x.z);
        keys[4 * u + 3] = __float_as_uint(x.w);
      }
#pragma unroll
      for (int e = 0; e < kSteps; ++e) cmask |= (((keys[e] & 0x7FFFFFFFu) >> kShift0) >= p0 ? 1u : 0u) << e;
    } else {
#pragma unroll
      for (int e = 0; e < kSteps; ++e) {
        const int64_t i = base + 4 * (threadIdx.x + kNT * (e >> 2)) + (e & 3);
        keys[e] = i < len ? __float_as_uint(row[i]) : 0u;
        cmask |= (i < len && ((keys[e] & 0x7FFFFFFFu) >> kShift0) >= p0 ? 1u : 0u) << e;
      }
    }
    unsigned long long pos = reserve_slots(__popc(cmask), st, s_wcnt, &s_base, &s_tot,
                                           &wk.tile_cbase[w * tiles + tile], &wk.tile_ccnt[w * tiles + tile]);
    while (cmask) {
      const int e = __ffs(cmask) - 1;
      cmask &= cmask - 1u;
      if (pos < static_cast<unsigned long long>(wk.cap)) {
        wk.cand_key[w * wk.cap + pos] = keys[e];
        wk.cand_idx[w * wk.cap + pos] = static_cast<unsigned int>(base + 4 * (threadIdx.x + kNT * (e >> 2)) + (e & 3));
      }
      ++pos;
    }
    __syncthreads();   // s_wcnt / s_base are reused by the next tile
  }
}

// Levels 1 and 2 over the candidates (grid-stride); on overflow, over the whole row.
__global__ void __launch_bounds__(kNT) cand_hist_kernel(Work wk, int level, int64_t len, const float *vals,
                                                        int64_t ld) {
  __shared__ unsigned int h[1024];
  const int w = blockIdx.y;
  for (int i = threadIdx.x; i < 1024; i += kNT) h[i] = 0;
  __syncthreads();
  const RowState &st = wk.state[w];
  const unsigned int prefix = st.prefix;
  const int64_t nc = static_cast<int64_t>(st.cand_count);
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kNT;
  if (nc <= wk.cap) {
    const unsigned int *ck = wk.cand_key + w * wk.cap;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < nc; e += stride) {
      const int b = bin_of(ck[e] & 0x7FFFFFFFu, level, prefix);
      if (b >= 0) atomicAdd(&h[b], 1u);
    }
  } else {
    const float *row = vals + w * ld;
    for (int64_t i = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; i < len; i += stride) {
      const int b = bin_of(key_of(row[i]), level, prefix);
      if (b >= 0) atomicAdd(&h[b], 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 1024; i += kNT)
    if (h[i]) atomicAdd(&wk.hist[w * kBins0 + i], h[i]);
}

// Tile counts of the candidates above / equal to T: one warp per tile walks the tile's segment
// (no atomics).  On overflow the counts come from the whole row.
__global__ void __launch_bounds__(kNT) cand_tile_kernel(Work wk, int64_t len, const float *vals, int64_t ld,
                                                        int64_t tiles) {
  const int w = blockIdx.y;
  const RowState &st = wk.state[w];
  const unsigned int T = st.thresh;
  const int64_t nc = static_cast<int64_t>(st.cand_count);
  if (nc <= wk.cap) {
    const int lane = threadIdx.x & 31;
    const unsigned int *ck = wk.cand_key + w * wk.cap;
    for (int64_t t = blockIdx.x * static_cast<int64_t>(kNT / 32) + (threadIdx.x >> 5); t < tiles;
         t += static_cast<int64_t>(gridDim.x) * (kNT / 32)) {
      const unsigned long long cb = wk.tile_cbase[w * tiles + t];
      const unsigned int cn = wk.tile_ccnt[w * tiles + t];
      unsigned int gt = 0, eq = 0;
      for (unsigned int e = lane; e < cn; e += 32) {
        const unsigned int key = ck[cb + e] & 0x7FFFFFFFu;
        gt += key > T;
        eq += key == T;
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        gt += __shfl_xor_sync(0xffffffffu, gt, o);
        eq += __shfl_xor_sync(0xffffffffu, eq, o);
      }
      if (lane == 0) {
        wk.tile_gt[w * tiles + t] = gt;
        wk.tile_eq[w * tiles + t] = eq;
      }
    }
    return;
  }
  const float *row = vals + w * ld;
  for (int64_t t = blockIdx.x; t < tiles; t += gridDim.x) {   // overflow: one CTA per tile
    const int64_t base = t * kTileE, end = min(base + kTileE, len);
    unsigned int gt = 0, eq = 0;
    for (int64_t i = base + threadIdx.x; i < end; i += kNT) {
      const unsigned int key = key_of(row[i]);
      gt += key > T;
      eq += key == T;
    }
    using R = cub::BlockReduce<unsigned int, kNT>;
    __shared__ typename R::TempStorage t1, t2;
    const unsigned int sgt = R(t1).Sum(gt);
    const unsigned int seq = R(t2).Sum(eq);
    if (threadIdx.x == 0) {
      wk.tile_gt[w * tiles + t] = sgt;
      wk.tile_eq[w * tiles + t] = seq;
    }
    __syncthreads();
  }
}

// One CTA per worker: find bin b (scanning bins from the top) with
// above < k_rem <= above + count[b]; extend the prefix; reset the histogram.
__global__ void __launch_bounds__(1024) find_kernel(Work wk, int level) {
  using Scan = cub::BlockScan<unsigned long long, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int found;
  __shared__ unsigned long long s_above, s_krem;
  const int w = blockIdx.x;
  RowState &s = wk.state[w];
  const int nb = level == 0 ? kBins0 : (level == 1 ? 1024 : 256);
  constexpr int kPerMax = kBins0 / 1024;
  const int per = nb >= 1024 ? nb / 1024 : 1;   // bins per thread, owned top-down
  if (threadIdx.x == 0) {
    found = -1;
    s_krem = static_cast<unsigned long long>(s.k_rem);
  }
  unsigned int *h = wk.hist + w * kBins0;
  unsigned int c[kPerMax] = {};
  unsigned long long local = 0;
#pragma unroll
  for (int j = 0; j < kPerMax; ++j) {
    const int bi = threadIdx.x * per + j;
    c[j] = (j < per && bi < nb) ? h[nb - 1 - bi] : 0u;
    local += c[j];
  }
  unsigned long long excl;
  Scan(tmp).ExclusiveSum(local, excl);
  __syncthreads();
  const unsigned long long k_rem = s_krem;
  unsigned long long run = excl;
#pragma unroll
  for (int j = 0; j < kPerMax; ++j) {
    if (j < per && run < k_rem && k_rem <= run + c[j]) {   // exactly one bin qualifies (c[j] > 0)
      found = nb - 1 - (threadIdx.x * per + j);
      s_above = run;
    }
    run += c[j];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int b = static_cast<unsigned int>(found);
    s.gt += static_cast<long long>(s_above);
    s.k_rem = static_cast<long long>(k_rem - s_above);
    s.prefix = (level == 0) ? b : (level == 1 ? ((s.prefix << 10) | b) : ((s.prefix << 8) | b));
    if (level == 0) {   // pass 1's candidates hold every bin >= guess: complete iff b >= guess
      const bool ok = s.guess != kNoGuess && b >= s.guess && s.cand_count <= static_cast<unsigned long long>(wk.cap);
      s.spec_ok = ok ? 1 : 0;
      if (s.guess != kNoGuess) s.spec_fail = ok ? 0u : s.spec_fail + 1u;
      if (!ok) s.cand_count = 0;   // pass 2 rebuilds the list
      s.hint2 = s.hint;
      s.hint = b + 1;
    }
    if (level == 2) {
      s.thresh = s.prefix;
      s.take_eq = s.k_rem;
    }
  }
  for (int i = threadIdx.x; i < kBins0; i += 1024) h[i] = 0;
}

// One CTA per worker: eq prefix (tie ranks) and selected-count prefix (output offsets).
__global__ void __launch_bounds__(1024) tile_scan_kernel(Work wk, int64_t tiles) {
  // kItems consecutive tiles per thread: a thread-local scan plus one block scan per 4096 tiles
  // (the block scans are the serial part: 7 steps instead of 27 at cfg3's 27K tiles).  Counts
  // and offsets fit int32: rows are shorter than 2^31 (gc_topk_select checks it).
  constexpr int kItems = 4;
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry_eq, carry_sel;
  const int w = blockIdx.x;
  const int m = static_cast<int>(wk.state[w].take_eq);
  if (threadIdx.x == 0) carry_eq = carry_sel = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < tiles; t0 += 1024 * kItems) {
    const int64_t tb = t0 + static_cast<int64_t>(threadIdx.x) * kItems;
    int eq[kItems], gt[kItems], eq_local = 0;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int64_t t = tb + j;
      eq[j] = t < tiles ? static_cast<int>(wk.tile_eq[w * tiles + t]) : 0;
      gt[j] = t < tiles ? static_cast<int>(wk.tile_gt[w * tiles + t]) : 0;
      eq_local += eq[j];
    }
    int eq_ex;
    Scan(tmp).ExclusiveSum(eq_local, eq_ex);
    __syncthreads();
    int eq_run = eq_ex + carry_eq, sel_local = 0, sel[kItems], eq_ofs[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      eq_ofs[j] = eq_run;
      int take = m - eq_run;
      take = take < 0 ? 0 : (take > eq[j] ? eq[j] : take);
      sel[j] = gt[j] + take;
      sel_local += sel[j];
      eq_run += eq[j];
    }
    int sel_ex, sel_tot;
    Scan(tmp).ExclusiveSum(sel_local, sel_ex, sel_tot);
    __syncthreads();
    int sel_run = sel_ex + carry_sel;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const int64_t t = tb + j;
      if (t < tiles) {
        wk.tile_eq_off[w * tiles + t] = eq_ofs[j];
        wk.tile_sel_off[w * tiles + t] = sel_run;
      }
      sel_run += sel[j];
    }
    __syncthreads();
    if (threadIdx.x == 1023) carry_eq = eq_run;
    if (threadIdx.x == 0) carry_sel += sel_tot;
    __syncthreads();
  }
}

// Emit selected indices in ascending order (and optionally fp16-rounded values).  Each warp
// owns kSteps groups of 32 consecutive elements; a group with no key >= T (most of them at
// 1 % density) costs one ballot.  Ties (key == T) are taken in index order up to m.
__global__ void __launch_bounds__(kNT) write_kernel(Work wk, int64_t len, const float *vals, int64_t ld,
                                                    int64_t tiles, int64_t k, int32_t *idx_out, float *val_out,
                                                    int fp16_vals, float *resid) {
  __shared__ unsigned int s_eq[kNT / 32], s_sel[kNT / 32];
  // fallback only: the candidate write (cand_write_kernel) covers every row that fit the list
  if (wk.state[blockIdx.y].cand_count <= static_cast<unsigned long long>(wk.cap)) return;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int w = blockIdx.y;
    const unsigned int T = wk.state[w].thresh;
    const long long m = wk.state[w].take_eq;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t base = static_cast<int64_t>(tile) * kTileE + warp * (kSteps * 32);
    const unsigned int lt_mask = (1u << lane) - 1u;
    const float *row = vals + w * ld;
    unsigned int keys[kSteps];
    if (base + kSteps * 32 <= len) {
  #pragma unroll
      for (int s = 0; s < kSteps; ++s) keys[s] = key_of(__ldcs(row + base + s * 32 + lane));
    } else {
  #pragma unroll
      for (int s = 0; s < kSteps; ++s) {
        const int64_t i = base + s * 32 + lane;
        keys[s] = i < len ? key_of(row[i]) : 0u;   // key 0 <= T: never selected past the end
      }
    }
    // masks per group: ge (key >= T) and eq (key == T); padding lanes read key 0
    unsigned int gem[kSteps], eqm[kSteps];
    unsigned int eq_tot = 0;
    const bool t_zero = T == 0u;
  #pragma unroll
    for (int s = 0; s < kSteps; ++s) {
      const bool valid = base + s * 32 + lane < len;
      gem[s] = __ballot_sync(0xffffffffu, valid && keys[s] >= T);
      eqm[s] = 0u;
      if (gem[s]) {
        eqm[s] = __ballot_sync(0xffffffffu, valid && keys[s] == T);
        eq_tot += __popc(eqm[s]);
      }
    }
    (void)t_zero;
    if (lane == 0) s_eq[warp] = eq_tot;
    __syncthreads();
    long long eq_run = wk.tile_eq_off[w * tiles + tile];
    for (int j = 0; j < warp; ++j) eq_run += s_eq[j];
    unsigned int sel_tot = 0;
  #pragma unroll
    for (int s = 0; s < kSteps; ++s) {
      unsigned int sm = gem[s] & ~eqm[s];   // strictly above T: always taken
      if (eqm[s]) {
        // ties: the first max(0, min(popc, m - eq_run)) set bits of eqm, in lane (= index) order
        const long long room = m - eq_run;
        const int take = room <= 0 ? 0 : (room >= 32 ? 32 : static_cast<int>(room));
        unsigned int e = eqm[s];
        for (int t = 0; t < take && e; ++t) {
          const unsigned int lowbit = e & (0u - e);
          sm |= lowbit;
          e ^= lowbit;
        }
        eq_run += __popc(eqm[s]);
      }
      gem[s] = sm;   // reuse as the selected mask
      sel_tot += __popc(sm);
    }
    if (lane == 0) s_sel[warp] = sel_tot;
    __syncthreads();
    long long out = wk.tile_sel_off[w * tiles + tile];
    for (int j = 0; j < warp; ++j) out += s_sel[j];
  #pragma unroll
    for (int s = 0; s < kSteps; ++s) {
      const unsigned int sm = gem[s];
      if (sm) {
        if ((sm >> lane) & 1u) {
          const long long pos = out + __popc(sm & lt_mask);
          const int64_t i = base + s * 32 + lane;
          if (pos < k) {
            idx_out[w * k + pos] = static_cast<int32_t>(i);
            if (val_out) {
              const float x = row[i];
              val_out[w * k + pos] = fp16_vals ? gc::fp16_round_trip(x) : x;
            }
            if (resid) {   // fused ef_update (the corrected row is resid itself)
              const float x = row[i];
              resid[w * ld + i] = x - (fp16_vals ? gc::fp16_round_trip(x) : x);
            }
          }
        }
        out += __popc(sm);
      }
    }
    __syncthreads();   // s_eq / s_sel are reused by the next tile
  }
}

// write_kernel with float4 loads (aligned rows): a warp owns 512 consecutive elements as 4
// steps of 128, lane l holding elements 128u + 4l .. 128u + 4l + 3 of step u (index order =
// step, lane, element).  Tie ranks and output positions come from warp scans per step, skipped
// (one ballot) when a step has no tie / no selected element.
__device__ __forceinline__ unsigned int warp_excl_scan(unsigned int v, int lane, unsigned int &total) {
  unsigned int incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  total = __shfl_sync(0xffffffffu, incl, 31);
  return incl - v;
}

__global__ void __launch_bounds__(kNT) write_vec_kernel(Work wk, int64_t len, const float *vals, int64_t ld,
                                                        int64_t tiles, int64_t k, int32_t *idx_out, float *val_out,
                                                        int fp16_vals, float *resid) {
  __shared__ unsigned int s_eq[kNT / 32], s_sel[kNT / 32];
  // fallback only: the candidate write (cand_write_kernel) covers every row that fit the list
  if (wk.state[blockIdx.y].cand_count <= static_cast<unsigned long long>(wk.cap)) return;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int w = blockIdx.y;
    const unsigned int T = wk.state[w].thresh;
    const long long m = wk.state[w].take_eq;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t wbase = static_cast<int64_t>(tile) * kTileE + warp * 512;
    const float *row = vals + w * ld;
    unsigned int keys[16];
    if (wbase + 512 <= len) {
  #pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 x = __ldcs(reinterpret_cast<const float4 *>(row + wbase + 128 * u) + lane);
        keys[4 * u] = key_of(x.x); keys[4 * u + 1] = key_of(x.y); keys[4 * u + 2] = key_of(x.z); keys[4 * u + 3] = key_of(x.w);
      }
    } else {
  #pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int64_t i = wbase + 128 * (e >> 2) + 4 * lane + (e & 3);
        keys[e] = i < len ? key_of(row[i]) : 0u;   // key 0 is never above T; never a tie past len
      }
    }
    auto valid = [&](int e) { return wbase + 128 * (e >> 2) + 4 * lane + (e & 3) < len; };
    unsigned int eqbits = 0, gtbits = 0;
  #pragma unroll
    for (int e = 0; e < 16; ++e) {
      const bool v = valid(e);
      eqbits |= (v && keys[e] == T) ? (1u << e) : 0u;
      gtbits |= (v && keys[e] > T) ? (1u << e) : 0u;
    }
    unsigned int weq = __popc(eqbits);
  #pragma unroll
    for (int o = 16; o; o >>= 1) weq += __shfl_xor_sync(0xffffffffu, weq, o);
    if (lane == 0) s_eq[warp] = weq;
    __syncthreads();
    long long eq_run = wk.tile_eq_off[w * tiles + tile];
    for (int j = 0; j < warp; ++j) eq_run += s_eq[j];
    unsigned int selbits = gtbits;
    if (__any_sync(0xffffffffu, eqbits != 0u)) {   // ties: the first m (index order) are taken
  #pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned int eu = (eqbits >> (4 * u)) & 0xFu;
        unsigned int tot;
        const unsigned int ex = warp_excl_scan(__popc(eu), lane, tot);
        long long rank = eq_run + ex;
  #pragma unroll
        for (int q = 0; q < 4; ++q)
          if ((eu >> q) & 1u) {
            if (rank < m) selbits |= 1u << (4 * u + q);
            ++rank;
          }
        eq_run += tot;
      }
    }
    unsigned int wsel = __popc(selbits);
  #pragma unroll
    for (int o = 16; o; o >>= 1) wsel += __shfl_xor_sync(0xffffffffu, wsel, o);
    if (lane == 0) s_sel[warp] = wsel;
    __syncthreads();
    long long out = wk.tile_sel_off[w * tiles + tile];
    for (int j = 0; j < warp; ++j) out += s_sel[j];
  #pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned int su = (selbits >> (4 * u)) & 0xFu;
      if (!__any_sync(0xffffffffu, su != 0u)) continue;
      unsigned int tot;
      long long pos = out + warp_excl_scan(__popc(su), lane, tot);
  #pragma unroll
      for (int q = 0; q < 4; ++q)
        if ((su >> q) & 1u) {
          const int64_t i = wbase + 128 * u + 4 * lane + q;
          if (pos < k) {
            idx_out[w * k + pos] = static_cast<int32_t>(i);
            if (val_out) {
              const float x = row[i];
              val_out[w * k + pos] = fp16_vals ? gc::fp16_round_trip(x) : x;
            }
            if (resid) {   // fused ef_update (the corrected row is resid itself)
              const float x = row[i];
              resid[w * ld + i] = x - (fp16_vals ? gc::fp16_round_trip(x) : x);
            }
          }
          ++pos;
        }
      out += tot;
    }
    __syncthreads();   // s_eq / s_sel are reused by the next tile
  }
}

// Pass 3 from the candidate segments, one warp per tile: tile t's selected elements are its
// segment's entries with key > T plus its ties (key == T) whose global tie rank (tile_eq_off +
// rank in the tile) is below m.  Index ranks come from two 4096-bit bitmaps per warp (ties,
// selected; lane l owns words 4l..4l+3) and a warp prefix popcount, so no sort is needed.
// With ef != 0 the own payload is subtracted in place: resid[i] = x - val (ef_update,
// compressors.py:629-631; x is the corrected value the candidate carries).
__global__ void __launch_bounds__(kNT) cand_write_kernel(Work wk, int64_t tiles, int64_t k, int32_t *idx_out,
                                                         float *val_out, int fp16_vals, float *resid, int64_t ld) {
  constexpr int kWords = kTileE / 32;   // 128
  __shared__ unsigned int s_bits[kNT / 32][2][kWords];
  const int w = blockIdx.y;
  const RowState &st = wk.state[w];
  if (st.cand_count > static_cast<unsigned long long>(wk.cap)) return;   // overflow: full-row write
  const unsigned int T = st.thresh;
  const long long m = st.take_eq;
  const unsigned int *ck = wk.cand_key + w * wk.cap, *ci = wk.cand_idx + w * wk.cap;
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  unsigned int *eqw = s_bits[wp][0], *selw = s_bits[wp][1];
  for (int64_t tile = blockIdx.x * static_cast<int64_t>(kNT / 32) + wp; tile < tiles;
       tile += static_cast<int64_t>(gridDim.x) * (kNT / 32)) {
    const unsigned long long cb = wk.tile_cbase[w * tiles + tile];
    const unsigned int cn = wk.tile_ccnt[w * tiles + tile];
    if (cn == 0) continue;
    const long long sel_off = wk.tile_sel_off[w * tiles + tile];
    const long long eq_off = wk.tile_eq_off[w * tiles + tile];
    const unsigned int tbase = static_cast<unsigned int>(tile * kTileE);
#pragma unroll
    for (int j = 0; j < 4; ++j) eqw[4 * lane + j] = 0u, selw[4 * lane + j] = 0u;
    __syncwarp();
    for (unsigned int e = lane; e < cn; e += 32) {
      const unsigned int key = ck[cb + e] & 0x7FFFFFFFu, pos = ci[cb + e] - tbase;
      if (key > T) atomicOr(&selw[pos >> 5], 1u << (pos & 31));
      else if (key == T) atomicOr(&eqw[pos >> 5], 1u << (pos & 31));
    }
    __syncwarp();
    unsigned int ew[4], sw[4], ec = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) ew[j] = eqw[4 * lane + j], sw[j] = selw[4 * lane + j], ec += __popc(ew[j]);
    if (__any_sync(0xffffffffu, ec != 0u)) {   // ties in index order up to m
      unsigned int incl = ec;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      long long rank = eq_off + (incl - ec);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        unsigned int e = ew[j];
        while (e && rank < m) {
          const unsigned int low = e & (0u - e);
          sw[j] |= low;
          e ^= low;
          ++rank;
        }
        rank += __popc(e);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) selw[4 * lane + j] = sw[j];
    }
    unsigned int sc = __popc(sw[0]) + __popc(sw[1]) + __popc(sw[2]) + __popc(sw[3]);
    unsigned int incl = sc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    // exclusive prefix of selected bits before each of the lane's words, published in eqw
    unsigned int ex = incl - sc;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      eqw[4 * lane + j] = ex;
      ex += __popc(sw[j]);
    }
    __syncwarp();
    for (unsigned int e = lane; e < cn; e += 32) {
      const unsigned int pos = ci[cb + e] - tbase, wd = pos >> 5, bit = 1u << (pos & 31);
      const unsigned int sword = selw[wd];
      if (sword & bit) {
        const long long o = sel_off + eqw[wd] + __popc(sword & (bit - 1u));
        if (o < k) {
          const float x = __uint_as_float(ck[cb + e]);
          const float v = fp16_vals ? gc::fp16_round_trip(x) : x;
          idx_out[w * k + o] = static_cast<int32_t>(tbase + pos);
          if (val_out) val_out[w * k + o] = v;
          if (resid) resid[w * ld + tbase + pos] = x - v;
        }
      }
    }
    __syncwarp();   // bitmaps are reused by the warp's next tile
  }
}

// ---------------------------------------------------------------- sparse aggregation
// estimate[idx] += val for one worker's payload (indices unique within a payload), launched
// once per worker in worker order: the f32 sum per coordinate follows the reference's
// np.add.at order (pipelines.py:206-209).
__global__ void scatter_add_kernel(int64_t k, const int32_t *idx, const float *val, float *acc) {
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < k;
       e += static_cast<int64_t>(gridDim.x) * kNT)
    acc[idx[e]] += val[e];
}

// Tiled sparse mean (pipelines.py:204-211 + the / n): one warp builds the estimate of a
// 1024-coordinate tile in shared memory from each worker's entries in [start[w][t],
// start[w][t+1]) -- worker by worker (__syncwarp between), so every coordinate sees the
// np.add.at order -- and writes it once, divided by n.  The payload indices are ascending per
// worker, so the tile starts come from one pass over them.
constexpr int kMeanTile = 1024;

__global__ void sparse_tile_starts_kernel(int L, int64_t k, const int32_t *idx, int64_t tiles, int32_t *start) {
  const int w = blockIdx.y;
  const int32_t *iw = idx + w * k;
  int32_t *sw = start + w * (tiles + 1);
  for (int64_t j = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; j <= k;
       j += static_cast<int64_t>(gridDim.x) * kNT) {
    // entry j opens tiles (tile(idx[j-1]), tile(idx[j])]; j == k closes the list
    const int64_t lo = j == 0 ? -1 : iw[j - 1] / kMeanTile;
    const int64_t hi = j == k ? tiles : iw[j] / kMeanTile;
    for (int64_t t = lo + 1; t <= hi; ++t) sw[t] = static_cast<int32_t>(j);
  }
}

__global__ void __launch_bounds__(kNT) sparse_mean_kernel(int L, int64_t k, const int32_t *idx, const float *val,
                                                          int64_t dim, int64_t tiles, const int32_t *start,
                                                          int divisor, float *est) {
  __shared__ __align__(16) float acc_all[kNT / 32][kMeanTile];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  float *acc = acc_all[wp];
  const gc::DivN dv(divisor);
  const bool a16 = (reinterpret_cast<uintptr_t>(est) & 15) == 0;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(kNT / 32) + wp; t < tiles;
       t += static_cast<int64_t>(gridDim.x) * (kNT / 32)) {
    const int64_t base = t * kMeanTile;
#pragma unroll
    for (int i = 0; i < kMeanTile / 128; ++i)
      reinterpret_cast<float4 *>(acc)[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
    __syncwarp();
    // one round trip for the tile's entry ranges of all workers (lane w < L), then the entries
    // of the concatenated worker-ordered list loaded in chunks of 32 * kE ahead of their adds
    for (int w0 = 0; w0 < L; w0 += 32) {   // groups of 32 workers
      const int nw = min(32, L - w0);
      int32_t my0 = 0, mycnt = 0;
      if (lane < nw) {
        my0 = start[(w0 + lane) * (tiles + 1) + t];
        mycnt = start[(w0 + lane) * (tiles + 1) + t + 1] - my0;
      }
      int32_t incl = mycnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const int32_t excl = incl - mycnt;
      constexpr int kE = 4;
      for (int32_t q0 = 0; q0 < total; q0 += 32 * kE) {
        int wq[kE];
        int32_t iq[kE];
        float vq[kE];
#pragma unroll
        for (int e = 0; e < kE; ++e) {
          const int32_t q = q0 + lane + 32 * e;
          int ww = 0;   // the worker whose [excl, excl + cnt) holds q (all lanes shuffle)
          for (int u = 1; u < nw; ++u)
            if (q >= __shfl_sync(0xffffffffu, excl, u)) ww = u;
          const int32_t j = __shfl_sync(0xffffffffu, my0, ww) + (q - __shfl_sync(0xffffffffu, excl, ww));
          wq[e] = q < total ? ww : -1;
          iq[e] = 0;
          vq[e] = 0.0f;
          if (q < total) {
            iq[e] = idx[(w0 + ww) * k + j];
            vq[e] = val[(w0 + ww) * k + j];
          }
        }
        for (int ww = 0; ww < nw; ++ww) {   // worker order; indices unique within a worker
#pragma unroll
          for (int e = 0; e < kE; ++e)
            if (wq[e] == ww) acc[iq[e] - base] += vq[e];
          __syncwarp();
        }
      }
    }
    if (a16 && base + kMeanTile <= dim) {
#pragma unroll
      for (int i = 0; i < kMeanTile / 128; ++i) {
        const float4 a = reinterpret_cast<const float4 *>(acc)[lane + 32 * i];
        __stcs(reinterpret_cast<float4 *>(est + base) + lane + 32 * i,
               make_float4(dv(a.x), dv(a.y), dv(a.z), dv(a.w)));
      }
    } else {
      for (int i = lane; i < kMeanTile && base + i < dim; i += 32) est[base + i] = dv(acc[i]);
    }
    __syncwarp();   // the tile buffer is reused by the warp's next tile
  }
}

// resid[idx] = resid[idx] - val (ef_update at the selected coordinates; elsewhere own = 0).
__global__ void sparse_ef_kernel(int L, int64_t k, const int32_t *idx, const float *val, float *resid, int64_t ld) {
  const int w = blockIdx.y;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < k;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const int64_t i = idx[w * k + e];
    resid[w * ld + i] = resid[w * ld + i] - val[w * k + e];
  }
}

// SparsePayload wire bytes (compressors.py:294-297): <B 1><I k><i4 idx * k><f2 val * k>, one
// row per worker; values are fp16-valued floats, so the half conversion is exact.
__global__ void encode_sparse_kernel(int L, int64_t k, const int32_t *idx, const float *val, uint8_t *out,
                                     int64_t stride) {
  const int64_t total = static_cast<int64_t>(L) * k;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = e / k, j = e - w * k;
    uint8_t *row = out + w * stride;
    if (j == 0) {
      row[0] = 1;
      for (int b = 0; b < 4; ++b) row[1 + b] = static_cast<uint8_t>(static_cast<uint64_t>(k) >> (8 * b));
    }
    const uint32_t iv = static_cast<uint32_t>(idx[e]);
    for (int b = 0; b < 4; ++b) row[5 + 4 * j + b] = static_cast<uint8_t>(iv >> (8 * b));
    // fp16 bits straight from cvt: nvcc 12.9 folds uint8_t(__half_as_ushort(h)) into a saturating
    // F2I.U8.F16 *value* conversion (also from a 16-bit cvt result), so the low byte would come out as 0 / 255
    uint32_t hv;   // packed cvt: fp16(val) in the low half of a 32-bit register
    asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(hv) : "f"(0.0f), "f"(val[e]));
    row[5 + 4 * k + 2 * j] = static_cast<uint8_t>(hv);
    row[5 + 4 * k + 2 * j + 1] = static_cast<uint8_t>(hv >> 8);
  }
}

// QuantPayload wire bytes (compressors.py:305-317): <B 3><B q><I block><I num_codes><I num_blocks>
// <i1 codes * num_codes><f4 ranges * 2 num_blocks><Q rotation_id>, one row per worker.  Codes /
// ranges past the given lengths (the all-zero padded tail the engine skips) are zero.  One thread
// per output byte: the row is HBM-bound byte traffic, the header costs nothing.
__global__ void encode_quant_kernel(int L, int q, int64_t block, int64_t num_codes, const int8_t *codes,
                                    int64_t codes_ld, int64_t codes_len, int64_t num_blocks, const float *ranges,
                                    int64_t ranges_len, unsigned long long rot, uint8_t *out, int64_t stride,
                                    int64_t row_bytes) {
  const int64_t total = static_cast<int64_t>(L) * row_bytes;
  const int64_t c0 = 14, r0 = c0 + num_codes, t0 = r0 + 8 * num_blocks;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = e / row_bytes, p = e - w * row_bytes;
    uint8_t b;
    if (p >= c0 && p < r0) {
      const int64_t i = p - c0;
      b = i < codes_len ? static_cast<uint8_t>(codes[w * codes_ld + i]) : 0;
    } else if (p >= r0 && p < t0) {
      const int64_t j = (p - r0) >> 2;   // float index into ranges [num_blocks][2]
      const uint32_t bits = j < 2 * ranges_len ? __float_as_uint(ranges[j]) : 0u;
      b = static_cast<uint8_t>(bits >> (8 * ((p - r0) & 3)));
    } else if (p >= t0) {
      b = static_cast<uint8_t>(rot >> (8 * (p - t0)));
    } else if (p == 0) {
      b = 3;
    } else if (p == 1) {
      b = static_cast<uint8_t>(q);
    } else {   // bytes 2..13: block, num_codes, num_blocks as little-endian u32
      const int64_t f = (p - 2) >> 2;
      const uint32_t v = static_cast<uint32_t>(f == 0 ? block : (f == 1 ? num_codes : num_blocks));
      b = static_cast<uint8_t>(v >> (8 * ((p - 2) & 3)));
    }
    out[w * stride + p] = b;
  }
}

int grid_for(int64_t work) {
  int64_t g = (work + kNT - 1) / kNT;
  if (g > 148 * 16) g = 148 * 16;
  return static_cast<int>(g < 1 ? 1 : g);
}

}  // namespace

extern "C" {

int64_t gc_topk_workspace_bytes(int32_t workers, int64_t len) {
  const int64_t tiles = (len + kTileE - 1) / kTileE;
  return ws_bytes(workers, tiles, len);
}

int gc_topk_select(int32_t workers, int64_t len, const float *values, int64_t ld, int64_t k, const float *grads,
                   float *resid, int32_t *idx_out, float *val_out, int32_t flags, void *workspace,
                   void *stream) {
  const int fp16_vals = flags & GC_TOPK_FP16_VALUES;
  const bool ef = (flags & GC_TOPK_EF_UPDATE) != 0;
  GC_REQUIRE(!ef || (grads && resid && !values), "GC_TOPK_EF_UPDATE needs grads and resid (fused ef_apply)");
  GC_REQUIRE(workers >= 1 && workers <= 65535 && len >= 1 && ld >= len, "invalid shape");
  GC_REQUIRE(k >= 1 && k <= len, "need 1 <= k <= len");
  GC_REQUIRE(len <= 0x7fffffff, "rows longer than 2^31-1 are not supported (int32 indices)");
  GC_REQUIRE(workspace && idx_out && (values || grads), "null argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t tiles = (len + kTileE - 1) / kTileE;
  Work wk = carve(workspace, workers, tiles, len);
  const dim3 grid(static_cast<unsigned>(tiles), workers);
  const float *src = grads ? grads : values;
  const bool vec = (ld % 4) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(resid)) & 15) == 0;
  init_kernel<<<grid_for(kBins0 * workers), kNT, 0, st>>>(wk, workers, k, vec ? 1 : 0);
  GC_LAUNCH_CHECK("init_kernel");
  // pass 1: level 0 (optionally fused with ef_apply: values then live in resid, or in grads if EF is off)
  if (vec)
    hist0_vec_kernel<<<dim3(static_cast<unsigned>(tiles < kH0Ctas ? tiles : kH0Ctas), workers), kNT, 0, st>>>(
        wk, len, values, ld, grads, resid, tiles);
  else
    hist_kernel<<<grid, kNT, 0, st>>>(wk, 0, len, values, ld, grads, resid);
  GC_LAUNCH_CHECK("hist_kernel");
  const float *vals = values ? values : (resid ? resid : grads);
  const int vec_vals = (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(vals) & 15) == 0;
  find_kernel<<<workers, 1024, 0, st>>>(wk, 0);
  // pass 2: tile counts above the boundary bin + the boundary bin's candidates
  const dim3 pgrid(static_cast<unsigned>(tiles < 8 * 148 ? tiles : 8 * 148), workers);
  collect_kernel<<<pgrid, kNT, 0, st>>>(wk, len, vals, ld, tiles, vec_vals);
  const dim3 cgrid(static_cast<unsigned>(tiles < 4 * 148 ? tiles : 4 * 148), workers);
  for (int level = 1; level <= 2; ++level) {
    cand_hist_kernel<<<cgrid, kNT, 0, st>>>(wk, level, len, vals, ld);
    find_kernel<<<workers, 1024, 0, st>>>(wk, level);
  }
  GC_LAUNCH_CHECK("radix select");
  cand_tile_kernel<<<cgrid, kNT, 0, st>>>(wk, len, vals, ld, tiles);
  tile_scan_kernel<<<workers, 1024, 0, st>>>(wk, tiles);
  // pass 3: ordered emission from the candidate segments; rows whose candidates overflowed the
  // list take the full-row write (each kernel returns at once for the other case)
  const dim3 wgrid(static_cast<unsigned>(tiles < 16 * 148 ? tiles : 16 * 148), workers);
  cand_write_kernel<<<wgrid, kNT, 0, st>>>(wk, tiles, k, idx_out, val_out, fp16_vals, ef ? resid : nullptr, ld);
  const dim3 fgrid(static_cast<unsigned>(tiles < 4 * 148 ? tiles : 4 * 148), workers);
  if (vec_vals)
    write_vec_kernel<<<fgrid, kNT, 0, st>>>(wk, len, vals, ld, tiles, k, idx_out, val_out, fp16_vals,
                                            ef ? resid : nullptr);
  else
    write_kernel<<<fgrid, kNT, 0, st>>>(wk, len, vals, ld, tiles, k, idx_out, val_out, fp16_vals,
                                        ef ? resid : nullptr);
  GC_LAUNCH_CHECK("topk write");
  return GC_OK;
}

int gc_sparse_accumulate(int32_t workers, int64_t k, const int32_t *idx, const float *val, int64_t dim,
                         float *estimate, void *stream) {
  GC_REQUIRE(workers >= 1 && k >= 0 && dim >= 1 && idx && val && estimate, "invalid argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  cudaMemsetAsync(estimate, 0, sizeof(float) * dim, st);
  for (int w = 0; w < workers; ++w) {   // worker-id order (pipelines.py:207)
    scatter_add_kernel<<<grid_for(k), kNT, 0, st>>>(k, idx + w * k, val + w * k, estimate);
  }
  GC_LAUNCH_CHECK("scatter_add_kernel");
  return GC_OK;
}

int64_t gc_sparse_mean_workspace_bytes(int32_t workers, int64_t dim) {
  return static_cast<int64_t>(workers) * ((dim + kMeanTile - 1) / kMeanTile + 1) * 4;
}

int gc_sparse_mean(int32_t workers, int64_t k, const int32_t *idx, const float *val, int64_t dim, int32_t divisor,
                   float *estimate, void *workspace, void *stream) {
  GC_REQUIRE(workers >= 1 && workers <= 65535 && k >= 0 && k <= 0x7fffffff && dim >= 1 && dim <= 0x7fffffff &&
                 divisor >= 1 && estimate && workspace && (k == 0 || (idx && val)),
             "invalid argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t tiles = (dim + kMeanTile - 1) / kMeanTile;
  int32_t *start = static_cast<int32_t *>(workspace);
  sparse_tile_starts_kernel<<<dim3(grid_for(k + 1), workers), kNT, 0, st>>>(workers, k, idx, tiles, start);
  const int64_t ctas = (tiles + kNT / 32 - 1) / (kNT / 32);
  sparse_mean_kernel<<<static_cast<unsigned>(ctas < 6 * 148 ? ctas : 6 * 148), kNT, 0, st>>>(
      workers, k, idx, val, dim, tiles, start, divisor, estimate);
  GC_LAUNCH_CHECK("sparse_mean_kernel");
  return GC_OK;
}

int gc_encode_sparse_payloads(int32_t workers, int64_t k, const int32_t *idx, const float *val, uint8_t *out,
                              int64_t stride, void *stream) {
  GC_REQUIRE(workers >= 1 && k >= 0 && k <= 0xffffffffll && (k == 0 || (idx && val)) && out && stride >= 5 + 6 * k,
             "invalid argument");
  const int64_t total = static_cast<int64_t>(workers) * (k > 0 ? k : 1);
  if (k == 0) {   // header only: <B 1><I 0>
    cudaMemsetAsync(out, 0, static_cast<size_t>(stride) * workers, static_cast<cudaStream_t>(stream));
    for (int w = 0; w < workers; ++w) cudaMemsetAsync(out + w * stride, 1, 1, static_cast<cudaStream_t>(stream));
    return GC_OK;
  }
  encode_sparse_kernel<<<grid_for(total), kNT, 0, static_cast<cudaStream_t>(stream)>>>(workers, k, idx, val, out,
                                                                                      stride);
  GC_LAUNCH_CHECK("encode_sparse_kernel");
  return GC_OK;
}

int64_t gc_quant_payload_nbytes(int64_t num_codes, int64_t num_blocks) { return 14 + num_codes + 8 * num_blocks + 8; }

int gc_encode_quant_payloads(int32_t workers, int32_t quant_bits, int64_t block_size, int64_t num_codes,
                             const int8_t *codes, int64_t codes_ld, int64_t codes_len, int64_t num_blocks,
                             const float *ranges, int64_t ranges_len, uint64_t rotation_id, uint8_t *out,
                             int64_t stride, void *stream) {
  const int64_t row = gc_quant_payload_nbytes(num_codes, num_blocks);
  GC_REQUIRE(workers >= 1 && quant_bits >= 2 && quant_bits <= 8 && block_size >= 1 && num_codes >= 0 &&
                 num_codes <= 0xffffffffll && num_blocks >= 0 && num_blocks * block_size == num_codes &&
                 codes_len >= 0 && codes_len <= num_codes && ranges_len >= 0 && ranges_len <= num_blocks &&
                 (codes_len == 0 || (codes && codes_ld >= codes_len)) && (ranges_len == 0 || ranges) && out &&
                 stride >= row,
             "invalid argument");
  encode_quant_kernel<<<grid_for(workers * row), kNT, 0, static_cast<cudaStream_t>(stream)>>>(
      workers, quant_bits, block_size, num_codes, codes, codes_ld, codes_len, num_blocks, ranges, ranges_len,
      static_cast<unsigned long long>(rotation_id), out, stride, row);
  GC_LAUNCH_CHECK("encode_quant_kernel");
  return GC_OK;
}

int gc_sparse_ef_update(int32_t workers, int64_t k, const int32_t *idx, const float *val, float *resid, int64_t ld,
                        void *stream) {
  GC_REQUIRE(workers >= 1 && k >= 0 && idx && val && resid, "invalid argument");
  if (k == 0) return GC_OK;
  sparse_ef_kernel<<<dim3(grid_for(k), workers), kNT, 0, static_cast<cudaStream_t>(stream)>>>(workers, k, idx, val,
                                                                                              resid, ld);
  GC_LAUNCH_CHECK("sparse_ef_kernel");
  return GC_OK;
}

}  // extern "C"
