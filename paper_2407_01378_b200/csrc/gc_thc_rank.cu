// Per-rank THC round of the distributed pipeline (one rank's L workers), tile-wise and fused.
//
// Reference round (pkg/src/gradcomp/pipelines.py:260-322) split at its two exchange points:
//
//   K1  gc_thc_rank_ranges   ef_apply + signs + fp64 WHT + chunk_ranges           (reads g, r)
//       (gc_thc_rank_ranges_signs: the round's rotation signs drawn here too and written for K2 / K3)
//       -- range consensus: NCCL all-reduce MAX of (-lo, hi) --
//   K2  gc_thc_rank_quant    ef_apply + WHT again + quantize_stochastic + own decode + ef_update:
//                            codes straight into the all-to-all send layout, r_new written
//       -- codes: all-to-all, ring-ordered saturating fold (gc_sat_fold), all-gather --
//   K3  gc_thc_rank_decode   dequantize_sum + inverse WHT + / n  -> estimate
//
// K2 recomputes the rotation instead of storing x_rot: the host runs K1 and K2 over L2-sized
// segments (K1 of segment s+1 overlaps the consensus all-reduce of segment s), so K2's re-read of
// g and r hits L2 and HBM sees g, r once, codes and r_new once, the summed codes and the estimate
// once: 16 + 2w bytes per coordinate for one worker.
//
// Every warp owns a contiguous run of tiles of one worker and never waits on another warp (no
// CTA-wide barriers): the coin chains of a run continue from tile to tile without a jump.
// Numerics are those of the fused single-GPU kernel (gc_thc_fused.cu, shared building blocks in
// gc_thc_tile.cuh): bit-exact codes, residuals and estimate.
#include <cuda_runtime.h>

#include <cstdlib>

#include "gc_device.cuh"
#include "gc_internal.h"
#include "gc_thc_tile.cuh"

namespace {

using namespace thc;

constexpr int kWarps = 4;      // independent warps per CTA
constexpr int kMaxL = 16;      // local workers per rank
constexpr int kLutMax = 256;   // doubles in a warp's own-decode table

struct RankArgs {
  int64_t dim, active, nb, tile_begin, tile_end, tpw, chunks;   // chunks of tpw tiles per worker
  int L, q, bits, n;
  double scale;
  const float *g;
  const float *r;
  float *rout;
  int64_t ld;
  int aligned;
  const uint32_t *signs;
  float *neg_ranges;          // K1: [L][nb][2] (-lo, hi)
  const float *shared;        // K2: [nb][2] (-lo, hi) consensus over all workers
  int8_t *send;               // K2: [W][L][slice] codes (or packed nibbles, halved offsets)
  int64_t slice;
  int nibble;
  unsigned long long *counters;   // K2: [1] sum z, [2] sum z^2
  const void *sums;           // K3: [active] saturated sums (sum_bytes each)
  int sum_bytes;
  float *est;                 // K3: [dim]
  // K1 with signs_out: the rotation signs are drawn here (gc_thc_signs' stream layout) and written
  // for K2 / K3; sign_jump = {mult_hi, mult_lo, c_hi, c_lo} advances a lane by 496 outputs (the
  // next tile's word of that lane), c = plus * inc of the stream
  uint32_t *signs_out;
  gc_pcg64 sign_stream;
  uint64_t sign_jump[4];
  gc_pcg64 streams[kMaxL];
};

// per-warp shared memory
struct WarpSmem {
  int scratch, cbuf, cod, bp, lut, total;
};

__host__ __device__ inline WarpSmem warp_smem(int nblk, int q) {
  WarpSmem S;
  S.scratch = 0;                               // fp64 transpose / x_rot staging (f32 [32][32])
  S.cbuf = S.scratch + kScrBytes;              // corrected, natural order (padded rows)
  // the tile's codes share the scratch rows behind x_rot: both live only between the forward and
  // the own-decode transposes (the codes are read into registers before that transpose), so the
  // warp needs 13 KB and four 4-warp CTAs fit an SM
  S.cod = S.scratch + kTileN * 4;
  S.bp = S.cbuf + kCBytes;                     // nblk x 8 doubles: block parameters
  S.lut = S.bp + nblk * 64;                    // dq(z, 1) table
  const int lut_n = nblk * ((1 << q) - 1);
  S.total = S.lut + ((lut_n < kLutMax ? lut_n : kLutMax) * 8 + 15) / 16 * 16;
  return S;
}

// The warp's run: worker l, tiles [t_lo, t_hi).  false when the warp has no work.
__device__ __forceinline__ bool warp_run(const RankArgs &a, int &l, int64_t &t_lo, int64_t &t_hi,
                                         int cta_warps = kWarps) {
  const int64_t gw = static_cast<int64_t>(blockIdx.x) * cta_warps + (threadIdx.x >> 5);
  if (gw >= a.L * a.chunks) return false;
  l = static_cast<int>(gw / a.chunks);
  t_lo = a.tile_begin + (gw % a.chunks) * a.tpw;
  t_hi = min(t_lo + a.tpw, a.tile_end);
  return t_lo < t_hi;
}

// corrected = f32(g + r) of one tile into cbuf (compressors.py:624-626), coalesced float4 loads in
// two batches of four.  K1 loads with the default policy so the segment stays in L2 for K2; K2's
// re-read is the last use (streaming loads).
template <bool LAST_USE>
__device__ __forceinline__ void load_corrected(const RankArgs &a, const float *gw, const float *rw, int64_t t0,
                                               float *cbuf, int lane) {
  if (a.aligned && t0 + kTileN <= a.dim) {
#pragma unroll
    for (int h = 0; h < 8; h += 4) {
      float4 gv[4], rv[4];
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const float4 *p = reinterpret_cast<const float4 *>(gw + t0 + (lane + 32 * (h + m)) * 4);
        gv[m] = LAST_USE ? __ldcs(p) : __ldg(p);
      }
      if (rw) {
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const float4 *p = reinterpret_cast<const float4 *>(rw + t0 + (lane + 32 * (h + m)) * 4);
          rv[m] = LAST_USE ? __ldcs(p) : __ldg(p);
        }
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          gv[m].x = gv[m].x + rv[m].x;
          gv[m].y = gv[m].y + rv[m].y;
          gv[m].z = gv[m].z + rv[m].z;
          gv[m].w = gv[m].w + rv[m].w;
        }
      }
#pragma unroll
      for (int m = 0; m < 4; ++m) *reinterpret_cast<float4 *>(cbuf + cidx((lane + 32 * (h + m)) * 4)) = gv[m];
    }
  } else {
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int e4 = (lane + 32 * m) * 4;
      float t[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = t0 + e4 + u;
        float v = 0.0f;
        if (i < a.dim) {
          v = gw[i];
          if (rw) v = v + rw[i];
        }
        t[u] = v;
      }
      *reinterpret_cast<float4 *>(cbuf + cidx(e4)) = make_float4(t[0], t[1], t[2], t[3]);
    }
  }
  __syncwarp();
}

// signs * corrected (transforms.py:115) in layout A, then the forward WHT (ends in layout B).
template <int K>
__device__ __forceinline__ void forward(double (&v)[32], const float *cbuf, uint32_t sign_word, double *scr,
                                        int lane) {
#pragma unroll
  for (int m = 0; m < 8; ++m) {
    const float4 c = *reinterpret_cast<const float4 *>(cbuf + cidx(lane * 32 + 4 * m));
    v[4 * m + 0] = apply_sign(static_cast<double>(c.x), (sign_word >> (4 * m + 0)) & 1u);
    v[4 * m + 1] = apply_sign(static_cast<double>(c.y), (sign_word >> (4 * m + 1)) & 1u);
    v[4 * m + 2] = apply_sign(static_cast<double>(c.z), (sign_word >> (4 * m + 2)) & 1u);
    v[4 * m + 3] = apply_sign(static_cast<double>(c.w), (sign_word >> (4 * m + 3)) & 1u);
  }
  wht_tile<K>(v, scr, lane);
}

// lane's sign "column" in layout B: bit j = sign of element 32j + lane
__device__ __forceinline__ uint32_t sign_column(uint32_t sign_word, int lane) {
  return bit_transpose32(sign_word, lane);
}

// ---------------------------------------------------------------- K1: ranges
template <int K>
__global__ void __launch_bounds__(kWarps * 32) rank_ranges_kernel(const __grid_constant__ RankArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int nblk = kTileN >> K;
  constexpr int rpb_log = K - 5;
  const int lane = threadIdx.x & 31;
  const WarpSmem S = warp_smem(nblk, a.q);
  unsigned char *ws = smem + (threadIdx.x >> 5) * S.total;
  double *scr = reinterpret_cast<double *>(ws + S.scratch);
  float *cbuf = reinterpret_cast<float *>(ws + S.cbuf);
  int l;
  int64_t t_lo, t_hi;
  if (!warp_run(a, l, t_lo, t_hi)) return;
  const float *gw = a.g + l * a.ld;
  const float *rw = a.r ? a.r + l * a.ld : nullptr;
  float *out = a.neg_ranges + static_cast<int64_t>(l) * a.nb * 2;
  // fused sign draw: the lane's word of tile t is outputs 16 (32 t + lane) .. + 15 of the
  // rotation-signs stream (transforms.py:80-82; numpy's bounded uint32 draws, two per next64)
  const bool gen = a.signs_out != nullptr;
  gc::u128 sstate = 0;
  if (gen) {
    gc::Pcg p;
    p.load(a.sign_stream);
    p.jump(static_cast<uint64_t>(t_lo) * 512 + static_cast<uint64_t>(lane) * 16);
    sstate = p.state;
  }
  for (int64_t t = t_lo; t < t_hi; ++t) {
    const int64_t t0 = t * kTileN;
    uint32_t sw;
    if (gen) {
      const gc::u128 inc = gc::mk128(a.sign_stream.inc_hi, a.sign_stream.inc_lo);
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        sstate = sstate * GC_PCG_MULT + inc;
        const uint64_t u = gc::Pcg::output(sstate);
        word |= static_cast<uint32_t>((u >> 31) & 1u) << (2 * j);
        word |= static_cast<uint32_t>((u >> 63) & 1u) << (2 * j + 1);
      }
      sstate = sstate * gc::mk128(a.sign_jump[0], a.sign_jump[1]) + gc::mk128(a.sign_jump[2], a.sign_jump[3]);
      if (l == 0) a.signs_out[(t0 >> 5) + lane] = word;
      sw = word;
    } else {
      sw = a.signs[(t0 >> 5) + lane];
    }
    load_corrected<false>(a, gw, rw, t0, cbuf, lane);
    double v[32];
    forward<K>(v, cbuf, sw, scr, lane);
    float blo = INFINITY, bhi = -INFINITY;
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const float f = static_cast<float>(v[j] * a.scale);   // x_rot (transforms.py:116)
      blo = fminf(blo, f);
      bhi = fmaxf(bhi, f);
      if (((j + 1) & ((1 << rpb_log) - 1)) == 0) {   // last register of block j >> rpb_log
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          blo = fminf(blo, __shfl_xor_sync(0xffffffffu, blo, o));
          bhi = fmaxf(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
        }
        const int64_t blk = (t0 >> K) + (j >> rpb_log);
        if (lane == 0 && blk < a.nb) *reinterpret_cast<float2 *>(out + 2 * blk) = make_float2(-blo, bhi);
        blo = INFINITY;
        bhi = -INFINITY;
      }
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- K2: quantize + own decode + EF
// WQ warps per CTA.  WQ = 16 (one CTA per SM, the default): the SM's warps start their ~90 KB
// straight-line tile bodies together and drift apart only slowly, so they share the instruction
// cache better than four independently scheduled 4-warp CTAs (ncu: no_instruction was K2's top
// stall; 4.00 -> 3.86 ms per 350M round).  A per-tile CTA barrier removes the fetch stalls entirely
// but makes every warp load its tile at once (long_scoreboard / lg_throttle): slower, not kept.
template <int K, int WQ>
__global__ void __launch_bounds__(WQ * 32, 16 / WQ) rank_quant_kernel(const __grid_constant__ RankArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int nblk = kTileN >> K;
  constexpr int rpb_log = K - 5;
  constexpr bool kPow2Scale = (K % 2) == 0;
  const int lane = threadIdx.x & 31;
  const int q = a.q;
  const WarpSmem S = warp_smem(nblk, q);
  unsigned char *ws = smem + (threadIdx.x >> 5) * S.total;
  double *scr = reinterpret_cast<double *>(ws + S.scratch);
  float *xs = reinterpret_cast<float *>(scr);
  float *cbuf = reinterpret_cast<float *>(ws + S.cbuf);
  int8_t *cod = reinterpret_cast<int8_t *>(ws + S.cod);
  double *bp = reinterpret_cast<double *>(ws + S.bp);
  double *lut = reinterpret_cast<double *>(ws + S.lut);
  int l;
  int64_t t_lo, t_hi;
  if (!warp_run(a, l, t_lo, t_hi, WQ)) return;

  const int ibound = (1 << (q - 1)) - 1;
  const double levels = static_cast<double>((1 << q) - 2);
  const int lut_span = 2 * ibound + 1;
  const bool use_lut = nblk * lut_span <= kLutMax;

  // coin chains: lane consumes positions t0 + lane + 1 + 32 j; chain c = j mod 4 jumps 128 steps
  const uint64_t inc_h = a.streams[l].inc_hi, inc_l = a.streams[l].inc_lo;
  uint32_t m128[4], c128[4], m32[4], c32[4];
  {
    uint64_t h, lo;
    limbs(gc::kPcgJump[7][0], gc::kPcgJump[7][1], m128);
    mul128(gc::kPcgJump[7][2], gc::kPcgJump[7][3], inc_h, inc_l, h, lo);
    limbs(h, lo, c128);
    limbs(gc::kPcgJump[5][0], gc::kPcgJump[5][1], m32);
    mul128(gc::kPcgJump[5][2], gc::kPcgJump[5][3], inc_h, inc_l, h, lo);
    limbs(h, lo, c32);
  }
  Lcg ch[4];
  {
    gc::Pcg p;
    p.load(a.streams[l]);
    p.jump(static_cast<uint64_t>(t_lo) * kTileN + lane + 1);
    ch[0].set(static_cast<uint64_t>(p.state >> 64), static_cast<uint64_t>(p.state));
#pragma unroll
    for (int c = 1; c < 4; ++c) {
      ch[c] = ch[c - 1];
      ch[c].step(m32, c32);
    }
  }

  const float *gw = a.g + l * a.ld;
  const float *rw = a.r ? a.r + l * a.ld : nullptr;
  float *ro = a.r ? a.rout + l * a.ld : nullptr;
  long long sz = 0, sz2 = 0;
  for (int64_t t = t_lo; t < t_hi; ++t) {
    const int64_t t0 = t * kTileN;
    const uint32_t sw = a.signs[(t0 >> 5) + lane];
    load_corrected<true>(a, gw, rw, t0, cbuf, lane);
    double v[32];
    forward<K>(v, cbuf, sw, scr, lane);
    const uint32_t sign_col = sign_column(sw, lane);
#pragma unroll
    for (int j = 0; j < 32; ++j) xs[j * 32 + lane] = static_cast<float>(v[j] * a.scale);
    // block parameters from the consensus grid (pipelines.py:271-288, compressors.py:481-488)
    if (lane < nblk) {
      const int64_t blk = (t0 >> K) + lane;
      double dlo = 0.0, dhi = 0.0;   // blocks past `active` are all-zero: range (0, 0)
      if (blk < a.nb) {
        const float2 rg = *reinterpret_cast<const float2 *>(a.shared + 2 * blk);
        dlo = static_cast<double>(-rg.x);
        dhi = static_cast<double>(rg.y);
      }
      const double step = (dhi - dlo) / levels;
      bp[8 * lane] = dlo;
      bp[8 * lane + 1] = dhi;
      bp[8 * lane + 2] = (dlo + dhi) / 2.0;
      bp[8 * lane + 3] = step;
      bp[8 * lane + 4] = 0.0;
      bp[8 * lane + 5] = dhi > dlo ? step : 0.0;   // dequantize_sum's step (compressors.py:520)
      *reinterpret_cast<float4 *>(bp + 8 * lane + 6) =
          screen_params((dlo + dhi) / 2.0, step, static_cast<double>(ibound));
    }
    __syncwarp();
    if (use_lut) {
      for (int e = lane; e < nblk * lut_span; e += 32) {
        const int b = e / lut_span, z = e - b * lut_span - ibound;
        lut[e] = static_cast<double>(static_cast<float>(1.0 * bp[8 * b + 2] + bp[8 * b + 5] * static_cast<double>(z))) *
                 (kPow2Scale ? a.scale : 1.0);
      }
    }
    // quantize_stochastic (compressors.py:473-498), layout B: e = 32 j + lane
    {
      int tz = 0, tz2 = 0;
      for (int j = 0; j < 32; j += 4) {
        int z[4];
        uint32_t hw[4], oa[4], ob[4], orot[4];
        float xv[4];
        bool safe = true;
        const float4 sp_j = *reinterpret_cast<const float4 *>(bp + 8 * (j >> rpb_log) + 6);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 sp = rpb_log >= 2 ? sp_j : *reinterpret_cast<const float4 *>(bp + 8 * ((j + c) >> rpb_log) + 6);
          hw[c] = ch[c].out_hi(oa[c], ob[c], orot[c]);
#if GC_THC_IMM
          ch[c].step128(c128);
#else
          ch[c].step(m128, c128);
#endif
          xv[c] = xs[(j + c) * 32 + lane];
          const float tq = (xv[c] - sp.x) * sp.y;
          const float sm = __fadd_rd(tq, 12582912.0f);
          const float f = tq - (sm - 12582912.0f);
          const float c23 = __uint_as_float(0x3f800000u | (hw[c] >> 9)) - 1.0f;
          safe = safe && fminf(fminf(f, 1.0f - f), fabsf(c23 - f)) > sp.z;
          z[c] = (__float_as_int(sm) - 0x4B400000) + (c23 < f ? 1 : 0);
        }
        if (__any_sync(0xffffffffu, !safe)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const double *pb = bp + 8 * ((j + c) >> rpb_log);
            const float4 sp = *reinterpret_cast<const float4 *>(pb + 6);
            const float tq = (xv[c] - sp.x) * sp.y;
            const float sm = __fadd_rd(tq, 12582912.0f);
            const float f = tq - (sm - 12582912.0f);
            const float c23 = __uint_as_float(0x3f800000u | (hw[c] >> 9)) - 1.0f;
            if (!(fminf(fminf(f, 1.0f - f), fabsf(c23 - f)) > sp.z))
              z[c] = quantize_ref(static_cast<double>(xv[c]), pb[0], pb[1], pb[2], pb[3], static_cast<double>(ibound),
                                  coin_from(hw[c], Lcg::lo_of(oa[c], ob[c], orot[c])));
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          cod[(j + c) * 32 + lane] = static_cast<int8_t>(z[c]);
          tz += z[c];
          tz2 += z[c] * z[c];
        }
      }
      sz += tz;
      sz2 += tz2;
    }
    __syncwarp();
    // codes -> the all-to-all send layout: slice t0 / S goes to that rank, worker row l
    {
      const int64_t dst = t0 / a.slice, off = t0 - dst * a.slice;
      const int64_t base = (dst * a.L + l) * a.slice + off + lane * 32;
      const int4 z0 = *reinterpret_cast<const int4 *>(cod + lane * 32);
      const int4 z1 = *reinterpret_cast<const int4 *>(cod + lane * 32 + 16);
      if (!a.nibble) {
        *reinterpret_cast<int4 *>(a.send + base) = z0;
        *reinterpret_cast<int4 *>(a.send + base + 16) = z1;
      } else {   // element 2i in the low nibble, 2i+1 in the high one (gc_pack_nibbles)
        const uint32_t zw[8] = {static_cast<uint32_t>(z0.x), static_cast<uint32_t>(z0.y), static_cast<uint32_t>(z0.z),
                                static_cast<uint32_t>(z0.w), static_cast<uint32_t>(z1.x), static_cast<uint32_t>(z1.y),
                                static_cast<uint32_t>(z1.z), static_cast<uint32_t>(z1.w)};
        uint32_t pk[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t o = 0;
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t x = zw[2 * u + h];
#pragma unroll
            for (int b = 0; b < 2; ++b) {
              const uint32_t lo4 = (x >> (16 * b)) & 0xfu, hi4 = (x >> (16 * b + 8)) & 0xfu;
              o |= (lo4 | (hi4 << 4)) << (8 * (2 * h + b));
            }
          }
          pk[u] = o;
        }
        *reinterpret_cast<uint4 *>(a.send + base / 2) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
    }
    // own decode + ef_update (pipelines.py:312-318, 168-170)
    if (rw) {
      const int blk = lane >> rpb_log;
      const int4 z0 = *reinterpret_cast<const int4 *>(cod + lane * 32);
      const int4 z1 = *reinterpret_cast<const int4 *>(cod + lane * 32 + 16);
      const int zw[8] = {z0.x, z0.y, z0.z, z0.w, z1.x, z1.y, z1.z, z1.w};
      const double mid = bp[8 * blk + 2], step = bp[8 * blk + 5];
      const double *tab = lut + blk * lut_span + ibound;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int z = static_cast<int8_t>((zw[j >> 2] >> (8 * (j & 3))) & 0xff);
        v[j] = use_lut ? tab[z]
                       : static_cast<double>(static_cast<float>(1.0 * mid + step * static_cast<double>(z))) *
                             (kPow2Scale ? a.scale : 1.0);
      }
      __syncwarp();   // every lane has read the tile's codes: the transpose rows below overlay them
      wht_tile<K>(v, scr, lane);
      if (t0 + kTileN <= a.dim) {
        float *rt = ro + t0 + lane;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float own = static_cast<float>(apply_sign(kPow2Scale ? v[j] : v[j] * a.scale, (sign_col >> j) & 1u));
          __stcs(rt + 32 * j, cbuf[cidx(j * 32 + lane)] - own);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const int e = j * 32 + lane;
          const float own = static_cast<float>(apply_sign(kPow2Scale ? v[j] : v[j] * a.scale, (sign_col >> j) & 1u));
          if (t0 + e < a.dim) __stcs(ro + t0 + e, cbuf[cidx(e)] - own);
        }
      }
    }
    __syncwarp();
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
    sz2 += __shfl_xor_sync(0xffffffffu, sz2, o);
  }
  if (lane == 0 && a.counters) {
    atomicAdd(&a.counters[1], static_cast<unsigned long long>(sz));
    atomicAdd(&a.counters[2], static_cast<unsigned long long>(sz2));
  }
}

// ---------------------------------------------------------------- K3: estimate decode
__device__ __forceinline__ void load_sums32(const RankArgs &a, int64_t e0, int (&z)[32]) {
  if (a.sum_bytes == 1) {
    const int4 *p = reinterpret_cast<const int4 *>(static_cast<const int8_t *>(a.sums) + e0);
    const int4 u0 = p[0], u1 = p[1];
    const int w[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
#pragma unroll
    for (int j = 0; j < 32; ++j) z[j] = static_cast<int8_t>((w[j >> 2] >> (8 * (j & 3))) & 0xff);
  } else if (a.sum_bytes == 2) {
    const int4 *p = reinterpret_cast<const int4 *>(static_cast<const int16_t *>(a.sums) + e0);
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int4 u = p[m];
      const int w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int h = 0; h < 8; ++h) z[8 * m + h] = static_cast<int16_t>((w[h >> 1] >> (16 * (h & 1))) & 0xffff);
    }
  } else {
    const int4 *p = reinterpret_cast<const int4 *>(static_cast<const int32_t *>(a.sums) + e0);
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int4 u = p[m];
      z[4 * m] = u.x;
      z[4 * m + 1] = u.y;
      z[4 * m + 2] = u.z;
      z[4 * m + 3] = u.w;
    }
  }
}

template <int K>
__global__ void __launch_bounds__(kWarps * 32) rank_decode_kernel(const __grid_constant__ RankArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  double *scr = reinterpret_cast<double *>(smem + (threadIdx.x >> 5) * kScrBytes);
  int l;
  int64_t t_lo, t_hi;
  if (!warp_run(a, l, t_lo, t_hi)) return;
  const double levels = static_cast<double>((1 << a.q) - 2);
  const double nd = static_cast<double>(a.n);
  const gc::DivN dn(a.n);   // / n: an exact reciprocal product for power-of-two n
  // one-byte sums (wire_bits <= 8): the next tile's sign word, 32 sums and block range are loaded
  // while this tile transforms, so the loop pays no global-load latency per tile
  const bool pf = a.sum_bytes == 1;
  int4 nu0 = make_int4(0, 0, 0, 0), nu1 = nu0;
  uint32_t nsw = 0;
  float2 nrg = make_float2(0.0f, 0.0f);
  auto fetch = [&](int64_t t) {
    const int64_t e0 = t * kTileN + lane * 32;
    nsw = a.signs[(t * kTileN >> 5) + lane];
    const int4 *p = reinterpret_cast<const int4 *>(static_cast<const int8_t *>(a.sums) + e0);
    nu0 = p[0];
    nu1 = p[1];
    const int64_t b = e0 >> K;
    nrg = b < a.nb ? *reinterpret_cast<const float2 *>(a.shared + 2 * b) : make_float2(-0.0f, 0.0f);
  };
  if (pf) fetch(t_lo);
  for (int64_t t = t_lo; t < t_hi; ++t) {
    const int64_t t0 = t * kTileN;
    uint32_t sw;
    int z[32];
    double dlo = 0.0, dhi = 0.0;
    if (pf) {
      sw = nsw;
      const int w[8] = {nu0.x, nu0.y, nu0.z, nu0.w, nu1.x, nu1.y, nu1.z, nu1.w};
#pragma unroll
      for (int j = 0; j < 32; ++j) z[j] = static_cast<int8_t>((w[j >> 2] >> (8 * (j & 3))) & 0xff);
      dlo = static_cast<double>(-nrg.x);
      dhi = static_cast<double>(nrg.y);
      if (t + 1 < t_hi) fetch(t + 1);
    } else {
      sw = a.signs[(t0 >> 5) + lane];
      load_sums32(a, t0 + lane * 32, z);
      // dequantize_sum(sums, ranges, q, n) (compressors.py:501-521): f32(n * mid + step * z)
      const int64_t blk = (t0 + lane * 32) >> K;   // a lane's 32 coordinates sit in one block (B >= 32)
      if (blk < a.nb) {
        const float2 rg = *reinterpret_cast<const float2 *>(a.shared + 2 * blk);
        dlo = static_cast<double>(-rg.x);
        dhi = static_cast<double>(rg.y);
      }
    }
    const double mid = (dlo + dhi) / 2.0;
    const double step = dhi > dlo ? (dhi - dlo) / levels : 0.0;
    double v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = static_cast<double>(static_cast<float>(nd * mid + step * static_cast<double>(z[j])));
    wht_tile<K>(v, scr, lane);
    const uint32_t sign_col = sign_column(sw, lane);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t i = t0 + 32 * j + lane;
      // rht_inverse (transforms.py:120-126) then / n (pipelines.py:308-311)
      const float f = dn(static_cast<float>(apply_sign(v[j] * a.scale, (sign_col >> j) & 1u)));
      if (i < a.dim) __stcs(a.est + i, f);
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------- L -> 1 range merge
__global__ void merge_neg_ranges_kernel(int L, int64_t nb, const float *in, float *out) {
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < nb;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float2 m = *reinterpret_cast<const float2 *>(in + 2 * b);
    for (int l = 1; l < L; ++l) {
      const float2 x = *reinterpret_cast<const float2 *>(in + (l * nb + b) * 2);
      m.x = fmaxf(m.x, x.x);
      m.y = fmaxf(m.y, x.y);
    }
    *reinterpret_cast<float2 *>(out + 2 * b) = m;
  }
}

int log2_block(const gc_thc_geom *g) {
  int k = 0;
  while ((int64_t{1} << k) < g->block) ++k;
  return k;
}

int prepare(RankArgs &a, const gc_thc_geom *g, int32_t L, int64_t tile_begin, int64_t tile_end, int &grid,
            int cta_warps = kWarps) {
  GC_REQUIRE(g != nullptr, "geometry is null");
  GC_REQUIRE(L >= 1 && L <= kMaxL, "per-rank THC kernels support 1..16 local workers");
  GC_REQUIRE(g->dim >= 1 && g->padded >= kTileN && (g->padded & (g->padded - 1)) == 0 && g->padded >= g->dim,
             "per-rank THC kernels need padded >= 1024 (power of two)");
  GC_REQUIRE(g->block >= 32 && g->block <= kTileN && (g->block & (g->block - 1)) == 0,
             "per-rank THC kernels need a rotation block in [32, 1024]");
  GC_REQUIRE(g->quant_bits >= 2 && g->quant_bits <= 8 && g->wire_bits >= g->quant_bits && g->wire_bits <= 32,
             "invalid quant/wire bits");
  a.dim = g->dim;
  a.active = ((g->dim + g->block - 1) / g->block) * g->block;
  a.nb = a.active / g->block;
  const int64_t all_tiles = (a.active + kTileN - 1) / kTileN;
  if (tile_end < 0 || tile_end > all_tiles) tile_end = all_tiles;
  GC_REQUIRE(tile_begin >= 0 && tile_begin <= tile_end, "invalid tile range");
  a.tile_begin = tile_begin;
  a.tile_end = tile_end;
  a.L = L;
  a.q = g->quant_bits;
  a.bits = g->wire_bits;
  a.scale = g->scale;
  const int64_t T = tile_end - tile_begin;
  if (T == 0) return 1;
  // contiguous runs of tiles per warp: about two waves of 148 SMs x 16 warps
  int64_t tpw = (T * L + 148 * 16 * 2 - 1) / (148 * 16 * 2);
  if (tpw < 1) tpw = 1;
  a.tpw = tpw;
  a.chunks = (T + tpw - 1) / tpw;
  const int64_t warps = a.chunks * L;
  grid = static_cast<int>((warps + cta_warps - 1) / cta_warps);
  return 0;
}

// warps per CTA of K2: 16 (one CTA per SM) unless GC_THC_K2_WARPS=4 (four independent CTAs)
int k2_cta_warps() {
  static const int w = [] {
    const char *e = getenv("GC_THC_K2_WARPS");
    return e && atoi(e) == 4 ? 4 : 16;
  }();
  return w;
}

template <typename F>
int set_smem(F fn, int bytes) {
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  return bytes;
}


// Host: the 496-step jump of a PCG64 stream (state -> m state + c), from the 2^k-step table.
void sign_jump_consts(const gc_pcg64 &st, uint64_t out[4]) {
  static const uint64_t table[128][4] = GC_PCG_TABLE_INIT;
  typedef unsigned __int128 h128;
  h128 am = 1, ap = 0;
  uint64_t delta = 512 - 16;
  for (int k = 0; delta; ++k, delta >>= 1) {
    if (delta & 1) {
      const h128 m = (static_cast<h128>(table[k][0]) << 64) | table[k][1];
      const h128 p = (static_cast<h128>(table[k][2]) << 64) | table[k][3];
      am *= m;
      ap = ap * m + p;
    }
  }
  const h128 inc = (static_cast<h128>(st.inc_hi) << 64) | st.inc_lo;
  const h128 c = ap * inc;
  out[0] = static_cast<uint64_t>(am >> 64);
  out[1] = static_cast<uint64_t>(am);
  out[2] = static_cast<uint64_t>(c >> 64);
  out[3] = static_cast<uint64_t>(c);
}

int rank_ranges_launch(const gc_thc_geom *g, int32_t L, const float *grads, const float *resid, int64_t ld,
                       int64_t tile_begin, int64_t tile_end, const uint32_t *sign_bits,
                       const gc_pcg64 *sign_stream, uint32_t *signs_out, float *neg_ranges, void *stream) {
  RankArgs a{};
  int grid = 0;
  const int st = prepare(a, g, L, tile_begin, tile_end, grid);
  if (st < 0) return st;
  if (st == 1) return GC_OK;
  GC_REQUIRE(grads && sign_bits && neg_ranges && ld >= g->dim, "invalid argument");
  a.g = grads;
  a.r = resid;
  a.ld = ld;
  a.aligned = ((reinterpret_cast<uintptr_t>(grads) | reinterpret_cast<uintptr_t>(resid)) & 15) == 0 && (ld % 4) == 0;
  a.signs = sign_bits;
  a.neg_ranges = neg_ranges;
  if (signs_out) {
    a.signs_out = signs_out;
    a.sign_stream = *sign_stream;
    sign_jump_consts(*sign_stream, a.sign_jump);
  }
  const int k = log2_block(g);
  const int smem = kWarps * warp_smem(kTileN >> k, a.q).total;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
#define GC_K1(KK) \
  case KK:        \
    rank_ranges_kernel<KK><<<grid, kWarps * 32, set_smem(rank_ranges_kernel<KK>, smem), s>>>(a); \
    break;
  switch (k) { GC_K1(5) GC_K1(6) GC_K1(7) GC_K1(8) GC_K1(9) GC_K1(10) default: return GC_ERR_INVALID; }
#undef GC_K1
  GC_LAUNCH_CHECK("rank_ranges_kernel");
  return GC_OK;
}


}  // namespace

extern "C" {

int gc_thc_rank_ranges_signs(const gc_thc_geom *g, int32_t L, const float *grads, const float *resid, int64_t ld,
                             int64_t tile_begin, int64_t tile_end, const gc_pcg64 *rotation_stream,
                             uint32_t *sign_bits, float *neg_ranges, void *stream) {
  GC_REQUIRE(rotation_stream && sign_bits, "invalid argument");
  return rank_ranges_launch(g, L, grads, resid, ld, tile_begin, tile_end, sign_bits, rotation_stream, sign_bits,
                            neg_ranges, stream);
}

int gc_thc_rank_ranges(const gc_thc_geom *g, int32_t L, const float *grads, const float *resid, int64_t ld,
                       int64_t tile_begin, int64_t tile_end, const uint32_t *sign_bits, float *neg_ranges,
                       void *stream) {
  return rank_ranges_launch(g, L, grads, resid, ld, tile_begin, tile_end, sign_bits, nullptr, nullptr, neg_ranges,
                            stream);
}

int gc_thc_merge_ranges(int32_t L, int64_t num_blocks, const float *neg_ranges_in, float *neg_ranges_out,
                        void *stream) {
  GC_REQUIRE(L >= 1 && num_blocks >= 0 && neg_ranges_in && neg_ranges_out, "invalid argument");
  if (num_blocks == 0) return GC_OK;
  int64_t grid = (num_blocks + 255) / 256;
  if (grid > 148 * 8) grid = 148 * 8;
  merge_neg_ranges_kernel<<<static_cast<int>(grid), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      L, num_blocks, neg_ranges_in, neg_ranges_out);
  GC_LAUNCH_CHECK("merge_neg_ranges_kernel");
  return GC_OK;
}

int gc_thc_rank_quant(const gc_thc_geom *g, int32_t L, const float *grads, const float *resid_in, float *resid_out,
                      int64_t ld, int64_t tile_begin, int64_t tile_end, const uint32_t *sign_bits,
                      const float *shared_neg_ranges, const gc_pcg64 *coin_streams, int8_t *send, int64_t slice,
                      int32_t nibble, int64_t *counters, void *stream) {
  RankArgs a{};
  int grid = 0;
  // 16-warp CTAs while their shared memory fits an SM (small rotation blocks need more per warp)
  int wq = k2_cta_warps();
  if (wq == 16 && g && g->block >= 32 && g->block <= kTileN &&
      16 * warp_smem(kTileN >> log2_block(g), g->quant_bits).total > 227 * 1024)
    wq = kWarps;
  const int st = prepare(a, g, L, tile_begin, tile_end, grid, wq);
  if (st < 0) return st;
  if (st == 1) return GC_OK;
  GC_REQUIRE(grads && sign_bits && shared_neg_ranges && coin_streams && send && ld >= g->dim, "invalid argument");
  GC_REQUIRE((resid_in == nullptr) == (resid_out == nullptr), "residual in/out must both be set or both NULL");
  GC_REQUIRE(slice >= kTileN && slice % kTileN == 0, "send slice must be a multiple of 1024 coordinates");
  GC_REQUIRE(!nibble || g->wire_bits <= 4, "nibble codes need wire_bits <= 4");
  GC_REQUIRE((reinterpret_cast<uintptr_t>(send) & 15) == 0, "send buffer must be 16-byte aligned");
  a.g = grads;
  a.r = resid_in;
  a.rout = resid_out;
  a.ld = ld;
  a.aligned = ((reinterpret_cast<uintptr_t>(grads) | reinterpret_cast<uintptr_t>(resid_in) |
                reinterpret_cast<uintptr_t>(resid_out)) & 15) == 0 && (ld % 4) == 0;
  a.signs = sign_bits;
  a.shared = shared_neg_ranges;
  a.send = send;
  a.slice = slice;
  a.nibble = nibble;
  a.counters = reinterpret_cast<unsigned long long *>(counters);
  for (int l = 0; l < L; ++l) a.streams[l] = coin_streams[l];
  const int k = log2_block(g);
  const int smem = wq * warp_smem(kTileN >> k, a.q).total;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
#define GC_K2(KK)                                                                                           \
  case KK:                                                                                                  \
    if (wq == 16)                                                                                           \
      rank_quant_kernel<KK, 16><<<grid, 16 * 32, set_smem(rank_quant_kernel<KK, 16>, smem), s>>>(a);        \
    else                                                                                                    \
      rank_quant_kernel<KK, kWarps><<<grid, kWarps * 32, set_smem(rank_quant_kernel<KK, kWarps>, smem), s>>>(a); \
    break;
  switch (k) { GC_K2(5) GC_K2(6) GC_K2(7) GC_K2(8) GC_K2(9) GC_K2(10) default: return GC_ERR_INVALID; }
#undef GC_K2
  GC_LAUNCH_CHECK("rank_quant_kernel");
  return GC_OK;
}

int gc_thc_rank_decode(const gc_thc_geom *g, int32_t n, const void *sums, int32_t sum_bytes,
                       const float *shared_neg_ranges, const uint32_t *sign_bits, float *estimate, void *stream) {
  RankArgs a{};
  int grid = 0;
  const int st = prepare(a, g, 1, 0, -1, grid);
  if (st < 0) return st;
  if (st == 1) return GC_OK;
  GC_REQUIRE(n >= 1 && sums && shared_neg_ranges && sign_bits && estimate, "invalid argument");
  GC_REQUIRE(sum_bytes == 1 || sum_bytes == 2 || sum_bytes == 4, "sum_bytes must be 1, 2 or 4");
  GC_REQUIRE((reinterpret_cast<uintptr_t>(sums) & 15) == 0, "sums must be 16-byte aligned");
  a.n = n;
  a.sums = sums;
  a.sum_bytes = sum_bytes;
  a.shared = shared_neg_ranges;
  a.signs = sign_bits;
  a.est = estimate;
  const int k = log2_block(g);
  const int smem = kWarps * kScrBytes;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
#define GC_K3(KK) \
  case KK:        \
    rank_decode_kernel<KK><<<grid, kWarps * 32, set_smem(rank_decode_kernel<KK>, smem), s>>>(a); \
    break;
  switch (k) { GC_K3(5) GC_K3(6) GC_K3(7) GC_K3(8) GC_K3(9) GC_K3(10) default: return GC_ERR_INVALID; }
#undef GC_K3
  GC_LAUNCH_CHECK("rank_decode_kernel");
  return GC_OK;
}

}  // extern "C"
