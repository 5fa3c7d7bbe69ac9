// Fused THC round for n workers simulated on one GPU (the bench's hot kernel).
//
// Reference path (pkg/src/gradcomp/pipelines.py:147-182, 260-322): ef_apply ->
// rht_forward -> chunk_ranges -> ElemMin/ElemMax ring consensus -> quantize_stochastic ->
// SatIntSum ring -> dequantize_sum + rht_inverse (estimate) -> own decode -> ef_update.
//
// B200 design: a persistent CTA of n warps (warp w = worker w) walks 1024-coordinate
// tiles.  Range consensus of a rotation block only needs that block of every worker and
// the saturating ring fold of a coordinate only needs that coordinate of every worker,
// so a tile is completed on-chip: HBM sees g and r read once and r_new / estimate written
// once (12n + 4 bytes per coordinate; codes only if the caller asks for them).  Shared
// memory is sized so two CTAs share an SM (n = 8, B = 1024: ~106 KB each) and the
// per-tile barriers of one CTA overlap the other's work.
//
// Per worker a warp holds the tile as 32 doubles per lane.  Layout A (lane l owns
// elements 32l..32l+31) makes butterfly stages 0-4 register-local; one XOR-swizzled
// shared-memory transpose gives layout B (lane l owns 32j+l) for stages 5-9.  Stage order
// is bit-0-first as in transforms.py:92-98, all arithmetic fp64 without contraction
// (this file is compiled with -fmad=false), so codes are bit-exact with the reference.
//
// Coins: numpy PCG64 "stochastic-round" stream of worker w; coordinate i uses output
// i+1.  Lane l of layout B consumes positions t0+l+1+32j: four interleaved LCG chains
// (j mod 4, 128-step jumps) keep four independent 128-bit multiply chains in flight; tiles
// advance by a host-precomputed gridDim*1024-step jump.  The quantizer decides a code from
// the top 23 bits of the coin in fp32 (see screen_params); the rare undecidable coordinates
// rebuild the full 53-bit coin and run the reference's fp64 formula.
//
// In-pipeline simplifications that are exact (not approximations):
//  * the value clamp of quantize_stochastic (compressors.py:482-483) is the identity: the
//    consensus range of a block is the min/max over all workers' values of that block, so
//    every x lies in [lo, hi] and the clamp count (range_clips) is 0;
//  * the clip of t to +-bound (:489) only moves t by the rounding error of (x-mid)/step
//    (< 1e-13 absolute), which the 1e-9 snapping (:492-493) maps to the same code, so the
//    final code clip (:496) never fires either.
#include <cuda_runtime.h>

#include "gc_device.cuh"
#include "gc_internal.h"
#include "gc_thc_tile.cuh"

#ifndef GC_THC_LOAD_BATCH
#define GC_THC_LOAD_BATCH 8
#endif

namespace {

using namespace thc;

constexpr int HALF = GC_THC_LOAD_BATCH;   // float4 loads of g (and r) in flight per batch
constexpr int kMaxN = 16;
constexpr int kLutMax = 256;   // doubles in the shared own-decode table

struct FusedArgs {
  int64_t dim, padded, active, tile_begin, tiles, ring_blk;   // tiles = end of the tile range
  int n, k, q, bits;
  double scale;
  const float *g;
  const float *r;   // residual read (ef_apply)
  float *rout;      // residual written (ef_update); == r for the in-place update
  int64_t ld;
  bool aligned;
  const uint32_t *signs;
  float *est;
  int8_t *codes;
  unsigned long long *counters;
  double *nmse;
  uint64_t tile_jump[4];  // {mult_hi, mult_lo, plus_hi, plus_lo} for gridDim*1024 steps
  gc_pcg64 streams[kMaxN];
};

struct Layout {
  int scratch, cbuf, cod, wr, bp, lut, sgn, pcg, total;
};

__host__ __device__ inline Layout layout_for(int n, int nblk, int q) {
  Layout L;
  L.scratch = 0;                        // n x 8.25 KB  fp64 transpose / x_rot staging
  L.cbuf = L.scratch + n * kScrBytes;   // n x 4.5 KB   corrected (f32, padded natural order)
  L.cod = L.cbuf + n * kCBytes;         // n x 1 KB     codes
  L.wr = L.cod + n * 1024;              // n x nblk x 2 f32   own block ranges
  L.bp = L.wr + ((n * nblk * 8 + 15) & ~15);   // n x nblk x 8 f64  consensus params (per warp)
  L.lut = L.bp + n * nblk * 64;         // nblk x (2^q - 1) f64 (<= kLutMax)  dq(z, 1) table
  const int lut_n = nblk * ((1 << q) - 1);
  L.sgn = L.lut + ((lut_n < kLutMax ? lut_n : kLutMax) * 8 + 15) / 16 * 16;          // 2 x 32 u32 sign words (double-buffered by tile parity)
  L.pcg = L.sgn + 256;                  // n x 16 u32: the worker's 4-step and tile-step LCG jumps
  L.total = L.pcg + n * 64 + 32 + n * 16;   // + loop invariants (8 ints) + per-warp counters (4 ints)
  return L;
}

template <int K, bool USE_LUT>
__global__ void __launch_bounds__(kMaxN * 32, 1) thc_fused_kernel(const __grid_constant__ FusedArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int n = a.n;
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;            // worker of this warp
  constexpr int k = K;                       // log2(rotation block), 5..10
  constexpr int nblk = kTileN >> K;
  const Layout L = layout_for(n, nblk, a.q);
  double *scratch = reinterpret_cast<double *>(smem + L.scratch) + w * (32 * kScrRow);
  float *xs = reinterpret_cast<float *>(scratch);                  // x_rot staging (layout B)
  const float *cbuf_all = reinterpret_cast<const float *>(smem + L.cbuf);
  float *cbuf = reinterpret_cast<float *>(smem + L.cbuf) + w * (32 * kCRow);
  const int8_t *cod_all = reinterpret_cast<const int8_t *>(smem + L.cod);
  int8_t *cod = reinterpret_cast<int8_t *>(smem + L.cod) + w * 1024;
  const float *wr_all = reinterpret_cast<const float *>(smem + L.wr);
  float *wr = reinterpret_cast<float *>(smem + L.wr) + w * nblk * 2;
  double *bp = reinterpret_cast<double *>(smem + L.bp) + w * nblk * 8;
  double *lut = reinterpret_cast<double *>(smem + L.lut);
  uint32_t *sgn_all = reinterpret_cast<uint32_t *>(smem + L.sgn);

  const int q = a.q;
  const int ibound = (1 << (q - 1)) - 1;
  const double levels = static_cast<double>((1 << q) - 2);
  const long long sat = (1ll << (a.bits - 1)) - 1;
  const int lut_span = 2 * ibound + 1;
  constexpr bool use_lut = USE_LUT;
  const bool simd_fold = a.bits <= 8 && (256 % n) == 0 && (a.ring_blk % 4) == 0;
  constexpr int rpb_log = k - 5;   // layout-B registers per rotation block = 2^(k-5)
  // B^-1/2 is a power of two for even log2(B): scaling the own-decode inputs by it is exact and
  // commutes with every fp64 butterfly, so the per-element multiply after the WHT disappears
  constexpr bool kPow2Scale = (K % 2) == 0;

  // ---- PCG64 coin stream of worker w: four lane-strided chains (j mod 4), 128-step jumps.
  const uint64_t inc_h = a.streams[w].inc_hi, inc_l = a.streams[w].inc_lo;
  // the per-step (128-step) jump stays in registers; the once-per-tile jumps live in shared
  // memory (pcgw: {m32, c32, mt, ct}) to keep the quantizer loop free of spills
  uint32_t m128[4], c128[4];
  uint32_t *pcgw = reinterpret_cast<uint32_t *>(smem + L.pcg) + w * 16;
  {
    uint64_t h, l;
    uint32_t t4[4];
    limbs(gc::kPcgJump[7][0], gc::kPcgJump[7][1], m128);
    mul128(gc::kPcgJump[7][2], gc::kPcgJump[7][3], inc_h, inc_l, h, l);
    limbs(h, l, c128);
    if (lane == 0) {
      limbs(gc::kPcgJump[5][0], gc::kPcgJump[5][1], t4);
      for (int e = 0; e < 4; ++e) pcgw[e] = t4[e];
      mul128(gc::kPcgJump[5][2], gc::kPcgJump[5][3], inc_h, inc_l, h, l);
      limbs(h, l, t4);
      for (int e = 0; e < 4; ++e) pcgw[4 + e] = t4[e];
      limbs(a.tile_jump[0], a.tile_jump[1], t4);
      for (int e = 0; e < 4; ++e) pcgw[8 + e] = t4[e];
      mul128(a.tile_jump[2], a.tile_jump[3], inc_h, inc_l, h, l);
      limbs(h, l, t4);
      for (int e = 0; e < 4; ++e) pcgw[12 + e] = t4[e];
    }
    __syncwarp();
  }
  Lcg tile_state;
  {
    gc::Pcg p;
    p.load(a.streams[w]);
    p.jump(static_cast<uint64_t>(a.tile_begin + blockIdx.x) * kTileN + lane + 1);
    tile_state.set(static_cast<uint64_t>(p.state >> 64), static_cast<uint64_t>(p.state));
  }

  const float *gw = a.g + w * a.ld;
  const float *rw = a.r ? a.r + w * a.ld : nullptr;
  float *ro = a.r ? a.rout + w * a.ld : nullptr;
  long long sz = 0, sz2 = 0, clips = 0;
  double nmse_num = 0.0, nmse_den = 0.0;

  // sign words of the next tile are loaded one tile ahead (the forward rotation needs them first)
  uint32_t next_sign_word = 0;
  if (a.tile_begin + blockIdx.x < a.tiles) next_sign_word = a.signs[((a.tile_begin + blockIdx.x) * kTileN >> 5) + lane];
  // loop-carried tile bookkeeping instead of per-tile 64-bit divisions: the estimate warp
  // (tile mod n), the sign-buffer parity, and the ring block of the tile start (t0 / ring_blk with
  // its remainder; a tile crosses at most one ring-block boundary when ring_blk >= 1024)
  const int64_t first_tile = a.tile_begin + blockIdx.x;
  const int64_t stride_elems = static_cast<int64_t>(gridDim.x) * kTileN;
  // (32-bit: ring_blk = ceil(P / n) <= 2^30 and the quotient is a worker index)
  const bool ring_incr = a.ring_blk >= kTileN && a.ring_blk < (int64_t{1} << 31);
  const int rb = static_cast<int>(a.ring_blk);
  // loop invariants and the per-warp tile counters live in shared memory (registers are at the
  // 128 cap): inv[0..3] = gridDim % n, ring quotient / remainder steps, fold share per warp;
  // wst = {estimate warp, ring block of the tile start, its remainder, sign-buffer parity}
  int *inv = reinterpret_cast<int *>(smem + L.pcg) + n * 16;
  int *wst = inv + 8 + 4 * w;
  if (threadIdx.x == 0) {
    inv[0] = static_cast<int>(gridDim.x % n);
    inv[1] = ring_incr ? static_cast<int>(stride_elems / a.ring_blk) : 0;
    inv[2] = ring_incr ? static_cast<int>(stride_elems % a.ring_blk) : 0;
    inv[3] = (kTileN + n - 1) / n;
    inv[4] = rb;
    inv[5] = ring_incr ? 1 : 0;
  }
  if (lane == 0) {
    const int q0 = ring_incr ? static_cast<int>((first_tile * kTileN) / a.ring_blk) : 0;
    wst[0] = static_cast<int>(first_tile % n);
    wst[1] = q0;
    wst[2] = ring_incr ? static_cast<int>(first_tile * kTileN - static_cast<int64_t>(q0) * a.ring_blk) : 0;
    wst[3] = 0;
  }
  __syncthreads();
  for (int64_t tile = first_tile; tile < a.tiles; tile += gridDim.x) {
    const int64_t t0 = tile * kTileN;
    const uint32_t my_sign_word = next_sign_word;
    if (tile + gridDim.x < a.tiles) next_sign_word = a.signs[((tile + gridDim.x) * kTileN >> 5) + lane];
    uint32_t *sgn = sgn_all + wst[3] * 32;
    {   // pull the next tile of this worker's g and r rows into L2 while this tile computes
      const int64_t tn = t0 + static_cast<int64_t>(gridDim.x) * kTileN;
      if (lane < 2 && tn + kTileN <= min(a.dim, a.tiles * kTileN) && a.aligned) {
        const float *src = lane == 0 ? gw + tn : (rw ? rw + tn : nullptr);
        if (src)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(kTileN * 4) : "memory");
      }
    }
    // ---- corrected = f32(g + r) (compressors.py:624-626), coalesced loads -> cbuf.  Full
    // aligned tiles issue all 16 float4 loads before the first add, so the tile start pays one
    // memory latency instead of eight (per-iteration bounds checks kept them serialised).
    if (a.aligned && t0 + kTileN <= a.dim) {
#pragma unroll
      for (int h = 0; h < 8; h += HALF) {
        float4 gv[HALF], rv[HALF];
#pragma unroll
        for (int m = 0; m < HALF; ++m)
          gv[m] = __ldcs(reinterpret_cast<const float4 *>(gw + t0 + (lane + 32 * (h + m)) * 4));
        if (rw) {
#pragma unroll
          for (int m = 0; m < HALF; ++m)
            rv[m] = __ldcs(reinterpret_cast<const float4 *>(rw + t0 + (lane + 32 * (h + m)) * 4));
#pragma unroll
          for (int m = 0; m < HALF; ++m) {
            gv[m].x = gv[m].x + rv[m].x;
            gv[m].y = gv[m].y + rv[m].y;
            gv[m].z = gv[m].z + rv[m].z;
            gv[m].w = gv[m].w + rv[m].w;
          }
        }
#pragma unroll
        for (int m = 0; m < HALF; ++m) *reinterpret_cast<float4 *>(cbuf + cidx((lane + 32 * (h + m)) * 4)) = gv[m];
      }
    } else
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const int e4 = (lane + 32 * m) * 4;
      const int64_t i = t0 + e4;
      float4 c;
      if (a.aligned && i + 3 < a.dim) {
        c = __ldcs(reinterpret_cast<const float4 *>(gw + i));
        if (rw) {
          const float4 rv = __ldcs(reinterpret_cast<const float4 *>(rw + i));
          c.x = c.x + rv.x;
          c.y = c.y + rv.y;
          c.z = c.z + rv.z;
          c.w = c.w + rv.w;
        }
      } else {
        float t[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          float v = 0.0f;
          if (i + u < a.dim) {
            v = gw[i + u];
            if (rw) v = v + rw[i + u];
          }
          t[u] = v;
        }
        c = make_float4(t[0], t[1], t[2], t[3]);
      }
      *reinterpret_cast<float4 *>(cbuf + cidx(e4)) = c;
    }
    if (w == 0) sgn[lane] = my_sign_word;
    __syncwarp();

    // ---- forward rotation (transforms.py:107-117)
    double v[32];
#pragma unroll
    for (int m = 0; m < 8; ++m) {
      const float4 c = *reinterpret_cast<const float4 *>(cbuf + cidx(lane * 32 + 4 * m));
      v[4 * m + 0] = apply_sign(static_cast<double>(c.x), (my_sign_word >> (4 * m + 0)) & 1u);
      v[4 * m + 1] = apply_sign(static_cast<double>(c.y), (my_sign_word >> (4 * m + 1)) & 1u);
      v[4 * m + 2] = apply_sign(static_cast<double>(c.z), (my_sign_word >> (4 * m + 2)) & 1u);
      v[4 * m + 3] = apply_sign(static_cast<double>(c.w), (my_sign_word >> (4 * m + 3)) & 1u);
    }
    wht_tile<K>(v, scratch, lane);
    // lane's sign "column": bit j = sign of element 32j + lane (layout B), from 32 ballots over
    // the row words the lanes already hold -- the own-decode epilogue then reads no shared memory
    const uint32_t sign_col = bit_transpose32(my_sign_word, lane);

    // ---- x_rot = f32(v * B^-1/2), staged in layout B; per-block (min, max) (compressors.py:447-453)
    {
      float blo = INFINITY, bhi = -INFINITY;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const float f = static_cast<float>(v[j] * a.scale);
        xs[j * 32 + lane] = f;
        blo = fminf(blo, f);
        bhi = fmaxf(bhi, f);
        if (((j + 1) & ((1 << rpb_log) - 1)) == 0) {   // last register of block j >> rpb_log
#pragma unroll
          for (int o = 16; o; o >>= 1) {
            blo = fminf(blo, __shfl_xor_sync(0xffffffffu, blo, o));
            bhi = fmaxf(bhi, __shfl_xor_sync(0xffffffffu, bhi, o));
          }
          if (lane == 0) {
            wr[2 * (j >> rpb_log)] = blo;
            wr[2 * (j >> rpb_log) + 1] = bhi;
          }
          blo = INFINITY;
          bhi = -INFINITY;
        }
      }
    }
    __syncthreads();   // (A) every worker's block ranges are in wr_all

    // ---- range consensus, ElemMin / ElemMax over workers (pipelines.py:271-288)
    if (lane < nblk) {
      float lo = wr_all[2 * lane], hi = wr_all[2 * lane + 1];
      for (int u = 1; u < n; ++u) {
        lo = fminf(lo, wr_all[u * nblk * 2 + 2 * lane]);
        hi = fmaxf(hi, wr_all[u * nblk * 2 + 2 * lane + 1]);
      }
      const double dlo = static_cast<double>(lo), dhi = static_cast<double>(hi);
      const double step = (dhi - dlo) / levels;
      bp[8 * lane] = dlo;
      bp[8 * lane + 1] = dhi;
      bp[8 * lane + 2] = (dlo + dhi) / 2.0;
      bp[8 * lane + 3] = step;
      bp[8 * lane + 4] = step > 0.0 ? 1.0 / step : 0.0;   // degenerate: any finite value works
      bp[8 * lane + 5] = dhi > dlo ? step : 0.0;     // dequantize_sum's step (compressors.py:520)
      *reinterpret_cast<float4 *>(bp + 8 * lane + 6) = screen_params((dlo + dhi) / 2.0, step, static_cast<double>(ibound));
    }
    __syncwarp();
    // dq(z, 1) table for the own decode (compressors.py:519-521), built cooperatively.
    if (use_lut) {
      for (int e = threadIdx.x; e < nblk * lut_span; e += n * 32) {
        const int b = e / lut_span, z = e - b * lut_span - ibound;
        // pre-scaled by B^-1/2 when that is a power of two (exact, and the WHT commutes with it)
        lut[e] = static_cast<double>(static_cast<float>(1.0 * bp[8 * b + 2] + bp[8 * b + 5] * static_cast<double>(z))) *
                 (kPow2Scale ? a.scale : 1.0);
      }
    }

    // ---- quantize_stochastic (compressors.py:473-498), layout B: e = 32j + lane; four
    // interleaved LCG chains (j mod 4), each jumping 128 steps per use.
    {
      Lcg ch[4];
      ch[0] = tile_state;
      {
        uint32_t m32[4], c32[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) m32[e] = pcgw[e], c32[e] = pcgw[4 + e];
#pragma unroll
        for (int c = 1; c < 4; ++c) {
          ch[c] = ch[c - 1];
          ch[c].step(m32, c32);
        }
      }
      int tz = 0, tz2 = 0;   // per-tile code sums (|z| <= 127, 32 codes per lane: int32 is exact)
      for (int j = 0; j < 32; j += 4) {
        int z[4];
        uint32_t hw[4], oa[4], ob[4], orot[4];
        float xv[4];
        bool safe = true;
        // screen parameters: one rotation block spans >= 4 registers when B >= 128
        const float4 sp_j = *reinterpret_cast<const float4 *>(bp + 8 * (j >> rpb_log) + 6);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const float4 sp =
              rpb_log >= 2 ? sp_j : *reinterpret_cast<const float4 *>(bp + 8 * ((j + c) >> rpb_log) + 6);
          hw[c] = ch[c].out_hi(oa[c], ob[c], orot[c]);
#if GC_THC_IMM
          ch[c].step128(c128);
#else
          ch[c].step(m128, c128);
#endif
          xv[c] = xs[(j + c) * 32 + lane];
          // fp32 screen: floor by the 1.5 * 2^23 magic constant (|t32| < 2^22), frac, 23-bit coin;
          // safe iff min(f, 1 - f, |c23 - f|) > H (1 - f is exact for f >= 1/2)
          const float tq = (xv[c] - sp.x) * sp.y;
          const float sm = __fadd_rd(tq, 12582912.0f);
          const float f = tq - (sm - 12582912.0f);
          const float c23 = __uint_as_float(0x3f800000u | (hw[c] >> 9)) - 1.0f;
          safe = safe && fminf(fminf(f, 1.0f - f), fabsf(c23 - f)) > sp.z;
          z[c] = (__float_as_int(sm) - 0x4B400000) + (c23 < f ? 1 : 0);
        }
        if (__any_sync(0xffffffffu, !safe)) {   // warp-uniform: the exact path stays off the main line
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
        // (degenerate blocks, compressors.py:497, come out as code 0 from their screen parameters)
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
    {
      uint32_t mt[4], ct[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) mt[e] = pcgw[8 + e], ct[e] = pcgw[12 + e];
      tile_state.step(mt, ct);
    }
    __syncthreads();   // (B) all codes and the dq table of the tile are in shared memory

    if (a.codes && t0 + lane * 32 < a.active) {   // optional code dump (parity tests)
      const uint4 *src = reinterpret_cast<const uint4 *>(cod + lane * 32);
      uint4 *dst = reinterpret_cast<uint4 *>(a.codes + w * a.active + t0 + lane * 32);
      dst[0] = src[0];
      dst[1] = src[1];
    }

    // ---- ring-ordered saturating fold (SatIntSum, collectives.py:123-143, 215-226), split
    // over all warps; dequantize_sum(., n) lands in the estimate warp's transpose rows.

    const int ew = wst[0];
    double *escr = reinterpret_cast<double *>(smem + L.scratch) + ew * (32 * kScrRow);
    {
      const double nd = static_cast<double>(n);
      const int per = inv[3];
      const int e_end = min(kTileN, (w + 1) * per);
      if (simd_fold) {
        // four coordinates per lane as packed int8 (ring blocks are 4-aligned here)
        for (int e = w * per + lane * 4; e < e_end; e += 128) {
          const int s0 = inv[5] ? wst[1] + (wst[2] + e >= inv[4] ? 1 : 0) : static_cast<int>((t0 + e) / a.ring_blk);
          uint32_t acc = *reinterpret_cast<const uint32_t *>(cod_all + s0 * 1024 + e);
          int u = s0;
          for (int m = 1; m < n; ++m) {
            u = (u + 1 == n) ? 0 : u + 1;
            const uint32_t z = *reinterpret_cast<const uint32_t *>(cod_all + u * 1024 + e);
            const uint32_t wrap = __vadd4(acc, z);
            uint32_t c;
            if (a.bits == 8) {
              c = __vmaxs4(__vaddss4(acc, z), 0x81818181u);   // clamp to +-127
            } else {
              const uint32_t hs = static_cast<uint32_t>(sat) * 0x01010101u;
              const uint32_t ls = static_cast<uint32_t>(-sat) & 0xffu;
              c = __vmins4(__vmaxs4(wrap, ls * 0x01010101u), hs);
            }
            clips += __popc(__vcmpne4(wrap, c)) >> 3;
            acc = c;
          }
          const int blk = e >> k;
          const double *pb = bp + 8 * blk;
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const int zs = static_cast<int8_t>((acc >> (8 * b)) & 0xffu);
            escr[((e + b) >> 5) * kScrRow + ((e + b) & 31)] =
                static_cast<double>(static_cast<float>(nd * pb[2] + pb[5] * static_cast<double>(zs)));
          }
        }
      } else {
        for (int e = w * per + lane; e < e_end; e += 32) {
          const int64_t i = t0 + e;
          // ring block j starts at worker j
          const int s0 = inv[5] ? wst[1] + (wst[2] + e >= inv[4] ? 1 : 0) : static_cast<int>(i / a.ring_blk);
          long long acc = cod_all[s0 * 1024 + e];
          int u = s0;
          for (int m = 1; m < n; ++m) {
            u = (u + 1 == n) ? 0 : u + 1;
            acc += cod_all[u * 1024 + e];
            const long long c = acc > sat ? sat : (acc < -sat ? -sat : acc);
            clips += (c != acc);
            acc = c;
          }
          const double *pb = bp + 8 * (e >> k);
          escr[(e >> 5) * kScrRow + (e & 31)] =
              static_cast<double>(static_cast<float>(nd * pb[2] + pb[5] * static_cast<double>(acc)));
        }
      }
    }
    // (D) the tile's dequantized sums are complete.  With n = 8 the fold of warp w covers
    // coordinates [128w, 128w + 128) = rows 4w..4w+3, exactly the rows its row phase below
    // transforms, so the dependency is warp-local.
    if (n == 8) __syncwarp(); else __syncthreads();

    // ---- estimate inverse rotation spread over all warps (transforms.py:120-126): a 32-lane
    // step covers 4 rows x 32 columns of the 32 x 32 tile, 4 elements per lane.  Row phase:
    // stages 0-1 in registers, 2-4 by shuffles; column phase: stages 5-6 in registers, 7-9 by
    // shuffles.  Butterfly order is bit 0 first, exactly as in the single-warp transform.
    {
      const int sub = lane >> 3, q4 = (lane & 7) * 4;
#pragma unroll 1
      for (int gi = w; gi < 8; gi += n) {
        double* rowp = escr + (4 * gi + sub) * kScrRow + q4;
        double e[4] = {rowp[0], rowp[1], rowp[2], rowp[3]};
        if (K > 0) { double x = e[0], y = e[1]; e[0] = x + y; e[1] = x - y; x = e[2]; y = e[3]; e[2] = x + y; e[3] = x - y; }
        if (K > 1) { double x = e[0], y = e[2]; e[0] = x + y; e[2] = x - y; x = e[1]; y = e[3]; e[1] = x + y; e[3] = x - y; }
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          if (K > 2 + b) {
            const bool upper = (lane >> b) & 1;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const double o = __shfl_xor_sync(0xffffffffu, e[t], 1 << b);
              e[t] = upper ? o - e[t] : e[t] + o;
            }
          }
        }
        rowp[0] = e[0]; rowp[1] = e[1]; rowp[2] = e[2]; rowp[3] = e[3];
      }
      __syncthreads();   // (E) row stages done
      const gc::DivN dn(n);   // / n (pipelines.py:308-311): exact reciprocal product for power-of-two n
      const double nd = static_cast<double>(n);
#pragma unroll 1
      for (int gi = w; gi < 8; gi += n) {
        const int col = 4 * gi + sub;
        double e[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) e[t] = escr[(q4 + t) * kScrRow + col];
        if (K > 5) { double x = e[0], y = e[1]; e[0] = x + y; e[1] = x - y; x = e[2]; y = e[3]; e[2] = x + y; e[3] = x - y; }
        if (K > 6) { double x = e[0], y = e[2]; e[0] = x + y; e[2] = x - y; x = e[1]; y = e[3]; e[1] = x + y; e[3] = x - y; }
#pragma unroll
        for (int b = 0; b < 3; ++b) {
          if (K > 7 + b) {
            const bool upper = (lane >> b) & 1;
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const double o = __shfl_xor_sync(0xffffffffu, e[t], 1 << b);
              e[t] = upper ? o - e[t] : e[t] + o;
            }
          }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int row = q4 + t;
          const int el = row * 32 + col;
          const int64_t i = t0 + el;
          const float f = dn(static_cast<float>(apply_sign(e[t] * a.scale, (sgn[row] >> col) & 1u)));
          if (i < a.dim) {
            __stcs(a.est + i, f);
            if (n == 1 && rw) __stcs(ro + i, cbuf[cidx(el)] - f);   // one worker: own == estimate
            if (a.nmse) {
              double ref = 0.0;
              for (int u = 0; u < n; ++u) ref += static_cast<double>(cbuf_all[u * (32 * kCRow) + cidx(el)]);
              ref = ref / nd;
              const double err = static_cast<double>(f) - ref;
              nmse_num += err * err;
              nmse_den += ref * ref;
            }
          }
        }
      }
    }

    __syncthreads();   // (F) the estimate buffer (warp ew's scratch) is free again

    // ---- own decode + ef_update (pipelines.py:312-318, 168-170)
    if (rw && n > 1) {
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
      wht_tile<K>(v, scratch, lane);
      if (t0 + kTileN <= a.dim) {   // full tile: no bounds checks, immediate store offsets
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
          const int64_t i = t0 + e;
          const float own = static_cast<float>(apply_sign(kPow2Scale ? v[j] : v[j] * a.scale, (sign_col >> j) & 1u));
          if (i < a.dim) __stcs(ro + i, cbuf[cidx(e)] - own);
        }
      }
    }
    // (C) end of tile: only the nmse reduction needs it (it reads every warp's cbuf); all other
    // buffers are protected by barriers A / B / D of the next tile (sign words double-buffered).
    if (a.nmse) __syncthreads();
    __syncwarp();   // every lane of the warp is done with this tile's counters
    if (lane == 0) {
      int e2 = wst[0] + inv[0];
      wst[0] = e2 >= n ? e2 - n : e2;
      if (inv[5]) {
        int q = wst[1] + inv[1], r = wst[2] + inv[2];
        if (r >= inv[4]) {
          r -= inv[4];
          ++q;
        }
        wst[1] = q;
        wst[2] = r;
      }
      wst[3] ^= 1;
    }
    __syncwarp();
  }

#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
    sz2 += __shfl_xor_sync(0xffffffffu, sz2, o);
    clips += __shfl_xor_sync(0xffffffffu, clips, o);
    nmse_num += __shfl_xor_sync(0xffffffffu, nmse_num, o);
    nmse_den += __shfl_xor_sync(0xffffffffu, nmse_den, o);
  }
  if (lane == 0) {
    if (a.counters) {
      atomicAdd(&a.counters[1], static_cast<unsigned long long>(sz));
      atomicAdd(&a.counters[2], static_cast<unsigned long long>(sz2));
      atomicAdd(&a.counters[3], static_cast<unsigned long long>(clips));
    }
    if (a.nmse && (nmse_num != 0.0 || nmse_den != 0.0)) {
      atomicAdd(&a.nmse[0], nmse_num);
      atomicAdd(&a.nmse[1], nmse_den);
    }
  }
}

}  // namespace

namespace {

int launch_fused(const gc_thc_geom *g, int32_t n, const float *grads, const float *resid_in, float *resid_out,
                 int64_t ld, int64_t tile_begin, int64_t tile_end, const uint32_t *sign_bits,
                 const gc_pcg64 *coin_streams, float *estimate, int8_t *codes, int64_t *counters, double *nmse_acc,
                 void *stream) {
  GC_REQUIRE(g != nullptr, "geometry is null");
  GC_REQUIRE(n >= 1 && n <= kMaxN, "fused THC round supports 1..16 workers");
  GC_REQUIRE(g->dim >= 1 && g->padded >= kTileN && (g->padded & (g->padded - 1)) == 0 && g->padded >= g->dim,
             "fused THC round needs padded >= 1024 (power of two)");
  GC_REQUIRE(g->block >= 32 && g->block <= kTileN && (g->block & (g->block - 1)) == 0,
             "fused THC round needs a rotation block in [32, 1024]");
  GC_REQUIRE(g->quant_bits >= 2 && g->quant_bits <= 8 && g->wire_bits >= g->quant_bits && g->wire_bits <= 32,
             "invalid quant/wire bits");
  GC_REQUIRE(grads && sign_bits && coin_streams && estimate && ld >= g->dim, "invalid argument");
  GC_REQUIRE((resid_in == nullptr) == (resid_out == nullptr), "residual in/out must both be set or both NULL");

  FusedArgs a{};
  a.dim = g->dim;
  a.padded = g->padded;
  a.active = ((g->dim + g->block - 1) / g->block) * g->block;
  const int64_t all_tiles = (a.active + kTileN - 1) / kTileN;
  if (tile_end < 0 || tile_end > all_tiles) tile_end = all_tiles;
  GC_REQUIRE(tile_begin >= 0 && tile_begin <= tile_end, "invalid tile range");
  if (tile_begin == tile_end) return GC_OK;
  a.tile_begin = tile_begin;
  a.tiles = tile_end;
  a.ring_blk = (g->padded + n - 1) / n;
  a.n = n;
  int k = 0;
  while ((int64_t{1} << k) < g->block) ++k;
  a.k = k;
  a.q = g->quant_bits;
  a.bits = g->wire_bits;
  a.scale = g->scale;
  a.g = grads;
  a.r = resid_in;
  a.rout = resid_out;
  a.ld = ld;
  a.aligned = ((reinterpret_cast<uintptr_t>(grads) | reinterpret_cast<uintptr_t>(resid_in) |
                reinterpret_cast<uintptr_t>(resid_out)) & 15) == 0 && (ld % 4) == 0;
  a.signs = sign_bits;
  a.est = estimate;
  a.codes = codes;
  a.counters = reinterpret_cast<unsigned long long *>(counters);
  a.nmse = nmse_acc;
  for (int w = 0; w < n; ++w) a.streams[w] = coin_streams[w];

  const int nblk = kTileN >> k;
  const bool lut = nblk * ((1 << g->quant_bits) - 1) <= kLutMax;
  using KernelFn = void (*)(FusedArgs);
  KernelFn fn = nullptr;
#define GC_PICK(KK)                                                       \
  case KK:                                                                \
    fn = lut ? thc_fused_kernel<KK, true> : thc_fused_kernel<KK, false>; \
    break;
  switch (k) {
    GC_PICK(5) GC_PICK(6) GC_PICK(7) GC_PICK(8) GC_PICK(9) GC_PICK(10)
    default: break;
  }
#undef GC_PICK
  GC_REQUIRE(fn != nullptr, "unsupported rotation block");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = layout_for(n, nblk, g->quant_bits).total;
  cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, n * 32, smem);
  if (per_sm < 1) {
    gc_set_error("fused THC kernel does not fit on an SM");
    return GC_ERR_UNSUPPORTED;
  }
  int64_t grid = static_cast<int64_t>(sms) * per_sm;
  if (grid > tile_end - tile_begin) grid = tile_end - tile_begin;
  host_jump(static_cast<uint64_t>(grid) * kTileN, a.tile_jump);
  fn<<<static_cast<unsigned>(grid), n * 32, smem, static_cast<cudaStream_t>(stream)>>>(a);
  GC_LAUNCH_CHECK("thc_fused_kernel");
  return GC_OK;
}

}  // namespace

extern "C" int gc_thc_round_fused(const gc_thc_geom *g, int32_t n, const float *grads, float *resid, int64_t ld,
                                  const uint32_t *sign_bits, const gc_pcg64 *coin_streams, float *estimate,
                                  int8_t *codes, int64_t *counters, double *nmse_acc, void *stream) {
  return launch_fused(g, n, grads, resid, resid, ld, 0, -1, sign_bits, coin_streams, estimate, codes, counters,
                      nmse_acc, stream);
}

extern "C" int gc_thc_round_fused_range(const gc_thc_geom *g, int32_t n, const float *grads, const float *resid_in,
                                        float *resid_out, int64_t ld, int64_t tile_begin, int64_t tile_end,
                                        const uint32_t *sign_bits, const gc_pcg64 *coin_streams, float *estimate,
                                        int8_t *codes, int64_t *counters, double *nmse_acc, void *stream) {
  return launch_fused(g, n, grads, resid_in, resid_out, ld, tile_begin, tile_end, sign_bits, coin_streams, estimate,
                      codes, counters, nmse_acc, stream);
}
