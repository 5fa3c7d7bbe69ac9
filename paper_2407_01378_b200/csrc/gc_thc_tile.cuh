// Building blocks of the tile-wise THC kernels (gc_thc_fused.cu: n workers simulated on one GPU;
// gc_thc_rank.cu: one rank's workers in the distributed round).  A warp holds one worker's
// 1024-coordinate tile as 32 doubles per lane; the fp64 blockwise WHT runs bit-0-first
// (transforms.py:92-98) in registers with one padded shared-memory transpose, the PCG64 coin
// streams advance as 128-bit LCG limbs, and the quantizer decides codes with an fp32 screen
// backed by the reference's IEEE fp64 formula (compressors.py:481-498).  Files including this
// are compiled with -fmad=false (bit-exact fp64).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "gc_device.cuh"

#ifndef GC_THC_IMM
#define GC_THC_IMM 1
#endif

namespace thc {

constexpr int kTileN = 1024;
constexpr int kScrRow = 33;   // fp64 transpose rows padded to 33: conflict-free, immediate offsets
constexpr int kCRow = 36;     // corrected-value rows padded to 36 floats (float4 reads stay aligned)
constexpr int kScrBytes = 32 * kScrRow * 8;
constexpr int kCBytes = 32 * kCRow * 4;

template <int COUNT>
__device__ __forceinline__ void stages_reg(double (&v)[32]) {
#pragma unroll
  for (int s = 0; s < 5; ++s) {
    if (s < COUNT) {
      const int h = 1 << s;
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        if (!(j & h)) {
          const double a = v[j], b = v[j | h];
          v[j] = a + b;
          v[j | h] = a - b;
        }
      }
    }
  }
}

// layout A (lane owns 32*lane + j) -> layout B (lane owns 32*j + lane) through rows padded
// to 33 doubles: both directions hit 2 wavefronts per 256 B (optimal) with static offsets.
__device__ __forceinline__ void transpose_ab(double (&v)[32], double *scr, int lane) {
#pragma unroll
  for (int j = 0; j < 32; ++j) scr[lane * kScrRow + j] = v[j];
  __syncwarp();
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = scr[j * kScrRow + lane];
  __syncwarp();
}

// Full blockwise WHT (stages 0..K-1) of one tile from layout-A registers; ends in layout B.
template <int K>
__device__ __forceinline__ void wht_tile(double (&v)[32], double *scr, int lane) {
  stages_reg<(K < 5 ? K : 5)>(v);
  transpose_ab(v, scr, lane);
  stages_reg<K - 5>(v);
}

// cbuf keeps the tile in natural order, rows of 32 floats padded to 36: layout-A float4
// reads, layout-B scalar reads and the coalesced float4 stores are all conflict-free.
__device__ __forceinline__ int cidx(int e) { return (e >> 5) * kCRow + (e & 31); }

// x * (+1 or -1) as a sign-bit flip (bit-identical to the fp64 multiply by +-1.0).
__device__ __forceinline__ double apply_sign(double x, uint32_t positive) {
  return __longlong_as_double(__double_as_longlong(x) ^ (static_cast<long long>(positive ^ 1u) << 63));
}

// 32 x 32 bit-matrix transpose across the warp (row = lane, column = bit): returns the word whose
// bit j is bit `lane` of lane j's w.  Five shuffle stages swapping the off-diagonal blocks
// (16, 8, 4, 2, 1) instead of 32 ballots; used for the layout-B sign "column" of a tile.
__device__ __forceinline__ uint32_t bit_transpose32(uint32_t x, int lane) {
  const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    const int sft = 16 >> k;
    const uint32_t m = masks[k];
    const uint32_t y = __shfl_xor_sync(0xffffffffu, x, sft);
    x = (lane & sft) ? ((x & ~m) | ((y >> sft) & m)) : ((x & m) | ((y << sft) & ~m));
  }
  return x;
}

// PCG64 state as four 32-bit limbs (s0 least significant).  step(): s = s * m + c mod 2^128 as
// a schoolbook column product with PTX carry chains (17 IMADs); output(): numpy's XSL-RR.
struct Lcg {
  uint32_t s0, s1, s2, s3;
  __device__ __forceinline__ void set(uint64_t hi, uint64_t lo) {
    s0 = static_cast<uint32_t>(lo);
    s1 = static_cast<uint32_t>(lo >> 32);
    s2 = static_cast<uint32_t>(hi);
    s3 = static_cast<uint32_t>(hi >> 32);
  }
  __device__ __forceinline__ void step(const uint32_t (&m)[4], const uint32_t (&c)[4]) {
    uint32_t r0, r1, r2, r3;
    asm("mad.lo.cc.u32  %0, %4, %8, %12;\n\t"
        "madc.hi.cc.u32 %1, %4, %8, %13;\n\t"
        "madc.hi.cc.u32 %2, %4, %9, %14;\n\t"
        "madc.hi.u32    %3, %4, %10, %15;\n\t"
        "mad.lo.cc.u32  %1, %4, %9, %1;\n\t"
        "madc.lo.cc.u32 %2, %4, %10, %2;\n\t"
        "madc.lo.u32    %3, %4, %11, %3;\n\t"
        "mad.lo.cc.u32  %1, %5, %8, %1;\n\t"
        "madc.hi.cc.u32 %2, %5, %8, %2;\n\t"
        "madc.hi.u32    %3, %5, %9, %3;\n\t"
        "mad.lo.cc.u32  %2, %5, %9, %2;\n\t"
        "madc.lo.u32    %3, %5, %10, %3;\n\t"
        "mad.lo.cc.u32  %2, %6, %8, %2;\n\t"
        "madc.hi.u32    %3, %6, %8, %3;\n\t"
        "mad.lo.u32     %3, %6, %9, %3;\n\t"
        "mad.lo.u32     %3, %7, %8, %3;"
        : "=&r"(r0), "=&r"(r1), "=&r"(r2), "=&r"(r3)
        : "r"(s0), "r"(s1), "r"(s2), "r"(s3), "r"(m[0]), "r"(m[1]), "r"(m[2]), "r"(m[3]), "r"(c[0]),
          "r"(c[1]), "r"(c[2]), "r"(c[3]));
    s0 = r0;
    s1 = r1;
    s2 = r2;
    s3 = r3;
  }

#if GC_THC_IMM
  // s = s * A^128 + c with the 128-step jump multiplier as instruction immediates
  // (kPcgJump[7] mult = 0x602167331d86cf56'84fe009a6d09de01); c stays per-stream.
  __device__ __forceinline__ void step128(const uint32_t (&c)[4]) {
    uint32_t r0, r1, r2, r3;
    asm("mad.lo.cc.u32  %0, %4, 0x6d09de01, %8;\n\t"
        "madc.hi.cc.u32 %1, %4, 0x6d09de01, %9;\n\t"
        "madc.hi.cc.u32 %2, %4, 0x84fe009a, %10;\n\t"
        "madc.hi.u32    %3, %4, 0x1d86cf56, %11;\n\t"
        "mad.lo.cc.u32  %1, %4, 0x84fe009a, %1;\n\t"
        "madc.lo.cc.u32 %2, %4, 0x1d86cf56, %2;\n\t"
        "madc.lo.u32    %3, %4, 0x60216733, %3;\n\t"
        "mad.lo.cc.u32  %1, %5, 0x6d09de01, %1;\n\t"
        "madc.hi.cc.u32 %2, %5, 0x6d09de01, %2;\n\t"
        "madc.hi.u32    %3, %5, 0x84fe009a, %3;\n\t"
        "mad.lo.cc.u32  %2, %5, 0x84fe009a, %2;\n\t"
        "madc.lo.u32    %3, %5, 0x1d86cf56, %3;\n\t"
        "mad.lo.cc.u32  %2, %6, 0x6d09de01, %2;\n\t"
        "madc.hi.u32    %3, %6, 0x6d09de01, %3;\n\t"
        "mad.lo.u32     %3, %6, 0x84fe009a, %3;\n\t"
        "mad.lo.u32     %3, %7, 0x6d09de01, %3;"
        : "=&r"(r0), "=&r"(r1), "=&r"(r2), "=&r"(r3)
        : "r"(s0), "r"(s1), "r"(s2), "r"(s3), "r"(c[0]), "r"(c[1]), "r"(c[2]), "r"(c[3]));
    s0 = r0;
    s1 = r1;
    s2 = r2;
    s3 = r3;
  }
#endif

  // the high half of the XSL-RR output; (a, b, rot) let lo_of() rebuild the low half on demand
  __device__ __forceinline__ uint32_t out_hi(uint32_t &a, uint32_t &b, uint32_t &rot) const {
    const uint32_t xl = s0 ^ s2, xh = s1 ^ s3;
    rot = s3 >> 26;
    const bool swap = rot & 32u;
    a = swap ? xh : xl;
    b = swap ? xl : xh;
    return __funnelshift_r(b, a, rot);
  }
  static __device__ __forceinline__ uint32_t lo_of(uint32_t a, uint32_t b, uint32_t rot) {
    return __funnelshift_r(a, b, rot);
  }
};

__device__ __forceinline__ void limbs(uint64_t hi, uint64_t lo, uint32_t (&o)[4]) {
  o[0] = static_cast<uint32_t>(lo);
  o[1] = static_cast<uint32_t>(lo >> 32);
  o[2] = static_cast<uint32_t>(hi);
  o[3] = static_cast<uint32_t>(hi >> 32);
}

__device__ __forceinline__ void mul128(uint64_t ah, uint64_t al, uint64_t bh, uint64_t bl, uint64_t &rh,
                                       uint64_t &rl) {
  rl = al * bl;
  rh = __umul64hi(al, bl) + al * bh + ah * bl;
}

// coin_from: numpy's random() double (next64 >> 11) * 2^-53 from the two output halves.
__device__ __forceinline__ double coin_from(uint32_t hi, uint32_t lo) {
  const uint64_t u = (static_cast<uint64_t>(hi) << 32) | lo;
  return static_cast<double>(u >> 11) * (1.0 / 9007199254740992.0);
}

// The reference quantizer for one value, IEEE fp64 step by step (compressors.py:481-498):
// the rare coordinates the fp32 screen below cannot decide come here.
static __device__ __noinline__ int quantize_ref(double x, double lo, double hi, double mid, double step, double bound,
                                         double coin) {
  x = fmin(fmax(x, lo), hi);
  double t = (x - mid) / step;
  t = fmin(fmax(t, -bound), bound);
  double low = floor(t);
  double frac = t - low;
  if (frac > 1.0 - 1e-9) {
    low += 1.0;
    frac = 0.0;
  } else if (frac < 1e-9) {
    frac = 0.0;
  }
  const int z = static_cast<int>(low) + (coin < frac ? 1 : 0);
  const int b = static_cast<int>(bound);
  return z < -b ? -b : (z > b ? b : z);
}

// Per-block fp32 screen parameters {mid32, 1/step as f32, H, 1 - H}.  With t32 = (x - mid32) *
// inv32 in fp32, |t32 - t| <= E = m + (bound + m) * 3.01 * 2^-24 (m = |mid| / step * 2^-24:
// the rounding of mid to f32; the other terms: the f32 subtract, inv32 and the multiply).
// H = E + 2^-22 also covers the 23-bit coin prefix (2^-23) and the f32 rounding of
// frac = t32 - floor(t32) (2^-25).  A coordinate whose f32 frac lies in [H, 1 - H] and more
// than H from the coin prefix has the reference's floor(t), no snapping and the same coin
// comparison, so its code is decided in fp32; the rest (probability ~6H) take quantize_ref.
// Degenerate blocks (step <= 0) always pass the screen with t32 = 0 and a coin test against
// frac = 0 that never fires, i.e. code 0 as the reference forces (compressors.py:497).
__device__ __forceinline__ float4 screen_params(double mid, double step, double bound) {
  if (!(step > 0.0)) return make_float4(0.0f, 0.0f, -1.0f, 2.0f);
  const double m = fabs(mid) / step * 0x1p-24;
  const double h = (m + (bound + m) * 3.01 * 0x1p-24 + 0x1p-40 + 0x1p-22) * 1.001;
  if (!(h < 0x1p-8)) return make_float4(0.0f, 0.0f, 2.0f, -1.0f);   // never passes: exact path
  return make_float4(static_cast<float>(mid), static_cast<float>(1.0 / step), static_cast<float>(h),
                     static_cast<float>(1.0 - h));
}

using u128h = unsigned __int128;

inline void host_jump(uint64_t delta, uint64_t out[4]) {
  const u128h mult = (static_cast<u128h>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
  u128h cm = mult, cp = 1, am = 1, ap = 0;
  while (delta) {
    if (delta & 1) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
  out[0] = static_cast<uint64_t>(am >> 64);
  out[1] = static_cast<uint64_t>(am);
  out[2] = static_cast<uint64_t>(ap >> 64);
  out[3] = static_cast<uint64_t>(ap);
}


}  // namespace thc
