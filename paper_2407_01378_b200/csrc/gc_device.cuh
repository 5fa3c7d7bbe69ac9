// Device-side building blocks shared by the kernels: PCG64 (numpy's BitGenerator)
// with jump-ahead, the fp16 wire rounding, and the fp64 Walsh-Hadamard stage loop.
#pragma once
#include <cuda_fp16.h>
#include <stdint.h>

#include "gc_pcg_tables.h"
#include "gradcomp_b200.h"

namespace gc {

typedef unsigned __int128 u128;

__device__ __forceinline__ u128 mk128(uint64_t hi, uint64_t lo) {
  return (static_cast<u128>(hi) << 64) | lo;
}

// PCG64 multiplier (numpy pcg64.h PCG_DEFAULT_MULTIPLIER_128).
#define GC_PCG_MULT (gc::mk128(0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull))

// {mult_hi, mult_lo, plus_hi, plus_lo} for 2^k steps (gen_pcg_tables.py).
static __constant__ uint64_t kPcgJump[128][4] = GC_PCG_TABLE_INIT;

struct Pcg {
  u128 state, inc;
  __device__ __forceinline__ void load(const gc_pcg64 &g) {
    state = mk128(g.state_hi, g.state_lo);
    inc = mk128(g.inc_hi, g.inc_lo);
  }
  // state <- state advanced by `delta` steps (delta < 2^64).
  __device__ __forceinline__ void jump(uint64_t delta) {
    u128 am = 1, ap = 0;
    for (int k = 0; delta; ++k, delta >>= 1) {
      if (delta & 1) {
        const u128 m = mk128(kPcgJump[k][0], kPcgJump[k][1]);
        const u128 p = mk128(kPcgJump[k][2], kPcgJump[k][3]);
        am *= m;
        ap = ap * m + p;
      }
    }
    state = am * state + ap * inc;
  }
  // numpy pcg64_next64: step, then XSL-RR output.
  __device__ __forceinline__ uint64_t next() {
    state = state * GC_PCG_MULT + inc;
    return output(state);
  }
  static __device__ __forceinline__ uint64_t output(u128 s) {
    const uint64_t hi = static_cast<uint64_t>(s >> 64);
    const uint64_t x = hi ^ static_cast<uint64_t>(s);
    const unsigned rot = static_cast<unsigned>(hi >> 58);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
};

// numpy Generator.random(): (next64 >> 11) * 2^-53.
__device__ __forceinline__ double coin_from(uint64_t u) {
  return static_cast<double>(u >> 11) * (1.0 / 9007199254740992.0);
}

// fp16_round_trip (vectors.py:136-152): RNE cast to binary16, overflow saturates to +-65504.
__device__ __forceinline__ float fp16_round_trip(float x) {
  const float y = __half2float(__float2half_rn(x));
  return isinf(y) ? copysignf(65504.0f, x) : y;
}

// One fp64 butterfly stage of the Sylvester WHT (transforms.py:92-98):
// pairs (i, i + 2^s) inside groups of 2^(s+1) -> (lo + hi, lo - hi).
// `buf` holds `count` doubles (a multiple of 2^(s+1)); NT threads cooperate.
template <int NT>
__device__ __forceinline__ void wht_stage_smem(double *buf, int count, int s) {
  const int half = 1 << s;
  for (int p = threadIdx.x; p < (count >> 1); p += NT) {
    const int i = ((p >> s) << (s + 1)) | (p & (half - 1));
    const double a = buf[i];
    const double b = buf[i + half];
    buf[i] = a + b;
    buf[i + half] = a - b;
  }
  __syncthreads();
}

__device__ __forceinline__ bool sign_positive(const uint32_t *bits, int64_t i) {
  return (bits[i >> 5] >> (i & 31)) & 1u;
}

// x / n in f32 with the IEEE quotient the reference computes: for a power-of-two n the product
// with the exact reciprocal is the same correctly rounded value (no division sequence).
struct DivN {
  float n, inv;
  bool pow2;
  __device__ __forceinline__ explicit DivN(int d) : n(static_cast<float>(d)), inv(1.0f / static_cast<float>(d)),
                                                    pow2(d > 0 && (d & (d - 1)) == 0) {}
  __device__ __forceinline__ float operator()(float x) const { return pow2 ? x * inv : x / n; }
};

// Order-preserving float <-> uint encoding for atomic min/max.
__device__ __forceinline__ unsigned int float_to_ordered(float f) {
  const unsigned int u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ordered_to_float(unsigned int u) {
  return __uint_as_float((u & 0x80000000u) ? (u & 0x7FFFFFFFu) : ~u);
}

}  // namespace gc
