// Microbenchmark: the PCG64 128-step LCG jump (s = s * A^128 + c mod 2^128) as the serial
// carry-flag chain of gc_thc_tile.cuh (16 dependent mad/madc) vs a 64-bit formulation whose
// partial products are independent (s_lo * m_lo full product, the two cross terms low halves,
// one carry): same integer result, shorter dependency chain.  Four chains per thread as in the
// THC quantizer, 256 threads, two CTAs per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lcg_ilp lcg_ilp.cu && ./lcg_ilp
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr uint64_t kMl = 0x84fe009a6d09de01ull, kMh = 0x602167331d86cf56ull;

__device__ __forceinline__ void step_chain(uint32_t &s0, uint32_t &s1, uint32_t &s2, uint32_t &s3, uint32_t c0,
                                           uint32_t c1, uint32_t c2, uint32_t c3) {
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
      : "r"(s0), "r"(s1), "r"(s2), "r"(s3), "r"(c0), "r"(c1), "r"(c2), "r"(c3));
  s0 = r0; s1 = r1; s2 = r2; s3 = r3;
}

__device__ __forceinline__ void step_u64(uint64_t &lo, uint64_t &hi, uint64_t cl, uint64_t ch) {
  const uint64_t plo = lo * kMl;
  const uint64_t phi = __umul64hi(lo, kMl);
  const uint64_t cross = lo * kMh + hi * kMl + ch;
  const uint64_t nlo = plo + cl;
  hi = phi + cross + (nlo < plo ? 1ull : 0ull);
  lo = nlo;
}

template <int V>
__global__ void __launch_bounds__(256, 2) lcg(uint64_t cl, uint64_t ch, int steps, uint32_t *out) {
  uint64_t lo[4], hi[4];
  for (int k = 0; k < 4; ++k) {
    lo[k] = (uint64_t(threadIdx.x) * 7 + blockIdx.x * 13 + k * 3) * 0x9e3779b97f4a7c15ull;
    hi[k] = (uint64_t(blockIdx.x) * 5 + k) * 0xbf58476d1ce4e5b9ull;
  }
  uint32_t acc = 0;
  for (int i = 0; i < steps; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (V == 0) {
        uint32_t s0 = uint32_t(lo[k]), s1 = uint32_t(lo[k] >> 32), s2 = uint32_t(hi[k]), s3 = uint32_t(hi[k] >> 32);
        step_chain(s0, s1, s2, s3, uint32_t(cl), uint32_t(cl >> 32), uint32_t(ch), uint32_t(ch >> 32));
        lo[k] = (uint64_t(s1) << 32) | s0;
        hi[k] = (uint64_t(s3) << 32) | s2;
      } else {
        step_u64(lo[k], hi[k], cl, ch);
      }
      // the THC quantizer consumes the XSL-RR high word of every state
      const uint64_t x = lo[k] ^ hi[k];
      const uint32_t rot = uint32_t(hi[k] >> 58);
      acc ^= uint32_t(((x >> rot) | (x << ((64 - rot) & 63))) >> 32);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ uint32_t(lo[0] ^ hi[3]);
}

int main() {
  uint32_t *out;
  const int blocks = 148 * 2, threads = 256, steps = 8192;
  cudaMalloc(&out, blocks * threads * 4);
  uint32_t *h[2];
  const char *name[2] = {"carry_chain", "u64_ilp"};
  for (int v = 0; v < 2; ++v) {
    h[v] = new uint32_t[blocks * threads];
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      if (v == 0) lcg<0><<<blocks, threads>>>(0x1234567890abcdefull, 0x0fedcba987654321ull, steps, out);
      else lcg<1><<<blocks, threads>>>(0x1234567890abcdefull, 0x0fedcba987654321ull, steps, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaMemcpy(h[v], out, blocks * threads * 4, cudaMemcpyDeviceToHost);
    const double tot = double(blocks) * threads * steps * 4;
    printf("{\"variant\": \"%s\", \"ms\": %.4f, \"gsteps_per_s\": %.1f}\n", name[v], best, tot / best / 1e6);
  }
  int same = 1;
  for (int i = 0; i < blocks * threads; ++i) same &= h[0][i] == h[1][i];
  printf("{\"same_result\": %d}\n", same);
  return 0;
}
