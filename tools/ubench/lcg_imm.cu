// Microbenchmark: the PCG64 128-bit LCG step (s = s * m + c mod 2^128) with the multiplier in
// registers vs as compile-time immediates (the THC coin streams' 128-step jump is a constant).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o lcg_imm lcg_imm.cu && ./lcg_imm
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define STEP_ASM(M0, M1, M2, M3)                                                              \
  asm("mad.lo.cc.u32  %0, %4, %8, %12;\n\t"                                                   \
      "madc.hi.cc.u32 %1, %4, %8, %13;\n\t"                                                   \
      "madc.hi.cc.u32 %2, %4, %9, %14;\n\t"                                                   \
      "madc.hi.u32    %3, %4, %10, %15;\n\t"                                                  \
      "mad.lo.cc.u32  %1, %4, %9, %1;\n\t"                                                    \
      "madc.lo.cc.u32 %2, %4, %10, %2;\n\t"                                                   \
      "madc.lo.u32    %3, %4, %11, %3;\n\t"                                                   \
      "mad.lo.cc.u32  %1, %5, %8, %1;\n\t"                                                    \
      "madc.hi.cc.u32 %2, %5, %8, %2;\n\t"                                                    \
      "madc.hi.u32    %3, %5, %9, %3;\n\t"                                                    \
      "mad.lo.cc.u32  %2, %5, %9, %2;\n\t"                                                    \
      "madc.lo.u32    %3, %5, %10, %3;\n\t"                                                   \
      "mad.lo.cc.u32  %2, %6, %8, %2;\n\t"                                                    \
      "madc.hi.u32    %3, %6, %8, %3;\n\t"                                                    \
      "mad.lo.u32     %3, %6, %9, %3;\n\t"                                                    \
      "mad.lo.u32     %3, %7, %8, %3;"                                                        \
      : "=&r"(r0), "=&r"(r1), "=&r"(r2), "=&r"(r3)                                            \
      : "r"(s0), "r"(s1), "r"(s2), "r"(s3), M0, M1, M2, M3, "r"(c0), "r"(c1), "r"(c2), "r"(c3))

template <bool IMM>
__global__ void lcg(const uint32_t *mreg, uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, int steps,
                    uint32_t *out) {
  uint32_t st[4][4];
  for (int k = 0; k < 4; ++k)
    for (int e = 0; e < 4; ++e) st[k][e] = threadIdx.x * 7 + blockIdx.x * 13 + k * 3 + e;
  const uint32_t m0 = mreg[0], m1 = mreg[1], m2 = mreg[2], m3 = mreg[3];
  uint32_t acc = 0;
  for (int i = 0; i < steps; ++i) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t s0 = st[k][0], s1 = st[k][1], s2 = st[k][2], s3 = st[k][3], r0, r1, r2, r3;
      if (IMM)
        STEP_ASM("n"(0x6d09de01u), "n"(0x84fe009au), "n"(0x1d86cf56u), "n"(0x60216733u));
      else
        STEP_ASM("r"(m0), "r"(m1), "r"(m2), "r"(m3));
      st[k][0] = r0; st[k][1] = r1; st[k][2] = r2; st[k][3] = r3;
      acc ^= r3;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
}

int main() {
  uint32_t *m, *out;
  cudaMalloc(&m, 16);
  const uint32_t mh[4] = {0x6d09de01u, 0x84fe009au, 0x1d86cf56u, 0x60216733u};
  cudaMemcpy(m, mh, 16, cudaMemcpyHostToDevice);
  const int blocks = 148 * 8, threads = 256, steps = 4096;
  cudaMalloc(&out, blocks * threads * 4);
  uint32_t h0[2];
  for (int imm = 0; imm < 2; ++imm) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      if (imm) lcg<true><<<blocks, threads>>>(m, 1, 2, 3, 4, steps, out);
      else lcg<false><<<blocks, threads>>>(m, 1, 2, 3, 4, steps, out);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double stepsTot = double(blocks) * threads * steps * 4;
      if (rep == 2) printf("%s: %.3f ms, %.1f Gstep/s, %.2f ps/step\n", imm ? "immediate" : "register", ms, stepsTot / ms / 1e6, ms * 1e9 / stepsTot);
    }
    cudaMemcpy(&h0[imm], out, 4, cudaMemcpyDeviceToHost);
  }
  printf("same result: %d\n", h0[0] == h0[1]);
  return 0;
}
