// Microbenchmark: tcgen05.mma kind::tf32 issue rate from shared memory, one CTA per SM, one thread
// issuing back-to-back MMAs into one TMEM accumulator, by M (64 / 128), N (8..256) and A major-ness
// (K-major SW128 / MN-major SW128 with 32-byte atoms).  Reports cycles per MMA and the fraction of
// the tf32 dense rate (1024 FMA per N column per cycle at M = 128, K = 8 ... measured, not assumed).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (static_cast<uint64_t>(lbo >> 4) << 16) |
         (static_cast<uint64_t>(sbo >> 4) << 32) | (1ull << 46) | (static_cast<uint64_t>(layout) << 61);
}

__global__ void __launch_bounds__(128, 1) rate_kernel(int m, int n, int mn_major, int iters, int kspread,
                                                      unsigned long long *cycles) {
  extern __shared__ unsigned char sm_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(sm_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t barp = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  // operands: A 128 x 32 fp32 (16 KB), B 256 x 32 fp32 (32 KB); small finite values
  for (int i = threadIdx.x; i < (16384 + 32768) / 4; i += blockDim.x)
    reinterpret_cast<float *>(sm_raw + (base - raw))[i] = 1.0f / (1 + (i & 7));
  if (threadIdx.x == 0) {
    mbar_init(barp, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(&tslot)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (mn_major ? (1u << 15) : 0u) |
                         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
  if (threadIdx.x == 0) {
    const uint32_t a0 = base, b0 = base + 16384;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const int ks = kspread ? (i & 3) : 0;
      const uint64_t a = mn_major ? desc(a0 + 1024 * ks, 4096, 512, 1) : desc(a0 + 32 * ks, 16, 1024, 2);
      const uint64_t b = desc(b0 + 32 * ks, 16, 1024, 2);
      const uint32_t acc = i ? 1u : 0u;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(a), "l"(b), "r"(idesc), "r"(acc)
          : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(barp) : "memory");
    mbar_wait(barp, 0);
    const long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = static_cast<unsigned long long>(t1 - t0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

int main() {
  unsigned long long *d_cycles, h = 0;
  cudaMalloc(&d_cycles, sizeof(unsigned long long));
  const int smem = 16384 + 32768 + 1024;
  cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int iters = 4096;
  for (int mn = 0; mn < 2; ++mn)
    for (int m : {64, 128})
      for (int n : {8, 16, 32, 64, 128, 256}) {
        if (m == 128 && n % 16) continue;
        rate_kernel<<<148, 128, smem>>>(m, n, mn, iters, 1, d_cycles);
        rate_kernel<<<148, 128, smem>>>(m, n, mn, iters, 1, d_cycles);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("m %d n %d mn %d: %s\n", m, n, mn, cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(&h, d_cycles, sizeof(h), cudaMemcpyDeviceToHost);
        const double cpm = static_cast<double>(h) / iters;
        printf("{\"a_major\": \"%s\", \"M\": %d, \"N\": %d, \"cycles_per_mma\": %.2f, \"fma_per_cycle\": %.0f}\n",
               mn ? "mn" : "k", m, n, cpm, m * n * 8.0 / cpm);
      }
  return 0;
}
