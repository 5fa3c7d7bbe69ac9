// Device helpers shared by the tcgen05 PowerSGD passes (gc_psgd_tma.cu, gc_psgd_async.cu):
// mbarriers, UMMA shared-memory descriptors, the 3xTF32 split, cp.async and the deferred-EF
// own term.  sm_100a only.
#pragma once

#include <cstdint>

namespace gcu {

// byte offset of (row, 16-byte chunk) in a K-major SWIZZLE_128B tile (8 rows x 128 B atoms,
// 16-byte chunks XOR-swizzled by row; 1024-byte aligned)
__device__ __forceinline__ uint32_t sw128(int row, int chunk) {
  return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4));
}

// UMMA shared-memory descriptor, K-major SWIZZLE_128B: LBO 16 B (unused), SBO 1024 B between
// 8-row groups, descriptor version 1 (sm_100)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

// instruction descriptor: D f32, A/B tf32, K-major unless a_mn, N x M
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n, bool a_mn = false) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn ? (1u << 15) : 0u) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

// 3xTF32 split by truncation: big keeps the top 10 mantissa bits (what kind::tf32 reads of an fp32
// pattern), small = tf32(c - big); c - (big + small) < 2^-20 |c|
__device__ __forceinline__ void split3(float c, float &big, float &small) {
  big = __uint_as_float(__float_as_uint(c) & 0xFFFFE000u);
  small = __uint_as_float(__float_as_uint(c - big) & 0xFFFFE000u);
}

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// 1-D TMA bulk copy global -> shared, completing bytes on the mbarrier (16-byte aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}

// 4-byte asynchronous global -> shared copy
__device__ __forceinline__ void cp_async4(uint32_t dst, const float *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// own = P_hat_prev[i,:] . Q_w_prev[j,:] exactly as the decode kernel forms it (fp32 product, then
// FMAs in rank order), so r = f32(c_prev - own) is the residual the three-pass schedule stores
template <int R>
__device__ __forceinline__ float own_of(const float *pa, const float *qv) {
  float v = __fmul_rn(pa[0], qv[0]);
#pragma unroll
  for (int b = 1; b < R; ++b) v = fmaf(pa[b], qv[b], v);
  return v;
}

// position k of a ring of n slots by counting: idx = k mod n, phase = (k / n) & 1
struct RingPos {
  int idx;
  uint32_t phase;
  __device__ __forceinline__ void step(int n) {
    if (++idx == n) {
      idx = 0;
      phase ^= 1u;
    }
  }
};

// tcgen05.ld 32 lanes x 16 columns (32-bit) of TMEM at taddr into x
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&x)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]), "=r"(x[8]),
        "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

}  // namespace gcu
