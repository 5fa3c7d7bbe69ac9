// PowerSGD P = M Q on the 5th-generation tensor cores (tcgen05, kind::tf32), fused with
// ef_apply.
//
// Reference: P_w = M_w @ Q (pipelines.py:348) with M_w = to_matrix(corrected_w)
// (compressors.py:530-548) and corrected_w = f32(g_w + r_w) (ef_apply, compressors.py:624-626).
//
// B200 design.  A CTA owns a 128-row band of M (UMMA M = 128) and a range of 32-column
// chunks.  Per chunk, 256 threads stream g and r (float4, coalesced rows), form the corrected
// values, write them back over r (the later passes read them there) and split each value
// three-way for 3xTF32: big = tf32(c), small = tf32(c - big); both go to shared memory in the
// canonical K-major SWIZZLE_128B layout (8 rows x 128 B atoms, 16-byte chunks XOR-swizzled by
// row), so the stores are conflict-free.  Q^T for the chunk (N = 16 rows, rank padded with
// zeros) is split the same way.  One elected thread issues, per 8-column k-step,
//     D += A_big B_big + A_big B_small + A_small B_big
// (tcgen05.mma.cta_group::1.kind::tf32, M = 128, N = 16) into a TMEM accumulator, and
// tcgen05.commit releases the stage (mbarrier) -- a 4-stage ring keeps the loads running while
// the tensor core works.  The dot products along K -- the cross-lane reductions a CUDA-core
// version pays in shuffles -- happen inside the MMA.  Every kGroup chunks (512 columns) the
// fp32 TMEM partial is read (tcgen05.ld 32x32b, warps 0-3: thread = row) and folded into fp64
// registers, alternating between two TMEM accumulators so the fold never stalls the MMA.  The
// fp64 split-K partials go through the existing ordered reduction (deterministic).
//
// Precision: 3xTF32 drops small * small and the bits below small (~2^-20 relative per product); fp32 accumulation
// spans at most 512 products before the fp64 fold.  Against the reference's fp32 BLAS the
// factors agree to ~1e-6 relative (the contract is 1e-5).
#include <cuda_runtime.h>

#include "gc_internal.h"

namespace {

#ifndef GC_MQ_M64
#define GC_MQ_M64 0
#endif
// M64: UMMA M = 64 rows per CTA with 64-column (two 128-byte swizzle atoms) stages -- the same
// shared memory per stage, 256-byte row segments per load and half the concurrent row streams
constexpr int kM = GC_MQ_M64 ? 64 : 128;   // UMMA M: rows per CTA
constexpr int kN = 16;           // UMMA N: rank padded to 16
constexpr int kKc = GC_MQ_M64 ? 64 : 32;   // columns per stage: 128-byte swizzle atoms of tf32
constexpr int kAtoms = kKc / 32;           // swizzle atoms along K per stage
constexpr int kF4Row = kKc / 4;            // float4 per row of a chunk
#ifndef GC_MQ_STAGES
#define GC_MQ_STAGES 2
#endif
constexpr int kStages = GC_MQ_STAGES;   // smem ring depth (36 KB per stage)
constexpr int kThreads = 256;
constexpr int kGroup = 512 / kKc;   // chunks per TMEM partial (512 columns) before the fp64 fold
constexpr int kATile = kM * kKc * 4;    // 16 KB
constexpr int kBTile = kN * kKc * 4;    // 2 KB
constexpr int kStageBytes = 2 * kATile + 2 * kBTile;
constexpr int kSmemBytes = kStages * kStageBytes + 1024 /*barriers*/ + 1024 /*alignment slack*/;

struct Rows {
  const int64_t *offs;
  int64_t ld;
  int n_per;
  __device__ __forceinline__ int64_t at(int v) const { return offs ? offs[v] : static_cast<int64_t>(v) * ld; }
  __device__ __forceinline__ int tensor(int v) const { return v / n_per; }
};

// byte offset of (row, 16-byte chunk) in a K-major SWIZZLE_128B tile (1024-byte aligned)
__device__ __forceinline__ uint32_t sw128(int row, int chunk) {
  return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4));
}
// (row, 16-byte chunk ch of the stage's kKc columns) in a tile of `rows` rows stored atom-major:
// swizzle atom ch / 8 occupies rows * 128 bytes
__device__ __forceinline__ uint32_t tile_off(int rows, int row, int ch) {
  return static_cast<uint32_t>((ch >> 3) * rows * 128) + sw128(row, ch & 7);
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, SBO = 1024 B between 8-row groups,
// descriptor version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}

// instruction descriptor: D f32, A/B tf32, both K-major, N = 16, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kN >> 3) << 17) | ((kM >> 4) << 24);

// 3xTF32 split by truncation: big keeps the top 10 mantissa bits (the tensor core reads a
// tf32 operand as the f32 pattern with the low 13 bits ignored), small = c - big is exact in
// f32 and is itself truncated to tf32.  c - (big + small) < 2^-20 |c|; two LOP3 + one FADD
// per value (cvt.rna.tf32.f32 is a 4-instruction sequence on sm_100).
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

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdesc), "r"(accumulate)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar)
               : "memory");
}

// A16: rows are 16-byte aligned and cols % 4 == 0 (float4 accesses); otherwise every thread's 4
// columns go as plain (L1-allocating) scalars masked to the row (nv = columns left in the row
// and before d): the 4 scalar instructions of a warp share sectors, so L1 absorbs the repeats.
template <int R, bool A16>
__global__ void __launch_bounds__(kThreads, 2) mq_umma_kernel(int64_t d, int64_t rows, int64_t cols, const float *g,
                                                              float *r, Rows rw_, const float *q, double *partial,
                                                              int splits, int64_t chunks_per_split) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char *sm = smem_raw + (base - raw);
  auto a_big = [&](int s) { return base + s * kStageBytes; };
  auto a_small = [&](int s) { return base + s * kStageBytes + kATile; };
  auto b_big = [&](int s) { return base + s * kStageBytes + 2 * kATile; };
  auto b_small = [&](int s) { return base + s * kStageBytes + 2 * kATile + kBTile; };
  const uint32_t bars = base + kStages * kStageBytes;   // empty[kStages], acc[2], full[kStages], tmem slot
  auto empty_bar = [&](int s) { return bars + 8 * s; };
  auto acc_bar = [&](int a) { return bars + 8 * (kStages + a); };
  auto full_bar = [&](int s) { return bars + 8 * (kStages + 2 + s); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + kStages * kStageBytes + 8 * (2 * kStages + 2));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int v = blockIdx.z;                      // (tensor, worker) row of the batch
  const int split = blockIdx.y;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kM;
  const int64_t nchunks_all = (cols + kKc - 1) / kKc;
  const int64_t c_begin = split * chunks_per_split;
  const int64_t c_end = min(nchunks_all, c_begin + chunks_per_split);
  const float *gw = g + rw_.at(v);
  float *rw = r ? r + rw_.at(v) : nullptr;
  q += static_cast<int64_t>(rw_.tensor(v)) * cols * R;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(empty_bar(s), 1);
    for (int s = 0; s < kStages; ++s) mbar_init(full_bar(s), kThreads);   // every producer arrives
    mbar_init(acc_bar(0), 1);
    mbar_init(acc_bar(1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {   // 32 TMEM columns: two 16-column fp32 accumulators
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // zero the B tiles once: rows >= R stay zero (padding of the rank to N = 16)
  for (int e = tid; e < kStages * 2 * kBTile / 16; e += kThreads) {
    const int s = e / (2 * kBTile / 16), o = e - s * (2 * kBTile / 16);
    *reinterpret_cast<uint4 *>(sm + (b_big(s) - base) + o * 16) = make_uint4(0, 0, 0, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  double acc64[R];
#pragma unroll
  for (int b = 0; b < R; ++b) acc64[b] = 0.0;

  // fold the fp32 TMEM partial of group gi into the fp64 accumulators (warps 0-3: thread = row)
  auto fold_group = [&](int64_t gi) {
    if (warp < 4) {
      mbar_wait(acc_bar(static_cast<int>(gi & 1)), static_cast<uint32_t>((gi >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      uint32_t x[16];
      const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>((gi & 1) * kN);
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]),
            "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      // M = 128: lane = row 32 warp + lane; M = 64: rows 16 warp + lane live in lanes 0-15
      if (kM == 128 || lane < 16) {
#pragma unroll
        for (int b = 0; b < R; ++b) acc64[b] += static_cast<double>(__uint_as_float(x[b]));
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
  };

  const int64_t nloc = c_end - c_begin;
  // chunk kk's g and r in registers: thread t covers float4 f = t + 256u (row f / 8, chunk f % 8);
  // the next chunk's loads are issued before this chunk's stores, so 8 float4 stay in flight
  float4 pg[4], pr[4];
  auto load_chunk = [&](int64_t kk) {
    const int64_t col0 = (c_begin + kk) * kKc;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int f = tid + kThreads * u;
      const int64_t grow = row0 + f / kF4Row, col = col0 + 4 * (f % kF4Row);
      const int64_t i = grow * cols + col;
      pg[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      pr[u] = pg[u];
      if (!A16 && grow < rows && col < cols) {
        const int nv = static_cast<int>(min(min(static_cast<int64_t>(4), cols - col), d - i));
        float t[4] = {0.f, 0.f, 0.f, 0.f}, t2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (e < nv) {
            t[e] = gw[i + e];
            if (rw) t2[e] = rw[i + e];
          }
        pg[u] = make_float4(t[0], t[1], t[2], t[3]);
        pr[u] = make_float4(t2[0], t2[1], t2[2], t2[3]);
      } else if (A16 && grow < rows && col < cols) {
        if (i + 3 < d) {
          pg[u] = __ldcs(reinterpret_cast<const float4 *>(gw + i));
          if (rw) pr[u] = __ldcs(reinterpret_cast<const float4 *>(rw + i));
        } else {
          float t[4] = {0.f, 0.f, 0.f, 0.f}, t2[4] = {0.f, 0.f, 0.f, 0.f};
          for (int e = 0; e < 4; ++e)
            if (i + e < d) {
              t[e] = gw[i + e];
              if (rw) t2[e] = rw[i + e];
            }
          pg[u] = make_float4(t[0], t[1], t[2], t[3]);
          pr[u] = make_float4(t2[0], t2[1], t2[2], t2[3]);
        }
      }
    }
  };
  if (nloc > 0) load_chunk(0);
  for (int64_t k = 0; k < nloc; ++k) {
    const int s = static_cast<int>(k % kStages);
    const int64_t col0 = (c_begin + k) * kKc;
    float4 cg[4], cr[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) cg[u] = pg[u], cr[u] = pr[u];
    if (k + 1 < nloc) load_chunk(k + 1);
    if (k >= kStages) mbar_wait(empty_bar(s), static_cast<uint32_t>(((k / kStages) - 1) & 1));
    // ---- A: corrected = f32(g + r) for 128 rows x 32 columns, written back over r, split
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int f = tid + kThreads * u;
      const int row = f / kF4Row, ch = f % kF4Row;
      const int64_t grow = row0 + row, col = col0 + 4 * ch;
      const int64_t i = grow * cols + col;
      float4 c = cg[u];
      if (rw) {
        c.x = c.x + cr[u].x; c.y = c.y + cr[u].y; c.z = c.z + cr[u].z; c.w = c.w + cr[u].w;
        if (!A16 && grow < rows && col < cols) {
          const int nv = static_cast<int>(min(min(static_cast<int64_t>(4), cols - col), d - i));
          const float cv[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
          for (int e = 0; e < 4; ++e)
            if (e < nv) rw[i + e] = cv[e];
        } else if (A16 && grow < rows && col < cols) {
          if (i + 3 < d) {
            __stcs(reinterpret_cast<float4 *>(rw + i), c);   // corrected kept in r for the later passes
          } else {
            const float cv[4] = {c.x, c.y, c.z, c.w};
            for (int e = 0; e < 4; ++e)
              if (i + e < d) rw[i + e] = cv[e];
          }
        }
      }
      float4 hb, hs;
      split3(c.x, hb.x, hs.x);
      split3(c.y, hb.y, hs.y);
      split3(c.z, hb.z, hs.z);
      split3(c.w, hb.w, hs.w);
      const uint32_t off = tile_off(kM, row, ch);
      *reinterpret_cast<float4 *>(sm + (a_big(s) - base) + off) = hb;
      *reinterpret_cast<float4 *>(sm + (a_small(s) - base) + off) = hs;
    }
    // ---- B = Q^T for the chunk (rows n < R; 8 threads per row, 4 columns each)
    if (tid < R * kF4Row) {
      const int n = tid / kF4Row, ch = tid % kF4Row;
      float t[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t col = col0 + 4 * ch + e;
        t[e] = col < cols ? q[col * R + n] : 0.0f;
      }
      float4 hb, hs;
      split3(t[0], hb.x, hs.x);
      split3(t[1], hb.y, hs.y);
      split3(t[2], hb.z, hs.z);
      split3(t[3], hb.w, hs.w);
      const uint32_t off = tile_off(kN, n, ch);
      *reinterpret_cast<float4 *>(sm + (b_big(s) - base) + off) = hb;
      *reinterpret_cast<float4 *>(sm + (b_small(s) - base) + off) = hs;
    }
    // the generic-proxy stores must be visible to the tensor core (async proxy).  Producers
    // publish the stage on a full barrier instead of a CTA-wide barrier: only the issuing
    // thread waits for all of them, the other warps run ahead to the next chunk
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full_bar(s)) : "memory");
    const int64_t gi = k / kGroup;
    if (tid == 0) {
      mbar_wait(full_bar(s), static_cast<uint32_t>((k / kStages) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t dcol = tmem + static_cast<uint32_t>((gi & 1) * kN);
#pragma unroll
      for (int kk = 0; kk < kKc / 8; ++kk) {
        const uint32_t ao = (kk >> 2) * kM * 128 + 32 * (kk & 3), bo = (kk >> 2) * kN * 128 + 32 * (kk & 3);
        const uint64_t ab = sdesc(a_big(s) + ao), as = sdesc(a_small(s) + ao);
        const uint64_t bb = sdesc(b_big(s) + bo), bs = sdesc(b_small(s) + bo);
        const uint32_t accum = (k % kGroup != 0 || kk != 0) ? 1u : 0u;
        umma_tf32(dcol, as, bb, accum);
        umma_tf32(dcol, ab, bs, 1u);
        umma_tf32(dcol, ab, bb, 1u);
      }
      umma_commit(empty_bar(s));
      if (k % kGroup == kGroup - 1 || k == nloc - 1) umma_commit(acc_bar(static_cast<int>(gi & 1)));
    }
    // fold the previous group's partial once this group's first chunk is issued
    if (k % kGroup == 0 && gi >= 1) fold_group(gi - 1);
  }
  if (nloc > 0) fold_group((nloc - 1) / kGroup);

  if (warp < 4 && (kM == 128 || lane < 16)) {
    const int64_t grow = row0 + warp * (kM / 4) + lane;
    if (grow < rows) {
#pragma unroll
      for (int b = 0; b < R; ++b)
        partial[((static_cast<int64_t>(v) * splits + split) * rows + grow) * R + b] = acc64[b];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

int grid_cap(int64_t g) { return static_cast<int>(g < 1 ? 1 : (g > 65535 ? 65535 : g)); }

}  // namespace

// Host side of the tcgen05 P = M Q pass; called by gc_psgd_mq_fused (gc_psgd.cu).  Writes fp64
// split-K partials partial[w][split][row][R]; returns the split count (<= ceil(cols / 1024), the
// workspace the caller sized) or a negative status.
int gc_psgd_mq_umma_launch(int32_t L, int32_t workers, const int64_t *row_offsets, int64_t ld, int64_t d,
                           int64_t rows, int64_t cols, int32_t rank, const float *grads, float *resid, const float *q,
                           double *partial, int a16, cudaStream_t st) {
  const int64_t row_blocks = (rows + kM - 1) / kM;
  const int64_t nchunks = (cols + kKc - 1) / kKc;
  const int64_t max_splits = (cols + 1023) / 1024;
  int64_t splits = (2 * 148 + row_blocks * L - 1) / (row_blocks * L);
  if (splits > max_splits) splits = max_splits;
  if (splits < 1) splits = 1;
  const int64_t per = (nchunks + splits - 1) / splits;
  splits = (nchunks + per - 1) / per;
  Rows rw{row_offsets, ld, workers};
  const dim3 grid(grid_cap(row_blocks), static_cast<unsigned>(splits), static_cast<unsigned>(L));
#define GC_UMMA_LAUNCH(RR, AA)                                                                             \
  cudaFuncSetAttribute(mq_umma_kernel<RR, AA>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);   \
  mq_umma_kernel<RR, AA><<<grid, kThreads, kSmemBytes, st>>>(d, rows, cols, grads, resid, rw, q, partial,   \
                                                             static_cast<int>(splits), per);
#define GC_UMMA_CASE(RR)        \
  case RR:                      \
    if (a16) {                  \
      GC_UMMA_LAUNCH(RR, true)  \
    } else {                    \
      GC_UMMA_LAUNCH(RR, false) \
    }                           \
    break;
  switch (rank) {
    GC_UMMA_CASE(1) GC_UMMA_CASE(2) GC_UMMA_CASE(3) GC_UMMA_CASE(4) GC_UMMA_CASE(5) GC_UMMA_CASE(6)
    GC_UMMA_CASE(7) GC_UMMA_CASE(8) GC_UMMA_CASE(16)
    default:
      gc_set_error("rank must be 1..8 or 16");
      return GC_ERR_UNSUPPORTED;
  }
#undef GC_UMMA_CASE
#undef GC_UMMA_LAUNCH
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gc_set_error(std::string("mq_umma_kernel: ") + cudaGetErrorString(e));
    return GC_ERR_CUDA;
  }
  return static_cast<int>(splits);
}
