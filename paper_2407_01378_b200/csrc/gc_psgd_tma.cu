// PowerSGD P = M Q on tcgen05 with TMA-fed operands and the error-feedback update folded in
// (single-matrix layout: worker w's matrix at w * ld, cols % 4 == 0, 16-byte aligned rows).
//
// Reference: P_w = M_w @ Q (pipelines.py:348), M_w = to_matrix(corrected_w) (compressors.py:530-548),
// corrected_w = f32(g_w + r_w) (ef_apply, compressors.py:624-626), and the previous round's
// r_w = f32(c_w - own_w), own_w = P_hat Q_w^T (pipelines.py:357-361, ef_update compressors.py:629-631).
//
// Deferred error feedback.  The previous round left its corrected matrix c_prev in the residual
// buffer together with its factors (P_hat_prev, Q_w_prev) instead of materialising
// r = c_prev - P_hat_prev Q_w_prev^T (that materialisation was a read-modify-write of M).  This
// pass forms, per element, own = P_hat_prev[i,:] . Q_w_prev[j,:] in the decode kernel's fp32 order
// (product, then FMAs), r = f32(c_prev - own), corrected = f32(g + r) -- the values the three-pass
// schedule produces, bit for bit -- so a round moves g and c_prev in, corrected out (12 B per
// element here), Mᵀ P_hat (4 B) and the estimate (4 B): 20 B per element instead of 28.
//
// B200 design.  One CTA (256 threads) per SM owns a 128-row band and a range of 32-column
// chunks.  The control thread (thread 0) keeps a 3-stage ring full with TMA: per chunk a
// 128 x 32 fp32 box of g and of the residual buffer (SWIZZLE_128B, i.e. already in the canonical
// K-major UMMA layout) plus the chunk's 32 x r rows of Q (and of Q_w_prev) by 1-D bulk copies, all
// on one mbarrier with expect-tx.  The producers (all 256 threads) turn the boxes into operands in
// place: corrected c into the residual box -- the TMA store source and, as is, A_big (kind::tf32
// reads the top 19 bits of an fp32 pattern: tf32(c) by truncation) -- and small = tf32(c - big)
// over the consumed g box; Q^T split into big / small 16 x 32 B tiles.  Two 16 KB boxes per stage
// let five stages (four chunks of loads in flight) share the SM.  The
// control thread then issues D += A_big B_big + A_big B_small + A_small B_big (kind::tf32,
// M = 128, N = 16) into TMEM, commits the stage's release, and TMA-stores the corrected box back
// over the residual buffer.  Every 512 columns the fp32 TMEM partial is folded into fp64
// registers (two accumulators alternate), as in gc_psgd_umma.cu.  A row that is only partly
// inside d (the zero-padded tail of to_matrix) is left to a one-row fix-up kernel; rows past it
// are zero padding.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>

#include "gc_internal.h"
#include "gc_umma.cuh"

namespace {

constexpr int kM = 128;        // UMMA M: rows per CTA
constexpr int kN = 16;         // UMMA N: rank padded to 16
constexpr int kKc = 32;        // columns per stage: one 128-byte swizzle atom of fp32
constexpr int kProducers = 512;            // 16 producer warps (2 float4 of a 128 x 32 box each)
constexpr int kThreads = kProducers + 32;  // + the control warp (TMA loads / MMA issue / TMA stores)
#ifndef GC_MQT_PAIR
#define GC_MQT_PAIR 0
#endif
constexpr int kPair = GC_MQT_PAIR ? 2 : 1;   // stages refilled together: 256-byte row bursts for DRAM
#ifndef GC_MQT_STAGES
#define GC_MQT_STAGES 5
#endif
constexpr int kStages = GC_MQT_STAGES;
constexpr int kGroup = 512 / kKc;          // chunks per TMEM partial before the fp64 fold
constexpr int kTile = kM * kKc * 4;        // 16 KB
constexpr int kBTile = kN * kKc * 4;       // 2 KB
constexpr int kRaw = kKc * 16 * 4;         // 2 KB: 32 rows of Q (or Q_w_prev), rank <= 16
// stage: G (g box -> small = tf32(c - tf32(c))) | C (residual box -> corrected c, which is also A_big:
// kind::tf32 reads an fp32 pattern's top 19 bits, i.e. tf32(c) by truncation) | Bb | Bs | Qraw | Wraw
constexpr int kOffG = 0, kOffC = kTile, kOffBb = 2 * kTile, kOffBs = 2 * kTile + kBTile,
              kOffQ = 2 * kTile + 2 * kBTile, kOffW = 2 * kTile + 2 * kBTile + kRaw;
constexpr int kStageBytes = 2 * kTile + 2 * kBTile + 2 * kRaw;
constexpr int kPhBytes = kM * 16 * 4;      // P_hat_prev rows of the band, rank <= 16
constexpr int kSmemBytes = kStages * kStageBytes + kPhBytes + 256 /*barriers*/ + 1024 /*alignment*/;

__device__ __forceinline__ uint32_t sw128(int row, int chunk) {
  return static_cast<uint32_t>((row >> 3) * 1024 + (row & 7) * 128 + ((chunk ^ (row & 7)) << 4));
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | ((kN >> 3) << 17) | ((kM >> 4) << 24);
#ifndef GC_MQT_PACK
#define GC_MQT_PACK 1
#endif
// P = M Q's B operand: with GC_MQT_PACK, [Q_big^T ; Q_small^T] packed along N (rows h < H the tf32
// heads, H + h the remainders; H = 8, or 16 for rank 16) so each k-step is two MMAs
//     D += A_small [B_big B_small] + A_big [B_big B_small]
// instead of three with N = 16 -- every MMA costs ~50 cycles up to N = 64 (profiles/r02_umma_rate.txt)
// and reads the 4 KB A slice from shared memory; columns h and H + h of D are summed in the fold
template <int R>
struct MqPack {
  static constexpr int H = GC_MQT_PACK ? (R <= 8 ? 8 : 16) : kN;
  static constexpr int N = GC_MQT_PACK ? 2 * H : kN;
  static constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((N >> 3) << 17) | ((kM >> 4) << 24);
};

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
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap *map, int c0, int c1, int c2,
                                            uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::
          "r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, uint32_t src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(src), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
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

// A batch of T same-shape tensors (the chunked PowerSGD of a model: one group per matrix shape):
// one 3-D tensor map [L workers][rows_full][cols] per tensor in each direction.
constexpr int kMaxMapT = 48;
struct MapSet {
  CUtensorMap g[kMaxMapT];
  CUtensorMap r[kMaxMapT];
};

struct TmaArgs {
  int64_t d, rows, cols, rows_full;
  int L;                   // workers per tensor: virtual row v = t * L + w
  int v_base;              // first virtual row of this launch (tensor chunks of <= kMaxMapT)
  const int64_t *row_start;   // device [T * L] element offset of each virtual row (tail-row kernel)
  const float *q;          // [cols][R] (one tensor)
  const float *ef_ph;      // deferred EF: P_hat_prev [rows][R] or NULL
  const float *ef_qw;      // deferred EF: Q_w_prev [L][cols][R]
  double *partial;         // [L][splits][rows][R]
  int splits;
  int64_t chunks_per_split;
  int has_resid;
  float *r_out;            // mq_pair_kernel: the residual buffer (odd rows' corrected values)
  int64_t ld;              // ... and its row pitch when row_start is null
};

// own = P_hat_prev[i,:] . Q_w_prev[j,:] exactly as decode_vec_kernel forms it (fp32 product then
// FMAs in rank order), so r = f32(c_prev - own) is the residual the three-pass schedule stores
template <int R>
__device__ __forceinline__ float own_of(const float *pa, const float *qv) {
  float v = __fmul_rn(pa[0], qv[0]);
#pragma unroll
  for (int b = 1; b < R; ++b) v = fmaf(pa[b], qv[b], v);
  return v;
}

template <int R, bool DEF>
__global__ void __launch_bounds__(kThreads, 1)
    mq_tma_kernel(const __grid_constant__ MapSet maps, const __grid_constant__ TmaArgs a) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char *sm = smem_raw + (base - raw);
  auto stage = [&](int s) { return base + static_cast<uint32_t>(s * kStageBytes); };
  float *ph_s = reinterpret_cast<float *>(sm + kStages * kStageBytes);
  const uint32_t bars = base + kStages * kStageBytes + kPhBytes;   // loaded[S], empty[S], full[S], acc[2]
  auto loaded_bar = [&](int s) { return bars + 8 * s; };
  auto empty_bar = [&](int s) { return bars + 8 * (kStages + s); };
  auto full_bar = [&](int s) { return bars + 8 * (2 * kStages + s); };
  auto acc_bar = [&](int x) { return bars + 8 * (3 * kStages + x); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + kStages * kStageBytes + kPhBytes + 8 * (3 * kStages + 2));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int vl = blockIdx.z;                 // virtual row within this launch
  const int v = a.v_base + vl;               // (tensor, worker) row of the batch
  const int tl = vl / a.L, w = vl - tl * a.L;   // tensor within the launch, worker
  const int t = v / a.L;                     // tensor within the batch
  const CUtensorMap *map_g = &maps.g[tl];
  const CUtensorMap *map_r = &maps.r[tl];
  const float *qt = a.q + static_cast<int64_t>(t) * a.cols * R;
  const float *pht = DEF ? a.ef_ph + static_cast<int64_t>(t) * a.rows * R : nullptr;
  const int split = blockIdx.y;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kM;
  const int64_t nchunks_all = (a.cols + kKc - 1) / kKc;
  const int64_t c_begin = split * a.chunks_per_split;
  const int64_t c_end = min(nchunks_all, c_begin + a.chunks_per_split);
  const int64_t nloc = c_end - c_begin;
  const float *qw_prev = DEF ? a.ef_qw + static_cast<int64_t>(v) * a.cols * R : nullptr;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(loaded_bar(s), 1);
      mbar_init(empty_bar(s), 1);
      mbar_init(full_bar(s), kProducers);
    }
    mbar_init(acc_bar(0), 1);
    mbar_init(acc_bar(1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  // B tiles: rows >= R stay zero (rank padded to N = 16)
  for (int e = tid; e < kStages * 2 * kBTile / 16; e += kThreads) {
    const int s = e / (2 * kBTile / 16), o = e - s * (2 * kBTile / 16);
    *reinterpret_cast<uint4 *>(sm + s * kStageBytes + kOffBb + o * 16) = make_uint4(0, 0, 0, 0);
  }
  if (DEF) {   // the band's P_hat_prev rows (rows past d's matrix are never used)
    for (int e = tid; e < kM * R; e += kThreads) {
      const int64_t i = row0 + e / R;
      ph_s[e] = i < a.rows ? pht[i * R + e % R] : 0.0f;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const uint32_t tx_bytes_box = static_cast<uint32_t>(kTile) * (a.has_resid ? 2u : 1u);
  // control warp: fill stage s with chunk k
  auto issue_load = [&](int64_t k) {
    const int s = static_cast<int>(k % kStages);
    const int64_t col0 = (c_begin + k) * kKc;
    const int64_t ncol = min(static_cast<int64_t>(kKc), a.cols - col0);
    const uint32_t qbytes = static_cast<uint32_t>(ncol * R * 4);
    mbar_expect_tx(loaded_bar(s), tx_bytes_box + qbytes * (DEF ? 2u : 1u));
    tma_load_3d(stage(s) + kOffG, map_g, static_cast<int>(col0), static_cast<int>(row0), w, loaded_bar(s));
    if (a.has_resid)
      tma_load_3d(stage(s) + kOffC, map_r, static_cast<int>(col0), static_cast<int>(row0), w, loaded_bar(s));
    bulk_load(stage(s) + kOffQ, qt + col0 * R, qbytes, loaded_bar(s));
    if (DEF) bulk_load(stage(s) + kOffW, qw_prev + col0 * R, qbytes, loaded_bar(s));
  };

  double acc64[R];
#pragma unroll
  for (int b = 0; b < R; ++b) acc64[b] = 0.0;
  auto fold_group = [&](int64_t gi) {
    if (warp < 4) {
      mbar_wait(acc_bar(static_cast<int>(gi & 1)), static_cast<uint32_t>((gi >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      constexpr int H = MqPack<R>::H, N = MqPack<R>::N;
      const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>((gi & 1) * N);
#pragma unroll
      for (int part = 0; part < N / 16; ++part) {
        uint32_t x[16];
        gcu::tmem_ld16(taddr + 16 * part, x);
#pragma unroll
        for (int j = 0; j < 16; ++j) {   // column 16 part + j is rank (16 part + j) mod H
          const int b = (16 * part + j) % H;
          if (b < R) acc64[b] += static_cast<double>(__uint_as_float(x[j]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
  };

  if (warp == kProducers / 32) {
    // ---- control warp (one elected lane): TMA ring, MMA issue, TMA stores.  It never produces, so
    // the producers' chunk time is not serialised behind the issue path.
    if (lane == 0) {
      for (int64_t k = 0; k < min(static_cast<int64_t>(kStages), nloc); ++k) issue_load(k);
      int64_t next = kStages;   // next chunk to load
      for (int64_t k = 0; k < nloc; ++k) {
        const int s = static_cast<int>(k % kStages);
        const int64_t col0 = (c_begin + k) * kKc;
        const int64_t gi = k / kGroup;
        mbar_wait(full_bar(s), static_cast<uint32_t>((k / kStages) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dcol = tmem + static_cast<uint32_t>((gi & 1) * MqPack<R>::N);
#pragma unroll
        for (int kk = 0; kk < kKc / 8; ++kk) {
          const uint64_t ab = sdesc(stage(s) + kOffC + 32 * kk), as = sdesc(stage(s) + kOffG + 32 * kk);
          const uint64_t bb = sdesc(stage(s) + kOffBb + 32 * kk), bs = sdesc(stage(s) + kOffBs + 32 * kk);
          const uint32_t accum = (k % kGroup != 0 || kk != 0) ? 1u : 0u;
          if (GC_MQT_PACK) {
            gcu::umma_tf32(dcol, as, bb, MqPack<R>::idesc, accum);
            gcu::umma_tf32(dcol, ab, bb, MqPack<R>::idesc, 1u);
          } else {
            umma_tf32(dcol, as, bb, accum);
            umma_tf32(dcol, ab, bs, 1u);
            umma_tf32(dcol, ab, bb, 1u);
          }
        }
        umma_commit(empty_bar(s));
        if (k % kGroup == kGroup - 1 || k == nloc - 1) umma_commit(acc_bar(static_cast<int>(gi & 1)));
        if (a.has_resid) {   // corrected box back over the residual buffer (clipped to the map)
          tma_store_3d(map_r, stage(s) + kOffC, static_cast<int>(col0), static_cast<int>(row0), w);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        // refill the stages of chunks next - S .. next - S + kPair - 1 (all older than k) once their
        // MMAs and stores are done, kPair at a time so each row's adjacent segments go out together
        if (next < nloc && next - kStages + kPair - 1 <= k - 1) {
          const int64_t batch = min(static_cast<int64_t>(kPair), nloc - next);
          for (int64_t pp = 0; pp < batch; ++pp) {
            const int64_t old = next + pp - kStages;
            mbar_wait(empty_bar(static_cast<int>(old % kStages)), static_cast<uint32_t>((old / kStages) & 1));
          }
          if (a.has_resid) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          for (int64_t pp = 0; pp < batch; ++pp) issue_load(next + pp);
          next += batch;
        }
      }
      if (a.has_resid) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else {
    // ---- producers: boxes -> operands (and the corrected values) in place
    const int ch = tid & 7;   // the thread's 16-byte chunk of a row (4 columns): the same in every pass
    for (int64_t k = 0; k < nloc; ++k) {
      const int s = static_cast<int>(k % kStages);
      const int64_t col0 = (c_begin + k) * kKc;
      unsigned char *st = sm + s * kStageBytes;
      const float *qraw = reinterpret_cast<const float *>(st + kOffQ);
      mbar_wait(loaded_bar(s), static_cast<uint32_t>((k / kStages) & 1));
      // this thread's 4 columns; columns past cols are zero in the boxes (TMA fill) and stay zero
      const int64_t cbase = col0 + 4 * ch;
      float wq[4][R];
      if (DEF) {
        const float *wraw = reinterpret_cast<const float *>(st + kOffW);
#pragma unroll
        for (int e = 0; e < 4; ++e)
#pragma unroll
          for (int b = 0; b < R; ++b) wq[e][b] = wraw[(4 * ch + e) * R + b];
      }
#pragma unroll
      for (int u = 0; u < kM * 8 / kProducers; ++u) {
        const int row = (tid >> 3) + (kProducers / 8) * u;
        const uint32_t off = sw128(row, ch);
        float4 gv = *reinterpret_cast<const float4 *>(st + kOffG + off);
        float4 c = gv;
        if (a.has_resid) {
          float4 rv = *reinterpret_cast<const float4 *>(st + kOffC + off);
          if (DEF) {
            float pa[R];
#pragma unroll
            for (int b = 0; b < R; ++b) pa[b] = ph_s[row * R + b];
            const bool live = row0 + row < a.rows_full;   // the partial row is the fix-up kernel's
            rv.x = live && cbase + 0 < a.cols ? rv.x - own_of<R>(pa, wq[0]) : 0.0f;
            rv.y = live && cbase + 1 < a.cols ? rv.y - own_of<R>(pa, wq[1]) : 0.0f;
            rv.z = live && cbase + 2 < a.cols ? rv.z - own_of<R>(pa, wq[2]) : 0.0f;
            rv.w = live && cbase + 3 < a.cols ? rv.w - own_of<R>(pa, wq[3]) : 0.0f;
          }
          c.x = gv.x + rv.x;
          c.y = gv.y + rv.y;
          c.z = gv.z + rv.z;
          c.w = gv.w + rv.w;
        }
        float4 hb, hs;
        split3(c.x, hb.x, hs.x);
        split3(c.y, hb.y, hs.y);
        split3(c.z, hb.z, hs.z);
        split3(c.w, hb.w, hs.w);
        *reinterpret_cast<float4 *>(st + kOffC + off) = c;    // A_big (truncated by the MMA) and the store source
        *reinterpret_cast<float4 *>(st + kOffG + off) = hs;   // A_small over the consumed g box
      }
      if (tid < R * 8) {   // B = Q^T of the chunk: row n (< R), 4 columns per thread
        const int n = tid >> 3;
        float t[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) t[e] = cbase + e < a.cols ? qraw[(4 * ch + e) * R + n] : 0.0f;
        float4 hb, hs;
        split3(t[0], hb.x, hs.x);
        split3(t[1], hb.y, hs.y);
        split3(t[2], hb.z, hs.z);
        split3(t[3], hb.w, hs.w);
        const uint32_t off = sw128(n, ch);
        *reinterpret_cast<float4 *>(st + kOffBb + off) = hb;
        // packed: the remainders are rows H.. of the same (contiguous, up to 32-row) B tile
        *reinterpret_cast<float4 *>(st + (GC_MQT_PACK ? kOffBb + sw128(MqPack<R>::H + n, ch) : kOffBs + off)) = hs;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full_bar(s)) : "memory");
      const int64_t gi = k / kGroup;
      if (k % kGroup == 0 && gi >= 1) fold_group(gi - 1);
    }
    if (nloc > 0) fold_group((nloc - 1) / kGroup);
  }

  if (warp < 4) {
    const int64_t grow = row0 + warp * 32 + lane;
    if (grow < a.rows) {
#pragma unroll
      for (int b = 0; b < R; ++b)
        a.partial[((static_cast<int64_t>(v) * a.splits + split) * a.rows + grow) * R + b] = acc64[b];
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

// The row of the matrix that is only partly inside d (to_matrix's zero padding starts in it):
// corrected values written, P row summed in fp64 (split 0; the other splits' partials zeroed).
constexpr int kTailThreads = 1024;

template <int R, bool DEF>
__global__ void __launch_bounds__(kTailThreads) mq_tail_row_kernel(const float *g, float *resid, int64_t ld,
                                                                  TmaArgs a) {
  __shared__ double red[kTailThreads / 32][R];
  const int v = a.v_base + blockIdx.x;
  const int t = v / a.L;
  const int64_t i = a.rows_full;
  const int64_t n_valid = a.d - i * a.cols;
  const int64_t rs = a.row_start ? a.row_start[v] : static_cast<int64_t>(v) * ld;
  const float *gw = g + rs + i * a.cols;
  float *rw = resid ? resid + rs + i * a.cols : nullptr;
  const float *qw_prev = DEF ? a.ef_qw + static_cast<int64_t>(v) * a.cols * R : nullptr;
  const float *qt = a.q + static_cast<int64_t>(t) * a.cols * R;
  float pa[R];
  if (DEF) {
#pragma unroll
    for (int b = 0; b < R; ++b) pa[b] = a.ef_ph[(static_cast<int64_t>(t) * a.rows + i) * R + b];
  }
  double acc[R];
#pragma unroll
  for (int b = 0; b < R; ++b) acc[b] = 0.0;
  for (int64_t j = threadIdx.x; j < n_valid; j += kTailThreads) {
    float c = gw[j];
    if (rw) {
      float r = rw[j];
      if (DEF) {
        float qv[R];
#pragma unroll
        for (int b = 0; b < R; ++b) qv[b] = qw_prev[j * R + b];
        r = r - own_of<R>(pa, qv);
      }
      c = c + r;
      rw[j] = c;
    }
#pragma unroll
    for (int b = 0; b < R; ++b) acc[b] += static_cast<double>(c) * static_cast<double>(qt[j * R + b]);
  }
#pragma unroll
  for (int b = 0; b < R; ++b) {
    double x = acc[b];
#pragma unroll
    for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5][b] = x;
  }
  __syncthreads();
  if (threadIdx.x < R) {
    double x = 0.0;
    for (int w = 0; w < kTailThreads / 32; ++w) x += red[w][threadIdx.x];
    for (int s = 0; s < a.splits; ++s)
      a.partial[((static_cast<int64_t>(v) * a.splits + s) * a.rows + i) * R + threadIdx.x] = s == 0 ? x : 0.0;
  }
}

// ------------------------------------------------------------------ Q_w = M_w^T P_hat (pipelines.py:354)
// Same TMA boxes (128 rows x 32 columns of M, SWIZZLE_128B) streamed by a producer warp, together
// with the box's 128 rows of P_hat (one bulk copy); a CTA owns a 32-column slab and a range of rows.
// Consumer thread (float4 column group g4, row group rg) forms, per row, the 4 columns x R
// products from one float4 of the box and one broadcast read of the P_hat row, in fp32 FMAs folded
// into fp64 after every box (4 rows per thread per box); the 32 row groups are reduced in order
// through shared memory and the split-K partials written as gc_psgd_mtp's, so the same ordered
// reduction finishes Q_w.  Ranks 1..4.
constexpr int kMtpStages = 4;
constexpr int kMtpConsumers = 256;
constexpr int kMtpThreads = kMtpConsumers + 32;
constexpr int kMtpPh = kM * 4 * 4;                  // 128 rows of P_hat, rank <= 4
constexpr int kMtpStage = kTile + kMtpPh;
constexpr int kMtpSmem = kMtpStages * kMtpStage + 64 + 1024;

struct MtpArgs {
  int64_t d, rows, cols, rows_full, ld;
  const float *c;          // corrected matrices (the partial row is read from here)
  const float *ph;         // P_hat [T][rows][R]
  double *partial;         // [V][splits][cols][R]
  int splits;
  int64_t rows_per_split;  // multiple of kM
  int stages, slots, stage_bytes, op_bytes;   // mtp_umma_kernel's rings
  int L, v_base;           // mtp_tma_kernel batches: virtual row v = v_base + blockIdx.z = t * L + w
  const int64_t *row_start;   // device [V] element offset of each virtual row, or null (v * ld)
};
// one tensor map [L workers][rows_full][cols] per tensor of a batch (<= kMaxMapT per launch)
struct MtpMaps {
  CUtensorMap m[kMaxMapT];
};

template <int R>
__global__ void __launch_bounds__(kMtpThreads, 1) mtp_tma_kernel(const __grid_constant__ MtpMaps maps,
                                                                const __grid_constant__ MtpArgs a) {
  static_assert(R <= 4, "rank <= 4");
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char *sm = smem_raw + (base - raw);
  const uint32_t bars = base + kMtpStages * kMtpStage;   // loaded[S], empty[S]
  __shared__ double red[kMtpConsumers / 8][32][R];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int vl = blockIdx.z, v = a.v_base + vl, split = blockIdx.y;
  const CUtensorMap *map_c = &maps.m[vl / a.L];
  const int w = vl % a.L;
  const float *ph = a.ph + static_cast<int64_t>(v / a.L) * a.rows * R;
  const int64_t col0 = static_cast<int64_t>(blockIdx.x) * kKc;
  const int64_t r_begin = split * a.rows_per_split;
  const int64_t r_end = min(a.rows_full, r_begin + a.rows_per_split);
  const int64_t nbox = r_end > r_begin ? (r_end - r_begin + kM - 1) / kM : 0;
  if (tid == 0) {
    for (int s = 0; s < kMtpStages; ++s) {
      mbar_init(bars + 8 * s, 1);
      mbar_init(bars + 8 * (kMtpStages + s), kMtpConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kMtpConsumers / 32) {   // producer warp: the TMA ring (box + its P_hat rows)
    if (lane == 0) {
      for (int64_t b = 0; b < nbox; ++b) {
        const int s = static_cast<int>(b % kMtpStages);
        const int64_t i0 = r_begin + b * kM;
        if (b >= kMtpStages)
          mbar_wait(bars + 8 * (kMtpStages + s), static_cast<uint32_t>(((b / kMtpStages) - 1) & 1));
        const bool full = i0 + kM <= r_end;   // partial boxes read P_hat with plain loads
        mbar_expect_tx(bars + 8 * s, kTile + (full ? kM * R * 4 : 0));
        tma_load_3d(base + s * kMtpStage, map_c, static_cast<int>(col0), static_cast<int>(i0), w, bars + 8 * s);
        if (full) bulk_load(base + s * kMtpStage + kTile, ph + i0 * R, kM * R * 4, bars + 8 * s);
      }
    }
    return;
  }
  const int g4 = tid & 7, rg = tid >> 3;   // float4 column group of the slab, row group (0..31)
  double acc64[4][R];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) acc64[t][b] = 0.0;
  for (int64_t bx = 0; bx < nbox; ++bx) {
    const int s = static_cast<int>(bx % kMtpStages);
    const int64_t i0 = r_begin + bx * kM;
    const bool full = i0 + kM <= r_end;
    mbar_wait(bars + 8 * s, static_cast<uint32_t>((bx / kMtpStages) & 1));
    const unsigned char *st = sm + s * kMtpStage;
    const float *phs = reinterpret_cast<const float *>(st + kTile);
    float acc[4][R];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int b = 0; b < R; ++b) acc[t][b] = 0.0f;
#pragma unroll
    for (int k = 0; k < kM / 32; ++k) {
      const int row = rg + 32 * k;
      const float4 m = *reinterpret_cast<const float4 *>(st + sw128(row, g4));
      float p[R];
      if (full) {
#pragma unroll
        for (int b = 0; b < R; ++b) p[b] = phs[row * R + b];
      } else {
#pragma unroll
        for (int b = 0; b < R; ++b) p[b] = i0 + row < r_end ? __ldg(ph + (i0 + row) * R + b) : 0.0f;
      }
      const float mv[4] = {m.x, m.y, m.z, m.w};
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int b = 0; b < R; ++b) acc[t][b] = fmaf(mv[t], p[b], acc[t][b]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int b = 0; b < R; ++b) acc64[t][b] += static_cast<double>(acc[t][b]);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bars + 8 * (kMtpStages + s)) : "memory");
  }
  // the row that is only partly inside d belongs to the last split (plain loads, fp64)
  if (rg == 0 && split == a.splits - 1 && a.rows_full < a.rows) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t col = col0 + 4 * g4 + t;
      const int64_t off = a.rows_full * a.cols + col;
      if (col < a.cols && off < a.d) {
        const int64_t rs = a.row_start ? a.row_start[v] : static_cast<int64_t>(v) * a.ld;
        const double m = static_cast<double>(a.c[rs + off]);
#pragma unroll
        for (int b = 0; b < R; ++b) acc64[t][b] += m * static_cast<double>(ph[a.rows_full * R + b]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) red[rg][4 * g4 + t][b] = acc64[t][b];
  asm volatile("bar.sync 1, %0;" ::"r"(kMtpConsumers) : "memory");   // consumers only
  for (int e = tid; e < 32 * R; e += kMtpConsumers) {
    const int cc = e / R, b = e - cc * R;
    double x = 0.0;
#pragma unroll 8
    for (int w = 0; w < kMtpConsumers / 8; ++w) x += red[w][cc][b];
    if (col0 + cc < a.cols)
      a.partial[((static_cast<int64_t>(v) * a.splits + split) * a.cols + col0 + cc) * R + b] = x;
  }
}

// ------------------------------------------------------------------ Q_w = M_w^T P_hat on tcgen05
// D[cols x r] = M^T P_hat with A = M^T MN-major, straight from the TMA boxes of M: a box is 32 rows
// (K) x 32 columns (MN, 128 bytes), loaded with the 128-byte swizzle of 32-byte atoms that MN-major
// tf32 operands require (descriptor layout type 1, 4 K-rows per 512-byte atom), and four boxes side
// by side are A for UMMA M = 128 columns (LBO = 4 KB between boxes, SBO = 512 B between K-row
// quads).  kind::tf32 reads the raw fp32 box as A_big (truncation); the producers write
// A_small = tf32(c - tf32(c)) at the same offsets and the K-major B tiles (P_hat^T of the chunk's
// 32 rows, split in two; the rows arrive by bulk copy with the box).  D += A_small B_big +
// A_big B_small + A_big B_big into TMEM, folded to fp64 every 512 rows.  A CTA owns 128 columns
// and a range of rows; its two producer halves take alternate chunks.
constexpr int kQtM = 128;                 // columns per CTA (UMMA M)
constexpr int kQtK = 32;                  // rows per chunk (4 k-steps of 8)
constexpr int kQtBox = kQtK * 128;        // one 32-row x 32-column box: 4 KB
constexpr int kQtA = 4 * kQtBox;          // 16 KB: the four column boxes
// load ring (held from the TMA issue to the chunk's MMAs): the raw boxes (= A_big) and the P_hat
// rows; operand slots (held from production to the chunk's MMAs): A_small and B.  One CTA per SM;
// the ring depths are launch arguments sized to fill shared memory (gc_psgd_mtp_umma_launch).
constexpr int kQtOffP = kQtA;                      // [32][R] fp32 P_hat rows
constexpr int kQtOffSmall = 0, kQtOffB = kQtA;
constexpr int kQtProducers = 256, kQtHalf = kQtProducers / 2;
constexpr int kQtThreads = kQtProducers + 64;   // + the TMA warp + the MMA warp
constexpr int kQtGroup = 512 / kQtK;      // chunks per TMEM partial
constexpr int kQtFoldLag = 4;             // group g-1 is folded at chunk 16 g + 4 (long retired)
constexpr int kQtBarBytes = 512;
// B = [P_hat_big^T ; P_hat_small^T]: rows 0..H-1 the tf32 heads, rows H..2H-1 the remainders
// (H = 8, or 16 for rank 16), so one MMA gives A x both halves: two MMAs per k-step for 3xTF32.
template <int R> struct QtShape {
  static constexpr int H = R <= 8 ? 8 : 16;
  static constexpr int N = 2 * H;
  static constexpr uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) /*A MN-major*/ |
                                    ((N >> 3) << 17) | ((kQtM >> 4) << 24);
};
static_assert(kQtFoldLag % 2 == 0 && kQtGroup % 2 == 0, "folds run on the even-chunk half (warps 0..3)");

__device__ __forceinline__ uint64_t sdesc_mn(uint32_t saddr) {
  return static_cast<uint64_t>((saddr & 0x3FFFF) >> 4) | (static_cast<uint64_t>(kQtBox >> 4) << 16) |
         (static_cast<uint64_t>(512 >> 4) << 32) | (1ull << 46) | (1ull << 61);
}

__device__ __forceinline__ void umma_tf32_desc(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate)
      : "memory");
}

struct RingPos {   // position k of a ring of n slots: idx = k mod n, phase = (k / n) & 1
  int idx;
  uint32_t phase;
  __device__ __forceinline__ void step(int n) {
    if (++idx == n) {
      idx = 0;
      phase ^= 1u;
    }
  }
};

template <int R>
__global__ void __launch_bounds__(kQtThreads, 1) mtp_umma_kernel(const __grid_constant__ CUtensorMap map_c,
                                                                 const __grid_constant__ MtpArgs a) {
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char *sm = smem_raw + (base - raw);
  const int kQtStages = a.stages, kQtSlots = a.slots, kQtStage = a.stage_bytes, kQtOp = a.op_bytes;
  auto stage = [&](int s) { return base + static_cast<uint32_t>(s * kQtStage); };
  auto op = [&](int h) { return base + static_cast<uint32_t>(kQtStages * kQtStage + h * kQtOp); };
  constexpr int H = QtShape<R>::H, N = QtShape<R>::N;
  const uint32_t bars = op(kQtSlots);   // loaded[S], empty[S], full[S], acc[2], op_free[slots]
  auto loaded_bar = [&](int s) { return bars + 8 * s; };
  auto empty_bar = [&](int s) { return bars + 8 * (kQtStages + s); };
  auto full_bar = [&](int s) { return bars + 8 * (2 * kQtStages + s); };
  auto acc_bar = [&](int x) { return bars + 8 * (3 * kQtStages + x); };
  auto op_bar = [&](int h) { return bars + 8 * (3 * kQtStages + 2 + h); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + (bars - base) + 8 * (3 * kQtStages + 2 + kQtSlots));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int v = blockIdx.z, split = blockIdx.y;
  const int64_t col0 = static_cast<int64_t>(blockIdx.x) * kQtM;
  const int64_t r_begin = split * a.rows_per_split;
  const int64_t r_end = min(a.rows_full, r_begin + a.rows_per_split);
  const int64_t nk = r_end > r_begin ? (r_end - r_begin + kQtK - 1) / kQtK : 0;
  if (tid == 0) {
    for (int s = 0; s < kQtStages; ++s) {
      mbar_init(loaded_bar(s), 1);
      mbar_init(empty_bar(s), 1);
      mbar_init(full_bar(s), kQtHalf);
    }
    for (int x = 0; x < 2; ++x) mbar_init(acc_bar(x), 1);
    for (int x = 0; x < kQtSlots; ++x) mbar_init(op_bar(x), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int e = tid; e < kQtSlots * N * 8; e += kQtThreads) {   // padding rows of B stay zero
    const int h = e / (N * 8), o = e - h * (N * 8);
    *reinterpret_cast<uint4 *>(sm + (op(h) - base) + kQtOffB + o * 16) = make_uint4(0, 0, 0, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  auto chunk_full = [&](int64_t k) { return r_begin + (k + 1) * kQtK <= r_end; };
  auto issue_load = [&](int64_t k, int s) {
    const int64_t row = r_begin + k * kQtK;
    const bool full = chunk_full(k);   // a partial chunk reads its P_hat rows with plain loads
    mbar_expect_tx(loaded_bar(s), kQtA + (full ? kQtK * R * 4 : 0));
#pragma unroll
    for (int j = 0; j < 4; ++j)
      tma_load_3d(stage(s) + j * kQtBox, &map_c, static_cast<int>(col0 + 32 * j), static_cast<int>(row),
                  v, loaded_bar(s));
    if (full) bulk_load(stage(s) + kQtOffP, a.ph + row * R, kQtK * R * 4, loaded_bar(s));
  };
  double acc64[R];
#pragma unroll
  for (int b = 0; b < R; ++b) acc64[b] = 0.0;
  auto fold_group = [&](int64_t gi) {   // warps 0..3: TMEM lanes = the CTA's 128 columns
    mbar_wait(acc_bar(static_cast<int>(gi & 1)), static_cast<uint32_t>((gi >> 1) & 1));
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>((gi & 1) * N);
#pragma unroll
    for (int part = 0; part < N / 16; ++part) {   // columns 16 part .. 16 part + 15
      uint32_t x[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(x[0]), "=r"(x[1]), "=r"(x[2]), "=r"(x[3]), "=r"(x[4]), "=r"(x[5]), "=r"(x[6]), "=r"(x[7]),
            "=r"(x[8]), "=r"(x[9]), "=r"(x[10]), "=r"(x[11]), "=r"(x[12]), "=r"(x[13]), "=r"(x[14]), "=r"(x[15])
          : "r"(taddr + 16 * part));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int j = 0; j < 16; ++j) {   // column c = 16 part + j is rank c mod H (head or remainder)
        const int b = (16 * part + j) % H;
        if (b < R) acc64[b] += static_cast<double>(__uint_as_float(x[j]));
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  };

  if (warp == kQtProducers / 32) {   // TMA warp: the load ring
    if (lane == 0) {
      RingPos rs{0, 0};   // ring positions by counting: no runtime divisions in the loops
      for (int64_t k = 0; k < nk; ++k, rs.step(kQtStages)) {
        if (k >= kQtStages) mbar_wait(empty_bar(rs.idx), rs.phase ^ 1u);
        issue_load(k, rs.idx);
      }
    }
  } else if (warp == kQtProducers / 32 + 1) {   // MMA warp: one elected lane issues
    if (lane == 0) {
      RingPos rs{0, 0}, ro{0, 0};
      for (int64_t k = 0; k < nk; ++k, rs.step(kQtStages), ro.step(kQtSlots)) {
        const int s = rs.idx;
        const int64_t gi = k / kQtGroup;
        mbar_wait(full_bar(s), rs.phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dcol = tmem + static_cast<uint32_t>((gi & 1) * N);
        const uint32_t o = op(ro.idx);
#pragma unroll
        for (int ks = 0; ks < kQtK / 8; ++ks) {
          const uint64_t ab = sdesc_mn(stage(s) + 1024 * ks), as = sdesc_mn(o + kQtOffSmall + 1024 * ks);
          const uint64_t bd = sdesc(o + kQtOffB + 32 * ks);
          const uint32_t accum = (k % kQtGroup != 0 || ks != 0) ? 1u : 0u;
          umma_tf32_desc(dcol, as, bd, QtShape<R>::idesc, accum);   // A_small [B_big B_small]
          umma_tf32_desc(dcol, ab, bd, QtShape<R>::idesc, 1u);      // A_big   [B_big B_small]
        }
        umma_commit(empty_bar(s));
        umma_commit(op_bar(ro.idx));
        if (k % kQtGroup == kQtGroup - 1 || k == nk - 1) umma_commit(acc_bar(static_cast<int>(gi & 1)));
      }
    }
  } else {
    const int half = tid / kQtHalf, ht = tid - half * kQtHalf;
    int64_t folded = 0;   // groups folded so far (warps 0..3)
    RingPos rs{0, 0}, ro{0, 0};
    if (half) {
      rs.step(kQtStages);
      ro.step(kQtSlots);
    }
    for (int64_t k = half; k < nk; k += 2, rs.step(kQtStages), rs.step(kQtStages), ro.step(kQtSlots), ro.step(kQtSlots)) {
      const int s = rs.idx;
      const int64_t k0 = r_begin + k * kQtK;
      unsigned char *st = sm + s * kQtStage;
      const int slot = ro.idx;
      unsigned char *ot = sm + (op(slot) - base);
      mbar_wait(loaded_bar(s), rs.phase);
      if (k >= kQtSlots)   // the slot's previous chunk (k - slots) has been consumed by its MMAs
        mbar_wait(op_bar(slot), ro.phase ^ 1u);
#pragma unroll
      for (int u = 0; u < kQtA / 16 / kQtHalf; ++u) {   // A_small at the raw box's offsets
        const int f = ht + kQtHalf * u;
        const float4 c = *reinterpret_cast<const float4 *>(st + 16 * f);
        float4 hb, hs;
        split3(c.x, hb.x, hs.x);
        split3(c.y, hb.y, hs.y);
        split3(c.z, hb.z, hs.z);
        split3(c.w, hb.w, hs.w);
        *reinterpret_cast<float4 *>(ot + kQtOffSmall + 16 * f) = hs;
      }
      if (ht < R * 8) {   // B = P_hat^T of the chunk's rows: row n (< R), 4 k per thread
        const int n = ht >> 3, ch = ht & 7;
        const float *prow = reinterpret_cast<const float *>(st + kQtOffP);
        const bool full = chunk_full(k);
        float t[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int kk = 4 * ch + e;
          t[e] = full ? prow[kk * R + n] : (k0 + kk < r_end ? __ldg(a.ph + (k0 + kk) * R + n) : 0.0f);
        }
        float4 hb, hs;
        split3(t[0], hb.x, hs.x);
        split3(t[1], hb.y, hs.y);
        split3(t[2], hb.z, hs.z);
        split3(t[3], hb.w, hs.w);
        *reinterpret_cast<float4 *>(ot + kQtOffB + sw128(n, ch)) = hb;
        *reinterpret_cast<float4 *>(ot + kQtOffB + sw128(H + n, ch)) = hs;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full_bar(s)) : "memory");
      if (warp < 4 && k % kQtGroup == kQtFoldLag && k >= kQtGroup) {
        fold_group(k / kQtGroup - 1);
        folded = k / kQtGroup;
      }
    }
    if (warp < 4) {
      for (int64_t g = folded; nk > 0 && g <= (nk - 1) / kQtGroup; ++g) fold_group(g);
      const int64_t col = col0 + warp * 32 + lane;
      if (split == a.splits - 1 && a.rows_full < a.rows && col < a.cols) {   // the partly filled row, fp64
        const int64_t off = a.rows_full * a.cols + col;
        if (off < a.d) {
          const double m = static_cast<double>(a.c[v * a.ld + off]);
#pragma unroll
          for (int b = 0; b < R; ++b) acc64[b] += m * static_cast<double>(a.ph[a.rows_full * R + b]);
        }
      }
      if (col < a.cols) {
#pragma unroll
        for (int b = 0; b < R; ++b)
          a.partial[((static_cast<int64_t>(v) * a.splits + split) * a.cols + col) * R + b] = acc64[b];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

// ------------------------------------------------------------------ P = M Q for cols = 2 (mod 4)
// GPT-2-medium's chunked PowerSGD matrices (1774 x 1774, 7174 x 7174) have a row pitch of
// 8 (mod 16) bytes, which no tensor map describes.  Row PAIRS do: a pair of rows is 2 cols floats
// = a multiple of 16 bytes.  Two maps per operand over the pair rows -- even rows at the tensor
// start, odd rows at start + (cols - 2) floats (16-byte aligned when the tensor start is) -- so an
// odd-row box at column c0 holds that row's columns c0 - 2 .. c0 + 29.  A CTA's 128-row band is
// tile rows 0..63 = its 64 even rows and 64..127 = its 64 odd rows; the odd half simply computes
// with a B shifted by two columns (Q rows c0 - 2 ..), as a second M = 64 MMA chain into its own
// TMEM accumulator.  Everything else is mq_tma_kernel's: TMA boxes (SWIZZLE_128B) formed in place,
// deferred EF, packed 3xTF32, fp64 folds; the even half's corrected box goes back by TMA store, the
// odd half's (and the last chunk's even half) by 16-byte stores (an odd box's first two columns of
// the first chunk are the even row's tail: neither used nor stored).  Ranks 4, 8, 16 (16-byte Q-row
// windows).
constexpr int kPrM = 64;                     // rows per half (UMMA M)
constexpr int kPrRaw = 36 * 16 * 4;          // Q (or Q_w_prev) rows c0 - 4 .. c0 + 31, rank <= 16
constexpr int kPrOffG = 0, kPrOffC = kTile, kPrOffBe = 2 * kTile, kPrOffBo = 2 * kTile + 4096,
              kPrOffQ = 2 * kTile + 8192, kPrOffW = kPrOffQ + kPrRaw;
constexpr int kPrStage = (kPrOffW + kPrRaw + 1023) / 1024 * 1024;
constexpr int kPrStages = 4;
constexpr int kPrSmem = kPrStages * kPrStage + kPhBytes + 512 + 1024;
struct PairMapSet {   // per tensor: g even / odd, residual even / odd
  CUtensorMap ge[kMaxMapT / 2], go[kMaxMapT / 2], re[kMaxMapT / 2], ro[kMaxMapT / 2];
};
template <int R>
struct PairShape {
  static constexpr int H = R <= 8 ? 8 : 16;
  static constexpr int N = 2 * H;
  static constexpr uint32_t idesc = gcu::idesc_tf32(kPrM, N);
};

template <int R, bool DEF>
__global__ void __launch_bounds__(kThreads, 1)
    mq_pair_kernel(const __grid_constant__ PairMapSet maps, const __grid_constant__ TmaArgs a) {
  static_assert(R % 4 == 0, "16-byte Q-row windows");
  constexpr int H = PairShape<R>::H, N = PairShape<R>::N;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char *sm = smem_raw + (base - raw);
  auto stage = [&](int s) { return base + static_cast<uint32_t>(s * kPrStage); };
  float *ph_s = reinterpret_cast<float *>(sm + kPrStages * kPrStage);
  const uint32_t bars = base + kPrStages * kPrStage + kPhBytes;   // loaded[S], empty[S], full[S], acc[2]
  auto loaded_bar = [&](int s) { return bars + 8 * s; };
  auto empty_bar = [&](int s) { return bars + 8 * (kPrStages + s); };
  auto full_bar = [&](int s) { return bars + 8 * (2 * kPrStages + s); };
  auto acc_bar = [&](int x) { return bars + 8 * (3 * kPrStages + x); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + kPrStages * kPrStage + kPhBytes + 8 * (3 * kPrStages + 2));

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int vl = blockIdx.z, v = a.v_base + vl;
  const int tl = vl / a.L, w = vl - tl * a.L, t = v / a.L;
  const float *qt = a.q + static_cast<int64_t>(t) * a.cols * R;
  const float *pht = DEF ? a.ef_ph + static_cast<int64_t>(t) * a.rows * R : nullptr;
  const float *qw_prev = DEF ? a.ef_qw + static_cast<int64_t>(v) * a.cols * R : nullptr;
  const int split = blockIdx.y;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * kM;   // even
  const int k0 = static_cast<int>(row0 / 2);                     // pair row
  const int64_t nchunks_all = (a.cols + kKc - 1) / kKc;
  const int64_t c_begin = split * a.chunks_per_split;
  const int64_t c_end = min(nchunks_all, c_begin + a.chunks_per_split);
  const int64_t nloc = c_end - c_begin;
  // matrix row of tile row tr: even half 2 tr, odd half 2 (tr - 64) + 1
  auto mrow = [&](int tr) { return row0 + (tr < kPrM ? 2 * tr : 2 * (tr - kPrM) + 1); };

  if (tid == 0) {
    for (int s = 0; s < kPrStages; ++s) {
      mbar_init(loaded_bar(s), 1);
      mbar_init(empty_bar(s), 1);
      mbar_init(full_bar(s), kProducers);
    }
    mbar_init(acc_bar(0), 1);
    mbar_init(acc_bar(1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {   // two groups x (even, odd) accumulators of N <= 32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int e = tid; e < kPrStages * 8192 / 16; e += kThreads) {   // both B tiles: padding rows stay zero
    const int s = e / (8192 / 16), o = e - s * (8192 / 16);
    *reinterpret_cast<uint4 *>(sm + s * kPrStage + kPrOffBe + o * 16) = make_uint4(0, 0, 0, 0);
  }
  if (DEF) {   // P_hat_prev rows in tile order
    for (int e = tid; e < kM * R; e += kThreads) {
      const int64_t i = mrow(e / R);
      ph_s[e] = i < a.rows ? pht[i * R + e % R] : 0.0f;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const uint32_t tx_box = static_cast<uint32_t>(kTile) * (a.has_resid ? 2u : 1u);
  auto issue_load = [&](int64_t k) {
    const int s = static_cast<int>(k % kPrStages);
    const int64_t col0 = (c_begin + k) * kKc;
    // Q rows col0 - 4 .. col0 + 31 (the window starts at col0 for the first chunk, 4 rows in)
    const int64_t q0 = col0 >= 4 ? col0 - 4 : 0;
    const int64_t qn = min(col0 + kKc, a.cols) - q0;
    const uint32_t qbytes = static_cast<uint32_t>(qn * R * 4), qdst = col0 >= 4 ? 0u : 4u * R * 4;
    mbar_expect_tx(loaded_bar(s), tx_box + qbytes * (DEF ? 2u : 1u));
    const int c0i = static_cast<int>(col0);
    tma_load_3d(stage(s) + kPrOffG, &maps.ge[tl], c0i, k0, w, loaded_bar(s));
    tma_load_3d(stage(s) + kPrOffG + kTile / 2, &maps.go[tl], c0i, k0, w, loaded_bar(s));
    if (a.has_resid) {
      tma_load_3d(stage(s) + kPrOffC, &maps.re[tl], c0i, k0, w, loaded_bar(s));
      tma_load_3d(stage(s) + kPrOffC + kTile / 2, &maps.ro[tl], c0i, k0, w, loaded_bar(s));
    }
    bulk_load(stage(s) + kPrOffQ + qdst, qt + q0 * R, qbytes, loaded_bar(s));
    if (DEF) bulk_load(stage(s) + kPrOffW + qdst, qw_prev + q0 * R, qbytes, loaded_bar(s));
  };

  double acc_e[R], acc_o[R];
#pragma unroll
  for (int b = 0; b < R; ++b) acc_e[b] = acc_o[b] = 0.0;
  auto fold_group = [&](int64_t gi) {   // M = 64: row r of a half at lane 32 (r / 16) + r % 16
    if (warp < 4) {
      mbar_wait(acc_bar(static_cast<int>(gi & 1)), static_cast<uint32_t>((gi >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>((gi & 1) * 2 * N);
#pragma unroll
      for (int half = 0; half < 2; ++half) {
#pragma unroll
        for (int part = 0; part < N / 16; ++part) {
          uint32_t x[16];
          gcu::tmem_ld16(taddr + half * N + 16 * part, x);
          if (lane < 16) {
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int b = (16 * part + j) % H;
              if (b < R) (half ? acc_o : acc_e)[b] += static_cast<double>(__uint_as_float(x[j]));
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    }
  };

  if (warp == kProducers / 32) {   // ---- control warp: TMA ring, MMA issue, TMA stores (even half)
    if (lane == 0) {
      for (int64_t k = 0; k < min(static_cast<int64_t>(kPrStages), nloc); ++k) issue_load(k);
      for (int64_t k = 0; k < nloc; ++k) {
        const int s = static_cast<int>(k % kPrStages);
        const int64_t col0 = (c_begin + k) * kKc;
        const int64_t gi = k / kGroup;
        mbar_wait(full_bar(s), static_cast<uint32_t>((k / kPrStages) & 1));
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t de = tmem + static_cast<uint32_t>((gi & 1) * 2 * N), dodd = de + N;
#pragma unroll
        for (int kk = 0; kk < kKc / 8; ++kk) {
          const uint32_t accum = (k % kGroup != 0 || kk != 0) ? 1u : 0u;
          const uint64_t abe = gcu::sdesc(stage(s) + kPrOffC + 32 * kk), ase = gcu::sdesc(stage(s) + kPrOffG + 32 * kk);
          const uint64_t abo = gcu::sdesc(stage(s) + kPrOffC + kTile / 2 + 32 * kk),
                         aso = gcu::sdesc(stage(s) + kPrOffG + kTile / 2 + 32 * kk);
          const uint64_t be = gcu::sdesc(stage(s) + kPrOffBe + 32 * kk), bo = gcu::sdesc(stage(s) + kPrOffBo + 32 * kk);
          gcu::umma_tf32(de, ase, be, PairShape<R>::idesc, accum);
          gcu::umma_tf32(de, abe, be, PairShape<R>::idesc, 1u);
          gcu::umma_tf32(dodd, aso, bo, PairShape<R>::idesc, accum);
          gcu::umma_tf32(dodd, abo, bo, PairShape<R>::idesc, 1u);
        }
        umma_commit(empty_bar(s));
        if (k % kGroup == kGroup - 1 || k == nloc - 1) umma_commit(acc_bar(static_cast<int>(gi & 1)));
        // the even half's corrected box back over the residual buffer -- except in the last chunk:
        // TMA clips the inner dimension at 16-byte granularity and cols * 4 = 8 (mod 16) bytes, so
        // a clipped store would also write the odd row's first two elements (the producers store it)
        if (a.has_resid && col0 + kKc <= a.cols) {
          tma_store_3d(&maps.re[tl], stage(s) + kPrOffC, static_cast<int>(col0), k0, w);
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        if (k >= 1 && k - 1 + kPrStages < nloc) {   // refill the stage of chunk k - 1
          const int64_t old = k - 1;
          mbar_wait(empty_bar(static_cast<int>(old % kPrStages)), static_cast<uint32_t>((old / kPrStages) & 1));
          if (a.has_resid) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
          issue_load(old + kPrStages);
        }
      }
      if (a.has_resid) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else {   // ---- producers: thread = 16-byte column chunk ch of row rg (even half) and 64 + rg (odd)
    const int ch = tid & 7, rg = tid >> 3;
    const int64_t rs = a.row_start ? a.row_start[v] : static_cast<int64_t>(v) * a.ld;
    for (int64_t k = 0; k < nloc; ++k) {
      const int s = static_cast<int>(k % kPrStages);
      const int64_t col0 = (c_begin + k) * kKc;
      unsigned char *st = sm + s * kPrStage;
      const float *qraw = reinterpret_cast<const float *>(st + kPrOffQ);   // window row = col - col0 + 4
      const float *wraw = reinterpret_cast<const float *>(st + kPrOffW);
      mbar_wait(loaded_bar(s), static_cast<uint32_t>((k / kPrStages) & 1));
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int tr = rg + kPrM * half;
        const int64_t m = mrow(tr);
        const int64_t cb = col0 + 4 * ch - 2 * half;   // the thread's first column
        const uint32_t off = sw128(tr, ch);
        float4 gv = *reinterpret_cast<const float4 *>(st + kPrOffG + off);
        float4 rv = a.has_resid ? *reinterpret_cast<const float4 *>(st + kPrOffC + off) : make_float4(0.f, 0.f, 0.f, 0.f);
        float g4[4] = {gv.x, gv.y, gv.z, gv.w}, r4[4] = {rv.x, rv.y, rv.z, rv.w}, c4[4];
        const bool live = m < a.rows_full;   // the partial row is the fix-up kernel's
        float pa[R];
        if (DEF) {   // the row's P_hat_prev and the 4 columns' Q_w_prev rows as 16-byte loads
#pragma unroll
          for (int j = 0; j < R / 4; ++j) {
            const float4 x = *reinterpret_cast<const float4 *>(ph_s + tr * R + 4 * j);
            pa[4 * j] = x.x, pa[4 * j + 1] = x.y, pa[4 * j + 2] = x.z, pa[4 * j + 3] = x.w;
          }
        }
        const float *wcol = wraw + (cb - col0 + 4) * R;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t col = cb + e;
          const bool ok = live && col >= 0 && col < a.cols;
          float r = r4[e];
          if (DEF && ok) {
            float wq[R];
#pragma unroll
            for (int j = 0; j < R / 4; ++j) {
              const float4 x = *reinterpret_cast<const float4 *>(wcol + e * R + 4 * j);
              wq[4 * j] = x.x, wq[4 * j + 1] = x.y, wq[4 * j + 2] = x.z, wq[4 * j + 3] = x.w;
            }
            r = r - own_of<R>(pa, wq);
          }
          c4[e] = ok ? (a.has_resid ? g4[e] + r : g4[e]) : 0.0f;
        }
        const float4 c = make_float4(c4[0], c4[1], c4[2], c4[3]);
        float4 hb, hs;
        split3(c.x, hb.x, hs.x);
        split3(c.y, hb.y, hs.y);
        split3(c.z, hb.z, hs.z);
        split3(c.w, hb.w, hs.w);
        *reinterpret_cast<float4 *>(st + kPrOffC + off) = c;
        *reinterpret_cast<float4 *>(st + kPrOffG + off) = hs;
        if (a.has_resid && live && (half == 1 || col0 + kKc > a.cols)) {   // 16-byte stores of the corrected values
          float *dst = a.r_out + rs + m * a.cols + cb;
          if (cb >= 0 && cb + 3 < a.cols) {
            *reinterpret_cast<float4 *>(dst) = c;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (cb + e >= 0 && cb + e < a.cols) dst[e] = c4[e];
          }
        }
      }
      // B tiles: threads 0 .. 8R - 1 the even half's (Q rows col0 ..), 256 .. 256 + 8R - 1 the odd
      // half's (Q rows col0 - 2 ..); row n (< R) and H + n, 4 k per thread
      if ((tid & 255) < R * 8) {
        const int half = tid >> 8, n = (tid & 255) >> 3, c8 = tid & 7;
        float tv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t col = col0 + 4 * c8 + e - 2 * half;
          tv[e] = col >= 0 && col < a.cols ? qraw[(col - col0 + 4) * R + n] : 0.0f;
        }
        float4 hb, hs;
        split3(tv[0], hb.x, hs.x);
        split3(tv[1], hb.y, hs.y);
        split3(tv[2], hb.z, hs.z);
        split3(tv[3], hb.w, hs.w);
        unsigned char *bt = st + (half ? kPrOffBo : kPrOffBe);
        *reinterpret_cast<float4 *>(bt + sw128(n, c8)) = hb;
        *reinterpret_cast<float4 *>(bt + sw128(H + n, c8)) = hs;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full_bar(s)) : "memory");
      const int64_t gi = k / kGroup;
      if (k % kGroup == 0 && gi >= 1) fold_group(gi - 1);
    }
    if (nloc > 0) fold_group((nloc - 1) / kGroup);
  }

  if (warp < 4 && lane < 16) {
    const int r16 = warp * 16 + lane;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int64_t grow = row0 + 2 * r16 + half;
      if (grow < a.rows) {
#pragma unroll
        for (int b = 0; b < R; ++b)
          a.partial[((static_cast<int64_t>(v) * a.splits + split) * a.rows + grow) * R + b] =
              half ? acc_o[b] : acc_e[b];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem) : "memory");
}

// ------------------------------------------------------------------ Q_w = M_w^T P_hat for cols = 2 (mod 4)
// mtp_tma_kernel's column slabs over the row-pair maps: per 128-row box an even box (32 columns x
// 64 pair rows) and an odd box 36 columns wide (the odd rows' columns c0 - 2 .. c0 + 33, no
// swizzle: 144-byte rows) so the odd rows' columns c0 .. c0 + 31 are read at +2 floats (two
// 8-byte loads); the thread's 4 columns are the same for both halves.  Ranks 1..4.
constexpr int kMpEven = kPrM * kKc * 4;           // 8 KB
constexpr int kMpOdd = kPrM * 36 * 4;             // 9 KB
constexpr int kMpStage = (kMpEven + kMpOdd + kMtpPh + 1023) / 1024 * 1024;
constexpr int kMpSmem = kMtpStages * kMpStage + 64 + 1024;

template <int R>
__global__ void __launch_bounds__(kMtpThreads, 1) mtp_pair_kernel(const __grid_constant__ PairMapSet maps,
                                                                 const __grid_constant__ MtpArgs a) {
  static_assert(R <= 4, "rank <= 4");
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char *sm = smem_raw + (base - raw);
  const uint32_t bars = base + kMtpStages * kMpStage;   // loaded[S], empty[S]
  __shared__ double red[kMtpConsumers / 8][32][R];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int vl = blockIdx.z, v = a.v_base + vl, split = blockIdx.y;
  const int tl = vl / a.L, w = vl % a.L;
  const float *ph = a.ph + static_cast<int64_t>(v / a.L) * a.rows * R;
  const int64_t col0 = static_cast<int64_t>(blockIdx.x) * kKc;
  const int64_t r_begin = split * a.rows_per_split;
  const int64_t r_end = min(a.rows_full, r_begin + a.rows_per_split);
  const int64_t nbox = r_end > r_begin ? (r_end - r_begin + kM - 1) / kM : 0;
  if (tid == 0) {
    for (int s = 0; s < kMtpStages; ++s) {
      mbar_init(bars + 8 * s, 1);
      mbar_init(bars + 8 * (kMtpStages + s), kMtpConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kMtpConsumers / 32) {   // producer warp: the TMA ring (even box, odd box, P_hat rows)
    if (lane == 0) {
      for (int64_t b = 0; b < nbox; ++b) {
        const int s = static_cast<int>(b % kMtpStages);
        const int64_t i0 = r_begin + b * kM;
        if (b >= kMtpStages)
          mbar_wait(bars + 8 * (kMtpStages + s), static_cast<uint32_t>(((b / kMtpStages) - 1) & 1));
        const bool full = i0 + kM <= r_end;
        mbar_expect_tx(bars + 8 * s, kMpEven + kMpOdd + (full ? kM * R * 4 : 0));
        const int k0 = static_cast<int>(i0 / 2);
        tma_load_3d(base + s * kMpStage, &maps.ge[tl], static_cast<int>(col0), k0, w, bars + 8 * s);
        tma_load_3d(base + s * kMpStage + kMpEven, &maps.go[tl], static_cast<int>(col0), k0, w, bars + 8 * s);
        if (full) bulk_load(base + s * kMpStage + kMpEven + kMpOdd, ph + i0 * R, kM * R * 4, bars + 8 * s);
      }
    }
    return;
  }
  const int g4 = tid & 7, rg = tid >> 3;   // float4 column group, pair-row group (pair rows rg + 32 k)
  double acc64[4][R];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) acc64[t][b] = 0.0;
  for (int64_t bx = 0; bx < nbox; ++bx) {
    const int s = static_cast<int>(bx % kMtpStages);
    const int64_t i0 = r_begin + bx * kM;
    const bool full = i0 + kM <= r_end;
    mbar_wait(bars + 8 * s, static_cast<uint32_t>((bx / kMtpStages) & 1));
    const unsigned char *st = sm + s * kMpStage;
    const float *phs = reinterpret_cast<const float *>(st + kMpEven + kMpOdd);
    float acc[4][R];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int b = 0; b < R; ++b) acc[t][b] = 0.0f;
#pragma unroll
    for (int k = 0; k < kPrM / 32; ++k) {
      const int pr = rg + 32 * k;
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int row = 2 * pr + half;   // row within the box
        float mv[4];
        if (half == 0) {
          const float4 m = *reinterpret_cast<const float4 *>(st + sw128(pr, g4));
          mv[0] = m.x, mv[1] = m.y, mv[2] = m.z, mv[3] = m.w;
        } else {   // odd rows: columns c0 .. at +2 floats in the 36-wide box
          const float *orow = reinterpret_cast<const float *>(st + kMpEven + pr * 144) + 2 + 4 * g4;
          const float2 x = *reinterpret_cast<const float2 *>(orow), y = *reinterpret_cast<const float2 *>(orow + 2);
          mv[0] = x.x, mv[1] = x.y, mv[2] = y.x, mv[3] = y.y;
        }
        float p[R];
        if (full) {
#pragma unroll
          for (int b = 0; b < R; ++b) p[b] = phs[row * R + b];
        } else {
#pragma unroll
          for (int b = 0; b < R; ++b) p[b] = i0 + row < r_end ? __ldg(ph + (i0 + row) * R + b) : 0.0f;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int b = 0; b < R; ++b) acc[t][b] = fmaf(mv[t], p[b], acc[t][b]);
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int b = 0; b < R; ++b) acc64[t][b] += static_cast<double>(acc[t][b]);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bars + 8 * (kMtpStages + s)) : "memory");
  }
  if (rg == 0 && split == a.splits - 1 && a.rows_full < a.rows) {   // the partly filled row, fp64
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t col = col0 + 4 * g4 + t;
      const int64_t off = a.rows_full * a.cols + col;
      if (col < a.cols && off < a.d) {
        const int64_t rs = a.row_start ? a.row_start[v] : static_cast<int64_t>(v) * a.ld;
        const double m = static_cast<double>(a.c[rs + off]);
#pragma unroll
        for (int b = 0; b < R; ++b) acc64[t][b] += m * static_cast<double>(ph[a.rows_full * R + b]);
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) red[rg][4 * g4 + t][b] = acc64[t][b];
  asm volatile("bar.sync 1, %0;" ::"r"(kMtpConsumers) : "memory");
  for (int e = tid; e < 32 * R; e += kMtpConsumers) {
    const int cc = e / R, b = e - cc * R;
    double x = 0.0;
#pragma unroll 8
    for (int q = 0; q < kMtpConsumers / 8; ++q) x += red[q][cc][b];
    if (col0 + cc < a.cols) a.partial[((static_cast<int64_t>(v) * a.splits + split) * a.cols + col0 + cc) * R + b] = x;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// [L][rows_full][cols] fp32 view of worker rows at base + w * ld, 32 x 128 boxes, SWIZZLE_128B
bool make_map(CUtensorMap *m, const float *base, int64_t L, int64_t rows_full, int64_t cols, int64_t ld,
              uint32_t box_rows = kM, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows_full), static_cast<cuuint64_t>(L)};
  // one worker: the worker stride is never used, any multiple of 16 bytes will do
  const int64_t ld_map = L == 1 ? (ld + 3) / 4 * 4 : ld;
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(cols * 4), static_cast<cuuint64_t>(ld_map * 4)};
  cuuint32_t box[3] = {kKc, box_rows, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// row-pair maps for cols = 2 (mod 4): pair rows of 2 cols floats; odd = the odd rows, shifted so an
// odd box at column c0 holds columns c0 - 2 .. c0 + 29 (boxes 32 columns x 64 pair rows)
bool make_map_pair(CUtensorMap *m, const float *base, bool odd, int64_t L, int64_t rows_full, int64_t cols,
                   int64_t ld, uint32_t box_cols = kKc, CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int64_t pairs = odd ? rows_full / 2 : (rows_full + 1) / 2;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(odd ? cols + 2 : cols), static_cast<cuuint64_t>(pairs),
                        static_cast<cuuint64_t>(L)};
  const int64_t ld_map = L == 1 ? (ld + 3) / 4 * 4 : ld;
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(2 * cols * 4), static_cast<cuuint64_t>(ld_map * 4)};
  cuuint32_t box[3] = {box_cols, kPrM, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(odd ? base + cols - 2 : base), dims, strides,
            box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int grid_cap(int64_t g) { return static_cast<int>(g < 1 ? 1 : (g > 65535 ? 65535 : g)); }

// column splits for a grid of ctas x splits one-CTA-per-SM blocks: the fewest splits whose last
// wave is nearly full (a 336-CTA grid runs 2.27 waves; x 2 splits, 4.54 -> 0.91 of 5 full waves)
// Column splits of P = M Q: a CTA is one (row block, split, tensor-worker) item and pays a fixed
// cost (TMEM alloc, ring fill, accumulator drain and fp64 fold) worth about kSplitOverhead chunks of
// streaming, so minimise waves x (chunks per item + overhead) rather than maximising wave fill alone
// (GPT-2-medium's 7174-column matrix: 18 splits of 13 chunks -> 5 splits of 45; 1774 columns x 24
// tensors: 7 -> 2).  GC_MQ_SPLIT_OVERHEAD overrides the overhead (in chunks); < 0 selects the
// fill-only rule.
int64_t wave_splits(int64_t ctas, int64_t max_splits, int64_t nchunks, int sms) {
  static const double overhead = [] {
    const char *e = getenv("GC_MQ_SPLIT_OVERHEAD");
    return e ? atof(e) : 3.0;
  }();
  int64_t best = 1;
  double best_cost = 0.0, best_eff = 0.0;
  for (int64_t s = 1; s <= max_splits && nchunks / s >= 4; ++s) {
    const int64_t items = ctas * s, waves = (items + sms - 1) / sms;
    if (overhead < 0.0) {
      const double eff = static_cast<double>(items) / static_cast<double>(waves * sms);
      if (eff > best_eff + 0.02) best = s, best_eff = eff;
      continue;
    }
    const double cost = static_cast<double>(waves) * (static_cast<double>((nchunks + s - 1) / s) + overhead);
    if (s == 1 || cost < best_cost * 0.98) best = s, best_cost = cost;
  }
  return best;
}


// Row splits of Q = M^T P_hat: `items` (column slab, tensor-worker) CTAs per split, each walking
// ceil(boxes / s) 128-row boxes plus a fixed cost worth ~kMtpOverhead boxes; pick s minimising
// waves x (boxes per CTA + overhead) with `occ` resident CTAs per SM.  GC_MTP_SPLIT_OVERHEAD
// overrides the overhead (in boxes); < 0 selects the old rule (about two CTAs per SM).
int64_t mtp_splits(int64_t items, int64_t boxes, int64_t max_splits, int sms, int occ) {
  static const double overhead = [] {
    const char *e = getenv("GC_MTP_SPLIT_OVERHEAD");
    return e ? atof(e) : 6.0;
  }();
  int64_t best = 1;
  if (overhead < 0.0) {
    best = (2 * sms + items - 1) / items;
  } else {
    const int64_t slots = static_cast<int64_t>(sms) * (occ < 1 ? 1 : occ);
    double best_cost = 0.0;
    for (int64_t s = 1; s <= max_splits && s <= boxes; ++s) {
      const int64_t waves = (items * s + slots - 1) / slots;
      const double cost = static_cast<double>(waves) * (static_cast<double>((boxes + s - 1) / s) + overhead);
      if (s == 1 || cost < best_cost * 0.98) best = s, best_cost = cost;
    }
  }
  if (best > max_splits) best = max_splits;
  if (best > boxes) best = boxes;
  return best < 1 ? 1 : best;
}

template <typename K>
int mtp_occupancy(K kernel, int smem) {   // resident CTAs per SM, queried once per kernel type
  static int cached = 0;
  if (cached > 0) return cached;
  int occ = 1;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kMtpThreads, smem) != cudaSuccess) {
    (void)cudaGetLastError();
    occ = 1;
  }
  cached = occ;
  return occ;
}

}  // namespace

int gc_psgd_mq_tma_supported_impl(int32_t tensors, int32_t workers, const int64_t *host_tensor_offsets, int64_t ld,
                                  int64_t d, int64_t rows, int64_t cols, int32_t rank, const void *grads,
                                  const void *resid) {
  if (tensors < 1 || (tensors > 1 && host_tensor_offsets == nullptr)) return 0;
  if (cols % 4 != 0 || ((workers > 1 || tensors > 1) && ld % 4 != 0) || cols > (int64_t{1} << 31) - 1 ||
      rows > (int64_t{1} << 31) - 1)
    return 0;
  if (d / cols < 1) return 0;
  if ((reinterpret_cast<uintptr_t>(grads) | reinterpret_cast<uintptr_t>(resid)) & 15) return 0;
  if (host_tensor_offsets)
    for (int t = 0; t < tensors; ++t)
      if (host_tensor_offsets[t] % 4 != 0) return 0;
  switch (rank) {
    case 1: case 2: case 3: case 4: case 5: case 6: case 7: case 8: case 16: break;
    default: return 0;
  }
  return encode_fn() != nullptr ? 1 : 0;
}

// TMA-fed Q_w = M_w^T P_hat: fp64 split-K partials partial[w][split][col][R] (max_splits slots
// sized by the caller); returns the split count or a negative status.
int gc_psgd_mtp_tma_launch(int32_t T, int32_t L, const int64_t *host_tensor_offsets, const int64_t *row_start,
                           int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
                           const float *p_hat, double *partial, int64_t max_splits, cudaStream_t st) {
  const int64_t rows_full = d / cols;
  const int64_t slabs = (cols + kKc - 1) / kKc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t boxes = (rows_full + kM - 1) / kM;
  const int64_t V = static_cast<int64_t>(T) * L;
  int64_t splits = mtp_splits(slabs * V, boxes, max_splits, sms, mtp_occupancy(mtp_tma_kernel<4>, kMtpSmem));
  const int64_t per = (boxes + splits - 1) / splits;
  splits = (boxes + per - 1) / per;
  MtpArgs a{};
  a.d = d;
  a.rows = rows;
  a.cols = cols;
  a.rows_full = rows_full;
  a.ld = ld;
  a.c = c;
  a.ph = p_hat;
  a.partial = partial;
  a.splits = static_cast<int>(splits);
  a.rows_per_split = per * kM;
  a.L = L;
  a.row_start = row_start;
  MtpMaps maps;
  for (int t0 = 0; t0 < T; t0 += kMaxMapT) {
    const int tc = T - t0 < kMaxMapT ? T - t0 : kMaxMapT;
    for (int k = 0; k < tc; ++k) {
      const int64_t off = host_tensor_offsets ? host_tensor_offsets[t0 + k] : 0;
      if (!make_map(&maps.m[k], c + off, L, rows_full, cols, ld)) {
        gc_set_error("cuTensorMapEncodeTiled failed for the Q = M^T P_hat operand");
        return GC_ERR_CUDA;
      }
    }
    a.v_base = t0 * L;
    const dim3 grid(static_cast<unsigned>(slabs), static_cast<unsigned>(splits), static_cast<unsigned>(tc * L));
#define GC_MTPT(RR)                                                                                    \
  case RR:                                                                                             \
    cudaFuncSetAttribute(mtp_tma_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMtpSmem);   \
    mtp_tma_kernel<RR><<<grid, kMtpThreads, kMtpSmem, st>>>(maps, a);                                 \
    break;
    switch (rank) {
      GC_MTPT(1) GC_MTPT(2) GC_MTPT(3) GC_MTPT(4)
      default:
        gc_set_error("the TMA Q = M^T P_hat pass takes ranks 1..4");
        return GC_ERR_UNSUPPORTED;
    }
#undef GC_MTPT
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      gc_set_error(std::string("mtp_tma_kernel: ") + cudaGetErrorString(e));
      return GC_ERR_CUDA;
    }
  }
  return static_cast<int>(splits);
}

// tcgen05 Q_w = M_w^T P_hat (MN-major A from the TMA boxes): fp64 split-K partials
// partial[w][split][col][R]; returns the split count or a negative status.
int gc_psgd_mtp_umma_launch(int32_t L, int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
                            const float *p_hat, double *partial, int64_t max_splits, cudaStream_t st) {
  const int64_t rows_full = d / cols;
  const int64_t cblocks = (cols + kQtM - 1) / kQtM;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t chunks = (rows_full + kQtK - 1) / kQtK;
  int64_t splits = sms / (cblocks * L);
  if (splits > max_splits) splits = max_splits;
  if (splits > chunks) splits = chunks;
  if (splits < 1) splits = 1;
  const int64_t per = (chunks + splits - 1) / splits;
  splits = (chunks + per - 1) / per;
  CUtensorMap mc;
  if (!make_map(&mc, c, L, rows_full, cols, ld, kQtK, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B)) {
    gc_set_error("cuTensorMapEncodeTiled failed for the Q = M^T P_hat operand");
    return GC_ERR_CUDA;
  }
  MtpArgs a{};
  a.d = d;
  a.rows = rows;
  a.cols = cols;
  a.rows_full = rows_full;
  a.ld = ld;
  a.c = c;
  a.ph = p_hat;
  a.partial = partial;
  a.splits = static_cast<int>(splits);
  a.rows_per_split = per * kQtK;
  const dim3 grid(static_cast<unsigned>(cblocks), static_cast<unsigned>(splits), static_cast<unsigned>(L));
  // rings: operand slots first (the producers wait on them), then as many load stages as fit
  const int n_cols = rank <= 8 ? 16 : 32;
  a.stage_bytes = kQtA + (kQtK * rank * 4 + 1023) / 1024 * 1024;
  a.op_bytes = kQtA + n_cols * 128;
  const char *e_slots = getenv("GC_MTPU_SLOTS");
  a.slots = e_slots ? atoi(e_slots) : (rank <= 8 ? 6 : 4);
  const int smem_cap = 232448 - 1024 - kQtBarBytes;
  a.stages = (smem_cap - a.slots * a.op_bytes) / a.stage_bytes;
  if (const char *e_st = getenv("GC_MTPU_STAGES")) a.stages = std::min(a.stages, atoi(e_st));
  if (a.stages > 16) a.stages = 16;
  if (a.slots < 2 || a.slots > 16 || a.stages < 2) {
    gc_set_error("mtp_umma_kernel: ring sizes do not fit shared memory");
    return GC_ERR_UNSUPPORTED;
  }
  const int smem = a.stages * a.stage_bytes + a.slots * a.op_bytes + kQtBarBytes + 1024;
#define GC_MTPU(RR)                                                                                 \
  case RR:                                                                                          \
    cudaFuncSetAttribute(mtp_umma_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);   \
    mtp_umma_kernel<RR><<<grid, kQtThreads, smem, st>>>(mc, a);                                    \
    break;
  switch (rank) {
    GC_MTPU(1) GC_MTPU(2) GC_MTPU(3) GC_MTPU(4) GC_MTPU(5) GC_MTPU(6) GC_MTPU(7) GC_MTPU(8) GC_MTPU(16)
    default:
      gc_set_error("rank must be 1..8 or 16");
      return GC_ERR_UNSUPPORTED;
  }
#undef GC_MTPU
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gc_set_error(std::string("mtp_umma_kernel: ") + cudaGetErrorString(e));
    return GC_ERR_CUDA;
  }
  return static_cast<int>(splits);
}

// TMA-fed tcgen05 P = M Q with ef_apply (and, with ef_ph / ef_qw, the previous round's deferred
// EF update).  fp64 split-K partials partial[w][split][row][R]; returns the split count or a
// negative status.
int gc_psgd_mq_tma_launch(int32_t T, int32_t L, const int64_t *host_tensor_offsets, const int64_t *row_start,
                          int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                          float *resid, const float *q, const float *ef_ph, const float *ef_qw, double *partial,
                          int64_t max_splits, cudaStream_t st) {
  const int64_t rows_full = d / cols;
  const int64_t row_blocks = (rows + kM - 1) / kM;
  const int64_t nchunks = (cols + kKc - 1) / kKc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t splits = wave_splits(row_blocks * L * T, max_splits, nchunks, sms);
  const int64_t per = (nchunks + splits - 1) / splits;
  splits = (nchunks + per - 1) / per;
  TmaArgs a{};
  a.d = d;
  a.rows = rows;
  a.cols = cols;
  a.rows_full = rows_full;
  a.L = L;
  a.row_start = row_start;
  a.q = q;
  a.ef_ph = ef_ph;
  a.ef_qw = ef_qw;
  a.partial = partial;
  a.splits = static_cast<int>(splits);
  a.chunks_per_split = per;
  a.has_resid = resid != nullptr;
  const bool def = resid != nullptr && ef_ph != nullptr && ef_qw != nullptr;
  const bool tail = rows_full < rows && d > rows_full * cols;
  MapSet maps;   // the launch's tensor maps, copied into the kernel parameter buffer at launch
  for (int t0 = 0; t0 < T; t0 += kMaxMapT) {
    const int tc = T - t0 < kMaxMapT ? T - t0 : kMaxMapT;
    std::memset(&maps, 0, sizeof(maps));
    for (int k = 0; k < tc; ++k) {
      const int64_t off = host_tensor_offsets ? host_tensor_offsets[t0 + k] : 0;
      if (!make_map(&maps.g[k], grads + off, L, rows_full, cols, ld) ||
          (resid && !make_map(&maps.r[k], resid + off, L, rows_full, cols, ld))) {
        gc_set_error("cuTensorMapEncodeTiled failed for the P = M Q operands");
        return GC_ERR_CUDA;
      }
    }
    a.v_base = t0 * L;
    const dim3 grid(grid_cap(row_blocks), static_cast<unsigned>(splits), static_cast<unsigned>(tc * L));
#define GC_TMA_LAUNCH(RR, DD)                                                                              \
  cudaFuncSetAttribute(mq_tma_kernel<RR, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);    \
  mq_tma_kernel<RR, DD><<<grid, kThreads, kSmemBytes, st>>>(maps, a);                                      \
  if (tail) mq_tail_row_kernel<RR, DD><<<tc * L, kTailThreads, 0, st>>>(grads, resid, ld, a);
#define GC_TMA_CASE(RR)        \
  case RR:                     \
    if (def) {                 \
      GC_TMA_LAUNCH(RR, true)  \
    } else {                   \
      GC_TMA_LAUNCH(RR, false) \
    }                          \
    break;
    switch (rank) {
      GC_TMA_CASE(1) GC_TMA_CASE(2) GC_TMA_CASE(3) GC_TMA_CASE(4) GC_TMA_CASE(5) GC_TMA_CASE(6)
      GC_TMA_CASE(7) GC_TMA_CASE(8) GC_TMA_CASE(16)
      default:
        gc_set_error("rank must be 1..8 or 16");
        return GC_ERR_UNSUPPORTED;
    }
#undef GC_TMA_CASE
#undef GC_TMA_LAUNCH
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gc_set_error(std::string("mq_tma_kernel: ") + cudaGetErrorString(e));
    return GC_ERR_CUDA;
  }
  return static_cast<int>(splits);
}

int gc_psgd_mq_pair_supported_impl(int32_t tensors, int32_t workers, const int64_t *host_tensor_offsets, int64_t ld,
                                   int64_t d, int64_t rows, int64_t cols, int32_t rank, const void *grads,
                                   const void *resid) {
  if (cols % 4 != 2 || rank % 4 != 0 || rank > 16 || d / cols < 2 || cols > (int64_t{1} << 30)) return 0;
  if (tensors > 1 && host_tensor_offsets == nullptr) return 0;
  if (workers > 1 && ld % 4 != 0) return 0;
  if ((reinterpret_cast<uintptr_t>(grads) | reinterpret_cast<uintptr_t>(resid)) & 15) return 0;
  if (host_tensor_offsets)
    for (int t = 0; t < tensors; ++t)
      if (host_tensor_offsets[t] % 4 != 0) return 0;
  (void)rows;
  return 1;
}

// P = M Q over row-pair tensor maps (cols = 2 mod 4); the same split-K partials as gc_psgd_mq_tma_launch
int gc_psgd_mq_pair_launch(int32_t T, int32_t L, const int64_t *host_tensor_offsets, const int64_t *row_start,
                           int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                           float *resid, const float *q, const float *ef_ph, const float *ef_qw, double *partial,
                           int64_t max_splits, cudaStream_t st) {
  const int64_t rows_full = d / cols;
  const int64_t row_blocks = (rows + kM - 1) / kM;
  const int64_t nchunks = (cols + kKc - 1) / kKc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t splits = wave_splits(row_blocks * L * T, max_splits, nchunks, sms);
  const int64_t per = (nchunks + splits - 1) / splits;
  splits = (nchunks + per - 1) / per;
  TmaArgs a{};
  a.d = d;
  a.rows = rows;
  a.cols = cols;
  a.rows_full = rows_full;
  a.L = L;
  a.row_start = row_start;
  a.q = q;
  a.ef_ph = ef_ph;
  a.ef_qw = ef_qw;
  a.partial = partial;
  a.splits = static_cast<int>(splits);
  a.chunks_per_split = per;
  a.has_resid = resid != nullptr;
  a.r_out = resid;
  a.ld = ld;
  const bool def = resid != nullptr && ef_ph != nullptr && ef_qw != nullptr;
  const bool tail = rows_full < rows && d > rows_full * cols;
  constexpr int kPerLaunch = kMaxMapT / 2;
  PairMapSet maps;
  for (int t0 = 0; t0 < T; t0 += kPerLaunch) {
    const int tc = T - t0 < kPerLaunch ? T - t0 : kPerLaunch;
    std::memset(&maps, 0, sizeof(maps));
    for (int k = 0; k < tc; ++k) {
      const int64_t off = host_tensor_offsets ? host_tensor_offsets[t0 + k] : 0;
      bool ok = make_map_pair(&maps.ge[k], grads + off, false, L, rows_full, cols, ld) &&
                make_map_pair(&maps.go[k], grads + off, true, L, rows_full, cols, ld);
      if (resid)
        ok = ok && make_map_pair(&maps.re[k], resid + off, false, L, rows_full, cols, ld) &&
             make_map_pair(&maps.ro[k], resid + off, true, L, rows_full, cols, ld);
      if (!ok) {
        gc_set_error("cuTensorMapEncodeTiled failed for the row-pair P = M Q operands");
        return GC_ERR_CUDA;
      }
    }
    a.v_base = t0 * L;
    const dim3 grid(grid_cap(row_blocks), static_cast<unsigned>(splits), static_cast<unsigned>(tc * L));
#define GC_PAIR_LAUNCH(RR, DD)                                                                            \
  cudaFuncSetAttribute(mq_pair_kernel<RR, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPrSmem);     \
  mq_pair_kernel<RR, DD><<<grid, kThreads, kPrSmem, st>>>(maps, a);                                       \
  if (tail) mq_tail_row_kernel<RR, DD><<<tc * L, kTailThreads, 0, st>>>(grads, resid, ld, a);
#define GC_PAIR_CASE(RR)        \
  case RR:                      \
    if (def) {                  \
      GC_PAIR_LAUNCH(RR, true)  \
    } else {                    \
      GC_PAIR_LAUNCH(RR, false) \
    }                           \
    break;
    switch (rank) {
      GC_PAIR_CASE(4) GC_PAIR_CASE(8) GC_PAIR_CASE(16)
      default:
        gc_set_error("the row-pair P = M Q pass takes ranks 4, 8, 16");
        return GC_ERR_UNSUPPORTED;
    }
#undef GC_PAIR_CASE
#undef GC_PAIR_LAUNCH
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gc_set_error(std::string("mq_pair_kernel: ") + cudaGetErrorString(e));
    return GC_ERR_CUDA;
  }
  return static_cast<int>(splits);
}

// Q_w = M_w^T P_hat over row-pair maps (cols = 2 mod 4, ranks 1..4): split-K partials as gc_psgd_mtp's
int gc_psgd_mtp_pair_launch(int32_t T, int32_t L, const int64_t *host_tensor_offsets, const int64_t *row_start,
                            int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
                            const float *p_hat, double *partial, int64_t max_splits, cudaStream_t st) {
  const int64_t rows_full = d / cols;
  const int64_t slabs = (cols + kKc - 1) / kKc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t boxes = (rows_full + kM - 1) / kM;
  const int64_t V = static_cast<int64_t>(T) * L;
  int64_t splits = mtp_splits(slabs * V, boxes, max_splits, sms, mtp_occupancy(mtp_pair_kernel<4>, kMpSmem));
  const int64_t per = (boxes + splits - 1) / splits;
  splits = (boxes + per - 1) / per;
  MtpArgs a{};
  a.d = d;
  a.rows = rows;
  a.cols = cols;
  a.rows_full = rows_full;
  a.ld = ld;
  a.c = c;
  a.ph = p_hat;
  a.partial = partial;
  a.splits = static_cast<int>(splits);
  a.rows_per_split = per * kM;
  a.L = L;
  a.row_start = row_start;
  constexpr int kPerLaunch = kMaxMapT / 2;
  PairMapSet maps;
  for (int t0 = 0; t0 < T; t0 += kPerLaunch) {
    const int tc = T - t0 < kPerLaunch ? T - t0 : kPerLaunch;
    std::memset(&maps, 0, sizeof(maps));
    for (int k = 0; k < tc; ++k) {
      const int64_t off = host_tensor_offsets ? host_tensor_offsets[t0 + k] : 0;
      if (!make_map_pair(&maps.ge[k], c + off, false, L, rows_full, cols, ld) ||
          !make_map_pair(&maps.go[k], c + off, true, L, rows_full, cols, ld, 36, CU_TENSOR_MAP_SWIZZLE_NONE)) {
        gc_set_error("cuTensorMapEncodeTiled failed for the row-pair Q = M^T P_hat operand");
        return GC_ERR_CUDA;
      }
    }
    a.v_base = t0 * L;
    const dim3 grid(static_cast<unsigned>(slabs), static_cast<unsigned>(splits), static_cast<unsigned>(tc * L));
#define GC_MTPP(RR)                                                                                   \
  case RR:                                                                                            \
    cudaFuncSetAttribute(mtp_pair_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMpSmem);  \
    mtp_pair_kernel<RR><<<grid, kMtpThreads, kMpSmem, st>>>(maps, a);                                \
    break;
    switch (rank) {
      GC_MTPP(1) GC_MTPP(2) GC_MTPP(3) GC_MTPP(4)
      default:
        gc_set_error("the row-pair Q = M^T P_hat pass takes ranks 1..4");
        return GC_ERR_UNSUPPORTED;
    }
#undef GC_MTPP
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      gc_set_error(std::string("mtp_pair_kernel: ") + cudaGetErrorString(e));
      return GC_ERR_CUDA;
    }
  }
  return static_cast<int>(splits);
}
