// PowerSGD P = M Q on tcgen05 for row pitches a tensor map cannot describe (cols % 4 != 0, or
// tensor starts that are not 16-byte aligned): the chunked PowerSGD of a model has them (GPT-2's
// 1024 x 3072 attention weights become 1774 x 1774 matrices, its 50257 x 1024 embedding 7174 x 7174).
// The same pass as gc_psgd_tma.cu's -- deferred error feedback folded in (the previous round's
// r = c_prev - P_hat_prev Q_w_prev^T formed per element in the decode's fp32 order), corrected
// written back over the residual buffer, 3xTF32 on the tensor core -- with the operand tiles
// filled by 4-byte cp.async instead of TMA boxes.
//
// Reference: P_w = M_w @ Q (pipelines.py:348), M_w = to_matrix(corrected_w) (compressors.py:530-548),
// corrected_w = f32(g_w + r_w) (ef_apply, compressors.py:624-626), r_w = f32(c_w - own_w) of the
// previous round (pipelines.py:357-361, ef_update compressors.py:629-631).
//
// B200 design.  Persistent CTAs (one per SM) walk work items (tensor-worker row, 128-row band,
// column split).  Each of the 512 producer threads owns one column (lane) of 8 rows of every
// 128 x 32 chunk and copies its g and r elements with cp.async straight to their positions in the
// canonical K-major SWIZZLE_128B tile (a warp writes one row's 128 contiguous bytes: no bank
// conflicts), three chunks ahead of the one it forms; a thread reads back only what it copied, so
// forming needs no barrier -- cp.async.wait_group is enough.  Forming, in place: corrected c over
// the residual tile (A_big: kind::tf32 reads an fp32 pattern's top 19 bits), small = tf32(c -
// tf32(c)) over the gradient tile, c stored to the residual buffer (coalesced 128-byte rows), and
// B = [Q_big^T ; Q_small^T] packed along N so each 8-column k-step is two MMAs,
//     D += A_small [B_big B_small] + A_big [B_big B_small]
// (columns h and H + h of D summed in the fold).  A dedicated warp issues the MMAs (M = 128,
// N = 16 or 32) and commits each stage's release; every 512 columns the fp32 TMEM partial is
// folded into fp64 (two accumulators alternate, folded four chunks into the next group).
// Elements past the row, past d (to_matrix's zero padding) or past the matrix copy as zeros.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "gc_internal.h"
#include "gc_umma.cuh"

namespace {
using namespace gcu;

constexpr int kM = 128;                    // UMMA M: rows per band
constexpr int kKc = 32;                    // columns per chunk: one 128-byte swizzle atom of fp32
constexpr int kTile = kM * kKc * 4;        // 16 KB
constexpr int kProducers = 512;            // 16 warps: warp w owns rows w + 16u, lane = column (W = 1)
constexpr int kPWarps = kProducers / 32;
constexpr int kThreads = kProducers + 32;  // + the MMA warp
constexpr int kGroup = 512 / kKc;          // chunks per TMEM partial
constexpr int kFoldLag = 4;                // group g - 1 is folded at chunk 16 g + 4 of the item
constexpr int kOffG = 0, kOffC = kTile, kOffB = 2 * kTile;
constexpr int kPhBytes = kM * 16 * 4;      // the band's P_hat_prev rows, rank <= 16
// 4- and 8-byte cp.async land through L1 (.ca is the only cache mode below 16 bytes), so the bytes
// in flight are bounded by the L1 the ring leaves free: a 3-stage ring (~115 KB of shared memory)
// runs 1.25x faster than a 6-stage one (tools/ubench/unaligned_stream.cu, profiles/)
#ifndef GC_MQA_SMEM
#define GC_MQA_SMEM 150000
#endif
constexpr int kSmemCap = GC_MQA_SMEM;      // shared memory the ring may take (the rest stays L1)

// per rank: B = [Q_big^T ; Q_small^T] has N = 2H rows (H = 8, or 16 for rank 16); a stage holds the
// gradient tile (-> A_small), the residual tile (-> corrected = A_big), B, and the chunk's 32 rows of
// Q and of Q_w_prev (cp.async with the tiles); as many stages as shared memory takes
template <int R>
struct Shape {
  static constexpr int H = R <= 8 ? 8 : 16;
  static constexpr int N = 2 * H;
  static constexpr uint32_t idesc = idesc_tf32(kM, N);
  static constexpr int kRawBytes = (kKc * R * 4 + 127) / 128 * 128;   // 32 rows of Q (or Q_w_prev)
  static constexpr int kOffQ = 2 * kTile + N * 128, kOffW = kOffQ + kRawBytes;
  static constexpr int kStage = (kOffW + kRawBytes + 1023) / 1024 * 1024;
  static constexpr int kStages = (kSmemCap - 1024 - 512 - kPhBytes) / kStage;
  static constexpr int kAhead = kStages - 2;   // chunks of copies in flight beyond the one being formed
  static constexpr int kSmem = kStages * kStage + kPhBytes + 512 + 1024;
  static_assert(kStages >= 3, "ring too shallow");
};

struct AsyncArgs {
  int64_t d, rows, cols;
  int64_t rows_full, tail_cols;   // d / cols; columns of the partly filled row (d - rows_full * cols)
  const float *g;
  float *r;                  // residual buffer (corrected written back), or null
  const int64_t *row_offs;   // device [V] element offset of each (tensor, worker) row, or null
  int64_t ld;                // ... else row v at v * ld
  int L;                     // workers per tensor: virtual row v = t * L + w
  const float *q;            // [T][cols][R]
  const float *ef_ph;        // deferred EF: P_hat_prev [T][rows][R] or null
  const float *ef_qw;        // deferred EF: Q_w_prev [V][cols][R]
  double *partial;           // [V][splits][rows][R]
  int splits;
  int64_t chunks_per_split, nchunks;
  int row_blocks;
  int64_t items;
};

struct Item {   // work item: (v, split, band)
  int v, split;
  int64_t row0, c_begin, nloc;
  __device__ __forceinline__ void set(const AsyncArgs &a, int64_t it) {
    const int64_t rb = it % a.row_blocks, rest = it / a.row_blocks;
    split = static_cast<int>(rest % a.splits);
    v = static_cast<int>(rest / a.splits);
    row0 = rb * kM;
    c_begin = split * a.chunks_per_split;
    nloc = min(a.nchunks, c_begin + a.chunks_per_split) - c_begin;
  }
};

// the stream of chunks a CTA works through: items blockIdx.x, + gridDim.x, ..., their chunks in order
struct ChunkIt {
  int64_t it, lk;
  Item item;
  __device__ __forceinline__ void start(const AsyncArgs &a) {
    it = blockIdx.x;
    lk = 0;
    if (it < a.items) item.set(a, it);
  }
  __device__ __forceinline__ bool valid(const AsyncArgs &a) const { return it < a.items; }
  __device__ __forceinline__ void next(const AsyncArgs &a) {
    if (++lk == item.nloc) {
      lk = 0;
      it += gridDim.x;
      if (it < a.items) item.set(a, it);
    }
  }
};

// the thread's elements of a chunk: W = 1: column lane, rows warp + 16u (u < 8); W = 2: columns
// 2 (lane & 15) + {0, 1}, rows 2 warp + (lane >> 4) + 32u (u < 4).  A warp instruction covers 128 or
// 256 contiguous bytes of the swizzled tile (no bank conflicts); rows + 16 W = 2048 W bytes.
template <int W>
struct Lanes {
  static constexpr int U = kM / (kPWarps * W);
  static constexpr int kRowStep = kPWarps * W;
  static constexpr uint32_t kRowBytes = 128 * kPWarps * W;
  __device__ static __forceinline__ int row(int warp, int lane) { return W == 1 ? warp : 2 * warp + (lane >> 4); }
  __device__ static __forceinline__ int col(int lane) { return W == 1 ? lane : 2 * (lane & 15); }
  __device__ static __forceinline__ void copy(uint32_t dst, const float *src) {
    if (W == 1)
      cp_async4(dst, src);
    else
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
  }
  __device__ static __forceinline__ void lds(const unsigned char *p, float (&v)[W]) {
    if constexpr (W == 1) {
      v[0] = *reinterpret_cast<const float *>(p);
    } else {
      const float2 x = *reinterpret_cast<const float2 *>(p);
      v[0] = x.x;
      v[1] = x.y;
    }
  }
  __device__ static __forceinline__ void sts(unsigned char *p, const float (&v)[W]) {
    if constexpr (W == 1)
      *reinterpret_cast<float *>(p) = v[0];
    else
      *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
  }
  __device__ static __forceinline__ void stg(float *p, const float (&v)[W]) {
    if constexpr (W == 1)
      *p = v[0];
    else
      *reinterpret_cast<float2 *>(p) = make_float2(v[0], v[1]);
  }
};

__device__ __forceinline__ void producers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kProducers) : "memory"); }

template <int R, bool DEF, int W>
__global__ void __launch_bounds__(kThreads, 1) mq_async_kernel(const __grid_constant__ AsyncArgs a) {
  using SH = Shape<R>;
  constexpr int H = SH::H, N = SH::N, kStage = SH::kStage, kStages = SH::kStages;
  extern __shared__ unsigned char smem_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  unsigned char *sm = smem_raw + (base - raw);
  auto stage = [&](int s) { return base + static_cast<uint32_t>(s * kStage); };
  float *ph_s = reinterpret_cast<float *>(sm + kStages * kStage);
  const uint32_t bars = base + kStages * kStage + kPhBytes;   // empty[S], full[S], small[S], acc[2]
  auto empty_bar = [&](int s) { return bars + 8 * s; };
  auto full_bar = [&](int s) { return bars + 8 * (kStages + s); };
  auto small_bar = [&](int s) { return bars + 8 * (2 * kStages + s); };
  auto acc_bar = [&](int x) { return bars + 8 * (3 * kStages + x); };
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(sm + kStages * kStage + kPhBytes + 8 * (3 * kStages + 2));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(empty_bar(s), 1);
      mbar_init(full_bar(s), kProducers);
      mbar_init(small_bar(s), 1);
    }
    mbar_init(acc_bar(0), 1);
    mbar_init(acc_bar(1), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {   // two accumulators of N <= 32 columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(tmem_slot)))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  for (int e = tid; e < kStages * N * 8; e += kThreads) {   // padding rows of B stay zero
    const int s = e / (N * 8), o = e - s * (N * 8);
    *reinterpret_cast<uint4 *>(sm + s * kStage + kOffB + o * 16) = make_uint4(0, 0, 0, 0);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  if (warp == kProducers / 32) {   // ---- MMA warp (one elected lane)
    if (lane == 0) {
      RingPos rs{0, 0};
      int64_t groups = 0;   // TMEM groups issued by earlier items
      ChunkIt c;
      for (c.start(a); c.valid(a); c.next(a), rs.step(kStages)) {
        const int64_t gi = groups + c.lk / kGroup;
        mbar_wait(full_bar(rs.idx), rs.phase);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t dcol = tmem + static_cast<uint32_t>((gi & 1) * N);
        const uint32_t st = stage(rs.idx);
#pragma unroll
        for (int ks = 0; ks < kKc / 8; ++ks) {
          const uint64_t ab = sdesc(st + kOffC + 32 * ks), as = sdesc(st + kOffG + 32 * ks);
          const uint64_t bd = sdesc(st + kOffB + 32 * ks);
          const uint32_t accum = (c.lk % kGroup != 0 || ks != 0) ? 1u : 0u;
          umma_tf32(dcol, as, bd, SH::idesc, accum);   // A_small [B_big B_small]
          umma_tf32(dcol, ab, bd, SH::idesc, 1u);      // A_big   [B_big B_small]
        }
        umma_commit(empty_bar(rs.idx));
        const bool last = c.lk == c.item.nloc - 1;
        if (c.lk % kGroup == kGroup - 1 || last) umma_commit(acc_bar(static_cast<int>(gi & 1)));
        if (last) groups += (c.item.nloc + kGroup - 1) / kGroup;
      }
    }
  } else {   // ---- producers
    const int64_t d = a.d, rows = a.rows, cols = a.cols;
    auto row_base = [&](int v) { return a.row_offs ? a.row_offs[v] : static_cast<int64_t>(v) * a.ld; };
    // the thread's elements of a 128 x 32 chunk: W adjacent columns (W = 2: 8-byte copies, when every
    // row start is 8-byte aligned) of rows row_t + 8 W u, u < U; valid rows form a prefix per column
    // (past the matrix, past d in the partly filled row: zeros)
    using LM = Lanes<W>;
    const int row_t = LM::row(warp, lane), col_t = LM::col(lane);
    const uint32_t off0 = sw128(row_t, col_t >> 2) + 4 * (col_t & 3);
    const int64_t rstride = static_cast<int64_t>(LM::kRowStep) * cols;
    // Q / Q_w_prev rows: TMA bulk copies into the stage when every tensor's rows are 16-byte aligned
    // (cols R % 4 == 0), else per-thread register loads (prefetched a chunk ahead for small ranks)
    const bool bulk_small = (cols * R) % 4 == 0;
    auto n_valid = [&](int64_t row0, int64_t col) -> int {
      if (col >= cols) return 0;
      const int64_t last = min(rows - 1, a.rows_full - (col >= a.tail_cols ? 1 : 0));   // last row with data
      const int64_t span = last - row0 - row_t;
      return span < 0 ? 0 : static_cast<int>(min(static_cast<int64_t>(LM::U), span / LM::kRowStep + 1));
    };
    // copy chunk (item, lk) into stage s
    auto copy_chunk = [&](const ChunkIt &c, int s) {
      const int64_t col = (c.item.c_begin + c.lk) * kKc + col_t;
      const int nv0 = n_valid(c.item.row0, col), nv1 = W == 2 ? n_valid(c.item.row0, col + 1) : nv0;
      const int64_t e0 = row_base(c.item.v) + (c.item.row0 + row_t) * cols + col;
      const float *pg = a.g + e0;
      const float *pr = a.r ? a.r + e0 : nullptr;
      unsigned char *dst = sm + s * kStage + off0;
      const uint32_t sdst = stage(s) + off0;
#pragma unroll
      for (int u = 0; u < LM::U; ++u) {
        const uint32_t o = LM::kRowBytes * u;
        if (u < nv1) {   // every element of the row is data
          LM::copy(sdst + kOffG + o, pg);
          if (pr) LM::copy(sdst + kOffC + o, pr);
        } else if (u < nv0) {   // W = 2 in the partly filled row: the first column only
          cp_async4(sdst + kOffG + o, pg);
          *reinterpret_cast<float *>(dst + kOffG + o + 4) = 0.0f;
          if (pr) cp_async4(sdst + kOffC + o, pr);
          *reinterpret_cast<float *>(dst + kOffC + o + 4) = 0.0f;
        } else {
#pragma unroll
          for (int e = 0; e < W; ++e) {
            *reinterpret_cast<float *>(dst + kOffG + o + 4 * e) = 0.0f;
            *reinterpret_cast<float *>(dst + kOffC + o + 4 * e) = 0.0f;
          }
        }
        pg += rstride;
        if (pr) pr += rstride;
      }
      if (bulk_small && tid == 0) {   // the chunk's 32 rows of Q and Q_w_prev: TMA bulk copies
        const int64_t col0 = (c.item.c_begin + c.lk) * kKc;
        const uint32_t bytes = static_cast<uint32_t>(min(static_cast<int64_t>(kKc), cols - col0) * R * 4);
        const uint32_t bar = small_bar(s);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes * (DEF ? 2u : 1u))
                     : "memory");
        bulk_g2s(stage(s) + SH::kOffQ, a.q + (static_cast<int64_t>(c.item.v / a.L) * cols + col0) * R, bytes, bar);
        if (DEF) bulk_g2s(stage(s) + SH::kOffW, a.ef_qw + (static_cast<int64_t>(c.item.v) * cols + col0) * R, bytes, bar);
      }
    };
    // the small operands of a chunk, fetched into registers one chunk ahead (a thread reads only
    // what it copied or loaded itself): Q_w_prev rows of its columns (deferred EF) and, for the
    // B builders (tid < 8 R), 4 columns of Q's rank row n
    constexpr bool kPre = R * W <= 8;
    float qv_nx[W][R], tq_nx[4];
    auto fetch_small = [&](const ChunkIt &c) {
      const int64_t col0 = (c.item.c_begin + c.lk) * kKc;
      if (DEF) {
#pragma unroll
        for (int e = 0; e < W; ++e)
#pragma unroll
          for (int b = 0; b < R; ++b)
            qv_nx[e][b] = col0 + col_t + e < cols
                              ? __ldg(a.ef_qw + (static_cast<int64_t>(c.item.v) * cols + col0 + col_t + e) * R + b)
                              : 0.0f;
      }
      if (tid < R * 8) {
        const int n = tid >> 3, ch = tid & 7;
        const float *qt = a.q + static_cast<int64_t>(c.item.v / a.L) * cols * R;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t cj = col0 + 4 * ch + e;
          tq_nx[e] = cj < cols ? __ldg(qt + cj * R + n) : 0.0f;
        }
      }
    };
    double acc64[R];
#pragma unroll
    for (int b = 0; b < R; ++b) acc64[b] = 0.0;
    auto fold_group = [&](int64_t gi) {   // warps 0..3: TMEM lane = row of the band
      mbar_wait(acc_bar(static_cast<int>(gi & 1)), static_cast<uint32_t>((gi >> 1) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t taddr = tmem + (static_cast<uint32_t>(warp * 32) << 16) + static_cast<uint32_t>((gi & 1) * N);
#pragma unroll
      for (int part = 0; part < N / 16; ++part) {
        uint32_t x[16];
        tmem_ld16(taddr + 16 * part, x);
#pragma unroll
        for (int j = 0; j < 16; ++j) {   // column 16 part + j is rank (16 part + j) mod H
          const int b = (16 * part + j) % H;
          if (b < R) acc64[b] += static_cast<double>(__uint_as_float(x[j]));
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    };

    ChunkIt cc, cf;   // copy stream (kAhead ahead), form stream
    cc.start(a);
    cf.start(a);
    RingPos rc{0, 0}, rf{0, 0};
    int64_t kc = 0;   // chunks copied so far
    for (int p = 0; p < SH::kAhead; ++p) {
      if (cc.valid(a)) {
        copy_chunk(cc, rc.idx);
        cc.next(a);
        rc.step(kStages);
        ++kc;
      }
      cp_async_commit();
    }
    if (kPre && !bulk_small && cf.valid(a)) fetch_small(cf);
    int64_t groups = 0, folded = 0;
    for (; cf.valid(a); cf.next(a), rf.step(kStages)) {
      const Item &it = cf.item;
      if (cf.lk == 0) {   // new item: its band's P_hat_prev rows (all producers are past the last item)
        producers_sync();
        if (DEF) {
          const float *pht = a.ef_ph + static_cast<int64_t>(it.v / a.L) * rows * R;
          for (int e = tid; e < kM * R; e += kProducers) {
            const int64_t i = it.row0 + e / R;
            ph_s[e] = i < rows ? pht[i * R + e % R] : 0.0f;
          }
        }
        producers_sync();
      }
      // keep kAhead chunks of copies in flight: the stage of chunk kc held chunk kc - kStages
      if (cc.valid(a)) {
        if (kc >= kStages) mbar_wait(empty_bar(rc.idx), rc.phase ^ 1u);
        copy_chunk(cc, rc.idx);
        cc.next(a);
        rc.step(kStages);
        ++kc;
      }
      cp_async_commit();
      cp_async_wait<SH::kAhead>();   // this thread's copies of the chunk to form have landed
      unsigned char *st = sm + rf.idx * kStage;
      float qv[W][R], tq[4];
      if (bulk_small) {
        mbar_wait(small_bar(rf.idx), rf.phase);
        const float *wraw = reinterpret_cast<const float *>(st + SH::kOffW);
        const float *qraw = reinterpret_cast<const float *>(st + SH::kOffQ);
        if (DEF) {   // only columns < cols are used (the rows past them are stale)
#pragma unroll
          for (int e = 0; e < W; ++e)
#pragma unroll
            for (int b = 0; b < R; ++b) qv[e][b] = wraw[(col_t + e) * R + b];
        }
        if (tid < R * 8) {
          const int n = tid >> 3, ch = tid & 7;
#pragma unroll
          for (int e = 0; e < 4; ++e)
            tq[e] = (it.c_begin + cf.lk) * kKc + 4 * ch + e < cols ? qraw[(4 * ch + e) * R + n] : 0.0f;
        }
      } else {
        if (!kPre) fetch_small(cf);
#pragma unroll
        for (int e = 0; e < W; ++e)
#pragma unroll
          for (int b = 0; b < R; ++b) qv[e][b] = qv_nx[e][b];
#pragma unroll
        for (int e = 0; e < 4; ++e) tq[e] = tq_nx[e];
        if (kPre) {
          ChunkIt nx = cf;
          nx.next(a);
          if (nx.valid(a)) fetch_small(nx);
        }
      }
      const int64_t col0 = (it.c_begin + cf.lk) * kKc;
      const int64_t col = col0 + col_t;
      const int t = it.v / a.L;
      const int nv0 = n_valid(it.row0, col), nv1 = W == 2 ? n_valid(it.row0, col + 1) : nv0;
      float *pr = a.r ? a.r + row_base(it.v) + (it.row0 + row_t) * cols + col : nullptr;
      unsigned char *sg = st + kOffG + off0, *sc = st + kOffC + off0;
#pragma unroll
      for (int u = 0; u < LM::U; ++u) {
        const uint32_t o = LM::kRowBytes * u;
        float gv[W], rv[W], c[W];
        LM::lds(sg + o, gv);
        LM::lds(sc + o, rv);
#pragma unroll
        for (int e = 0; e < W; ++e) {
          c[e] = gv[e];
          if (pr && u < (e == 0 ? nv0 : nv1)) {
            if (DEF) rv[e] = rv[e] - own_of<R>(ph_s + (row_t + LM::kRowStep * u) * R, qv[e]);
            c[e] = gv[e] + rv[e];
          }
        }
        if (pr) {
          if (u < nv1) LM::stg(pr, c);
          else if (u < nv0) pr[0] = c[0];
          pr += rstride;
        }
        float hs[W];
#pragma unroll
        for (int e = 0; e < W; ++e) {
          float hb;
          split3(c[e], hb, hs[e]);
        }
        LM::sts(sc + o, c);    // A_big (truncated by the MMA)
        LM::sts(sg + o, hs);   // A_small over the consumed g
      }
      if (tid < R * 8) {   // B = [Q_big^T ; Q_small^T] of the chunk: row n (< R), 4 columns per thread
        const int n = tid >> 3, ch = tid & 7;
        const float (&tv)[4] = tq;
        float4 hb, hs;
        split3(tv[0], hb.x, hs.x);
        split3(tv[1], hb.y, hs.y);
        split3(tv[2], hb.z, hs.z);
        split3(tv[3], hb.w, hs.w);
        *reinterpret_cast<float4 *>(st + kOffB + sw128(n, ch)) = hb;
        *reinterpret_cast<float4 *>(st + kOffB + sw128(H + n, ch)) = hs;
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(full_bar(rf.idx));
      if (warp < 4) {
        if (cf.lk % kGroup == kFoldLag && cf.lk >= kGroup) {
          fold_group(groups + cf.lk / kGroup - 1);
          folded = groups + cf.lk / kGroup;
        }
        if (cf.lk == it.nloc - 1) {   // item done: remaining groups, then the band's partials
          const int64_t ng = groups + (it.nloc + kGroup - 1) / kGroup;
          for (int64_t g = folded; g < ng; ++g) fold_group(g);
          const int64_t grow = it.row0 + warp * 32 + lane;
          if (grow < rows) {
#pragma unroll
            for (int b = 0; b < R; ++b)
              a.partial[((static_cast<int64_t>(it.v) * a.splits + it.split) * rows + grow) * R + b] = acc64[b];
          }
#pragma unroll
          for (int b = 0; b < R; ++b) acc64[b] = 0.0;
          groups = folded = ng;
        }
      } else if (cf.lk == it.nloc - 1) {
        groups += (it.nloc + kGroup - 1) / kGroup;
        folded = groups;
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

// ------------------------------------------------------------------ Q_w = M_w^T P_hat (pipelines.py:354)
// for batches of tensors and row pitches TMA cannot describe: the CUDA-core column slabs of
// gc_psgd_tma.cu's mtp_tma_kernel (a CTA owns 32 columns and a range of rows; thread = float4 column
// group x row group; 4 columns x R products per row in fp32, folded into fp64 per 128-row box,
// the 32 row groups reduced in order) fed by cp.async: every thread copies exactly the elements it
// reads -- 16-byte cp.async.cg (no L1 allocation) when its rows are 16-byte aligned, else 8- or
// 4-byte copies -- so a per-thread cp.async.wait_group is the only synchronisation.  The width is
// picked per (tensor, worker) row at run time from its offset.  Elements past d (the partly filled
// last row) or past the matrix copy as zeros.  Ranks 1..4.
constexpr int kMtaThreads = 256;
constexpr int kMtaAhead = 3;
constexpr int kMtaStages = kMtaAhead + 1;
constexpr int kMtaStage = kM * kKc * 4;   // 16 KB: 128 rows x 32 columns, row-major

template <int R>
__global__ void __launch_bounds__(kMtaThreads) mtp_async_kernel(int64_t d, int64_t rows, int64_t cols, const float *c,
                                                                const int64_t *row_offs, int64_t ld, int L,
                                                                const float *ph, int64_t rows_per_split,
                                                                double *partial, int splits) {
  static_assert(R <= 4, "rank <= 4");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ double red[kMtaThreads / 8][32][R];
  const int tid = threadIdx.x;
  const int v = blockIdx.z, split = blockIdx.y;
  const int64_t col0 = static_cast<int64_t>(blockIdx.x) * kKc;
  const int64_t r_begin = split * rows_per_split;
  const int64_t r_end = min(rows, r_begin + rows_per_split);
  const int64_t nbox = r_end > r_begin ? (r_end - r_begin + kM - 1) / kM : 0;
  const int g4 = tid & 7, rg = tid >> 3;   // float4 column group, row group (rows rg + 32 k)
  const int64_t rb = row_offs ? row_offs[v] : static_cast<int64_t>(v) * ld;
  const float *cw = c + rb;
  const float *pht = ph + static_cast<int64_t>(v / L) * rows * R;
  const int64_t col = col0 + 4 * g4;
  const int ncol = static_cast<int>(max(static_cast<int64_t>(0), min(static_cast<int64_t>(4), cols - col)));
  // copy width from the alignment of this row's elements (uniform over the CTA)
  const uintptr_t base_addr = reinterpret_cast<uintptr_t>(cw);
  const int width = (cols % 4 == 0 && base_addr % 16 == 0) ? 4 : ((cols % 2 == 0 && base_addr % 8 == 0) ? 2 : 1);
  const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(smem_raw));
  auto copy_box = [&](int64_t bx, int s) {
    const int64_t i0 = r_begin + bx * kM;
#pragma unroll
    for (int k = 0; k < kM / 32; ++k) {
      const int row = rg + 32 * k;
      const int64_t grow = i0 + row;
      const int64_t e = grow * cols + col;
      const uint32_t dst = sbase + s * kMtaStage + row * 128 + g4 * 16;
      // elements of this float4 that are data: columns < cols, index < d, row < r_end
      const int64_t left = grow < r_end ? min(static_cast<int64_t>(ncol), d - e) : 0;
      if (left == 4 && width == 4) {
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(cw + e) : "memory");
      } else if (left == 4 && width == 2) {
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(cw + e) : "memory");
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst + 8), "l"(cw + e + 2) : "memory");
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          if (t < left)
            cp_async4(dst + 4 * t, cw + e + t);
          else
            *reinterpret_cast<float *>(smem_raw + s * kMtaStage + row * 128 + g4 * 16 + 4 * t) = 0.0f;
        }
      }
    }
  };
  double acc64[4][R];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) acc64[t][b] = 0.0;
  for (int p = 0; p < kMtaAhead; ++p) {
    if (p < nbox) copy_box(p, p);
    cp_async_commit();
  }
  for (int64_t bx = 0; bx < nbox; ++bx) {
    const int s = static_cast<int>(bx % kMtaStages);
    if (bx + kMtaAhead < nbox) copy_box(bx + kMtaAhead, static_cast<int>((bx + kMtaAhead) % kMtaStages));
    cp_async_commit();
    cp_async_wait<kMtaAhead>();   // this thread's elements of box bx have landed
    const int64_t i0 = r_begin + bx * kM;
    float acc[4][R];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int b = 0; b < R; ++b) acc[t][b] = 0.0f;
#pragma unroll
    for (int k = 0; k < kM / 32; ++k) {
      const int row = rg + 32 * k;
      const float4 m = *reinterpret_cast<const float4 *>(smem_raw + s * kMtaStage + row * 128 + g4 * 16);
      float p[R];
#pragma unroll
      for (int b = 0; b < R; ++b) p[b] = i0 + row < r_end ? __ldg(pht + (i0 + row) * R + b) : 0.0f;
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
  }
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) red[rg][4 * g4 + t][b] = acc64[t][b];
  __syncthreads();
  for (int e = tid; e < 32 * R; e += kMtaThreads) {
    const int cc = e / R, b = e - cc * R;
    double x = 0.0;
#pragma unroll 8
    for (int w = 0; w < kMtaThreads / 8; ++w) x += red[w][cc][b];
    if (col0 + cc < cols) partial[((static_cast<int64_t>(v) * splits + split) * cols + col0 + cc) * R + b] = x;
  }
}

}  // namespace

int gc_psgd_mq_async_supported_impl(int32_t rank, const void *grads, const void *resid) {
  if ((reinterpret_cast<uintptr_t>(grads) | reinterpret_cast<uintptr_t>(resid)) & 3) return 0;
  switch (rank) {
    case 1: case 2: case 3: case 4: case 5: case 6: case 7: case 8: case 16: return 1;
    default: return 0;
  }
}

// fp64 split-K partials partial[v][split][row][R] of P = M Q for V = T * L virtual rows (deferred
// EF when ef_ph / ef_qw are given); returns the split count (<= max_splits) or a negative status.
int gc_psgd_mq_async_launch(int32_t T, int32_t L, const int64_t *row_offsets, const int64_t *host_tensor_offsets,
                            int64_t ld, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                            float *resid, const float *q, const float *ef_ph, const float *ef_qw, double *partial,
                            int64_t max_splits, cudaStream_t st) {
  // 8-byte copies when every row start is 8-byte aligned (GPT-2's cols % 4 == 2 matrices)
  bool w8 = cols % 2 == 0 && ((reinterpret_cast<uintptr_t>(grads) | reinterpret_cast<uintptr_t>(resid)) & 7) == 0 &&
            (L == 1 || ld % 2 == 0) && (row_offsets == nullptr || host_tensor_offsets != nullptr);
  if (w8 && row_offsets != nullptr)
    for (int t = 0; t < T; ++t) w8 = w8 && host_tensor_offsets[t] % 2 == 0;
  if (const char *e = getenv("GC_PSGD_ASYNC_W")) w8 = w8 && atoi(e) != 1;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  AsyncArgs a{};
  a.d = d;
  a.rows = rows;
  a.cols = cols;
  a.rows_full = d / cols;
  a.tail_cols = d - a.rows_full * cols;
  a.g = grads;
  a.r = resid;
  a.row_offs = row_offsets;
  a.ld = ld;
  a.L = L;
  a.q = q;
  a.ef_ph = ef_ph;
  a.ef_qw = ef_qw;
  a.partial = partial;
  const int64_t V = static_cast<int64_t>(T) * L;
  a.row_blocks = static_cast<int>((rows + kM - 1) / kM);
  a.nchunks = (cols + kKc - 1) / kKc;
  // split the columns until there are a few items per SM (the ring runs across item boundaries)
  int64_t splits = 1;
  while (splits < max_splits && a.row_blocks * V * splits < 4 * sms && (a.nchunks + splits) / (splits + 1) >= 8)
    ++splits;
  const int64_t per = (a.nchunks + splits - 1) / splits;
  splits = (a.nchunks + per - 1) / per;
  a.splits = static_cast<int>(splits);
  a.chunks_per_split = per;
  a.items = a.row_blocks * V * splits;
  const unsigned grid = static_cast<unsigned>(std::min<int64_t>(a.items, sms));
#define GC_MQA_GO(RR, DD, WW)                                                                          \
  cudaFuncSetAttribute(mq_async_kernel<RR, DD, WW>, cudaFuncAttributeMaxDynamicSharedMemorySize,         \
                       Shape<RR>::kSmem);                                                                 \
  mq_async_kernel<RR, DD, WW><<<grid, kThreads, Shape<RR>::kSmem, st>>>(a);
#define GC_MQA(RR)                    \
  case RR:                            \
    if (ef_ph && w8) {                \
      GC_MQA_GO(RR, true, 2)          \
    } else if (ef_ph) {               \
      GC_MQA_GO(RR, true, 1)          \
    } else if (w8) {                  \
      GC_MQA_GO(RR, false, 2)         \
    } else {                          \
      GC_MQA_GO(RR, false, 1)         \
    }                                 \
    break;
  switch (rank) {
    GC_MQA(1) GC_MQA(2) GC_MQA(3) GC_MQA(4) GC_MQA(5) GC_MQA(6) GC_MQA(7) GC_MQA(8) GC_MQA(16)
    default:
      gc_set_error("rank must be 1..8 or 16");
      return GC_ERR_UNSUPPORTED;
  }
#undef GC_MQA
#undef GC_MQA_GO
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gc_set_error(std::string("mq_async_kernel: ") + cudaGetErrorString(e));
    return GC_ERR_CUDA;
  }
  return static_cast<int>(splits);
}

// fp64 split-K partials partial[v][split][col][R] of Q_w = M_w^T P_hat for V = T * L virtual rows
// (rank <= 4, any layout); returns the split count (<= max_splits) or a negative status.
int gc_psgd_mtp_async_launch(int32_t V, int32_t L, const int64_t *row_offsets, int64_t ld, int64_t d, int64_t rows,
                             int64_t cols, int32_t rank, const float *c, const float *p_hat, double *partial,
                             int64_t max_splits, cudaStream_t st) {
  const int64_t slabs = (cols + kKc - 1) / kKc;
  const int64_t boxes = (rows + kM - 1) / kM;
  int64_t splits = (4 * 148 + slabs * V - 1) / (slabs * V);
  if (splits > max_splits) splits = max_splits;
  if (splits > boxes) splits = boxes;
  if (splits < 1) splits = 1;
  const int64_t per = (boxes + splits - 1) / splits;
  splits = (boxes + per - 1) / per;
  const dim3 grid(static_cast<unsigned>(slabs), static_cast<unsigned>(splits), static_cast<unsigned>(V));
  const int smem = kMtaStages * kMtaStage;
#define GC_MTA(RR)                                                                                      \
  case RR:                                                                                              \
    cudaFuncSetAttribute(mtp_async_kernel<RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);      \
    mtp_async_kernel<RR><<<grid, kMtaThreads, smem, st>>>(d, rows, cols, c, row_offsets, ld, L, p_hat, per * kM, \
                                                          partial, static_cast<int>(splits));           \
    break;
  switch (rank) {
    GC_MTA(1) GC_MTA(2) GC_MTA(3) GC_MTA(4)
    default:
      gc_set_error("rank must be 1..4");
      return GC_ERR_UNSUPPORTED;
  }
#undef GC_MTA
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    gc_set_error(std::string("mtp_async_kernel: ") + cudaGetErrorString(e));
    return GC_ERR_CUDA;
  }
  return static_cast<int>(splits);
}
