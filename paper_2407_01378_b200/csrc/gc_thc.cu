// THC (rotated stochastic quantization with saturation) -- generic kernels.
//
// These are the building blocks used by the distributed pipeline (ranks exchange
// ranges and codes between them) and by the parity path.  They cover every
// rotation block size the reference accepts (RotatedQuantConfig, compressors.py:79-97):
//   * B <= 4096: one CTA per 4096-coordinate tile, all butterfly stages in shared memory;
//   * B  > 4096: fp64 scratch in HBM, stages 0-11 in a tile pass, then strided passes of
//     up to 8 stages, then an elementwise epilogue.
// The single-GPU fused round (all workers of a block in one CTA) lives in gc_thc_fused.cu.
//
// Bit-exactness: the WHT runs in fp64 with stages in bit-0-first
// order (transforms.py:92-98); the file is compiled with -fmad=false so no product is
// contracted into an FMA; divisions are IEEE.
#include <cuda_runtime.h>

#include "gc_device.cuh"
#include "gc_internal.h"

namespace {

constexpr int kTile = 4096;   // coordinates per shared-memory tile
constexpr int kLogTile = 12;
constexpr int kNT = 256;      // threads per CTA
constexpr int kMaxWorkers = 64;

enum Mode { kFwd = 0, kEst = 1, kEf = 2 };

struct ThcArgs {
  int64_t dim, active, nb;
  int block, log_block, q, mode, workers, addends;
  double scale;
  const float *grads;       // [L][ld] (kFwd, kEf)
  const float *resid;       // [L][ld] (kFwd: r_old; may be null)
  float *resid_out;         // [L][ld] (kEf)
  int64_t ld;
  const uint32_t *bits;     // sign bitmask
  float *x_rot;             // [L][active] (kFwd, optional)
  float *ranges;            // [L][nb][2]   (kFwd)
  unsigned int *ranges_enc; // [L][nb][2] ordered-uint scratch (global path, kFwd)
  const float *shared;      // [nb][2] consensus ranges (kEst, kEf)
  const void *sums;         // kEst: summed codes
  int sum_bytes;
  const int8_t *codes;      // kEf: [L][active]
  float *est;               // kEst: [dim]
  double *ws;               // [L][active] fp64 scratch (global path)
};

struct CoinStreams {
  gc_pcg64 s[kMaxWorkers];
};

__device__ __forceinline__ int64_t load_sum(const void *p, int bytes, int64_t i) {
  if (bytes == 1) return static_cast<const int8_t *>(p)[i];
  if (bytes == 2) return static_cast<const int16_t *>(p)[i];
  return static_cast<const int32_t *>(p)[i];
}

// dequantize_sum (compressors.py:501-521) for one coordinate, returned as the fp64
// value rht_inverse starts from (the f32 result widened again, transforms.py:124).
__device__ __forceinline__ double dequant(const float *shared, int64_t blk, int q, int addends, int64_t z) {
  const double lo = static_cast<double>(shared[2 * blk]);
  const double hi = static_cast<double>(shared[2 * blk + 1]);
  const double mid = (lo + hi) / 2.0;
  const double step = hi > lo ? (hi - lo) / static_cast<double>((1 << q) - 2) : 0.0;
  const float f = static_cast<float>(static_cast<double>(addends) * mid + step * static_cast<double>(z));
  return static_cast<double>(f);
}

// Prologue: value entering the butterflies for coordinate i of worker w.
__device__ __forceinline__ double prologue(const ThcArgs &a, int w, int64_t i) {
  if (a.mode == kFwd) {
    float c = 0.0f;
    if (i < a.dim) {
      c = a.grads[w * a.ld + i];
      if (a.resid) c = c + a.resid[w * a.ld + i];   // ef_apply, compressors.py:626
    }
    const double v = static_cast<double>(c);
    return gc::sign_positive(a.bits, i) ? v : -v;   // values * signs (transforms.py:115)
  }
  const int64_t blk = i >> a.log_block;
  if (a.mode == kEst) return dequant(a.shared, blk, a.q, a.addends, load_sum(a.sums, a.sum_bytes, i));
  return dequant(a.shared, blk, a.q, 1, a.codes[w * a.active + i]);
}

// Epilogue for the inverse modes (transforms.py:124-126, pipelines.py:308-318, 168-170).
__device__ __forceinline__ void inverse_epilogue(const ThcArgs &a, int w, int64_t i, double v) {
  if (i >= a.dim) return;
  const double sg = gc::sign_positive(a.bits, i) ? 1.0 : -1.0;
  const float f = static_cast<float>((v * a.scale) * sg);
  if (a.mode == kEst) {
    a.est[i] = f / static_cast<float>(a.addends);
  } else {
    float c = a.grads[w * a.ld + i];
    c = c + a.resid_out[w * a.ld + i];
    a.resid_out[w * a.ld + i] = c - f;
  }
}

// ---------------------------------------------------------------- B <= 4096
__global__ void __launch_bounds__(kNT) wht_local_kernel(ThcArgs a) {
  __shared__ double buf[kTile];
  __shared__ float fbuf[kTile];
  const int w = blockIdx.y;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  const int count = static_cast<int>(min(static_cast<int64_t>(kTile), a.active - base));
  for (int e = threadIdx.x; e < count; e += kNT) buf[e] = prologue(a, w, base + e);
  __syncthreads();
  for (int s = 0; s < a.log_block; ++s) gc::wht_stage_smem<kNT>(buf, count, s);

  if (a.mode != kFwd) {
    for (int e = threadIdx.x; e < count; e += kNT) inverse_epilogue(a, w, base + e, buf[e]);
    return;
  }
  float *xr = a.x_rot ? a.x_rot + w * a.active : nullptr;
  for (int e = threadIdx.x; e < count; e += kNT) {
    const float f = static_cast<float>(buf[e] * a.scale);   // transforms.py:116-117
    fbuf[e] = f;
    if (xr) xr[base + e] = f;
  }
  __syncthreads();
  // chunk_ranges (compressors.py:447-453): one warp per rotation block.
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nblk = count >> a.log_block;
  for (int b = warp; b < nblk; b += kNT / 32) {
    float lo = INFINITY, hi = -INFINITY;
    for (int e = lane; e < a.block; e += 32) {
      const float f = fbuf[(b << a.log_block) + e];
      lo = fminf(lo, f);
      hi = fmaxf(hi, f);
    }
    for (int o = 16; o; o >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      const int64_t gb = (base >> a.log_block) + b;
      a.ranges[(w * a.nb + gb) * 2] = lo;
      a.ranges[(w * a.nb + gb) * 2 + 1] = hi;
    }
  }
}

// ---------------------------------------------------------------- B > 4096
// Pass 1: prologue + stages 0..11 per 4096 tile -> fp64 scratch.
__global__ void __launch_bounds__(kNT) wht_first_pass(ThcArgs a) {
  __shared__ double buf[kTile];
  const int w = blockIdx.y;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  for (int e = threadIdx.x; e < kTile; e += kNT) buf[e] = prologue(a, w, base + e);
  __syncthreads();
  for (int s = 0; s < kLogTile; ++s) gc::wht_stage_smem<kNT>(buf, kTile, s);
  double *out = a.ws + w * a.active + base;
  for (int e = threadIdx.x; e < kTile; e += kNT) out[e] = buf[e];
}

// Strided pass: stages s0 .. s0+nst-1 (nst <= 8).  A CTA owns 16 contiguous low
// indices x 2^nst positions along the stage axis: i = hi*2^(s0+nst) + m*2^s0 + lo.
__global__ void __launch_bounds__(kNT) wht_strided_pass(double *ws, int64_t active, int s0, int nst) {
  __shared__ double buf[kTile];
  const int w = blockIdx.y;
  const int64_t lo_chunks = (int64_t{1} << s0) / 16;
  const int64_t hi = blockIdx.x / lo_chunks;
  const int64_t lo0 = (blockIdx.x % lo_chunks) * 16;
  const int span = 1 << nst;
  const int count = 16 * span;
  double *base = ws + w * active + hi * (int64_t{1} << (s0 + nst)) + lo0;
  for (int e = threadIdx.x; e < count; e += kNT) {
    const int m = e >> 4, l = e & 15;
    buf[e] = base[(static_cast<int64_t>(m) << s0) + l];
  }
  __syncthreads();
  for (int k = 0; k < nst; ++k) {
    const int half = 1 << k;
    for (int p = threadIdx.x; p < count / 2; p += kNT) {
      const int l = p & 15, pm = p >> 4;
      const int m = ((pm >> k) << (k + 1)) | (pm & (half - 1));
      const double x = buf[(m << 4) | l];
      const double y = buf[((m + half) << 4) | l];
      buf[(m << 4) | l] = x + y;
      buf[((m + half) << 4) | l] = x - y;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < count; e += kNT) {
    const int m = e >> 4, l = e & 15;
    base[(static_cast<int64_t>(m) << s0) + l] = buf[e];
  }
}

__global__ void init_ranges_enc(unsigned int *enc, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    enc[i] = (i & 1) ? gc::float_to_ordered(-INFINITY) : gc::float_to_ordered(INFINITY);
}

__global__ void __launch_bounds__(kNT) wht_final_pass(ThcArgs a) {
  const int w = blockIdx.y;
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kTile;
  const double *src = a.ws + w * a.active + base;
  if (a.mode != kFwd) {
    for (int e = threadIdx.x; e < kTile; e += kNT) inverse_epilogue(a, w, base + e, src[e]);
    return;
  }
  // A 4096 tile lies inside one rotation block (B > 4096).
  float lo = INFINITY, hi = -INFINITY;
  for (int e = threadIdx.x; e < kTile; e += kNT) {
    const float f = static_cast<float>(src[e] * a.scale);
    if (a.x_rot) a.x_rot[w * a.active + base + e] = f;
    lo = fminf(lo, f);
    hi = fmaxf(hi, f);
  }
  for (int o = 16; o; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    const int64_t gb = base >> a.log_block;
    atomicMin(&a.ranges_enc[(w * a.nb + gb) * 2], gc::float_to_ordered(lo));
    atomicMax(&a.ranges_enc[(w * a.nb + gb) * 2 + 1], gc::float_to_ordered(hi));
  }
}

__global__ void decode_ranges_enc(const unsigned int *enc, float *ranges, int64_t count) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < count;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    ranges[i] = gc::ordered_to_float(enc[i]);
}

int grid_for(int64_t work, int per_cta) {
  int64_t g = (work + per_cta - 1) / per_cta;
  if (g > 148 * 32) g = 148 * 32;
  return static_cast<int>(g < 1 ? 1 : g);
}

// Run the blockwise WHT for all L workers with the configured prologue/epilogue.
int run_wht(ThcArgs a, cudaStream_t st, void *workspace) {
  const int64_t tiles = (a.active + kTile - 1) / kTile;
  const int L = a.workers;
  if (a.block <= kTile) {
    wht_local_kernel<<<dim3(static_cast<unsigned>(tiles), L), kNT, 0, st>>>(a);
    GC_LAUNCH_CHECK("wht_local_kernel");
    return GC_OK;
  }
  if (!workspace) {
    gc_set_error("rotation block > 4096 needs a workspace (gc_thc_workspace_bytes)");
    return GC_ERR_INVALID;
  }
  a.ws = static_cast<double *>(workspace);
  a.ranges_enc = reinterpret_cast<unsigned int *>(a.ws + static_cast<int64_t>(L) * a.active);
  wht_first_pass<<<dim3(static_cast<unsigned>(tiles), L), kNT, 0, st>>>(a);
  GC_LAUNCH_CHECK("wht_first_pass");
  for (int s0 = kLogTile; s0 < a.log_block; s0 += 8) {
    const int nst = min(8, a.log_block - s0);
    const int64_t ctas = a.active / (16 * (int64_t{1} << nst));
    wht_strided_pass<<<dim3(static_cast<unsigned>(ctas), L), kNT, 0, st>>>(a.ws, a.active, s0, nst);
    GC_LAUNCH_CHECK("wht_strided_pass");
  }
  if (a.mode == kFwd) {
    const int64_t cnt = static_cast<int64_t>(L) * a.nb * 2;
    init_ranges_enc<<<grid_for(cnt, 256), 256, 0, st>>>(a.ranges_enc, cnt);
    GC_LAUNCH_CHECK("init_ranges_enc");
  }
  wht_final_pass<<<dim3(static_cast<unsigned>(tiles), L), kNT, 0, st>>>(a);
  GC_LAUNCH_CHECK("wht_final_pass");
  if (a.mode == kFwd) {
    const int64_t cnt = static_cast<int64_t>(L) * a.nb * 2;
    decode_ranges_enc<<<grid_for(cnt, 256), 256, 0, st>>>(a.ranges_enc, a.ranges, cnt);
    GC_LAUNCH_CHECK("decode_ranges_enc");
  }
  return GC_OK;
}

// ---------------------------------------------------------------- quantize
constexpr int kRun = 16;  // consecutive coordinates per thread (one PCG jump per run)

__global__ void __launch_bounds__(kNT) quantize_kernel(int64_t active, int log_block, int q, int workers,
                                                       const float *x_rot, const float *shared,
                                                       CoinStreams streams, int8_t *codes,
                                                       unsigned long long *counters) {
  const double bound = static_cast<double>((1 << (q - 1)) - 1);
  const int64_t runs_w = (active + kRun - 1) / kRun;
  const int64_t total = runs_w * workers;
  long long clamped = 0, sz = 0, sz2 = 0;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; r < total;
       r += static_cast<int64_t>(gridDim.x) * kNT) {
    const int w = static_cast<int>(r / runs_w);
    const int64_t i0 = (r % runs_w) * kRun;
    gc::Pcg g;
    g.load(streams.s[w]);
    g.jump(static_cast<uint64_t>(i0));
    for (int k = 0; k < kRun; ++k) {
      const int64_t i = i0 + k;
      if (i >= active) break;
      const uint64_t u = g.next();
      const int64_t blk = i >> log_block;
      // quantize_stochastic, compressors.py:473-498 (all fp64, no contraction)
      const double v = static_cast<double>(x_rot[w * active + i]);
      const double lo = static_cast<double>(shared[2 * blk]);
      const double hi = static_cast<double>(shared[2 * blk + 1]);
      const double m1 = v > lo ? v : lo;                 // np.clip = min(max(x, lo), hi)
      const double cl = m1 < hi ? m1 : hi;
      clamped += (cl != v);
      const double mid = (lo + hi) / 2.0;
      const double step = (hi - lo) / static_cast<double>((1 << q) - 2);
      const bool degenerate = step <= 0.0;
      const double safe = degenerate ? 1.0 : step;
      double t = (cl - mid) / safe;
      t = t > -bound ? t : -bound;
      t = t < bound ? t : bound;
      double low = floor(t);
      double frac = t - low;
      if (frac > 1.0 - 1e-9) low += 1.0;
      if (frac < 1e-9 || frac > 1.0 - 1e-9) frac = 0.0;
      const double coin = gc::coin_from(u);
      long long z = static_cast<long long>(low + (coin < frac ? 1.0 : 0.0));
      const long long b = static_cast<long long>(bound);
      z = z < -b ? -b : (z > b ? b : z);
      if (degenerate) z = 0;
      codes[w * active + i] = static_cast<int8_t>(z);
      sz += z;
      sz2 += z * z;
    }
  }
  for (int o = 16; o; o >>= 1) {
    clamped += __shfl_xor_sync(0xffffffffu, clamped, o);
    sz += __shfl_xor_sync(0xffffffffu, sz, o);
    sz2 += __shfl_xor_sync(0xffffffffu, sz2, o);
  }
  if ((threadIdx.x & 31) == 0 && counters) {
    atomicAdd(&counters[0], static_cast<unsigned long long>(clamped));
    atomicAdd(&counters[1], static_cast<unsigned long long>(sz));
    atomicAdd(&counters[2], static_cast<unsigned long long>(sz2));
  }
}

// ---------------------------------------------------------------- saturating fold
template <typename T>
__global__ void __launch_bounds__(kNT) sat_fold_kernel(int n, int64_t len, const int8_t *codes, int64_t ld,
                                                       int64_t offset, int64_t ring_block, int bits, T *out,
                                                       unsigned long long *clips) {
  const long long hi = (1ll << (bits - 1)) - 1;
  long long nclip = 0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(kNT) + threadIdx.x; e < len;
       e += static_cast<int64_t>(gridDim.x) * kNT) {
    const int s = static_cast<int>((offset + e) / ring_block);   // block j starts at worker j
    long long acc = codes[s * ld + e];
    int w = s;
    for (int k = 1; k < n; ++k) {
      w = (w + 1 == n) ? 0 : w + 1;
      acc += codes[w * ld + e];
      if (acc > hi) { acc = hi; ++nclip; }
      else if (acc < -hi) { acc = -hi; ++nclip; }
    }
    out[e] = static_cast<T>(acc);
  }
  for (int o = 16; o; o >>= 1) nclip += __shfl_xor_sync(0xffffffffu, nclip, o);
  if ((threadIdx.x & 31) == 0 && clips) atomicAdd(clips, static_cast<unsigned long long>(nclip));
}

__global__ void range_consensus_kernel(int L, int64_t nb, const float *in, float *out) {
  for (int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; b < nb;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float lo = in[2 * b], hi = in[2 * b + 1];
    for (int w = 1; w < L; ++w) {
      lo = fminf(lo, in[(w * nb + b) * 2]);
      hi = fmaxf(hi, in[(w * nb + b) * 2 + 1]);
    }
    out[2 * b] = lo;
    out[2 * b + 1] = hi;
  }
}

// words per thread: one PCG jump amortised over 8..64 words (128..1024 steps), as many as keeps
// ~2 threads per core busy (small vectors need the threads more than the amortisation)
inline int sign_words_per_thread(int64_t words) {
  int64_t w = words / (148 * 2048);
  return static_cast<int>(w < 8 ? 8 : (w > 64 ? 64 : w));
}

__global__ void signs_kernel(gc_pcg64 stream, int64_t count, uint32_t *bits, int wpt) {
  // Sign i = top bit of u32 word i; u32 words are the low then high half of each next64 output
  // (numpy buffered bounded uint32, Lemire with range 2).  Thread t writes words
  // [t*8, t*8 + 8): 128 consecutive outputs after one jump.
  const int64_t words = (count + 31) / 32;
  const int64_t groups = (words + wpt - 1) / wpt;
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < groups;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    gc::Pcg g;
    g.load(stream);
    g.jump(static_cast<uint64_t>(t) * wpt * 16);
    const int64_t w0 = t * wpt;
    const int nw = static_cast<int>(min(static_cast<int64_t>(wpt), words - w0));
#pragma unroll 2
    for (int k = 0; k < nw; ++k) {
      uint32_t word = 0;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint64_t u = g.next();
        word |= static_cast<uint32_t>((u >> 31) & 1u) << (2 * j);
        word |= static_cast<uint32_t>((u >> 63) & 1u) << (2 * j + 1);
      }
      bits[w0 + k] = word;
    }
  }
}

int check_geom(const gc_thc_geom *g) {
  GC_REQUIRE(g != nullptr, "geometry is null");
  GC_REQUIRE(g->dim >= 1, "dim must be positive");
  GC_REQUIRE(g->padded >= g->dim && (g->padded & (g->padded - 1)) == 0, "padded must be a power of two >= dim");
  GC_REQUIRE(g->block >= 1 && (g->block & (g->block - 1)) == 0 && g->block <= g->padded,
             "block must be a power of two <= padded");
  GC_REQUIRE(g->quant_bits >= 2 && g->quant_bits <= 8, "quant_bits must be in [2, 8]");
  GC_REQUIRE(g->wire_bits >= g->quant_bits && g->wire_bits <= 32, "wire_bits must be in [quant_bits, 32]");
  return GC_OK;
}

int log2_exact(int64_t x) {
  int l = 0;
  while ((int64_t{1} << l) < x) ++l;
  return l;
}

ThcArgs base_args(const gc_thc_geom *g, int mode, int workers) {
  ThcArgs a{};
  a.dim = g->dim;
  a.block = static_cast<int>(g->block);
  a.log_block = log2_exact(g->block);
  a.nb = (g->dim + g->block - 1) / g->block;
  a.active = a.nb * g->block;
  a.q = g->quant_bits;
  a.scale = g->scale;
  a.mode = mode;
  a.workers = workers;
  a.addends = 1;
  return a;
}

// Nibble wire for b <= 4: codes and saturated sums lie in [-7, 7], two per byte (element 2i in
// the low nibble, 2i + 1 in the high one; unpacking sign-extends).
__global__ void pack_nibbles_kernel(int64_t pairs, const int8_t *in, uint8_t *out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < pairs;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<uint8_t>((static_cast<uint8_t>(in[2 * i]) & 0xFu) | (static_cast<uint8_t>(in[2 * i + 1]) << 4));
}

__global__ void unpack_nibbles_kernel(int64_t pairs, const uint8_t *in, int8_t *out) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < pairs;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int v = in[i];
    out[2 * i] = static_cast<int8_t>(static_cast<int8_t>(v << 4) >> 4);
    out[2 * i + 1] = static_cast<int8_t>(static_cast<int8_t>(v) >> 4);
  }
}

int nibble_grid(int64_t pairs) {
  const int64_t g = (pairs + 255) / 256;
  return static_cast<int>(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

}  // namespace

extern "C" {

int gc_pack_nibbles(int64_t len, const int8_t *codes, uint8_t *packed, void *stream) {
  GC_REQUIRE(len >= 0 && len % 2 == 0 && (len == 0 || (codes && packed)), "need an even length and buffers");
  if (len == 0) return GC_OK;
  pack_nibbles_kernel<<<nibble_grid(len / 2), 256, 0, static_cast<cudaStream_t>(stream)>>>(len / 2, codes, packed);
  GC_LAUNCH_CHECK("pack_nibbles_kernel");
  return GC_OK;
}

int gc_unpack_nibbles(int64_t len, const uint8_t *packed, int8_t *codes, void *stream) {
  GC_REQUIRE(len >= 0 && len % 2 == 0 && (len == 0 || (codes && packed)), "need an even length and buffers");
  if (len == 0) return GC_OK;
  unpack_nibbles_kernel<<<nibble_grid(len / 2), 256, 0, static_cast<cudaStream_t>(stream)>>>(len / 2, packed, codes);
  GC_LAUNCH_CHECK("unpack_nibbles_kernel");
  return GC_OK;
}

int64_t gc_thc_active_len(const gc_thc_geom *g) {
  if (!g || g->block < 1) return 0;
  return ((g->dim + g->block - 1) / g->block) * g->block;
}

int64_t gc_thc_workspace_bytes(const gc_thc_geom *g, int32_t workers) {
  if (!g || g->block <= kTile) return 0;
  const int64_t active = gc_thc_active_len(g);
  const int64_t nb = active / g->block;
  return static_cast<int64_t>(workers) * active * 8 + static_cast<int64_t>(workers) * nb * 2 * 4;
}

int gc_thc_signs(const gc_pcg64 *rotation_stream, int64_t count, uint32_t *bits, void *stream) {
  GC_REQUIRE(rotation_stream && bits, "null argument");
  GC_REQUIRE(count >= 0, "count must be non-negative");
  if (count == 0) return GC_OK;
  const int64_t words = (count + 31) / 32;
  const int wpt = sign_words_per_thread(words);
  const int64_t groups = (words + wpt - 1) / wpt;
  signs_kernel<<<grid_for(groups, 128), 128, 0, static_cast<cudaStream_t>(stream)>>>(*rotation_stream, count, bits,
                                                                                       wpt);
  GC_LAUNCH_CHECK("signs_kernel");
  return GC_OK;
}

int gc_thc_rotate(const gc_thc_geom *g, int32_t workers, const float *grads, const float *resid, int64_t ld,
                  const uint32_t *sign_bits, float *x_rot, float *ranges, void *workspace, void *stream) {
  if (int rc = check_geom(g)) return rc;
  GC_REQUIRE(workers >= 1 && workers <= 65535, "workers out of range");
  GC_REQUIRE(grads && sign_bits && ranges, "null argument");
  GC_REQUIRE(ld >= g->dim, "ld must be >= dim");
  ThcArgs a = base_args(g, kFwd, workers);
  a.grads = grads;
  a.resid = resid;
  a.ld = ld;
  a.bits = sign_bits;
  a.x_rot = x_rot;
  a.ranges = ranges;
  return run_wht(a, static_cast<cudaStream_t>(stream), workspace);
}

int gc_range_consensus(int32_t workers, int64_t num_blocks, const float *ranges_in, float *ranges_out,
                       void *stream) {
  GC_REQUIRE(workers >= 1 && num_blocks >= 0 && ranges_in && ranges_out, "invalid argument");
  if (num_blocks == 0) return GC_OK;
  range_consensus_kernel<<<grid_for(num_blocks, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      workers, num_blocks, ranges_in, ranges_out);
  GC_LAUNCH_CHECK("range_consensus_kernel");
  return GC_OK;
}

int gc_thc_quantize(const gc_thc_geom *g, int32_t workers, const float *x_rot, const float *shared_ranges,
                    const gc_pcg64 *coin_streams, int8_t *codes, int64_t *counters, void *stream) {
  if (int rc = check_geom(g)) return rc;
  GC_REQUIRE(workers >= 1 && workers <= kMaxWorkers, "workers must be in [1, 64]");
  GC_REQUIRE(x_rot && shared_ranges && coin_streams && codes, "null argument");
  CoinStreams cs{};
  for (int w = 0; w < workers; ++w) cs.s[w] = coin_streams[w];
  const int64_t active = gc_thc_active_len(g);
  const int64_t runs = (active + kRun - 1) / kRun * workers;
  quantize_kernel<<<grid_for(runs, kNT), kNT, 0, static_cast<cudaStream_t>(stream)>>>(
      active, log2_exact(g->block), g->quant_bits, workers, x_rot, shared_ranges, cs, codes,
      reinterpret_cast<unsigned long long *>(counters));
  GC_LAUNCH_CHECK("quantize_kernel");
  return GC_OK;
}

int gc_sat_fold(int32_t n, int64_t len, const int8_t *codes, int64_t ld, int64_t offset, int64_t ring_block,
                int32_t bits, void *sums, int64_t *clip_counter, void *stream) {
  GC_REQUIRE(n >= 1 && len >= 0 && codes && sums, "invalid argument");
  GC_REQUIRE(bits >= 2 && bits <= 32, "bits must be in [2, 32]");
  GC_REQUIRE(ring_block >= 1 && ld >= len, "invalid ring block / leading dimension");
  if (len == 0) return GC_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  auto *clips = reinterpret_cast<unsigned long long *>(clip_counter);
  const int grid = grid_for(len, kNT);
  if (bits <= 8)
    sat_fold_kernel<int8_t><<<grid, kNT, 0, st>>>(n, len, codes, ld, offset, ring_block, bits,
                                                  static_cast<int8_t *>(sums), clips);
  else if (bits <= 16)
    sat_fold_kernel<int16_t><<<grid, kNT, 0, st>>>(n, len, codes, ld, offset, ring_block, bits,
                                                   static_cast<int16_t *>(sums), clips);
  else
    sat_fold_kernel<int32_t><<<grid, kNT, 0, st>>>(n, len, codes, ld, offset, ring_block, bits,
                                                   static_cast<int32_t *>(sums), clips);
  GC_LAUNCH_CHECK("sat_fold_kernel");
  return GC_OK;
}

int gc_thc_decode_estimate(const gc_thc_geom *g, int32_t n, const void *sums, int32_t sum_bytes,
                           const float *shared_ranges, const uint32_t *sign_bits, float *estimate,
                           void *workspace, void *stream) {
  if (int rc = check_geom(g)) return rc;
  GC_REQUIRE(n >= 1, "n must be positive");
  GC_REQUIRE(sum_bytes == 1 || sum_bytes == 2 || sum_bytes == 4, "sum_bytes must be 1, 2 or 4");
  GC_REQUIRE(sums && shared_ranges && sign_bits && estimate, "null argument");
  ThcArgs a = base_args(g, kEst, 1);
  a.addends = n;
  a.sums = sums;
  a.sum_bytes = sum_bytes;
  a.shared = shared_ranges;
  a.bits = sign_bits;
  a.est = estimate;
  return run_wht(a, static_cast<cudaStream_t>(stream), workspace);
}

int gc_thc_decode_ef(const gc_thc_geom *g, int32_t workers, const int8_t *codes, const float *shared_ranges,
                     const uint32_t *sign_bits, const float *grads, float *resid, int64_t ld, void *workspace,
                     void *stream) {
  if (int rc = check_geom(g)) return rc;
  if (!resid) return GC_OK;
  GC_REQUIRE(workers >= 1 && workers <= 65535, "workers out of range");
  GC_REQUIRE(codes && shared_ranges && sign_bits && grads, "null argument");
  GC_REQUIRE(ld >= g->dim, "ld must be >= dim");
  ThcArgs a = base_args(g, kEf, workers);
  a.codes = codes;
  a.shared = shared_ranges;
  a.bits = sign_bits;
  a.grads = grads;
  a.resid_out = resid;
  a.ld = ld;
  return run_wht(a, static_cast<cudaStream_t>(stream), workspace);
}

}  // extern "C"
