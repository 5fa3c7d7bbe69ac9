// PowerSGD (rank-r factorisation with error feedback) on B200.
//
// Reference: _round_powersgd (pipelines.py:324-368) with matrix_shape_for / to_matrix
// (compressors.py:530-548), orthonormalize (compressors.py:555-588), warm start (:366).
// M_w = corrected_w zero-padded to rows x cols (row-major); P_w = M_w Q; P_hat =
// orthonormalize(sum_w P_w); Q_w = M_w^T P_hat; own_w = P_hat Q_w^T; estimate =
// P_hat (sum_w Q_w)^T / n; warm Q = sum_w Q_w / n.
//
// B200 design: with r = 4 both products are matrix-vector-like (about 1 flop per byte), so
// they are HBM-bound streams over M, not tensor-core work.  Each is one pass over M with
// fp64 accumulation (more accurate than the reference's fp32 BLAS; results agree to
// ~1e-7 relative):
//   * mq:  a CTA owns a band of 64 rows, stages Q in 1024-column chunks in shared memory
//          (Q is read from L2 once per band), a warp accumulates 8 rows x r in registers;
//   * mtp: a CTA owns 1024 columns x a row range (thread = 4 columns, coalesced row reads,
//          the P_hat rows broadcast from shared memory); row ranges are reduced in a fixed order;
//   * decode: a CTA owns 1024 columns x 64 rows and writes r_new = c - own for every worker
//          and the estimate in one pass.
// mtp and decode use float4 accesses when cols % 4 == 0 and rows are 16-byte aligned, and the
// same kernels with coalesced scalar accesses otherwise (e.g. GPT-2's 1774 x 1774 matrices).
// MGS runs in one CTA in fp64 (column-by-column projections, block reductions), including
// the reference's canonical-basis completion of degenerate columns.
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <string>

#include "gc_device.cuh"
#include "gc_internal.h"

namespace {

constexpr int kMaxRank = 16;

int grid_cap(int64_t g) { return static_cast<int>(g < 1 ? 1 : (g > 65535 ? 65535 : g)); }

// Batched layout: virtual row v = t * n_per + w (tensor t, worker w).  Row v of M starts at
// offs[v] (a tensor's slice of the flat gradient) or v * ld when offs is NULL; per-tensor
// factors are strided by tensor.  The single-matrix path is n_per = L, one tensor.
struct Rows {
  const int64_t *offs;
  int64_t ld;
  int n_per;
  __device__ __forceinline__ int64_t at(int v) const { return offs ? offs[v] : static_cast<int64_t>(v) * ld; }
  __device__ __forceinline__ int tensor(int v) const { return v / n_per; }
};

// ------------------------------------------------------------------ P = M Q
template <int R>
struct MqShape {
  static constexpr int kRowsPerWarp = R <= 4 ? 8 : 32 / R;   // register budget: rows x R doubles
  static constexpr int kRowsPerCta = 8 * kRowsPerWarp;
  static constexpr int kChunk = 4096 / R;                     // 16 KB of Q per stage
};

template <int R>
__global__ void __launch_bounds__(256) mq_kernel(int64_t d, int64_t rows, int64_t cols, const float *c, Rows rw_,
                                                 const float *q, float *p) {
  constexpr int kRowsPerWarp = MqShape<R>::kRowsPerWarp, kChunk = MqShape<R>::kChunk;
  __shared__ float qs[kChunk * R];
  const int w = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t row0 = static_cast<int64_t>(blockIdx.x) * MqShape<R>::kRowsPerCta + warp * kRowsPerWarp;
  const float *cw = c + rw_.at(w);
  q += static_cast<int64_t>(rw_.tensor(w)) * cols * R;
  double acc[kRowsPerWarp][R];
#pragma unroll
  for (int a = 0; a < kRowsPerWarp; ++a)
#pragma unroll
    for (int b = 0; b < R; ++b) acc[a][b] = 0.0;
  for (int64_t j0 = 0; j0 < cols; j0 += kChunk) {
    const int nj = static_cast<int>(min(static_cast<int64_t>(kChunk), cols - j0));
    __syncthreads();
    for (int e = threadIdx.x; e < nj * R; e += 256) qs[e] = q[j0 * R + e];
    __syncthreads();
    for (int jj = lane; jj < nj; jj += 32) {
      float qv[R];
#pragma unroll
      for (int b = 0; b < R; ++b) qv[b] = qs[jj * R + b];
#pragma unroll
      for (int a = 0; a < kRowsPerWarp; ++a) {
        const int64_t i = (row0 + a) * cols + j0 + jj;   // flat index into the padded matrix
        const double m = (row0 + a < rows && i < d) ? static_cast<double>(cw[i]) : 0.0;
#pragma unroll
        for (int b = 0; b < R; ++b) acc[a][b] += m * static_cast<double>(qv[b]);
      }
    }
  }
#pragma unroll
  for (int a = 0; a < kRowsPerWarp; ++a)
#pragma unroll
    for (int b = 0; b < R; ++b) {
      double v = acc[a][b];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && row0 + a < rows) p[(w * rows + row0 + a) * R + b] = static_cast<float>(v);
    }
}

// ------------------------------------------------------------------ Q = M^T P_hat
// partial[w][s][col][R] over row range s; then reduced in order s = 0, 1, ...

__global__ void mtp_reduce_kernel(int L, int splits, int64_t cols, int R, const double *partial, float *q) {
  const int64_t total = static_cast<int64_t>(L) * cols * R;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = e / (cols * R), rest = e - w * cols * R;
    double v = 0.0;
    for (int s = 0; s < splits; ++s) v += partial[(w * splits + s) * cols * R + rest];
    q[e] = static_cast<float>(v);
  }
}

// ------------------------------------------------------------------ MGS (compressors.py:555-588)
__device__ double block_sum(double v, double *red) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

// a: [rows][R] fp64 workspace (row-major, like the reference's (rows, r) array).
__global__ void __launch_bounds__(1024) mgs_kernel(int64_t rows, int R, const float *in, double *a, float *out,
                                                   int *status) {
  __shared__ double red[33];
  {   // one CTA per tensor of the batch
    const int64_t t = blockIdx.x;
    in += t * rows * R;
    a += t * rows * R;
    out += t * rows * R;
    status += t;
  }
  double fro = 0.0;
  for (int64_t i = threadIdx.x; i < rows * R; i += blockDim.x) {
    const double v = static_cast<double>(in[i]);
    a[i] = v;
    fro += v * v;
  }
  fro = block_sum(fro, red);
  const double scale = sqrt(fro) / fmax(1.0, sqrt(static_cast<double>(R)));
  const double floor_ = fmax(scale * 1e-8, 1e-300);
  for (int c = 0; c < R; ++c) {
    for (int p = 0; p < c; ++p) {   // col -= (a_p . col) a_p, modified Gram-Schmidt
      double dot = 0.0;
      for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) dot += a[i * R + p] * a[i * R + c];
      dot = block_sum(dot, red);
      for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) a[i * R + c] -= dot * a[i * R + p];
      __syncthreads();
    }
    double nn = 0.0;
    for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) nn += a[i * R + c] * a[i * R + c];
    const double norm = sqrt(block_sum(nn, red));
    if (norm > floor_) {
      for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) a[i * R + c] /= norm;
      __syncthreads();
      continue;
    }
    // canonical completion: first e_basis whose residual after projection has norm > 0.5
    bool done = false;
    for (int64_t basis = 0; basis < rows && !done; ++basis) {
      // cand = e_basis, then cand -= (a_p . cand) a_p for p < c (recomputed after each step)
      double cn = 0.0;
      for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) a[i * R + c] = (i == basis) ? 1.0 : 0.0;
      __syncthreads();
      for (int p = 0; p < c; ++p) {
        double dot = 0.0;
        for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) dot += a[i * R + p] * a[i * R + c];
        dot = block_sum(dot, red);
        for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) a[i * R + c] -= dot * a[i * R + p];
        __syncthreads();
      }
      for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) cn += a[i * R + c] * a[i * R + c];
      const double cnorm = sqrt(block_sum(cn, red));
      if (cnorm > 0.5) {
        for (int64_t i = threadIdx.x; i < rows; i += blockDim.x) a[i * R + c] /= cnorm;
        done = true;
      }
      __syncthreads();
    }
    if (!done && threadIdx.x == 0) *status = 1;   // DegenerateMatrixError
    __syncthreads();
  }
  for (int64_t i = threadIdx.x; i < rows * R; i += blockDim.x) out[i] = static_cast<float>(a[i]);
}


// Orthonormalization for any rank <= kMaxOrthRank (compressors.py:555-588), one CTA per tensor
// (the dot-product buffers are dynamic shared memory, (kOrthThreads / 32 + 1) x R doubles).
// Column c is projected against all previous columns with classical Gram-Schmidt applied twice
// (CGS2: as stable as the reference's MGS; both give the Q factor of the same nested column
// spaces, agreeing to O(cond * eps) in fp64 -- far inside the 1e-5 contract).  The c dot products
// of a pass are formed together: a thread accumulates 8 of them over its rows, each warp reduces
// them with shuffles and the warps' partials are summed in a fixed order (deterministic), so a
// column costs 2 x (ceil(c / 8) + 1) row sweeps and 3 block reductions instead of MGS's c + 1
// sequential block reductions -- the difference that matters at r = 64.  A column
// whose residual norm is at or below 1e-8 * scale takes the reference's canonical-basis
// completion (the sequential path of mgs_kernel); none left -> status = 1 (DegenerateMatrixError).
constexpr int kMaxOrthRank = 1024;   // 9 x 1024 doubles = 72 KB of dynamic shared memory
constexpr int kOrthThreads = 256;

__device__ void orth_dots(int64_t rows, int R, const double *a, int c, double *dots, double *wred) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int p0 = 0; p0 < c; p0 += 8) {
    double part[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int64_t i = threadIdx.x; i < rows; i += kOrthThreads) {
      const double x = a[i * R + c];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        if (p0 + k < c) part[k] += a[i * R + p0 + k] * x;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double v = part[k];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && p0 + k < c) wred[warp * R + p0 + k] = v;
    }
  }
  __syncthreads();
  for (int p = threadIdx.x; p < c; p += kOrthThreads) {
    double v = 0.0;
    for (int w = 0; w < kOrthThreads / 32; ++w) v += wred[w * R + p];
    dots[p] = v;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kOrthThreads) orth_kernel(int64_t rows, int R, const float *in, double *a,
                                                            float *out, int *status, const int *fast) {
  __shared__ double red[33];
  extern __shared__ double orth_smem[];
  double *dots = orth_smem;        // [R]
  double *wred = orth_smem + R;    // [kOrthThreads / 32][R]
  if (fast && fast[blockIdx.x]) return;   // the Cholesky path already wrote this tensor's P_hat
  {
    const int64_t t = blockIdx.x;
    in += t * rows * R;
    a += t * rows * R;
    out += t * rows * R;
    status += t;
  }
  double fro = 0.0;
  for (int64_t i = threadIdx.x; i < rows * R; i += kOrthThreads) {
    const double v = static_cast<double>(in[i]);
    a[i] = v;
    fro += v * v;
  }
  fro = block_sum(fro, red);
  const double scale = sqrt(fro) / fmax(1.0, sqrt(static_cast<double>(R)));
  const double floor_ = fmax(scale * 1e-8, 1e-300);
  for (int c = 0; c < R; ++c) {
    for (int pass = 0; pass < 2 && c > 0; ++pass) {
      orth_dots(rows, R, a, c, dots, wred);
      for (int64_t i = threadIdx.x; i < rows; i += kOrthThreads) {
        double x = a[i * R + c];
        for (int p = 0; p < c; ++p) x -= dots[p] * a[i * R + p];
        a[i * R + c] = x;
      }
      __syncthreads();
    }
    double nn = 0.0;
    for (int64_t i = threadIdx.x; i < rows; i += kOrthThreads) nn += a[i * R + c] * a[i * R + c];
    const double norm = sqrt(block_sum(nn, red));
    if (norm > floor_) {
      for (int64_t i = threadIdx.x; i < rows; i += kOrthThreads) a[i * R + c] /= norm;
      __syncthreads();
      continue;
    }
    bool done = false;   // canonical completion, as mgs_kernel
    for (int64_t basis = 0; basis < rows && !done; ++basis) {
      for (int64_t i = threadIdx.x; i < rows; i += kOrthThreads) a[i * R + c] = (i == basis) ? 1.0 : 0.0;
      __syncthreads();
      for (int p = 0; p < c; ++p) {
        double dot = 0.0;
        for (int64_t i = threadIdx.x; i < rows; i += kOrthThreads) dot += a[i * R + p] * a[i * R + c];
        dot = block_sum(dot, red);
        for (int64_t i = threadIdx.x; i < rows; i += kOrthThreads) a[i * R + c] -= dot * a[i * R + p];
        __syncthreads();
      }
      double cn = 0.0;
      for (int64_t i = threadIdx.x; i < rows; i += kOrthThreads) cn += a[i * R + c] * a[i * R + c];
      const double cnorm = sqrt(block_sum(cn, red));
      if (cnorm > 0.5) {
        for (int64_t i = threadIdx.x; i < rows; i += kOrthThreads) a[i * R + c] /= cnorm;
        done = true;
      }
      __syncthreads();
    }
    if (!done && threadIdx.x == 0) *status = 1;
    __syncthreads();
  }
  for (int64_t i = threadIdx.x; i < rows * R; i += kOrthThreads) out[i] = static_cast<float>(a[i]);
}

// Fast path of the orthonormalization for tall factors (rank <= 16).  In exact arithmetic the
// reference's MGS (compressors.py:555-588) produces the Q factor of P = Q R with a positive
// diagonal, and R is the Cholesky factor of the Gram matrix G = P^T P; column c's residual norm
// after projection is R[c][c].  So: (A) G in fp64 from row slices spread over the GPU, (B) per
// tensor the slices summed in a fixed order, R = chol(G) and R^-1, (C) P_hat = P R^-1 row by row.
// (B) takes the fast path only when every pivot is far from the reference's degeneracy floor
// (R[c][c] > 1e3 * floor) and from cancellation (R[c][c] > 1e-4 * |p_c|, so the fp64 result is
// within ~1e-8 of MGS's); otherwise the tensor's flag stays 0 and orth_kernel (CGS2 with the
// canonical completion) runs it.  One pass over P instead of 2 r + 2 single-CTA sweeps.
constexpr int kOrthSlicesMax = 148;

template <int R>
__global__ void __launch_bounds__(256) tall_gram_kernel(int64_t rows, const float *p, double *partial, int slices) {
  constexpr int NP = R * (R + 1) / 2;
  __shared__ double red[8][NP];
  const int t = blockIdx.y, sl = blockIdx.x;
  p += static_cast<int64_t>(t) * rows * R;
  double acc[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) acc[k] = 0.0;
  for (int64_t i = static_cast<int64_t>(sl) * 256 + threadIdx.x; i < rows; i += static_cast<int64_t>(slices) * 256) {
    double x[R];
#pragma unroll
    for (int a = 0; a < R; ++a) x[a] = static_cast<double>(p[i * R + a]);
    int k = 0;
#pragma unroll
    for (int a = 0; a < R; ++a)
#pragma unroll
      for (int b = a; b < R; ++b) acc[k++] += x[a] * x[b];
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < NP; k += 256) {
    double v = 0.0;
    for (int w = 0; w < 8; ++w) v += red[w][k];
    partial[(static_cast<int64_t>(t) * slices + sl) * NP + k] = v;
  }
}

// one thread per tensor: G from the slices (fixed order), Cholesky, pivot checks, R^-1
__global__ void orth_chol_kernel(int T, int R, int slices, const double *partial, double *rinv, int *fast) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const int NP = R * (R + 1) / 2;
  double g[16][16], r[16][16], ri[16][16];
  for (int a = 0, k = 0; a < R; ++a)
    for (int b = a; b < R; ++b, ++k) {
      double v = 0.0;
      for (int sl = 0; sl < slices; ++sl) v += partial[(static_cast<int64_t>(t) * slices + sl) * NP + k];
      g[a][b] = v;
      g[b][a] = v;
    }
  double fro2 = 0.0;
  for (int a = 0; a < R; ++a) fro2 += g[a][a];
  const double scale = sqrt(fro2) / fmax(1.0, sqrt(static_cast<double>(R)));
  const double floor_ = fmax(scale * 1e-8, 1e-300);
  bool ok = true;
  for (int c = 0; c < R && ok; ++c) {
    for (int p = 0; p < c; ++p) {
      double v = g[p][c];
      for (int k = 0; k < p; ++k) v -= r[k][p] * r[k][c];
      r[p][c] = v / r[p][p];
    }
    double dd = g[c][c];
    for (int k = 0; k < c; ++k) dd -= r[k][c] * r[k][c];
    if (!(dd > 0.0)) {
      ok = false;
      break;
    }
    r[c][c] = sqrt(dd);
    if (!(r[c][c] > 1e3 * floor_) || !(r[c][c] > 1e-4 * sqrt(g[c][c]))) ok = false;
  }
  if (ok) {   // upper-triangular inverse, column by column
    for (int b = 0; b < R; ++b) {
      for (int a = R - 1; a >= 0; --a) {
        double v = a == b ? 1.0 : 0.0;
        for (int k = a + 1; k <= b; ++k) v -= r[a][k] * ri[k][b];
        ri[a][b] = a <= b ? v / r[a][a] : 0.0;
      }
    }
    for (int a = 0; a < R; ++a)
      for (int b = 0; b < R; ++b) rinv[(static_cast<int64_t>(t) * R + a) * R + b] = a <= b ? ri[a][b] : 0.0;
  }
  fast[t] = ok ? 1 : 0;
}

template <int R>
__global__ void __launch_bounds__(256) orth_apply_kernel(int64_t rows, const float *p, const double *rinv,
                                                         const int *fast, float *out) {
  const int t = blockIdx.y;
  if (!fast[t]) return;
  __shared__ double ri[R * R];
  for (int e = threadIdx.x; e < R * R; e += 256) ri[e] = rinv[static_cast<int64_t>(t) * R * R + e];
  __syncthreads();
  p += static_cast<int64_t>(t) * rows * R;
  out += static_cast<int64_t>(t) * rows * R;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x; i < rows;
       i += static_cast<int64_t>(gridDim.x) * 256) {
    double x[R];
#pragma unroll
    for (int a = 0; a < R; ++a) x[a] = static_cast<double>(p[i * R + a]);
#pragma unroll
    for (int b = 0; b < R; ++b) {
      double y = 0.0;
#pragma unroll
      for (int a = 0; a <= b; ++a) y += x[a] * ri[a * R + b];
      out[i * R + b] = static_cast<float>(y);
    }
  }
}

// ------------------------------------------------------------------ vectorised kernels
// Used when cols % 4 == 0 and the buffers are 16-byte aligned (cfg4: 18709 x 18708).
//
// P = M Q fused with ef_apply.  Column-slab split-K: a CTA owns 1024 columns (a thread 4
// columns with its Q rows in registers) x a chunk of kMqRows rows; per row the corrected
// values f32(g + r) are formed from float4 loads, written over r (EF on) and dotted with Q;
// warp shuffles + a shared-memory pass give the CTA's partial P[row] for its slab, written
// to partial[w][slab][row][R] and reduced over slabs in a fixed order (deterministic).
constexpr int kMqRows = 32;

template <int R>
__global__ void __launch_bounds__(256) mq_fused_kernel(int64_t d, int64_t rows, int64_t cols, const float *g,
                                                       float *r, Rows rw_, const float *q, double *partial,
                                                       int slabs) {
  __shared__ double red[kMqRows][8][R];
  const int w = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slab = blockIdx.x;
  const int64_t col = (static_cast<int64_t>(slab) * 256 + threadIdx.x) * 4;
  const int64_t row0 = static_cast<int64_t>(blockIdx.y) * kMqRows;
  const float *gw = g + rw_.at(w);
  float *rw = r ? r + rw_.at(w) : nullptr;
  q += static_cast<int64_t>(rw_.tensor(w)) * cols * R;
  float qv[4][R];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) qv[t][b] = col + t < cols ? q[(col + t) * R + b] : 0.0f;
  const int nrows = static_cast<int>(min(static_cast<int64_t>(kMqRows), rows - row0));
#pragma unroll 4
  for (int a = 0; a < nrows; ++a) {
    const int64_t i = (row0 + a) * cols + col;
    float c4[4] = {0.f, 0.f, 0.f, 0.f};
    if (col < cols) {
      if (i + 3 < d) {
        float4 c = __ldcs(reinterpret_cast<const float4 *>(gw + i));
        if (rw) {
          const float4 rv = __ldcs(reinterpret_cast<const float4 *>(rw + i));
          c.x = c.x + rv.x; c.y = c.y + rv.y; c.z = c.z + rv.z; c.w = c.w + rv.w;
          *reinterpret_cast<float4 *>(rw + i) = c;   // corrected kept in r for the later passes
        }
        c4[0] = c.x; c4[1] = c.y; c4[2] = c.z; c4[3] = c.w;
      } else {
        for (int t = 0; t < 4; ++t)
          if (i + t < d) {
            float v = gw[i + t];
            if (rw) {
              v = v + rw[i + t];
              rw[i + t] = v;
            }
            c4[t] = v;
          }
      }
    }
#pragma unroll
    for (int b = 0; b < R; ++b) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < 4; ++t) v += static_cast<double>(c4[t]) * static_cast<double>(qv[t][b]);
#pragma unroll
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0) red[a][warp][b] = v;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nrows * R; e += 256) {
    const int a = e / R, b = e - a * R;
    double v = 0.0;
    for (int k = 0; k < 8; ++k) v += red[a][k][b];
    partial[((static_cast<int64_t>(w) * slabs + slab) * rows + row0 + a) * R + b] = v;
  }
}

__global__ void mq_reduce_kernel(int L, int slabs, int64_t rows, int R, const double *partial, float *p) {
  const int64_t total = static_cast<int64_t>(L) * rows * R;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t w = e / (rows * R), rest = e - w * rows * R;
    double v = 0.0;
    for (int s = 0; s < slabs; ++s) v += partial[(w * slabs + s) * rows * R + rest];
    p[e] = static_cast<float>(v);
  }
}

// Q = M^T P_hat: a thread owns 4 consecutive columns (a CTA 1024) and streams the rows of its
// split.  Products accumulate in fp32 FMAs over 32-row groups that are folded into fp64
// registers (per element: one float4 lane and 4 FFMA -- no fp32->fp64 conversions, which run
// at a quarter of the FMA rate and capped the fp64 version at ~40% of HBM); the P_hat rows are
// broadcast from shared memory as float4.  Accuracy: 32 fp32 terms per group, fp64 across
// groups (~1e-7 relative, the reference itself is fp32 BLAS).
constexpr int kMtpFold = 32;

// A thread's 4 columns of one row.  A16 (cols % 4 == 0, 16-byte aligned rows): 4 consecutive
// columns as one float4.  Otherwise columns base + 256k (k = 0..3), so every scalar access of a
// warp covers 32 consecutive columns (coalesced); vm bit k = column k exists.
template <bool A16>
__device__ __forceinline__ int64_t col_off(int k) { return A16 ? k : 256 * k; }
template <bool A16>
__device__ __forceinline__ float4 ldc(const float *p, unsigned vm) {
  if (A16) return __ldcs(reinterpret_cast<const float4 *>(p));
  return make_float4(vm & 1u ? __ldcs(p) : 0.0f, vm & 2u ? __ldcs(p + 256) : 0.0f, vm & 4u ? __ldcs(p + 512) : 0.0f,
                     vm & 8u ? __ldcs(p + 768) : 0.0f);
}
template <bool A16>
__device__ __forceinline__ void stc(float *p, float4 v, unsigned vm) {
  if (A16) {
    __stcs(reinterpret_cast<float4 *>(p), v);
    return;
  }
  if (vm & 1u) __stcs(p, v.x);
  if (vm & 2u) __stcs(p + 256, v.y);
  if (vm & 4u) __stcs(p + 512, v.z);
  if (vm & 8u) __stcs(p + 768, v.w);
}
// the thread's first column, its valid-column mask and the offset of its last valid column
template <bool A16>
__device__ __forceinline__ int64_t thread_cols(int64_t cols, unsigned &vm, int64_t &last) {
  const int64_t col = A16 ? (static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x) * 4
                          : static_cast<int64_t>(blockIdx.x) * 1024 + threadIdx.x;
  vm = 0;
  last = 0;
#pragma unroll
  for (int k = 0; k < 4; ++k)
    if (col + col_off<A16>(k) < cols) vm |= 1u << k, last = col_off<A16>(k);
  return col;
}

template <int R, bool A16>
__global__ void __launch_bounds__(256) mtp_vec_kernel(int64_t d, int64_t rows, int64_t cols, const float *c,
                                                      Rows rw_, const float *ph, int64_t rows_per_split,
                                                      double *partial, int splits) {
  constexpr int kChunk = R <= 8 ? 512 : 256;
  constexpr int RP = R <= 4 ? 4 : (R <= 8 ? 8 : 16);   // P_hat rows padded for float4 reads
  __shared__ __align__(16) float ps[kChunk * RP];
  const int w = blockIdx.z;
  const int s = blockIdx.y;
  unsigned vm;
  int64_t lastoff;
  const int64_t col = thread_cols<A16>(cols, vm, lastoff);
  const int64_t r0 = s * rows_per_split;
  const int64_t r1 = min(rows, r0 + rows_per_split);
  const float *cw = c + rw_.at(w);
  ph += static_cast<int64_t>(rw_.tensor(w)) * rows * R;
  double acc[4][R];
  float a32[4][R];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) acc[t][b] = 0.0, a32[t][b] = 0.0f;
  for (int64_t i0 = r0; i0 < r1; i0 += kChunk) {
    const int ni = static_cast<int>(min(static_cast<int64_t>(kChunk), r1 - i0));
    __syncthreads();
    for (int e = threadIdx.x; e < ni * RP; e += 256) {
      const int ii = e / RP, b = e - ii * RP;
      ps[e] = b < R ? ph[(i0 + ii) * R + b] : 0.0f;
    }
    __syncthreads();
    if (vm) {
      // rows whose columns all lie below d load without per-row checks, so the unrolled loads
      // of a fold group are all in flight together (a per-row branch serialised them)
      const bool full = (i0 + ni - 1) * cols + col + lastoff < d;
      for (int g0 = 0; g0 < ni; g0 += kMtpFold) {
        const int g1 = min(ni, g0 + kMtpFold);
        auto row_fma = [&](int ii, const float4 m) {
          const float m4[4] = {m.x, m.y, m.z, m.w};
          float pv[RP];
#pragma unroll
          for (int b4 = 0; b4 < RP; b4 += 4) {
            const float4 p4 = *reinterpret_cast<const float4 *>(ps + ii * RP + b4);
            pv[b4] = p4.x; pv[b4 + 1] = p4.y; pv[b4 + 2] = p4.z; pv[b4 + 3] = p4.w;
          }
#pragma unroll
          for (int t = 0; t < 4; ++t)
#pragma unroll
            for (int b = 0; b < R; ++b) a32[t][b] = fmaf(m4[t], pv[b], a32[t][b]);
        };
        if (full && g1 - g0 == kMtpFold) {
          // branch-free group: all kMtpFold row loads are independent and issue back to back
          const float *src = cw + (i0 + g0) * cols + col;
#pragma unroll 8
          for (int ii = 0; ii < kMtpFold; ++ii)
            row_fma(g0 + ii, ldc<A16>(src + ii * cols, vm));
        } else {
          for (int ii = g0; ii < g1; ++ii) {
            const int64_t i = (i0 + ii) * cols + col;
            float4 m;
            if (i + lastoff < d) {
              m = ldc<A16>(cw + i, vm);
            } else {
              float t4[4] = {0.f, 0.f, 0.f, 0.f};
              for (int t = 0; t < 4; ++t)
                if (((vm >> t) & 1u) && i + col_off<A16>(t) < d) t4[t] = cw[i + col_off<A16>(t)];
              m = make_float4(t4[0], t4[1], t4[2], t4[3]);
            }
            row_fma(ii, m);
          }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int b = 0; b < R; ++b) {
            acc[t][b] += static_cast<double>(a32[t][b]);
            a32[t][b] = 0.0f;
          }
      }
    }
  }
#pragma unroll
  for (int t = 0; t < 4; ++t)
    if ((vm >> t) & 1u) {
#pragma unroll
      for (int b = 0; b < R; ++b)
        partial[((static_cast<int64_t>(w) * splits + s) * cols + col + col_off<A16>(t)) * R + b] = acc[t][b];
    }
}

// Decode with a CTA per (1024-column slab, 64-row chunk): a thread keeps the Q rows of its 4
// columns in registers and streams its rows -- per worker r_new = c - P_hat Q_w^T (c held in
// resid), then estimate = P_hat Q_sum^T / n.  Float4 loads/stores, Q read from L2 once per CTA.
constexpr int kDecRows = 64;
#ifndef GC_PSGD_DEC_BATCH
#define GC_PSGD_DEC_BATCH 8
#endif
constexpr int kDecBatch = GC_PSGD_DEC_BATCH;   // rows whose loads are in flight together

template <int R, bool A16>
__global__ void __launch_bounds__(256) decode_vec_kernel(int L, int n, int64_t d, int64_t rows, int64_t cols,
                                                         const float *ph, const float *qw, const float *qsum,
                                                         float *resid, Rows rw_, float *est, const int64_t *est_offs,
                                                         int est_acc) {
  __shared__ float ps[kDecRows * R];
  {   // tensor t of a batch: its factors, workers t*L .. t*L+L-1, its slice of the estimate
    const int t = blockIdx.z;
    ph += static_cast<int64_t>(t) * rows * R;
    qw += static_cast<int64_t>(t) * L * cols * R;
    qsum += static_cast<int64_t>(t) * cols * R;
    if (est) est += est_offs ? est_offs[t] : 0;
  }
  unsigned vm;
  int64_t lastoff;
  const int64_t col = thread_cols<A16>(cols, vm, lastoff);
  const int64_t row0 = static_cast<int64_t>(blockIdx.y) * kDecRows;
  const int nrows = static_cast<int>(min(static_cast<int64_t>(kDecRows), rows - row0));
  for (int e = threadIdx.x; e < nrows * R; e += 256) ps[e] = ph[row0 * R + e];
  __syncthreads();
  if (!vm) return;
  const gc::DivN dn(n);
  for (int w = 0; w <= L; ++w) {   // w == L: the estimate with Q_sum
    const float *qsrc = w < L ? qw + static_cast<int64_t>(w) * cols * R : qsum;
    float qv[4][R];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int b = 0; b < R; ++b) qv[t][b] = ((vm >> t) & 1u) ? qsrc[(col + col_off<A16>(t)) * R + b] : 0.0f;
    if (w < L && !resid) continue;
    if (w == L && !est) continue;
    float *dst = w < L ? resid + rw_.at(blockIdx.z * L + w) : est;
    if ((row0 + nrows - 1) * cols + col + lastoff < d) {   // whole block in range: branch-free
      // rows go in batches of 8: the 8 loads of c are issued before any store (the compiler
      // cannot prove that a store to row a does not alias the load of row a + 1)
      for (int a0 = 0; a0 < nrows; a0 += kDecBatch) {
        const int nb = min(kDecBatch, nrows - a0);
        float4 cv[kDecBatch];
        if (w < L) {
#pragma unroll
          for (int u = 0; u < kDecBatch; ++u)
            if (u < nb) cv[u] = ldc<A16>(dst + (row0 + a0 + u) * cols + col, vm);
        }
#pragma unroll
        for (int u = 0; u < kDecBatch; ++u) {
          if (u >= nb) break;
          const int a = a0 + u;
          float o4[4];
          float pa[R];
#pragma unroll
          for (int b = 0; b < R; ++b) pa[b] = ps[a * R + b];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            float v = __fmul_rn(pa[0], qv[t][0]);   // no contraction into the subtraction below
#pragma unroll
            for (int b = 1; b < R; ++b) v = fmaf(pa[b], qv[t][b], v);
            o4[t] = v;
          }
          float *o = dst + (row0 + a) * cols + col;
          if (w < L)
            stc<A16>(o, make_float4(cv[u].x - o4[0], cv[u].y - o4[1], cv[u].z - o4[2], cv[u].w - o4[3]), vm);
          else {
            float4 e = make_float4(dn(o4[0]), dn(o4[1]), dn(o4[2]), dn(o4[3]));
            if (est_acc) {   // rank chunks after the first: estimate += this chunk's part
              const float4 pv = ldc<A16>(o, vm);
              e.x += pv.x; e.y += pv.y; e.z += pv.z; e.w += pv.w;
            }
            stc<A16>(o, e, vm);
          }
        }
      }
      continue;
    }
#pragma unroll 8
    for (int a = 0; a < nrows; ++a) {
      const int64_t i = (row0 + a) * cols + col;
      if (i >= d) break;
      float o4[4];
      float pa[R];
#pragma unroll
      for (int b = 0; b < R; ++b) pa[b] = ps[a * R + b];
#pragma unroll
      for (int t = 0; t < 4; ++t) {   // fp32 FMAs, as the reference's fp32 p_hat @ q.T (K = r)
        float v = __fmul_rn(pa[0], qv[t][0]);   // no contraction into the subtraction below
#pragma unroll
        for (int b = 1; b < R; ++b) v = fmaf(pa[b], qv[t][b], v);
        o4[t] = v;
      }
      if (A16 && i + 3 < d) {
        if (w < L) {
          const float4 c = *reinterpret_cast<const float4 *>(dst + i);
          __stcs(reinterpret_cast<float4 *>(dst + i), make_float4(c.x - o4[0], c.y - o4[1], c.z - o4[2], c.w - o4[3]));
        } else {
          float4 e = make_float4(dn(o4[0]), dn(o4[1]), dn(o4[2]), dn(o4[3]));
          if (est_acc) {
            const float4 pv = *reinterpret_cast<const float4 *>(dst + i);
            e.x += pv.x; e.y += pv.y; e.z += pv.z; e.w += pv.w;
          }
          __stcs(reinterpret_cast<float4 *>(dst + i), e);
        }
      } else {
        for (int t = 0; t < 4; ++t) {
          const int64_t it = i + col_off<A16>(t);
          if (((vm >> t) & 1u) && it < d) dst[it] = w < L ? dst[it] - o4[t] : (est_acc ? dst[it] + dn(o4[t]) : dn(o4[t]));
        }
      }
    }
  }
}

// Q_w = M_w^T P_hat fused with the EF update r_w = c_w - P_hat Q_w^T: one read and one write of
// M instead of mtp's read plus decode's read-modify-write.  A cluster of kEfCta CTAs owns a
// kEfCols-column strip of one worker's matrix; each CTA stages its rows of the strip in shared
// memory (cp.async, all loads in flight), forms its partial Q in fp32 FMAs folded to fp64, the
// cluster sums the partials over distributed shared memory in rank order, and every CTA then
// writes its rows' residuals straight from shared memory.  Aligned shapes (cols % 4 == 0,
// 16-byte rows) whose strip fits the shared-memory budget; the estimate stays in decode.
// Opt-in: exactly the algorithmic DRAM bytes, but the strided 128-byte segments run at ~1.7 TB/s.
constexpr int kEfCta = 16;          // CTAs per cluster (row slices of a strip)
#ifndef GC_PSGD_EF_COLS
#define GC_PSGD_EF_COLS 32
#endif
constexpr int kEfCols = GC_PSGD_EF_COLS;   // strip width (kEfQ float4 per row)
constexpr int kEfQ = kEfCols / 4;
constexpr int kEfThreads = 256;            // kEfThreads / kEfQ rows per sweep
constexpr int64_t kEfSmemRows = 196608 / (kEfCols * 4);   // rows a CTA stages (192 KB)

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}

template <int R>
__global__ void __launch_bounds__(kEfThreads) mtp_ef_kernel(int64_t d, int64_t rows, int64_t cols, float *resid,
                                                            Rows rw_, const float *ph, float *qw,
                                                            int64_t rows_per_cta) {
  namespace cgr = cooperative_groups;
  cgr::cluster_group cl = cgr::this_cluster();
  extern __shared__ __align__(16) unsigned char ef_smem[];
  double *qp = reinterpret_cast<double *>(ef_smem);               // [kEfCols][R] CTA partial
  double *wred = qp + kEfCols * R;                                 // [8 warps][kEfCols][R]
  float *qf = reinterpret_cast<float *>(wred + 8 * kEfCols * R);   // [kEfCols][R] Q_w strip
  float4 *ms = reinterpret_cast<float4 *>(qf + kEfCols * R);       // [rows_per_cta][kEfQ]
  const int crank = static_cast<int>(cl.block_rank());
  const int v = blockIdx.y;
  const int64_t col0 = static_cast<int64_t>(blockIdx.x / kEfCta) * kEfCols;
  const int64_t r0 = crank * rows_per_cta;
  const int64_t r1 = min(rows, r0 + rows_per_cta);
  const int nr = r1 > r0 ? static_cast<int>(r1 - r0) : 0;
  float *cw = resid + rw_.at(v);
  ph += static_cast<int64_t>(rw_.tensor(v)) * rows * R;
  constexpr int kSweep = kEfThreads / kEfQ;
  const int qd = threadIdx.x % kEfQ, rg = threadIdx.x / kEfQ;
  const int64_t col = col0 + 4 * qd;
  const bool colok = col < cols;
  // stage: element (i, col..col+3) of the padded matrix; entries at flat index >= d are zero
  for (int a = rg; a < nr; a += kSweep) {
    const int64_t i = (r0 + a) * cols + col;
    float4 *dst = ms + a * kEfQ + qd;
    if (colok && i + 3 < d) {
      cp_async16(dst, cw + i);
    } else {
      float t4[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) t4[t] = colok && i + t < d ? cw[i + t] : 0.0f;
      *dst = make_float4(t4[0], t4[1], t4[2], t4[3]);
    }
  }
  asm volatile("cp.async.wait_all;\n" ::: "memory");
  __syncthreads();
  // partial Q over this CTA's rows: fp32 FMAs per thread, folded to fp64
  double acc[4][R];
  {
    float a32[4][R];
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int b = 0; b < R; ++b) a32[t][b] = 0.0f;
    for (int a = rg; a < nr; a += kSweep) {
      const float4 m = ms[a * kEfQ + qd];
      const float m4[4] = {m.x, m.y, m.z, m.w};
      const float *pr = ph + (r0 + a) * R;
      float pv[R];
#pragma unroll
      for (int b = 0; b < R; ++b) pv[b] = __ldg(pr + b);
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int b = 0; b < R; ++b) a32[t][b] = fmaf(m4[t], pv[b], a32[t][b]);
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int b = 0; b < R; ++b) acc[t][b] = static_cast<double>(a32[t][b]);
  }
  // lanes sharing qd (lane bits 2..4) -> warp sums -> CTA partial in warp order
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) {
      double s = acc[t][b];
      for (int o = kEfQ; o < 32; o <<= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      acc[t][b] = s;
    }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane < kEfQ) {
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int b = 0; b < R; ++b) wred[(warp * kEfCols + 4 * lane + t) * R + b] = acc[t][b];
  }
  __syncthreads();
  for (int e = threadIdx.x; e < kEfCols * R; e += kEfThreads) {
    double s = 0.0;
    for (int wp = 0; wp < kEfThreads / 32; ++wp) s += wred[wp * kEfCols * R + e];
    qp[e] = s;
  }
  cl.sync();
  // Q_w strip: the cluster's partials summed in rank order (identical in every CTA)
  for (int e = threadIdx.x; e < kEfCols * R; e += kEfThreads) {
    double s = 0.0;
    for (int k = 0; k < kEfCta; ++k) s += cl.map_shared_rank(qp, k)[e];
    qf[e] = static_cast<float>(s);
    if (crank == 0 && col0 + e / R < cols) qw[(static_cast<int64_t>(v) * cols + col0) * R + e] = qf[e];
  }
  cl.sync();   // no CTA leaves while a peer may still read its partial
  if (!colok) return;
  float qv[4][R];
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int b = 0; b < R; ++b) qv[t][b] = qf[(4 * qd + t) * R + b];
  // r = c - P_hat Q_w^T in fp32 FMAs (the decode's formula), c from shared memory
  for (int a = rg; a < nr; a += kSweep) {
    const int64_t i = (r0 + a) * cols + col;
    if (i >= d) break;
    const float4 m = ms[a * kEfQ + qd];
    const float *pr = ph + (r0 + a) * R;
    float pa[R];
#pragma unroll
    for (int b = 0; b < R; ++b) pa[b] = __ldg(pr + b);
    float o4[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      float x = pa[0] * qv[t][0];
#pragma unroll
      for (int b = 1; b < R; ++b) x = fmaf(pa[b], qv[t][b], x);
      o4[t] = x;
    }
    const float4 out = make_float4(m.x - o4[0], m.y - o4[1], m.z - o4[2], m.w - o4[3]);
    if (i + 3 < d) {
      __stcs(reinterpret_cast<float4 *>(cw + i), out);
    } else {
      const float o[4] = {out.x, out.y, out.z, out.w};
      for (int t = 0; t < 4; ++t)
        if (i + t < d) cw[i + t] = o[t];
    }
  }
}

// Gram matrix Q^T Q (fp64) for the rank check of ensure_full_rank (compressors.py:595-603).
// Gram Q^T Q per tensor (fp64): the columns are split over kGramSlices CTAs; a thread owns
// (a, b) pairs of the upper triangle and sums its slice's rows; the slices are added in order.
constexpr int kGramSlices = 32;

__global__ void __launch_bounds__(256) gram_partial_kernel(int64_t cols, int R, const float *q, double *partial) {
  const int t = blockIdx.x, sl = blockIdx.y;
  q += static_cast<int64_t>(t) * cols * R;
  const int P = R * (R + 1) / 2;
  const int64_t per = (cols + kGramSlices - 1) / kGramSlices;
  const int64_t j0 = sl * per, j1 = min(cols, j0 + per);
  for (int pi = threadIdx.x; pi < P; pi += 256) {
    int a = 0, rem = pi;   // pair index -> (a, b >= a)
    while (rem >= R - a) {
      rem -= R - a;
      ++a;
    }
    const int b = a + rem;
    double v = 0.0;
    for (int64_t j = j0; j < j1; ++j) v += static_cast<double>(q[j * R + a]) * static_cast<double>(q[j * R + b]);
    partial[(static_cast<int64_t>(t) * kGramSlices + sl) * P + pi] = v;
  }
}

__global__ void gram_reduce_kernel(int R, const double *partial, double *gram) {
  const int t = blockIdx.x;
  const int P = R * (R + 1) / 2;
  for (int pi = threadIdx.x; pi < P; pi += blockDim.x) {
    int a = 0, rem = pi;
    while (rem >= R - a) {
      rem -= R - a;
      ++a;
    }
    const int b = a + rem;
    double v = 0.0;
    for (int sl = 0; sl < kGramSlices; ++sl) v += partial[(static_cast<int64_t>(t) * kGramSlices + sl) * P + pi];
    gram[(static_cast<int64_t>(t) * R + a) * R + b] = v;
    gram[(static_cast<int64_t>(t) * R + b) * R + a] = v;
  }
}

#define GC_RANK_SWITCH(rank, CALL)                                                      \
  switch (rank) {                                                                        \
    case 1: { constexpr int R = 1; CALL; } break;                                        \
    case 2: { constexpr int R = 2; CALL; } break;                                        \
    case 3: { constexpr int R = 3; CALL; } break;                                        \
    case 4: { constexpr int R = 4; CALL; } break;                                        \
    case 5: { constexpr int R = 5; CALL; } break;                                        \
    case 6: { constexpr int R = 6; CALL; } break;                                        \
    case 7: { constexpr int R = 7; CALL; } break;                                        \
    case 8: { constexpr int R = 8; CALL; } break;                                        \
    case 16: { constexpr int R = 16; CALL; } break;                                      \
    default: gc_set_error("rank must be 1..8 or 16"); return GC_ERR_UNSUPPORTED;          \
  }

int check_batch(const gc_psgd_batch *b) {
  GC_REQUIRE(b != nullptr, "batch descriptor is null");
  GC_REQUIRE(b->tensors >= 1 && b->workers >= 1 && static_cast<int64_t>(b->tensors) * b->workers <= 65535,
             "batch must have 1..65535 (tensor, worker) rows");
  GC_REQUIRE(b->row_offsets != nullptr || b->ld >= 1, "need row_offsets or ld");
  GC_REQUIRE(!b->rows_aligned || b->row_offsets != nullptr || static_cast<int64_t>(b->tensors) * b->workers == 1 ||
                 b->ld % 4 == 0,
             "rows_aligned is set but the row pitch ld is not a multiple of 4 floats");
  return GC_OK;
}

std::string getenv_str(const char *name) {
  const char *v = getenv(name);
  return v ? v : "";
}

Rows rows_of(const gc_psgd_batch *b) { return Rows{b->row_offsets, b->ld, b->workers}; }

}  // namespace

extern "C" {

int gc_psgd_splits(int32_t rows_total, int64_t cols) {
  const int64_t slabs = (cols % 4 == 0 ? (cols + 1023) / 1024 : (cols + 255) / 256) * rows_total;
  int s = static_cast<int>((8 * 148 + slabs - 1) / slabs);
  return s < 1 ? 1 : (s > 64 ? 64 : s);
}

int64_t gc_psgd_workspace_bytes(int32_t rows_total, int64_t rows, int64_t cols, int32_t rank) {
  const int64_t splits = gc_psgd_splits(rows_total, cols);
  const int64_t mtp = 8 * (static_cast<int64_t>(rows_total) * splits * cols * rank);
  const int64_t mq = 8 * (static_cast<int64_t>(rows_total) * gc_psgd_mq_max_splits(cols) * rows * rank);
  return (mtp > mq ? mtp : mq) + 256;
}

int gc_psgd_vectorizable(int64_t cols, const void *a, const void *b, int64_t ld) {
  return cols % 4 == 0 && ld % 4 == 0 && ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b)) & 15) == 0;
}

int gc_psgd_mq(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
               const float *q, float *p, void *stream) {
  if (int rc = check_batch(b)) return rc;
  GC_REQUIRE(d >= 1 && rows * cols >= d && c && q && p, "invalid argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int L = b->tensors * b->workers;
  GC_RANK_SWITCH(rank, ({
    constexpr int rpc = MqShape<R>::kRowsPerCta;
    mq_kernel<R><<<dim3(grid_cap((rows + rpc - 1) / rpc), L), 256, 0, st>>>(d, rows, cols, c, rows_of(b), q, p);
  }));
  GC_LAUNCH_CHECK("mq_kernel");
  return GC_OK;
}

int gc_psgd_mq_fused(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                     float *resid, const float *q, float *p, void *workspace, void *stream) {
  if (int rc = check_batch(b)) return rc;
  GC_REQUIRE(d >= 1 && rows * cols >= d && grads && q && p && workspace, "invalid argument");
  const bool a16 = cols % 4 == 0 && b->rows_aligned;   // else the masked-scalar producer
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int L = b->tensors * b->workers;
  int slabs = static_cast<int>((cols + 1023) / 1024);
  double *partial = static_cast<double *>(workspace);
  const char *impl = getenv("GC_PSGD_MQ");
  if (impl && std::string(impl) == "cores" && a16) {
    GC_RANK_SWITCH(rank, ({
      mq_fused_kernel<R><<<dim3(slabs, grid_cap((rows + kMqRows - 1) / kMqRows), L), 256, 0, st>>>(
          d, rows, cols, grads, resid, rows_of(b), q, partial, slabs);
    }));
    GC_LAUNCH_CHECK("mq_fused_kernel");
  } else {
    // tcgen05 (kind::tf32, 3xTF32) band GEMM fused with ef_apply (gc_psgd_umma.cu)
    slabs = gc_psgd_mq_umma_launch(L, b->workers, b->row_offsets, b->ld, d, rows, cols, rank, grads, resid, q,
                                   partial, a16 ? 1 : 0, st);
    if (slabs < 0) return slabs;
  }
  const int64_t total = static_cast<int64_t>(L) * rows * rank;
  mq_reduce_kernel<<<grid_cap((total + 255) / 256 > 148 * 8 ? 148 * 8 : (total + 255) / 256), 256, 0, st>>>(
      L, slabs, rows, rank, partial, p);
  GC_LAUNCH_CHECK("mq_reduce_kernel");
  return GC_OK;
}

int gc_psgd_mq_tma_supported(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank,
                             const void *grads, const void *resid) {
  if (b == nullptr || d < 1 || rows * cols < d || b->tensors != 1 || b->row_offsets != nullptr) return 0;
  return gc_psgd_mq_tma_supported_impl(1, b->workers, nullptr, b->ld, d, rows, cols, rank, grads, resid);
}

int gc_psgd_mq_tma_supported_batched(const gc_psgd_batch *b, const int64_t *host_tensor_offsets, int64_t d,
                                     int64_t rows, int64_t cols, int32_t rank, const void *grads, const void *resid) {
  if (b == nullptr || d < 1 || rows * cols < d) return 0;
  // a batch with row offsets needs the host copy of its tensor offsets (one tensor map per tensor)
  if ((b->tensors > 1 || b->row_offsets != nullptr) && (host_tensor_offsets == nullptr || b->row_offsets == nullptr))
    return 0;
  return gc_psgd_mq_tma_supported_impl(b->tensors, b->workers, host_tensor_offsets, b->ld, d, rows, cols, rank, grads,
                                       resid);
}

int gc_psgd_mq_deferred_supported(const gc_psgd_batch *b, const int64_t *host_tensor_offsets, int64_t d,
                                  int64_t rows, int64_t cols, int32_t rank, const void *grads, const void *resid) {
  if (b == nullptr || d < 1 || rows * cols < d || d < cols) return 0;
  if (gc_psgd_mq_tma_supported_batched(b, host_tensor_offsets, d, rows, cols, rank, grads, resid)) return 1;
  if (b->tensors > 1 && b->row_offsets == nullptr) return 0;
  return gc_psgd_mq_async_supported_impl(rank, grads, resid);
}

int gc_psgd_mq_deferred_batched(const gc_psgd_batch *b, const int64_t *host_tensor_offsets, int64_t d, int64_t rows,
                                int64_t cols, int32_t rank, const float *grads, float *resid, const float *q,
                                const float *ef_p_hat, const float *ef_q_workers, float *p, void *workspace,
                                void *stream) {
  if (int rc = check_batch(b)) return rc;
  GC_REQUIRE(d >= 1 && rows * cols >= d && grads && q && p && workspace, "invalid argument");
  GC_REQUIRE((ef_p_hat == nullptr) == (ef_q_workers == nullptr), "deferred EF needs both factors or neither");
  GC_REQUIRE(ef_p_hat == nullptr || resid != nullptr, "deferred EF needs the residual buffer");
  if (!gc_psgd_mq_deferred_supported(b, host_tensor_offsets, d, rows, cols, rank, grads, resid)) {
    gc_set_error("deferred P = M Q needs 4-byte aligned buffers, d >= cols and a compiled rank");
    return GC_ERR_UNSUPPORTED;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int L = b->tensors * b->workers;
  // TMA boxes when a tensor map describes the rows, else the cp.async-fed pass (gc_psgd_async.cu)
  const bool tma = gc_psgd_mq_tma_supported_batched(b, host_tensor_offsets, d, rows, cols, rank, grads, resid) &&
                   getenv_str("GC_PSGD_MQ_FEED") != "async";
  // cols = 2 (mod 4) with aligned tensor starts: tensor maps over row pairs (GPT-2's shapes)
  const bool pair = !tma && getenv_str("GC_PSGD_MQ_FEED") != "async" &&
                    (b->tensors == 1 && b->row_offsets == nullptr ? true : host_tensor_offsets != nullptr) &&
                    gc_psgd_mq_pair_supported_impl(b->tensors, b->workers, host_tensor_offsets, b->ld, d, rows, cols,
                                                   rank, grads, resid);
  const int slabs =
      pair ? gc_psgd_mq_pair_launch(b->tensors, b->workers, host_tensor_offsets, b->row_offsets, b->ld, d, rows, cols,
                                    rank, grads, resid, q, ef_p_hat, ef_q_workers, static_cast<double *>(workspace),
                                    gc_psgd_mq_max_splits(cols), st)
      : tma ? gc_psgd_mq_tma_launch(b->tensors, b->workers, host_tensor_offsets, b->row_offsets, b->ld, d, rows, cols,
                                  rank, grads, resid, q, ef_p_hat, ef_q_workers, static_cast<double *>(workspace),
                                  gc_psgd_mq_max_splits(cols), st)
          : gc_psgd_mq_async_launch(b->tensors, b->workers, b->row_offsets, host_tensor_offsets, b->ld, d, rows, cols,
                                    rank, grads, resid, q, ef_p_hat, ef_q_workers, static_cast<double *>(workspace),
                                    gc_psgd_mq_max_splits(cols), st);
  if (slabs < 0) return slabs;
  const int64_t total = static_cast<int64_t>(L) * rows * rank;
  mq_reduce_kernel<<<grid_cap((total + 255) / 256 > 148 * 8 ? 148 * 8 : (total + 255) / 256), 256, 0, st>>>(
      L, slabs, rows, rank, static_cast<const double *>(workspace), p);
  GC_LAUNCH_CHECK("mq_reduce_kernel");
  return GC_OK;
}

int gc_psgd_mq_deferred(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                        float *resid, const float *q, const float *ef_p_hat, const float *ef_q_workers, float *p,
                        void *workspace, void *stream) {
  if (b != nullptr && (b->tensors != 1 || b->row_offsets != nullptr)) {
    gc_set_error("gc_psgd_mq_deferred takes one tensor without row offsets; see gc_psgd_mq_deferred_batched");
    return GC_ERR_UNSUPPORTED;
  }
  return gc_psgd_mq_deferred_batched(b, nullptr, d, rows, cols, rank, grads, resid, q, ef_p_hat, ef_q_workers, p,
                                     workspace, stream);
}

int gc_psgd_mtp(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
                const float *p_hat, float *q, void *workspace, void *stream) {
  return gc_psgd_mtp_batched(b, nullptr, d, rows, cols, rank, c, p_hat, q, workspace, stream);
}

int gc_psgd_mtp_batched(const gc_psgd_batch *b, const int64_t *host_tensor_offsets, int64_t d, int64_t rows,
                        int64_t cols, int32_t rank, const float *c, const float *p_hat, float *q, void *workspace,
                        void *stream) {
  if (int rc = check_batch(b)) return rc;
  GC_REQUIRE(d >= 1 && rows * cols >= d && c && p_hat && q && workspace, "invalid argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int L = b->tensors * b->workers;
  int splits = gc_psgd_splits(L, cols);
  const int64_t per = (rows + splits - 1) / splits;
  double *partial = static_cast<double *>(workspace);
  const bool vec = cols % 4 == 0 && b->rows_aligned && (reinterpret_cast<uintptr_t>(c) & 15) == 0;
  // TMA-fed passes (gc_psgd_tma.cu), the same split-K partials and ordered reduction.  Default:
  // ranks 5..16 on tcgen05 (MN-major A straight from the TMA boxes; 2.3x the CUDA-core pass at
  // ranks 8 and 16), ranks 1..4 on the CUDA-core TMA slabs (the 3xTF32 MMAs' shared-memory
  // traffic costs more than rank-4 FFMA); layouts without a tensor map (batches, unaligned rows)
  // on cp.async-fed slabs for ranks 1..4.  GC_PSGD_MTP=umma | async | cores | vec forces a path.
  const char *impl_env = getenv("GC_PSGD_MTP");
  const std::string impl = impl_env ? impl_env : "";
  const bool single = b->tensors == 1 && b->row_offsets == nullptr;
  // a batch with row offsets takes tensor maps only with its host tensor offsets
  // (P_hat of tensor t starts t rows R floats in: 16-byte aligned for the bulk copies iff rows R % 4 == 0)
  const bool maps_ok = (single || (host_tensor_offsets != nullptr && b->row_offsets != nullptr &&
                                   (rows * rank) % 4 == 0)) &&
                       gc_psgd_mq_tma_supported_impl(b->tensors, b->workers, single ? nullptr : host_tensor_offsets,
                                                     b->ld, d, rows, cols, rank, c, c);
  const bool tma_ok = single && maps_ok;
  if (tma_ok && (impl == "umma" || (impl.empty() && rank > 4))) {
    splits = gc_psgd_mtp_umma_launch(L, b->ld, d, rows, cols, rank, c, p_hat, partial, splits, st);
    if (splits < 0) return splits;
  } else if (maps_ok && rank <= 4 && impl != "cores" && impl != "async") {
    splits = gc_psgd_mtp_tma_launch(b->tensors, b->workers, single ? nullptr : host_tensor_offsets, b->row_offsets,
                                    b->ld, d, rows, cols, rank, c, p_hat, partial, splits, st);
    if (splits < 0) return splits;
  } else if (rank <= 4 && impl != "cores" && impl != "vec" && impl != "async" &&
             (single || (host_tensor_offsets && (rows * rank) % 4 == 0)) && cols % 4 == 2 && d / cols >= 2 &&
             (b->workers == 1 || b->ld % 4 == 0) &&
             gc_psgd_mq_pair_supported_impl(b->tensors, b->workers, single ? nullptr : host_tensor_offsets, b->ld, d,
                                            rows, cols, 4, c, c)) {
    // cols = 2 (mod 4): the row-pair tensor maps (gc_psgd_tma.cu)
    splits = gc_psgd_mtp_pair_launch(b->tensors, b->workers, single ? nullptr : host_tensor_offsets, b->row_offsets,
                                     b->ld, d, rows, cols, rank, c, p_hat, partial, splits, st);
    if (splits < 0) return splits;
  } else if (rank <= 4 && impl != "cores" && impl != "vec") {
    // batches of tensors and unaligned row pitches: the cp.async-fed slabs (gc_psgd_async.cu)
    splits = gc_psgd_mtp_async_launch(L, b->workers, b->row_offsets, b->ld, d, rows, cols, rank, c, p_hat, partial,
                                      splits, st);
    if (splits < 0) return splits;
  } else if (vec) {
    GC_RANK_SWITCH(rank, ({
      mtp_vec_kernel<R, true><<<dim3(grid_cap((cols + 1023) / 1024), splits, L), 256, 0, st>>>(
          d, rows, cols, c, rows_of(b), p_hat, per, partial, splits);
    }));
  } else {   // unaligned rows: the same kernel with coalesced scalar loads
    GC_RANK_SWITCH(rank, ({
      mtp_vec_kernel<R, false><<<dim3(grid_cap((cols + 1023) / 1024), splits, L), 256, 0, st>>>(
          d, rows, cols, c, rows_of(b), p_hat, per, partial, splits);
    }));
  }
  GC_LAUNCH_CHECK("mtp_kernel");
  const int64_t total = static_cast<int64_t>(L) * cols * rank;
  mtp_reduce_kernel<<<grid_cap((total + 255) / 256 > 148 * 8 ? 148 * 8 : (total + 255) / 256), 256, 0, st>>>(
      L, splits, cols, rank, partial, q);
  GC_LAUNCH_CHECK("mtp_reduce_kernel");
  return GC_OK;
}

int gc_psgd_mtp_ef_supported(int64_t rows, int64_t cols, int32_t rank, int32_t rows_aligned) {
  return rows_aligned && cols % 4 == 0 && rank >= 1 && rank <= 8 && rows >= kEfCta &&
         (rows + kEfCta - 1) / kEfCta <= kEfSmemRows;
}

// Q_w = M_w^T P_hat and r_w = c_w - P_hat Q_w^T in one pass over M (c held in resid).
int gc_psgd_mtp_ef(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, float *resid,
                   const float *p_hat, float *q, void *stream) {
  if (int rc = check_batch(b)) return rc;
  GC_REQUIRE(d >= 1 && rows * cols >= d && resid && p_hat && q, "invalid argument");
  if (!gc_psgd_mtp_ef_supported(rows, cols, rank, b->rows_aligned) || (reinterpret_cast<uintptr_t>(resid) & 15)) {
    gc_set_error("gc_psgd_mtp_ef: shape not supported (see gc_psgd_mtp_ef_supported)");
    return GC_ERR_UNSUPPORTED;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int L = b->tensors * b->workers;
  const int64_t per = (rows + kEfCta - 1) / kEfCta;
  const int64_t strips = (cols + kEfCols - 1) / kEfCols;
  GC_REQUIRE(strips * kEfCta < (int64_t{1} << 31) && L <= 65535, "invalid argument");
  cudaError_t err = cudaSuccess;
  GC_RANK_SWITCH(rank, ({
    const size_t smem = kEfCols * R * (8 + 64 + 4) + static_cast<size_t>(per) * kEfCols * 4;
    static bool attr_done = false;
    if (!attr_done) {
      cudaFuncSetAttribute(mtp_ef_kernel<R>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaFuncSetAttribute(mtp_ef_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(kEfCols * R * 76 + kEfSmemRows * kEfCols * 4));
      attr_done = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(strips * kEfCta), static_cast<unsigned>(L), 1);
    cfg.blockDim = dim3(kEfThreads, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = kEfCta;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    err = cudaLaunchKernelEx(&cfg, mtp_ef_kernel<R>, d, rows, cols, resid, rows_of(b), p_hat, q, per);
  }));
  if (err != cudaSuccess) {
    gc_set_error(std::string("mtp_ef_kernel launch: ") + cudaGetErrorString(err));
    return GC_ERR_CUDA;
  }
  GC_LAUNCH_CHECK("mtp_ef_kernel");
  return GC_OK;
}

int64_t gc_psgd_orth_workspace_bytes(int32_t tensors, int64_t rows, int32_t rank) {
  const int64_t np = static_cast<int64_t>(rank) * (rank + 1) / 2;
  return 8 * (static_cast<int64_t>(tensors) * rows * rank + static_cast<int64_t>(tensors) * kOrthSlicesMax * np +
              static_cast<int64_t>(tensors) * rank * rank) +
         4 * static_cast<int64_t>(tensors) + 64;
}

int gc_psgd_orthonormalize(int32_t tensors, int64_t rows, int32_t rank, const float *p, float *p_hat, void *workspace,
                           int32_t *status, void *stream) {
  GC_REQUIRE(tensors >= 1 && tensors <= 65535 && rows >= rank && rank >= 1 && rank <= kMaxOrthRank && p && p_hat &&
                 workspace && status,
             "invalid argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *a = static_cast<double *>(workspace);
  const int *fast = nullptr;
  if (rank <= 8 || rank == 16) {   // Cholesky fast path (flags per tensor), CGS2 kernel for the rest
    const int64_t np = static_cast<int64_t>(rank) * (rank + 1) / 2;
    double *partial = a + static_cast<int64_t>(tensors) * rows * rank;
    double *rinv = partial + static_cast<int64_t>(tensors) * kOrthSlicesMax * np;
    int *flags = reinterpret_cast<int *>(rinv + static_cast<int64_t>(tensors) * rank * rank);
    int64_t slices = (rows + 2047) / 2048;
    if (slices > kOrthSlicesMax) slices = kOrthSlicesMax;
    const int sl = static_cast<int>(slices);
    const dim3 g2(sl, tensors);
    GC_RANK_SWITCH(rank, ({ tall_gram_kernel<R><<<g2, 256, 0, st>>>(rows, p, partial, sl); }));
    GC_LAUNCH_CHECK("tall_gram_kernel");
    orth_chol_kernel<<<(tensors + 63) / 64, 64, 0, st>>>(tensors, rank, sl, partial, rinv, flags);
    GC_LAUNCH_CHECK("orth_chol_kernel");
    const dim3 g3(grid_cap((rows + 255) / 256 > 148 ? 148 : (rows + 255) / 256), tensors);
    GC_RANK_SWITCH(rank, ({ orth_apply_kernel<R><<<g3, 256, 0, st>>>(rows, p, rinv, flags, p_hat); }));
    GC_LAUNCH_CHECK("orth_apply_kernel");
    fast = flags;
  }
  const size_t orth_smem = static_cast<size_t>(kOrthThreads / 32 + 1) * rank * sizeof(double);
  if (orth_smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(orth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               static_cast<int>(orth_smem));
    GC_REQUIRE(e == cudaSuccess, "orth_kernel: cannot opt in to the shared memory this rank needs");
  }
  orth_kernel<<<tensors, kOrthThreads, orth_smem, st>>>(rows, rank, p, a, p_hat, status, fast);
  GC_LAUNCH_CHECK("orth_kernel");
  return GC_OK;
}

int gc_psgd_decode_fused(const gc_psgd_batch *b, int32_t n, int64_t d, int64_t rows, int64_t cols, int32_t rank,
                         const float *p_hat, const float *q_workers, const float *q_sum, float *resid, float *estimate,
                         void *stream);

// Either output may be NULL: estimate only, EF update only, or both in one pass.
int gc_psgd_decode(const gc_psgd_batch *b, int32_t n, int64_t d, int64_t rows, int64_t cols, int32_t rank,
                   const float *p_hat, const float *q_workers, const float *q_sum, float *resid, float *estimate,
                   void *stream) {
  return gc_psgd_decode_fused(b, n, d, rows, cols, rank, p_hat, q_workers, q_sum, resid, estimate, stream);
}

int gc_psgd_decode_fused(const gc_psgd_batch *b, int32_t n, int64_t d, int64_t rows, int64_t cols, int32_t rank,
                         const float *p_hat, const float *q_workers, const float *q_sum, float *resid, float *estimate,
                         void *stream) {
  if (int rc = check_batch(b)) return rc;
  GC_REQUIRE(n >= 1 && d >= 1 && p_hat && q_workers && q_sum, "invalid argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // float4 accesses need cols % 4 == 0 and 16-byte aligned rows; otherwise coalesced scalars
  const bool a16 = cols % 4 == 0 && b->rows_aligned;
  const dim3 grid(grid_cap((cols + 1023) / 1024), grid_cap((rows + kDecRows - 1) / kDecRows), b->tensors);
  GC_RANK_SWITCH(rank, ({
    if (a16)
      decode_vec_kernel<R, true><<<grid, 256, 0, st>>>(b->workers, n, d, rows, cols, p_hat, q_workers, q_sum, resid,
                                                       rows_of(b), estimate, b->est_offsets,
                                                       b->est_accumulate);
    else
      decode_vec_kernel<R, false><<<grid, 256, 0, st>>>(b->workers, n, d, rows, cols, p_hat, q_workers, q_sum, resid,
                                                        rows_of(b), estimate, b->est_offsets,
                                                        b->est_accumulate);
  }));
  GC_LAUNCH_CHECK("decode_vec_kernel");
  return GC_OK;
}

int64_t gc_psgd_gram_workspace_bytes(int32_t tensors, int32_t rank) {
  return 8 * static_cast<int64_t>(tensors) * kGramSlices * rank * (rank + 1) / 2;
}

int gc_psgd_gram(int32_t tensors, int64_t cols, int32_t rank, const float *q, double *gram, void *workspace,
                 void *stream) {
  GC_REQUIRE(tensors >= 1 && tensors <= 65535 && cols >= 1 && rank >= 1 && rank <= kMaxOrthRank && q && gram &&
                 workspace,
             "invalid argument");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  double *partial = static_cast<double *>(workspace);
  if (rank <= 8 || rank == 16) {   // row-parallel: every thread sums all pairs of its rows
    const dim3 g2(kGramSlices, tensors);
    GC_RANK_SWITCH(rank, ({ tall_gram_kernel<R><<<g2, 256, 0, st>>>(cols, q, partial, kGramSlices); }));
    GC_LAUNCH_CHECK("tall_gram_kernel");
  } else {
    gram_partial_kernel<<<dim3(tensors, kGramSlices), 256, 0, st>>>(cols, rank, q, partial);
    GC_LAUNCH_CHECK("gram_partial_kernel");
  }
  gram_reduce_kernel<<<tensors, 256, 0, st>>>(rank, partial, gram);
  GC_LAUNCH_CHECK("gram_reduce_kernel");
  return GC_OK;
}

int gc_fill_zero(void *ptr, int64_t bytes, void *stream) {
  GC_REQUIRE(bytes >= 0 && (ptr || bytes == 0), "invalid argument");
  if (bytes && cudaMemsetAsync(ptr, 0, static_cast<size_t>(bytes), static_cast<cudaStream_t>(stream)) != cudaSuccess) {
    gc_set_error("cudaMemsetAsync failed");
    return GC_ERR_CUDA;
  }
  return GC_OK;
}

}  // extern "C"
