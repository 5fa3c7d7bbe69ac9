// Microbenchmark: streaming 128-row x 32-column chunks of a row-major fp32 matrix whose row pitch
// is not a multiple of 16 bytes (cols % 4 == 2, GPT-2's 1774 x 1774 / 7174 x 7174 PowerSGD
// matrices), one CTA per SM, a ring of stages.  Feeds compared (GB/s of one read of the matrix):
//   bulk  : one 1-D cp.async.bulk per row segment, widened to the enclosing 16-byte-aligned window
//           (144 B), completion on the stage's mbarrier (the TMA engine, no L1 miss tracking)
//   async4: 4-byte cp.async per element (LDGSTS through L1), wait_group per stage
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o unaligned_stream unaligned_stream.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}

constexpr int kRows = 128, kCols = 32, kRowSlot = 48;   // staging row: 48 floats (192 B) >= 144 B window
constexpr int kStageBytes = kRows * kRowSlot * 4;       // 24 KB

// chunk c of CTA b: band (c / nchunk_cols) of rows, column chunk (c % nchunk_cols)
__global__ void __launch_bounds__(256, 1) bulk_kernel(const float *m, int64_t rows, int64_t cols, int stages,
                                                      int chunks_per_cta, float *sink) {
  extern __shared__ unsigned char sm_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(sm_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  const uint32_t bars = base + stages * kStageBytes;
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < stages; ++s) mbar_init(bars + 8 * s, kRows);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int64_t ncc = (cols + kCols - 1) / kCols;
  const int64_t nb = (rows + kRows - 1) / kRows;
  float acc = 0.f;
  auto issue = [&](int64_t k, int s) {   // threads 0..127: one row each
    const int64_t c = blockIdx.x + k * gridDim.x;
    const int64_t band = (c / ncc) % nb, cc = c % ncc;
    if (tid < kRows) {
      const int64_t row = band * kRows + tid;
      const int64_t e0 = row * cols + cc * kCols;
      const int64_t e1 = min(e0 + kCols, row * cols + cols);
      const uint64_t a0 = reinterpret_cast<uint64_t>(m + e0) & ~15ull;
      const uint64_t a1 = (reinterpret_cast<uint64_t>(m + e1) + 15ull) & ~15ull;
      const uint32_t bytes = row < rows ? static_cast<uint32_t>(a1 - a0) : 0u;
      const uint32_t bar = bars + 8 * s;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      if (bytes)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         base + s * kStageBytes + tid * kRowSlot * 4),
                     "l"(a0), "r"(bytes), "r"(bar)
                     : "memory");
    }
  };
  for (int k = 0; k < stages - 1 && k < chunks_per_cta; ++k) issue(k, k);
  for (int k = 0; k < chunks_per_cta; ++k) {
    const int s = k % stages;
    if (k + stages - 1 < chunks_per_cta) {
      __syncthreads();   // stage (k - 1) % stages consumed by everyone
      issue(k + stages - 1, (k + stages - 1) % stages);
    }
    mbar_wait(bars + 8 * s, (k / stages) & 1);
    const float *st = reinterpret_cast<const float *>(sm_raw + (base - raw) + s * kStageBytes);
    for (int e = tid; e < kRows * kCols; e += 256) acc += st[(e / kCols) * kRowSlot + e % kCols];
  }
  if (acc == 12345.f) *sink = acc;
}

__global__ void __launch_bounds__(256, 1) async4_kernel(const float *m, int64_t rows, int64_t cols, int stages,
                                                        int chunks_per_cta, float *sink) {
  extern __shared__ unsigned char sm_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(sm_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ncc = (cols + kCols - 1) / kCols;
  const int64_t nb = (rows + kRows - 1) / kRows;
  float acc = 0.f;
  auto issue = [&](int64_t k, int s) {
    const int64_t c = blockIdx.x + k * gridDim.x;
    const int64_t band = (c / ncc) % nb, cc = c % ncc;
    const int64_t col = cc * kCols + lane;
    for (int u = 0; u < kRows / 8; ++u) {
      const int64_t row = band * kRows + warp + 8 * u;
      if (row < rows && col < cols)
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(base + s * kStageBytes +
                                                                      ((warp + 8 * u) * kRowSlot + lane) * 4),
                     "l"(m + row * cols + col)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int k = 0; k < stages - 1; ++k) {
    if (k < chunks_per_cta) issue(k, k);
    else asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int k = 0; k < chunks_per_cta; ++k) {
    const int s = k % stages;
    if (k + stages - 1 < chunks_per_cta) issue(k + stages - 1, (k + stages - 1) % stages);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(0) : "memory");   // simple: see the variant below
    const float *st = reinterpret_cast<const float *>(sm_raw + (base - raw) + s * kStageBytes);
    for (int u = 0; u < kRows / 8; ++u) acc += st[(warp + 8 * u) * kRowSlot + lane];
  }
  if (acc == 12345.f) *sink = acc;
}

template <int AHEAD>
__global__ void __launch_bounds__(256, 1) async4w_kernel(const float *m, int64_t rows, int64_t cols,
                                                         int chunks_per_cta, float *sink) {
  constexpr int stages = AHEAD + 1;
  extern __shared__ unsigned char sm_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(sm_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ncc = (cols + kCols - 1) / kCols;
  const int64_t nb = (rows + kRows - 1) / kRows;
  float acc = 0.f;
  auto issue = [&](int64_t k, int s) {
    if (k < chunks_per_cta) {
      const int64_t c = blockIdx.x + k * gridDim.x;
      const int64_t band = (c / ncc) % nb, cc = c % ncc;
      const int64_t col = cc * kCols + lane;
      for (int u = 0; u < kRows / 8; ++u) {
        const int64_t row = band * kRows + warp + 8 * u;
        if (row < rows && col < cols)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(base + s * kStageBytes +
                                                                        ((warp + 8 * u) * kRowSlot + lane) * 4),
                       "l"(m + row * cols + col)
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int k = 0; k < AHEAD; ++k) issue(k, k % stages);
  for (int k = 0; k < chunks_per_cta; ++k) {
    issue(k + AHEAD, (k + AHEAD) % stages);
    asm volatile("cp.async.wait_group %0;" ::"n"(AHEAD) : "memory");
    const float *st = reinterpret_cast<const float *>(sm_raw + (base - raw) + (k % stages) * kStageBytes);
    for (int u = 0; u < kRows / 8; ++u) acc += st[(warp + 8 * u) * kRowSlot + lane];
  }
  if (acc == 12345.f) *sink = acc;
}

// 16-byte cp.async.cg of the 16-byte-aligned window around each row segment (9 x 16 B for a
// 2-element misalignment), 1152 copies per chunk spread over the 256 threads
template <int AHEAD>
__global__ void __launch_bounds__(256, 1) async16win_kernel(const float *m, int64_t rows, int64_t cols,
                                                            int chunks_per_cta, float *sink) {
  constexpr int stages = AHEAD + 1;
  constexpr int kWin = 9;   // 16-byte pieces per row window
  extern __shared__ unsigned char sm_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(sm_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  const int tid = threadIdx.x;
  const int64_t ncc = (cols + kCols - 1) / kCols;
  const int64_t nb = (rows + kRows - 1) / kRows;
  float acc = 0.f;
  auto issue = [&](int64_t k, int s) {
    if (k < chunks_per_cta) {
      const int64_t c = blockIdx.x + k * gridDim.x;
      const int64_t band = (c / ncc) % nb, cc = c % ncc;
      for (int p = tid; p < kRows * kWin; p += 256) {
        const int r = p / kWin, w = p - r * kWin;
        const int64_t row = band * kRows + r;
        const int64_t e0 = row * cols + cc * kCols;
        const uint64_t a0 = (reinterpret_cast<uint64_t>(m + e0) & ~15ull) + 16 * w;
        if (row < rows && a0 < reinterpret_cast<uint64_t>(m + rows * cols))
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + s * kStageBytes + (r * kRowSlot) * 4 + 16 * w),
                       "l"(a0)
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int k = 0; k < AHEAD; ++k) issue(k, k % stages);
  for (int k = 0; k < chunks_per_cta; ++k) {
    issue(k + AHEAD, (k + AHEAD) % stages);
    asm volatile("cp.async.wait_group %0;" ::"n"(AHEAD) : "memory");
    __syncthreads();
    const float *st = reinterpret_cast<const float *>(sm_raw + (base - raw) + (k % stages) * kStageBytes);
    for (int e = tid; e < kRows * kCols; e += 256) acc += st[(e / kCols) * kRowSlot + e % kCols + 2];
    __syncthreads();
  }
  if (acc == 12345.f) *sink = acc;
}

// the same with 8-byte cp.async.ca (rows 8-byte aligned when cols % 4 == 2): 16 lanes per row
template <int AHEAD>
__global__ void __launch_bounds__(256, 1) async8_kernel(const float *m, int64_t rows, int64_t cols,
                                                        int chunks_per_cta, float *sink) {
  constexpr int stages = AHEAD + 1;
  extern __shared__ unsigned char sm_raw[];
  const uint32_t raw = static_cast<uint32_t>(__cvta_generic_to_shared(sm_raw));
  const uint32_t base = (raw + 1023u) & ~1023u;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t ncc = (cols + kCols - 1) / kCols;
  const int64_t nb = (rows + kRows - 1) / kRows;
  float acc = 0.f;
  auto issue = [&](int64_t k, int s) {
    if (k < chunks_per_cta) {
      const int64_t c = blockIdx.x + k * gridDim.x;
      const int64_t band = (c / ncc) % nb, cc = c % ncc;
      const int64_t col = cc * kCols + 2 * (lane & 15);
      for (int u = 0; u < kRows / 16; ++u) {
        const int r = 2 * warp + (lane >> 4) + 16 * u;
        const int64_t row = band * kRows + r;
        if (row < rows && col < cols)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(base + s * kStageBytes + (r * kRowSlot + 2 * (lane & 15)) * 4),
                       "l"(m + row * cols + col)
                       : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int k = 0; k < AHEAD; ++k) issue(k, k % stages);
  for (int k = 0; k < chunks_per_cta; ++k) {
    issue(k + AHEAD, (k + AHEAD) % stages);
    asm volatile("cp.async.wait_group %0;" ::"n"(AHEAD) : "memory");
    const float *st = reinterpret_cast<const float *>(sm_raw + (base - raw) + (k % stages) * kStageBytes);
    for (int u = 0; u < kRows / 16; ++u) {
      const int r = 2 * warp + (lane >> 4) + 16 * u;
      acc += st[r * kRowSlot + 2 * (lane & 15)] + st[r * kRowSlot + 2 * (lane & 15) + 1];
    }
  }
  if (acc == 12345.f) *sink = acc;
}

int main() {
  const int64_t rows = 7174, cols = 7174;
  float *m, *sink;
  cudaMalloc(&m, rows * cols * 4 + 64);
  cudaMalloc(&sink, 4);
  cudaMemset(m, 0, rows * cols * 4);
  const int64_t chunks = ((rows + kRows - 1) / kRows) * ((cols + kCols - 1) / kCols);
  const int cpc = static_cast<int>(chunks / 148);
  const double bytes = static_cast<double>(cpc) * 148 * kRows * kCols * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char *name, int stages, auto launch) {
    const int smem = stages * kStageBytes + 1024 + 256;
    launch(smem);
    cudaEventRecord(e0);
    for (int i = 0; i < 5; ++i) launch(smem);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t e = cudaGetLastError();
    printf("{\"feed\": \"%s\", \"stages\": %d, \"GBps\": %.1f, \"err\": \"%s\"}\n", name, stages,
           bytes / (ms / 5 * 1e-3) / 1e9, cudaGetErrorString(e));
  };
  for (int st : {4, 6, 8}) {
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, st * kStageBytes + 1280);
    run("bulk", st, [&](int smem) { bulk_kernel<<<148, 256, smem>>>(m, rows, cols, st, cpc, sink); });
  }
  for (int st : {4, 8}) {
    cudaFuncSetAttribute(async4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, st * kStageBytes + 1280);
    run("async4_wait0", st, [&](int smem) { async4_kernel<<<148, 256, smem>>>(m, rows, cols, st, cpc, sink); });
  }
  cudaFuncSetAttribute(async4w_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kStageBytes + 1280);
  run("async4_ahead3", 4, [&](int smem) { async4w_kernel<3><<<148, 256, smem>>>(m, rows, cols, cpc, sink); });
  cudaFuncSetAttribute(async4w_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kStageBytes + 1280);
  run("async4_ahead7", 8, [&](int smem) { async4w_kernel<7><<<148, 256, smem>>>(m, rows, cols, cpc, sink); });
  cudaFuncSetAttribute(async16win_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kStageBytes + 1280);
  run("async16win_ahead3", 4, [&](int smem) { async16win_kernel<3><<<148, 256, smem>>>(m, rows, cols, cpc, sink); });
  cudaFuncSetAttribute(async16win_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kStageBytes + 1280);
  run("async16win_ahead7", 8, [&](int smem) { async16win_kernel<7><<<148, 256, smem>>>(m, rows, cols, cpc, sink); });
  cudaFuncSetAttribute(async8_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kStageBytes + 1280);
  run("async8_ahead3", 4, [&](int smem) { async8_kernel<3><<<148, 256, smem>>>(m, rows, cols, cpc, sink); });
  cudaFuncSetAttribute(async8_kernel<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * kStageBytes + 1280);
  run("async8_ahead7", 8, [&](int smem) { async8_kernel<7><<<148, 256, smem>>>(m, rows, cols, cpc, sink); });
  return 0;
}
