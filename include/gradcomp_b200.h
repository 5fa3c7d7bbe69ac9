/*
 * gradcomp_b200.h -- C ABI of the B200-native gradient-compression engine.
 *
 * Drop-in boundary: the reference `gradcomp` package (pure NumPy) has no FFI;
 * its seam is the Python class `GradientPipeline` (pkg/src/gradcomp/pipelines.py:97-393)
 * and the codec functions it calls.  Every entry point below replaces one
 * piece of that path and cites the reference code it restates.  The Python
 * package `paper_2407_01378_b200` binds these symbols with ctypes (see
 * INTEGRATION.md for the binding a maintainer of the reference would add).
 *
 * Conventions
 *  - Every device buffer is caller-owned (torch tensors in the Python host).
 *    The library never allocates device memory and never synchronises the host.
 *  - `stream` is a cudaStream_t passed as void*; all work is stream-ordered.
 *  - Return value: GC_OK (0) or a negative status; gc_last_error() gives a
 *    thread-local message.  Argument checks happen before any launch.
 *  - Reentrant: no mutable global state besides the per-thread error string.
 */
#ifndef GRADCOMP_B200_H
#define GRADCOMP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GC_OK 0
#define GC_ERR_INVALID (-1)
#define GC_ERR_CUDA (-2)
#define GC_ERR_UNSUPPORTED (-3)

/* numpy PCG64 BitGenerator state (128-bit LCG state and increment). */
typedef struct gc_pcg64 {
  uint64_t state_hi, state_lo, inc_hi, inc_lo;
} gc_pcg64;

int gc_version(void);
const char *gc_last_error(void);

/* ---------------------------------------------------------------- seeding
 * vectors.py:26-39 (splitmix64, fnv1a64), vectors.py:64-76 (SeedSpec.stream_seed / rng)
 * plus numpy's SeedSequence -> PCG64 initialisation (numpy 2.3, bit_generator.pyx /
 * pcg64.c), restated natively so kernels can regenerate the reference's draws. */
uint64_t gc_splitmix64(uint64_t value);
uint64_t gc_fnv1a64(const char *text, size_t len);
/* worker < 0 means "no worker component" (shared stream). */
uint64_t gc_stream_seed(uint64_t experiment_seed, const char *tag, size_t tag_len,
                        uint64_t round_index, int64_t worker);
/* np.random.PCG64(seed).state  (SeedSequence(seed) -> pcg64_set_seed). */
void gc_pcg64_from_seed(uint64_t seed, gc_pcg64 *out);
/* bit_generator.advance(delta) with delta = (delta_hi << 64) | delta_lo. */
void gc_pcg64_advance(gc_pcg64 *g, uint64_t delta_hi, uint64_t delta_lo);
/* next_uint64 (step, then XSL-RR output). */
uint64_t gc_pcg64_next(gc_pcg64 *g);


/* ---------------------------------------------------------------- round utilities */
/* GradientPipeline._checked (pipelines.py:184-197): *count += number of non-finite
 * entries of a [rows][cols] f32 matrix with leading dimension ld. */
int gc_check_finite(int64_t rows, const float *data, int64_t ld, int64_t cols, int64_t *count, void *stream);
/* RoundResult.nmse (pipelines.py:172-179, metrics.py:22-37): with ref = fp64 mean over the
 * n corrected inputs (g + resid, resid may be NULL), acc[0] += sum (est-ref)^2, acc[1] += sum ref^2. */
int gc_nmse_accumulate(int32_t n, int64_t d, const float *grads, const float *resid, int64_t ld,
                       const float *estimate, double *acc, void *stream);

/* ---------------------------------------------------------------- THC
 * RotatedQuantConfig round: pipelines.py:260-322. */
typedef struct gc_thc_geom {
  int64_t dim;        /* logical length d */
  int64_t padded;     /* P = next power of two >= d (pipelines.py:263, transforms.py:74-83) */
  int64_t block;      /* rotation block B = min(rotation_block, P) (transforms.py:78) */
  int32_t quant_bits; /* q (compressors.py:92) */
  int32_t wire_bits;  /* b, saturating aggregation width (compressors.py:94) */
  double scale;       /* float(B) ** -0.5 (transforms.py:116) */
} gc_thc_geom;

/* Coordinates that can hold non-zero data: ceil(d/B)*B.  Blocks past it are
 * all-zero in every worker: range (0,0), code 0, decode 0. */
int64_t gc_thc_active_len(const gc_thc_geom *g);
/* Device scratch (bytes) the THC entry points need for L workers (0 when B <= 4096). */
int64_t gc_thc_workspace_bytes(const gc_thc_geom *g, int32_t workers);

/* Rotation signs for one round as a bitmask (bit i of word i/32 set <=> sign +1):
 * RotationSpec.for_round, transforms.py:60-83 (PCG64.integers(0,2,P), Lemire on u32 halves). */
int gc_thc_signs(const gc_pcg64 *rotation_stream, int64_t count, uint32_t *bits, void *stream);

/* Forward rotation of L workers: corrected = f32(g + r) (compressors.py:624-626),
 * x_rot = f32(fp64 blockwise WHT(signs * corrected) * scale) (transforms.py:86-117),
 * ranges[w][blk] = (min, max) (compressors.py:447-453).
 * grads/resid rows have leading dimension ld (elements); resid may be NULL (EF off).
 * x_rot: [L][active] f32 (may be NULL if only ranges are wanted), ranges: [L][nb][2] f32. */
int gc_thc_rotate(const gc_thc_geom *g, int32_t workers, const float *grads, const float *resid,
                  int64_t ld, const uint32_t *sign_bits, float *x_rot, float *ranges,
                  void *workspace, void *stream);

/* Elementwise min of lo / max of hi over L range tables (ElemMin/ElemMax,
 * collectives.py:146-161; order-free, exact). in: [L][nb][2], out: [nb][2]. */
int gc_range_consensus(int32_t workers, int64_t num_blocks, const float *ranges_in,
                       float *ranges_out, void *stream);

/* quantize_stochastic (compressors.py:456-498) for L workers on the shared grid.
 * coin_streams: host array of L PCG64 states ("stochastic-round", round, worker),
 * coin for coordinate i = (next64 at step i+1) >> 11 * 2^-53.
 * codes: [L][active] int8.  counters (device int64[4], accumulated):
 * [0] clamp count, [1] sum z, [2] sum z^2. */
int gc_thc_quantize(const gc_thc_geom *g, int32_t workers, const float *x_rot,
                    const float *shared_ranges, const gc_pcg64 *coin_streams, int8_t *codes,
                    int64_t *counters, void *stream);

/* Nibble wire of the distributed THC exchange for wire_bits <= 4 (codes and saturated sums in
 * [-7, 7]): two values per byte, element 2i low nibble, 2i+1 high; len even.  The transport then
 * carries the ledger's b = 4 bits per coordinate (collectives.py:209-233). */
int gc_pack_nibbles(int64_t len, const int8_t *codes, uint8_t *packed, void *stream);
int gc_unpack_nibbles(int64_t len, const uint8_t *packed, int8_t *codes, void *stream);
/* Ordered saturating fold (SatIntSum.combine in ring order, collectives.py:123-143,215-226):
 * for element e (global index offset+e) start worker s = floor((offset+e)/ring_block);
 * acc = z[s]; acc = clip(acc + z[(s+k)%n], +-(2^(bits-1)-1)) for k=1..n-1.
 * codes: n rows of `len` int8 with leading dimension ld.  sums: int8 (bits<=8),
 * int16 (bits<=16) or int32.  counters[0] += clip events. */
int gc_sat_fold(int32_t n, int64_t len, const int8_t *codes, int64_t ld, int64_t offset,
                int64_t ring_block, int32_t bits, void *sums, int64_t *clip_counter, void *stream);

/* Decode of summed codes: estimate = f32(f32(inv_WHT(f32(n*mu + delta*z_sum))) / n)
 * (dequantize_sum compressors.py:501-521, rht_inverse transforms.py:120-126,
 * pipelines.py:307-311).  sums element size is sum_bytes (1, 2 or 4). estimate: [d] f32. */
int gc_thc_decode_estimate(const gc_thc_geom *g, int32_t n, const void *sums, int32_t sum_bytes,
                           const float *shared_ranges, const uint32_t *sign_bits,
                           float *estimate, void *workspace, void *stream);

/* Own decode + error-feedback update for L workers (pipelines.py:312-318,168-170):
 * resid[w] = f32((g[w] + resid[w]) - inv_WHT(dequantize_sum(z_w, ranges, q, 1))).
 * codes: [L][active] int8.  When resid is NULL nothing is written (EF off). */
int gc_thc_decode_ef(const gc_thc_geom *g, int32_t workers, const int8_t *codes,
                     const float *shared_ranges, const uint32_t *sign_bits, const float *grads,
                     float *resid, int64_t ld, void *workspace, void *stream);


/* Per-rank THC round of the distributed pipeline (one rank's L local workers), split at the
 * reference round's two exchange points (pipelines.py:260-322).  Tiles are 1024 coordinates;
 * [tile_begin, tile_end) restricts a call to a segment (tile_end < 0: to the end), so the host
 * can run K1 of segment s+1 while segment s's range all-reduce is in flight and K2 of segment s
 * re-reads g and r from L2.  Requires 32 <= B <= 1024, 1 <= L <= 16.
 *
 * K1 gc_thc_rank_ranges: corrected = f32(g + r), signs, fp64 WHT, per-block (min, max) stored as
 *    (-lo, hi) pairs: neg_ranges [L][nb][2] (nb = active / B), ready for one MAX all-reduce
 *    (ElemMin/ElemMax consensus, pipelines.py:271-288).  gc_thc_merge_ranges folds L tables.
 * K2 gc_thc_rank_quant: with the consensus table shared_neg_ranges [nb][2] (-lo, hi): the same
 *    rotation again, quantize_stochastic with worker l's coin stream coin_streams[l]
 *    (compressors.py:456-498), codes written straight into the all-to-all send buffer
 *    [W][L][slice] (slice a multiple of 1024; nibble != 0: packed nibbles, element 2i low, for
 *    wire_bits <= 4), then own decode + ef_update: resid_out = corrected - inv_WHT(dq(z, 1))
 *    (pipelines.py:312-318, 168-170; resid_in/out may alias; both NULL = EF off).
 *    counters[1] += sum z, counters[2] += sum z^2.
 * K3 gc_thc_rank_decode: estimate = f32(inv_WHT(f32(n mid + step z_sum)) * signs) / n
 *    (dequantize_sum + rht_inverse + / n, pipelines.py:307-311) from the all-gathered saturated
 *    sums (sum_bytes 1, 2 or 4; >= ceil(active/1024)*1024 entries, 16-byte aligned).
 * All three reproduce the reference bit for bit (codes, sums, residuals, estimate). */
int gc_thc_rank_ranges(const gc_thc_geom *g, int32_t L, const float *grads, const float *resid, int64_t ld,
                       int64_t tile_begin, int64_t tile_end, const uint32_t *sign_bits, float *neg_ranges,
                       void *stream);
/* K1 with the rotation signs drawn inside it: the words of tiles [tile_begin, tile_end) are generated
 * from rotation_stream exactly as gc_thc_signs would (transforms.py:80-82) and written to sign_bits
 * for K2 / K3 -- no separate gc_thc_signs pass over the vector. */
int gc_thc_rank_ranges_signs(const gc_thc_geom *g, int32_t L, const float *grads, const float *resid, int64_t ld,
                             int64_t tile_begin, int64_t tile_end, const gc_pcg64 *rotation_stream,
                             uint32_t *sign_bits, float *neg_ranges, void *stream);
int gc_thc_merge_ranges(int32_t L, int64_t num_blocks, const float *neg_ranges_in, float *neg_ranges_out,
                        void *stream);
int gc_thc_rank_quant(const gc_thc_geom *g, int32_t L, const float *grads, const float *resid_in, float *resid_out,
                      int64_t ld, int64_t tile_begin, int64_t tile_end, const uint32_t *sign_bits,
                      const float *shared_neg_ranges, const gc_pcg64 *coin_streams, int8_t *send, int64_t slice,
                      int32_t nibble, int64_t *counters, void *stream);
int gc_thc_rank_decode(const gc_thc_geom *g, int32_t n, const void *sums, int32_t sum_bytes,
                       const float *shared_neg_ranges, const uint32_t *sign_bits, float *estimate, void *stream);

/* ---------------------------------------------------------------- float ring folds
 * FloatSum ring_all_reduce (collectives.py:112-120, 177-236) as an ordered fold per element:
 * element e (global index offset+e) starts at worker (offset+e)/ring_block and folds in ring
 * order; wire_fp16 rounds every transmitted partial and the final value through binary16
 * (fp16_round_trip, vectors.py:136-152); round_inputs first rounds the inputs to fp16
 * (DenseConfig(16), pipelines.py:373); divisor > 0 divides the result (estimate = sum / n).
 * Used for the dense FP16/FP32 baselines (pipelines.py:370-393), TopK-Chunked's norm and chunk
 * aggregation (pipelines.py:224-244) and PowerSGD's factor sums (pipelines.py:327-363). */
int gc_float_fold(int32_t n, int64_t len, const float *inputs, int64_t ld, int64_t offset, int64_t ring_block,
                  int32_t wire_fp16, int32_t round_inputs, int32_t divisor, float *out, void *stream);
/* Batched form: B independent folds, inputs [B][n][len] (row stride ld, batch stride
 * in_stride), outputs [B][len] (batch stride out_stride). */
int gc_float_fold_batched(int32_t batch, int32_t n, int64_t len, const float *inputs, int64_t ld, int64_t in_stride,
                          int32_t wire_fp16, int32_t round_inputs, int32_t divisor, float *out, int64_t out_stride,
                          void *stream);
/* The batched fold of a slice: elements [offset, offset + len) of B same-length ring reductions
 * whose ring blocks are ring_block long (element i starts at worker floor(i / ring_block)); inputs
 * hold only the slice.  The per-tensor factor exchange of chunked PowerSGD across ranks. */
int gc_float_fold_batched_slice(int32_t batch, int32_t n, int64_t len, const float *inputs, int64_t ld,
                                int64_t in_stride, int64_t offset, int64_t ring_block, int32_t wire_fp16,
                                int32_t round_inputs, int32_t divisor, float *out, int64_t out_stride, void *stream);
/* Dense-fp32 bypass of many small tensors in one launch (pipelines.py:326-336): for segment s
 * (offsets/lengths device int64 [nseg]) of the flat [n][ld] corrected vectors, estimate =
 * ring-ordered fp32 sum / n, and resid = 0 there (own == corrected; resid may alias corrected
 * or be NULL). */
int gc_segment_fold_ef(int32_t n, int32_t nseg, const int64_t *seg_off, const int64_t *seg_len,
                       const float *corrected, float *resid, int64_t ld, float *estimate, void *stream);
/* Same with ef_apply fused (compressors.py:624-626): corrected = f32(grads + resid) is formed in
 * the kernel; resid (required) leaves as 0 on the segments. */
int gc_segment_ef_fold(int32_t n, int32_t nseg, const int64_t *seg_off, const int64_t *seg_len,
                       const float *grads, float *resid, int64_t ld, float *estimate, void *stream);
/* out = in / divisor (f32, may alias). */
int gc_scale_div(int64_t len, const float *in, int32_t divisor, float *out, void *stream);
/* FP16 bar across ranks (pipelines.py:370-393 with NCCL's half sum standing in for the ring):
 * gc_fold_to_half folds this rank's L rows [L][ld] with fp16 inputs and fp16 wire per hop into
 * binary16 (out_half: uint16 [len]); after the NCCL half all-reduce, gc_half_mean_sat maps the
 * sums back to f32 / divisor, saturating partial sums that overflowed to +-inf to +-65504 as the
 * reference's fp16 wire does (vectors.py:136-152). */
int gc_fold_to_half(int32_t L, int64_t len, const float *inputs, int64_t ld, void *out_half, void *stream);
int gc_half_mean_sat(int64_t len, const void *in_half, int32_t divisor, float *out, void *stream);
/* out = fp16_round_trip(in) (vectors.py:136-152; may alias). */
int gc_fp16_round(int64_t len, const float *in, float *out, void *stream);

/* ---------------------------------------------------------------- TopK
 * topk_indices / topk_compress (compressors.py:387-403): per row, the k largest |x| with the
 * lower index winning ties, emitted in ascending index order (idx_out [L][k] int32) with the
 * values (val_out [L][k], optional; fp16-rounded with GC_TOPK_FP16_VALUES).
 * Values come from `values`, or when values is NULL from grads (+ resid): with resid != NULL the
 * selection is fused with ef_apply and the corrected vector f32(g + r) is written over resid.
 * GC_TOPK_EF_UPDATE (needs grads + resid) also applies ef_update in place (compressors.py:629-631:
 * resid[i] -= val at the selected i), so resid leaves as r_new and gc_sparse_ef_update is not needed.
 * The workspace carries the previous call's boundary radix bin as a hint (zero it before first use;
 * any content is safe): when a call's boundary bin is at or above (hint - 1), the candidate
 * collection rides on the level-0 pass and the second full-row pass is skipped. */
#define GC_TOPK_FP16_VALUES 1
#define GC_TOPK_EF_UPDATE 2
int64_t gc_topk_workspace_bytes(int32_t workers, int64_t len);
int gc_topk_select(int32_t workers, int64_t len, const float *values, int64_t ld, int64_t k, const float *grads,
                   float *resid, int32_t *idx_out, float *val_out, int32_t flags, void *workspace,
                   void *stream);
/* TopK aggregation (pipelines.py:206-209): estimate = 0; estimate[idx_w] += val_w for w in
 * worker order (f32, the np.add.at order).  Dividing by n is gc_scale_div. */
int gc_sparse_accumulate(int32_t workers, int64_t k, const int32_t *idx, const float *val, int64_t dim,
                         float *estimate, void *stream);
/* The same aggregation with the mean in one dense pass: estimate = (worker-order f32 sums) /
 * divisor, every coordinate written once (pipelines.py:204-211).  idx ascending per worker (as
 * gc_topk_select emits); workspace: gc_sparse_mean_workspace_bytes (per-tile entry starts). */
int64_t gc_sparse_mean_workspace_bytes(int32_t workers, int64_t dim);
int gc_sparse_mean(int32_t workers, int64_t k, const int32_t *idx, const float *val, int64_t dim, int32_t divisor,
                   float *estimate, void *workspace, void *stream);
/* QuantPayload wire bytes (compressors.py:305-317) for L workers: row w = <B 3><B quant_bits>
 * <I block_size><I num_codes><I num_blocks> codes[w] (int8, num_codes; entries past codes_len are 0)
 * ranges (f32 [num_blocks][2], shared; blocks past ranges_len are (0, 0)) <Q rotation_id>.
 * Rows are gc_quant_payload_nbytes(num_codes, num_blocks) bytes at `stride`. */
int64_t gc_quant_payload_nbytes(int64_t num_codes, int64_t num_blocks);
int gc_encode_quant_payloads(int32_t workers, int32_t quant_bits, int64_t block_size, int64_t num_codes,
                             const int8_t *codes, int64_t codes_ld, int64_t codes_len, int64_t num_blocks,
                             const float *ranges, int64_t ranges_len, uint64_t rotation_id, uint8_t *out,
                             int64_t stride, void *stream);
/* ef_update with a sparse own payload (compressors.py:629-631, 406-409): resid[w][idx] -= val. */
int gc_sparse_ef_update(int32_t workers, int64_t k, const int32_t *idx, const float *val, float *resid, int64_t ld,
                        void *stream);

/* ---------------------------------------------------------------- TopK-Chunked
 * _round_chunked building blocks (pipelines.py:213-258).  `perm` (nullable, int64 [d]) is the
 * shared coordinate permutation of the ablation (transforms.py:129-151): the chunked vector is
 * work[i] = vals[perm[i]] and results are scattered back through it. */
/* ef_apply (compressors.py:624-626): out[w] = f32(g[w] + resid[w]) (resid NULL: copy). */
int gc_ef_apply(int32_t workers, int64_t d, const float *grads, const float *resid, int64_t ld, float *out,
                int64_t ld_out, void *stream);
/* fp16(f32(chunk_sq_norms)) per worker (vectors.py:180-192, pipelines.py:221-223), numpy's
 * pairwise fp64 order: norms [L][ceil(d/chunk)]. */
int gc_chunk_norms(int32_t workers, int64_t d, int64_t chunk, const float *vals, int64_t ld, const int64_t *perm,
                   float *norms, void *stream);
/* Same norms with ef_apply fused (no permutation, chunk % 8 == 0, chunk <= 128): corrected =
 * f32(g + r) is written over resid (resid NULL: EF off, norms of g). */
int gc_chunk_norms_ef(int32_t workers, int64_t d, int64_t chunk, const float *grads, float *resid, int64_t ld,
                      float *norms, void *stream);
/* chunk_values (compressors.py:417-430): packs[w][j*chunk + t] = fp16(work_w[sel[j]*chunk + t]). */
int gc_chunk_pack(int32_t workers, int64_t d, int64_t chunk, int64_t selected, const int32_t *sel,
                  const float *vals, int64_t ld, const int64_t *perm, float *packs, void *stream);
/* chunkset_to_dense / n (compressors.py:433-438, pipelines.py:246-247): estimate zeroed, then
 * estimate[sel[j]*chunk + t] = summed[j*chunk + t] / divisor. */
int gc_chunk_scatter(int64_t d, int64_t chunk, int64_t selected, const int32_t *sel, const float *summed,
                     int32_t divisor, const int64_t *perm, float *estimate, void *stream);
/* ef_update with own = the worker's chunk values (pipelines.py:248-251, 168-170): resid holds the
 * corrected vector; resid[w][sel chunk coords] -= packs[w]. */
int gc_chunk_ef_update(int32_t workers, int64_t d, int64_t chunk, int64_t selected, const int32_t *sel,
                       const float *packs, const int64_t *perm, float *resid, int64_t ld, void *stream);

/* ---------------------------------------------------------------- PowerSGD
 * _round_powersgd (pipelines.py:324-368).  Matrices are the corrected vectors zero-padded to
 * rows x cols (matrix_shape_for, compressors.py:530-548), row-major.  Supported ranks: 1..8, 16.
 * Products accumulate in fp64 and round to f32.
 *
 * A batch is T independent tensors of the same length d (so the same rows x cols), each with L
 * workers: virtual row v = t*L + w.  Row v of M starts at row_offsets[v] in the flat buffers
 * (device int64, e.g. tensor t's slice of worker w's flat gradient) or at v*ld when row_offsets
 * is NULL (the single-matrix reference path: T = 1).  Factors are per tensor: Q [T][cols][r]
 * (mq input), P [T*L][rows][r], P_hat [T][rows][r], Q_w [T*L][cols][r], Q_sum [T][cols][r];
 * tensor t's estimate starts at est_offsets[t] (NULL: 0).  This is the "chunked PowerSGD" of
 * one reference pipeline per layer tensor, batched by shape. */
typedef struct gc_psgd_batch {
  int32_t tensors;
  int32_t workers;
  const int64_t *row_offsets;
  int64_t ld;
  const int64_t *est_offsets;
  int32_t rows_aligned;   /* 1 if every row start (and the estimate slices) is 16-byte aligned */
  int32_t est_accumulate; /* decode: estimate += P_hat Q_sum^T / n instead of = (rank chunks after the first) */
} gc_psgd_batch;

int gc_psgd_splits(int32_t rows_total, int64_t cols);
int64_t gc_psgd_workspace_bytes(int32_t rows_total, int64_t rows, int64_t cols, int32_t rank);
int gc_psgd_vectorizable(int64_t cols, const void *a, const void *b, int64_t ld);
/* P_w = M_w Q (pipelines.py:348). */
int gc_psgd_mq(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
               const float *q, float *p, void *stream);
/* ef_apply fused into P = M Q (cols % 4 == 0, 16-byte aligned rows): corrected f32(g + r) is
 * written over resid (when non-NULL) in the same pass; split-K partials in the workspace. */
int gc_psgd_mq_fused(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                     float *resid, const float *q, float *p, void *workspace, void *stream);
/* TMA-fed tcgen05 P = M Q with ef_apply, and the previous round's EF update deferred into it
 * (pipelines.py:348 with compressors.py:624-631).  With ef_p_hat / ef_q_workers NULL: resid holds
 * the residuals r and corrected f32(g + r) is written over them (as gc_psgd_mq_fused).  With the
 * previous round's factors: resid holds that round's corrected matrices c_prev, and the pass uses
 * r = f32(c_prev - P_hat_prev Q_w_prev^T) (gc_psgd_decode's arithmetic, bit for bit) -- the
 * decode then only writes the estimate (gc_psgd_decode with resid NULL), and a residual read in
 * between materialises r with gc_psgd_decode(..., resid, NULL).  One tensor (row_offsets NULL),
 * cols % 4 == 0, ld % 4 == 0, 16-byte aligned rows, d >= cols, rank 1..8 or 16:
 * gc_psgd_mq_tma_supported; GC_ERR_UNSUPPORTED otherwise. */
int gc_psgd_mq_tma_supported(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank,
                             const void *grads, const void *resid);
int gc_psgd_mq_deferred(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *grads,
                        float *resid, const float *q, const float *ef_p_hat, const float *ef_q_workers, float *p,
                        void *workspace, void *stream);
/* The same for a batch of T same-shape tensors (chunked PowerSGD: one group per matrix shape; row
 * v = t * workers + w at row_offsets[v] = w * ld + host_tensor_offsets[t]): one tensor map per
 * tensor (the host needs the tensor offsets, host_tensor_offsets[T]; each a multiple of 4). */
int gc_psgd_mq_tma_supported_batched(const gc_psgd_batch *b, const int64_t *host_tensor_offsets, int64_t d,
                                     int64_t rows, int64_t cols, int32_t rank, const void *grads, const void *resid);
int gc_psgd_mq_deferred_batched(const gc_psgd_batch *b, const int64_t *host_tensor_offsets, int64_t d, int64_t rows,
                                int64_t cols, int32_t rank, const float *grads, float *resid, const float *q,
                                const float *ef_p_hat, const float *ef_q_workers, float *p, void *workspace,
                                void *stream);
/* 1 when gc_psgd_mq_deferred_batched accepts the layout: TMA-fed as above, or -- for row pitches a
 * tensor map cannot describe (cols % 4 != 0, unaligned tensor starts) -- fed by 4-byte cp.async
 * (any 4-byte aligned grads / resid, row_offsets or ld, rank 1..8 or 16; host_tensor_offsets may
 * then be NULL).  Same arithmetic, same outputs. */
int gc_psgd_mq_deferred_supported(const gc_psgd_batch *b, const int64_t *host_tensor_offsets, int64_t d,
                                  int64_t rows, int64_t cols, int32_t rank, const void *grads, const void *resid);
/* Q_w = M_w^T P_hat (pipelines.py:354). */
int gc_psgd_mtp(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, const float *c,
                const float *p_hat, float *q, void *workspace, void *stream);
/* The same for a batch of T same-shape tensors with row offsets, given the host copy of the tensor
 * offsets (host_tensor_offsets[T], as gc_psgd_mq_deferred_batched): one tensor map per tensor when
 * the rows are 16-byte aligned; NULL (or unaligned rows) takes the cp.async-fed pass. */
int gc_psgd_mtp_batched(const gc_psgd_batch *b, const int64_t *host_tensor_offsets, int64_t d, int64_t rows,
                        int64_t cols, int32_t rank, const float *c, const float *p_hat, float *q, void *workspace,
                        void *stream);
/* Q_w = M_w^T P_hat (pipelines.py:354) fused with the EF update r_w = c_w - P_hat Q_w^T
 * (pipelines.py:357-361, the own-decode half of gc_psgd_decode): resid holds the corrected
 * matrices on entry and the residuals on return, q receives Q_w.  One read and one write of M
 * (a 16-CTA cluster per 32-column strip, partial Q summed over distributed shared memory).
 * GC_ERR_UNSUPPORTED unless gc_psgd_mtp_ef_supported(rows, cols, rank, rows_aligned).
 * Moves the algorithmic bytes only, but measured slower than gc_psgd_mtp + gc_psgd_decode on
 * B200 (strided 128-byte segments); the host uses it only with GC_PSGD_MTP_EF=1. */
int gc_psgd_mtp_ef_supported(int64_t rows, int64_t cols, int32_t rank, int32_t rows_aligned);
int gc_psgd_mtp_ef(const gc_psgd_batch *b, int64_t d, int64_t rows, int64_t cols, int32_t rank, float *resid,
                   const float *p_hat, float *q, void *stream);
/* orthonormalize (compressors.py:555-588) for T tensors, rank <= 1024.  Ranks 1..8 and 16 first try
 * the Cholesky-QR fast path (fp64 Gram of P over the whole GPU, R = chol(G) whose pivots are MGS's
 * residual norms, P_hat = P R^-1) and keep it only when every pivot is far from the degeneracy
 * floor and from cancellation; every other tensor runs fp64 Gram-Schmidt (CGS2, the c dot products
 * of a column formed in one sweep) with the reference's canonical-basis completion; status[t] = 1
 * if completion failed (DegenerateMatrixError).  workspace: gc_psgd_orth_workspace_bytes. */
int64_t gc_psgd_orth_workspace_bytes(int32_t tensors, int64_t rows, int32_t rank);
int gc_psgd_orthonormalize(int32_t tensors, int64_t rows, int32_t rank, const float *p, float *p_hat, void *workspace,
                           int32_t *status, void *stream);
/* own_w = P_hat Q_w^T, resid_w -= own_w (resid holds the corrected matrix; NULL skips);
 * estimate = P_hat Q_sum^T / n (NULL skips) (pipelines.py:355, 365, 168-170). */
int gc_psgd_decode(const gc_psgd_batch *b, int32_t n, int64_t d, int64_t rows, int64_t cols, int32_t rank,
                   const float *p_hat, const float *q_workers, const float *q_sum, float *resid, float *estimate,
                   void *stream);
/* The same entry (kept for the fused call sites): both outputs in one pass over the rows, float4
 * accesses when cols % 4 == 0 and rows are 16-byte aligned, coalesced scalars otherwise. */
int gc_psgd_decode_fused(const gc_psgd_batch *b, int32_t n, int64_t d, int64_t rows, int64_t cols, int32_t rank,
                         const float *p_hat, const float *q_workers, const float *q_sum, float *resid, float *estimate,
                         void *stream);
/* gram[t] = Q_t^T Q_t in fp64 (rank check of ensure_full_rank, compressors.py:595-603), rank <= 1024;
 * workspace: gc_psgd_gram_workspace_bytes(tensors, rank) (column-slice partials, summed in order). */
int64_t gc_psgd_gram_workspace_bytes(int32_t tensors, int32_t rank);
int gc_psgd_gram(int32_t tensors, int64_t cols, int32_t rank, const float *q, double *gram, void *workspace,
                 void *stream);
/* cudaMemsetAsync wrapper (residual reset of the dense bypass, pipelines.py:336). */
int gc_fill_zero(void *ptr, int64_t bytes, void *stream);
/* rows x row_bytes strided copy in either direction (cudaMemcpy2DAsync): one PCIe transfer for the
 * same segment of all n worker rows of a host-fed round (pinned [n][d] host gradients). */
int gc_copy_rows_async(void *dst, int64_t dst_pitch, const void *src, int64_t src_pitch, int64_t row_bytes,
                       int64_t rows, void *stream);

/* SparsePayload wire bytes (encode_payload, compressors.py:292-297) for each worker's TopK
 * payload: out row w (stride >= 5 + 6k bytes) = <u8 1><u32 k><i32 idx[k]><f16 val[k]>, little endian. */
int gc_encode_sparse_payloads(int32_t workers, int64_t k, const int32_t *idx, const float *val, uint8_t *out,
                              int64_t stride, void *stream);

/* Whole THC round for n workers simulated on one GPU, fused into one kernel per
 * rotation block (pipelines.py:260-322 + EF 148-151,168-170): every CTA owns one block of
 * all n workers, so range consensus, quantization, the ring-ordered saturating fold,
 * the estimate decode and the own-decode + residual update never leave the SM.
 * Requires B <= 1024.  grads/resid: [n][ld] (resid NULL = EF off, updated in place);
 * estimate: [d]; codes: optional [n][active] int8; counters (device int64[4], accumulated):
 * [0] clamp count, [1] sum z, [2] sum z^2, [3] clip events; nmse_acc optional double[2]. */
int gc_thc_round_fused(const gc_thc_geom *g, int32_t n, const float *grads, float *resid, int64_t ld,
                       const uint32_t *sign_bits, const gc_pcg64 *coin_streams, float *estimate,
                       int8_t *codes, int64_t *counters, double *nmse_acc, void *stream);
/* The same round restricted to tiles [tile_begin, tile_end) of 1024 coordinates (tile_end < 0:
 * to the end), with the residual read from resid_in and written to resid_out (equal pointers:
 * in place).  Tiles are independent, so a host-fed round can stream: copy a segment of every
 * worker's gradient, run its tiles, copy its estimate back -- and keep the previous residual
 * intact until the whole round validated (pipelines.py:184-197 raises before any state change). */
int gc_thc_round_fused_range(const gc_thc_geom *g, int32_t n, const float *grads, const float *resid_in,
                             float *resid_out, int64_t ld, int64_t tile_begin, int64_t tile_end,
                             const uint32_t *sign_bits, const gc_pcg64 *coin_streams, float *estimate,
                             int8_t *codes, int64_t *counters, double *nmse_acc, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GRADCOMP_B200_H */
