/*
 * ckv.h — C-ABI of the B200-native Cocktail chunk-level KV-cache hot path.
 *
 * The reference's operator boundary is the Python facade `chunkkv.kernels`
 * (/root/reference/pkg/src/chunkkv/kernels/__init__.py:9-57) plus the callers
 * it serves (quantizer.py, retrieval.py, kv_store.py, attention.py).  Every
 * entry point below names the reference function it replaces.
 *
 * Conventions
 *   - All pointers are DEVICE pointers unless the name ends in `_host`.
 *   - No entry point allocates or synchronises; the caller owns every buffer
 *     (outputs and workspace) and passes the CUDA stream as `void* stream`.
 *   - Return 0 (CKV_OK) on success, a negative CKV_ERR_* on a bad argument.
 *     Data-dependent errors (non-finite input, zero-norm query, crossing
 *     thresholds) are reported through an int32 device flag word the caller
 *     reads after the stream completes (bits CKV_FLAG_*), mirroring the
 *     reference's ValueError sites.
 *   - Re-entrant per stream; one process per GPU.
 */
#ifndef CKV_H_
#define CKV_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes ------------------------------------------------------ */
#define CKV_OK 0
#define CKV_ERR_BITS (-1)        /* bitwidth not in {2,4}      (_core.pyx:21-24)      */
#define CKV_ERR_GROUP (-2)       /* group_size < 1            (_core.pyx:29-31)      */
#define CKV_ERR_SHAPE (-3)       /* dimension mismatch        (_core.pyx:156-159)    */
#define CKV_ERR_CAPACITY (-4)    /* count beyond packed words (_core.pyx:104-105)    */
#define CKV_ERR_UNSUPPORTED (-5) /* shape outside the specialised D=128/G=32 path    */
#define CKV_ERR_ARG (-6)         /* null pointer / negative size / bad alpha,beta    */
#define CKV_ERR_CUDA (-7)        /* kernel launch failed                             */

/* ---- device error-flag bits ---------------------------------------------- */
#define CKV_FLAG_NONFINITE 1     /* quantizer.py:71-72                      */
#define CKV_FLAG_ZERO_QUERY 2    /* retrieval.py:212-213                    */
#define CKV_FLAG_CROSSING 4      /* retrieval.py:231-234                    */
#define CKV_FLAG_EMPTY_SCORES 8  /* retrieval.py:225-226                    */
#define CKV_FLAG_NONFINITE_FP16 16 /* informational: inf/nan in a row copied to the FP16
                                      region (the reference accepts those, kv_store.py:199-202) */

/* tier codes (tiers.py:6-15) */
#define CKV_TIER_INT2 0
#define CKV_TIER_INT4 1
#define CKV_TIER_FP16 2

int32_t ckv_abi_version(void);
const char* ckv_status_string(int32_t status);

/* ======================================================================
 * Generic per-block kernels: the five callables of kernels/__init__.py:43-47.
 * float64 in / float64 out with the reference's expression trees, so codes,
 * words and metadata are bit-identical to _numpy.py / _core.pyx.
 * ==================================================================== */

/* kernels.quantize_groups (_numpy.py:27-67, _core.pyx:27-79).
 * x f64[rows, cols] row-major -> codes u8[rows*cols], scales/zero_points f64[rows*ceil(cols/gs)].
 * Sets CKV_FLAG_NONFINITE in *flag when x holds inf/nan (quantizer.py:71-72). */
int32_t ckv_quantize_groups_f64(const double* x, int64_t rows, int64_t cols, int32_t bits,
                                int64_t group_size, uint8_t* codes, double* scales,
                                double* zero_points, int32_t* flag, void* stream);

/* Same contract for float16 input (bit patterns as uint16); metadata still f64. */
int32_t ckv_quantize_groups_f16(const uint16_t* x, int64_t rows, int64_t cols, int32_t bits,
                                int64_t group_size, uint8_t* codes, double* scales,
                                double* zero_points, int32_t* flag, void* stream);

/* kernels.pack_codes (_numpy.py:70-86, _core.pyx:82-97): u8[n] -> u32[ceil(n*bits/32)]. */
int32_t ckv_pack_codes(const uint8_t* codes, int64_t n, int32_t bits, uint32_t* packed,
                       void* stream);

/* kernels.unpack_codes (_numpy.py:89-99, _core.pyx:100-116). */
int32_t ckv_unpack_codes(const uint32_t* packed, int64_t n_words, int32_t bits, int64_t count,
                         uint8_t* codes, void* stream);

/* kernels.dequantize_codes (_numpy.py:102-112, _core.pyx:119-145): zp + scale*code, no FMA. */
int32_t ckv_dequantize_codes_f64(const uint32_t* packed, int64_t n_words, const double* scales,
                                 const double* zero_points, int64_t rows, int64_t cols,
                                 int32_t bits, int64_t group_size, double* out, void* stream);

/* kernels.matmul_packed (_numpy.py:115-125, _core.pyx:148-192).
 * transpose!=0: out f64[m, rows] = a f64[m, cols] . deq^T ; else out f64[m, cols] = a[m, rows] . deq.
 * `accumulate`!=0 adds into out instead of overwriting (used to fuse the per-tier PV sum). */
int32_t ckv_matmul_packed_f64(const double* a, int64_t m, int64_t a_cols, int64_t lda,
                              const uint32_t* packed, int64_t n_words, const double* scales,
                              const double* zero_points, int64_t rows, int64_t cols, int32_t bits,
                              int64_t group_size, int32_t transpose, double* out, int64_t ldo,
                              int32_t accumulate, void* stream);

/* Dense f64 products used by attention.py:77,90,104,112 on the float regions:
 * transpose!=0: out[m, n] (+)= a[m, k] . b[n, k]^T ; else out[m, n] (+)= a[m, k] . b[k, n]. */
int32_t ckv_matmul_f64(const double* a, int64_t m, int64_t k, int64_t lda, const double* b,
                       int64_t n, int64_t ldb, int32_t transpose, double* out, int64_t ldo,
                       int32_t accumulate, void* stream);

/* attention.stable_softmax (attention.py:24-31) fused with `att *= scale; att += mask`
 * (attention.py:79-81).  x f64[m, n] in place; mask may be NULL. */
int32_t ckv_scale_mask_softmax_f64(double* x, int64_t m, int64_t n, double scale,
                                   const double* mask, void* stream);

/* kv_store.reconstruct scatter (kv_store.py:236-253): dst[order[r]] = src[r] rows of width cols. */
int32_t ckv_scatter_rows_f64(const double* src, int64_t rows, int64_t cols, const int64_t* order,
                             double* dst, void* stream);

/* ======================================================================
 * Batched hot path: fp16 K/V, head_dim 128, group 32, chunk 32.
 * ==================================================================== */

/* (0) Text encoders upstream of the search (retrieval.py:70-138).  They replace
 * the reference's per-text Python encode() calls (HashedBowEncoder.encode retrieval.py:87-100,
 * TfidfEncoder.encode retrieval.py:122-138) with one launch over all texts; the output rows are
 * ckv_search's emb / q inputs.
 * ckv_bow_encode: text = UTF-8 bytes of n_texts texts back to back, offsets i64[n_texts + 1]
 *   (device); key = HOST bytes of the BLAKE2b key (the seed's decimal ASCII), key_len <= 64;
 *   -> vectors f64[n_texts, dim], norms f64[n_texts] (1.0, or 0.0 for a text without words or
 *   with all buckets cancelled).  Words split at str.isspace() characters; dim <= 8192.
 *   Bit-identical to the reference.
 * ckv_tfidf_encode: vocabulary ids i32 (the caller maps words through the fitted sorted
 *   vocabulary, dropping unknown words), offsets i64[n_texts + 1], idf f64[vocab] -> vectors
 *   f64[n_texts, ld] (columns >= vocab zero), norms f64[n_texts].  Within a few ulp (the norm's
 *   summation order is not BLAS's). */
int32_t ckv_bow_encode(const uint8_t* text, const int64_t* offsets, int32_t n_texts, int32_t dim,
                       const uint8_t* key, int32_t key_len, double* vectors, double* norms,
                       void* stream);
int32_t ckv_tfidf_encode(const int32_t* ids, const int64_t* offsets, int32_t n_texts, const double* idf,
                         int32_t vocab, int32_t ld, double* vectors, double* norms, void* stream);

/* (1) Chunk-level quantization search (retrieval.py:199-250 + kv_store.py:190-206).
 * Per sequence b: cosine of q[b] with each chunk embedding (zero-norm chunks take the
 * minimum valid score, retrieval.py:217-219), thresholds (retrieval.py:222-237), strict
 * three-way tier rule (retrieval.py:240-250), stable INT2||INT4||FP16 permutation.
 *   emb f64[B, n_chunks, dim], emb_norm f64[B, n_chunks], q f64[B, dim], q_norm f64[B]
 *   -> scores f64[B, n_chunks], stats f64[B, 4] = (s_min, s_max, t_low, t_high),
 *      tiers u8[B, n_chunks], perm u32[B, n_chunks], seg_counts i32[B, 3], flags i32[B].
 * seq_chunks (nullable) i32[B]: per-sequence chunk count <= n_chunks (ragged batches).
 * emb == NULL selects the scores-given mode: `scores` is read as input and only
 * compute_thresholds / assign_tiers / the stable permutation run (retrieval.py:222-250). */
int32_t ckv_search(const double* emb, const double* emb_norm, const double* q,
                   const double* q_norm, const int32_t* seq_chunks, int32_t batch,
                   int32_t n_chunks, int32_t dim,
                   double alpha, double beta, double* scores, double* stats, uint8_t* tiers,
                   uint32_t* perm, int32_t* seg_counts, int32_t* flags, void* stream);

/* assign_tiers with caller-given thresholds (retrieval.py:240-250) plus the stable grouping:
 * scores f64[B, n_chunks] (read only), thresholds f64[B, 2] = (t_low, t_high)
 *   -> tiers u8[B, n_chunks], perm u32[B, n_chunks], seg_counts i32[B, 3], stats f64[B, 4],
 *      flags i32[B]. */
int32_t ckv_assign_tiers(const double* scores, const double* thresholds,
                         const int32_t* seq_chunks, int32_t batch, int32_t n_chunks,
                         uint8_t* tiers, uint32_t* perm, int32_t* seg_counts, double* stats,
                         int32_t* flags, void* stream);

/* Arena set for one of K or V over [layers, kv_heads]; rows are concatenated over the
 * batch (varlen; every segment starts at a multiple of 32 rows).  The quantized arenas are
 * TILE-NATIVE: each 16-row tile holds exactly the bits of the reference's row packing (one
 * D=128 row packs into 8 (INT2) / 16 (INT4) little-endian u32 words, _numpy.py:70-86) and
 * the rows' fp16 (lo, hi) group metadata, permuted (INT2: in bytes, INT4: in 16-bit pieces)
 * into the order the decode kernel's MMA fragments consume them: every 32-element group is its
 * own pair of k-steps (K) / m-tiles (V) (layout functions tile_byte_* / tile_off_* in
 * csrc/ckv_common.cuh; K and V tiles differ).  K and V share one interleaved tile buffer per
 * tier: tile t of the INT2 arenas is the 1536-byte block [K codes 512 | V codes 512 | K meta
 * 256 | V meta 256] at t * 1536 (INT4: 2560-byte blocks [K codes 1024 | V codes 1024 | K meta
 * 256 | V meta 256]), tiles indexed ([L][H] slab) * rows / 16 + row / 16.  So the K arena's
 * codes2 / meta2 point at block offsets 0 / 1024 and the V arena's at 512 / 1280 (INT4: 0 /
 * 2048 and 1024 / 2304); ckv_decode_attention checks this.  A decode tile is then one
 * contiguous block (3 / 5 coalesced 16-byte copies per lane).  ckv_arena_export restores
 * reference rows. */
typedef struct ckv_arena {
  uint32_t* codes2;   /* tile t at +t*1536: 512 B (16 rows x 8 u32)             */
  uint32_t* meta2;    /* tile t at +t*1536: 256 B (16 rows x 4 (lo, hi) half2)    */
  uint32_t* codes4;   /* tile t at +t*2560: 1024 B (16 rows x 16 u32)            */
  uint32_t* meta4;    /* tile t at +t*2560: 256 B                                 */
  uint16_t* fp;       /* fp16 [L][H][rows_fp][128] (FP16 chunks || tail || decode) */
  uint32_t* span_flags; /* u32 [L][H][B], zero-filled before build: bit0/bit1 set when an
                           INT2/INT4 group's scale exceeds 4000 (diagnostic; nullable) */
  uint32_t* span_max; /* f32 bits [L][H][B], zero-filled before build: the largest quantized
                         group span (hi - lo) of the unit's rows.  Decode sizes the unit's V
                         operand scaling 2^F from the V arena's (required there when the
                         arenas hold quantized rows; the K arena's is informational) */
  int64_t rows2, rows4, rows_fp;
} ckv_arena;

/* Per-sequence segment table (device, int32 [B][8]):
 *   off2, len2, off4, len4, off_fp, len_fp, tail_src, context_len
 * Offsets are rows into the arenas; len_fp grows with decode appends (kv_store.py:135-148).
 * context_len = 32 * (chunks in perm) + tail; tail_src is the source token index of the tail
 * (normally 32 * n_chunks; differs for a sequence-split shard that owns the global tail). */
#define CKV_SEQ_FIELDS 8

/* (2) Chunk-level reorder + quantize + pack (kv_store.build_cache, kv_store.py:169-219 with
 * quantizer.quantize / kernels.quantize_groups / pack_codes).  One pass over fp16 K and V:
 *   k, v fp16 element strides (layer, batch, token, head), all multiples of 8 (16-byte rows);
 *   head_dim contiguous; 0 < s_token <= INT32_MAX (CKV_ERR_UNSUPPORTED otherwise).
 *   perm u32[B, max_chunks] (from ckv_search), seq i32[B][8].
 * Writes codes/meta to the INT arenas and verbatim rows to the FP16 region (FP16-tier
 * chunks, then the context tail).  Sets CKV_FLAG_NONFINITE on inf/nan in a quantized (INT2 /
 * INT4) row, as quantizer.quantize does (quantizer.py:71-72); inf/nan in FP16-region rows only
 * sets the informational CKV_FLAG_NONFINITE_FP16. */
int32_t ckv_reorder_quantize_pack(const uint16_t* k, const uint16_t* v, int32_t layers,
                                  int32_t batch, int32_t kv_heads, int64_t s_layer,
                                  int64_t s_batch, int64_t s_token, int64_t s_head,
                                  const uint32_t* perm, int32_t max_chunks, const int32_t* seq,
                                  int32_t max_ctx, ckv_arena k_arena, ckv_arena v_arena,
                                  int32_t* flag, void* stream);

/* Decode-token append into the FP16 region (kv_store.append_decode_token, kv_store.py:222-224):
 * k_new, v_new fp16 [L][B][H][128]; each row lands at off_fp + len_fp of its sequence, then
 * len_fp += 1 (stream-ordered second kernel).  The caller checks len_fp < cap_fp on its host
 * mirror of the segment table before calling (capacity growth is a host decision). */
int32_t ckv_append_tokens(const uint16_t* k_new, const uint16_t* v_new, int32_t layers,
                          int32_t batch, int32_t kv_heads, int32_t* seq, ckv_arena k_arena,
                          ckv_arena v_arena, void* stream);

/* Arena metadata (lo, hi) fp16 pairs -> the reference's float64 scale = (hi - lo) / qmax and
 * zero_point = lo (quantize_groups, _numpy.py:65-66); exact because fp16 differences are exact
 * in f64.  Used to export arenas as reference QuantizedBlocks (quantizer.py:20-57). */
int32_t ckv_expand_meta(const uint32_t* meta, int64_t n_groups, int32_t bits, double* scales,
                        double* zero_points, void* stream);

/* kv_store.reconstruct + token_order (kv_store.py:227-253) on the tile-native arenas, on the
 * device: every row of layers [0, layers) of the arena views (ckv_arena at a layer offset), all
 * sequences and kv heads, dequantized as the reference's dequantize_codes does (zp + scale code
 * in f64, _numpy.py:102-112; FP16-region rows widened) and written to its ORIGINAL token position
 * t (the build permutation perm u32[batch][max_chunks]; the tail and decode tokens follow the
 * chunks in order): out_k / out_v f64 elements at l s_layer + b s_batch + t s_token + h s_head +
 * d (d contiguous); rows with t >= t_out are skipped.  max_rows = the largest len2 + len4 +
 * len_fp over the sequences. */
int32_t ckv_reconstruct(ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq, const uint32_t* perm,
                        int32_t max_chunks, int32_t layers, int32_t batch, int32_t kv_heads, int32_t max_rows,
                        double* out_k, double* out_v, int64_t s_layer, int64_t s_batch, int64_t s_token,
                        int64_t s_head, int32_t t_out, void* stream);

/* Tile-native arena rows -> reference format (export / verification, quantizer.py:20-57):
 * `rows` (a multiple of 16) rows starting at a tile boundary of one arena (codes + meta of
 * the K arena when is_v == 0, of the V arena otherwise; consecutive tiles `tile_stride` bytes
 * apart, 1536 / 2560 for the interleaved INT2 / INT4 buffers) -> out_codes u32 [rows][8 or 16]
 * (pack_codes row format, _numpy.py:70-86) and out_meta half2 (lo, hi) [rows][4]. */
int32_t ckv_arena_export(const uint32_t* codes, const uint32_t* meta, int64_t rows, int32_t bits,
                         int32_t is_v, int64_t tile_stride, uint32_t* out_codes,
                         uint32_t* out_meta, void* stream);

/* (3) Mixed-precision decode attention (attention.mixed_decode_attention, attention.py:63-90,
 * for every (layer, sequence, kv-head) unit at once).  q fp16 [L][B][H*m][128] (strides
 * q_s_layer, q_s_batch in elements; out strides o_s_layer, o_s_batch likewise multiples of 8,
 * out 16-byte aligned), m = q heads per kv head (1..8).  Online softmax over the
 * virtual sequence INT2 || INT4 || FP16 with split-KV; scale = softmax scale (1/sqrt(128)).
 * Output fp16 [L][B][H*m][128].  Workspace: ckv_decode_workspace_bytes() bytes, zero-filled
 * once before first use (it holds self-resetting split arrival counters; the last CTA of
 * each unit merges the split partials inside the same launch).  partial_out (nullable):
 * write unnormalised f32 [L][B][H*m][130] = (acc[128], m (log2 domain), l) instead of out,
 * for a cross-GPU split-KV merge with ckv_lse_merge. */
int64_t ckv_decode_workspace_bytes(int32_t layers, int32_t batch, int32_t kv_heads, int32_t m,
                                   int32_t splits);
/* Resident decode CTAs per SM on the current device (for sizing `splits` to whole waves). */
int32_t ckv_decode_ctas_per_sm(void);
#define CKV_DECODE_PDL 1  /* flags bit: launch as a programmatic dependent of the preceding
                             kernel, which must not write the quantized arenas or the immutable
                             seq fields (e.g. the previous layer's decode).  The kernel prefetches
                             its first K/V tiles, then waits on the preceding grid before it
                             reads q, len_fp or the FP16 region. */
int32_t ckv_decode_attention(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                             ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                             int32_t layers, int32_t batch, int32_t kv_heads, int32_t m,
                             float scale, int32_t splits, void* workspace, uint16_t* out,
                             int64_t o_s_layer, int64_t o_s_batch, float* partial_out,
                             int32_t flags, void* stream);
/* The same over sequences [seq_begin, seq_begin + seq_count) of the cache's `batch` only
 * (q, out, partial_out and the workspace keep their full-batch layout; a launch touches only
 * its sequences' rows and counters, so launches over disjoint sequence ranges may run
 * concurrently on different streams, e.g. two micro-batch chains of per-layer launches whose
 * layer boundaries overlap each other's work). */
int32_t ckv_decode_attention_seqs(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                                  ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                                  int32_t layers, int32_t batch, int32_t seq_begin, int32_t seq_count,
                                  int32_t kv_heads, int32_t m, float scale, int32_t splits,
                                  void* workspace, uint16_t* out, int64_t o_s_layer, int64_t o_s_batch,
                                  float* partial_out, int32_t flags, void* stream);
/* The same over kv heads [head_begin, head_begin + head_count) of sequences [seq_begin,
 * seq_begin + seq_count) (micro-batch chains over heads, e.g. a batch-1 128K context as 8
 * chains of 5 heads): rows of other heads and sequences in out / partial_out are left
 * untouched; the workspace is the whole cache's (ckv_decode_workspace_bytes), so concurrent
 * launches over disjoint ranges never share a counter. */
int32_t ckv_decode_attention_range(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                                   ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                                   int32_t layers, int32_t batch, int32_t seq_begin, int32_t seq_count,
                                   int32_t kv_heads, int32_t head_begin, int32_t head_count, int32_t m,
                                   float scale, int32_t splits, void* workspace, uint16_t* out,
                                   int64_t o_s_layer, int64_t o_s_batch, float* partial_out, int32_t flags,
                                   void* stream);

/* Warp-plan schedule of the same computation (whole-batch launches): unit u = b * kv_heads + h
 * of every layer takes unit_warps[u] >= 1 warps (their sum = 16 * ctas); CTA c (16 warps, one
 * per SM) runs warps [16c, 16c + 16).  ckv_decode_wp_plan builds, on the host from the host
 * copy of the seq table, the plan table the kernel reads (ckv_decode_wp_plan_ints(ctas) int32:
 * per-warp tile ranges, per-CTA unit slots; upload it to device memory) and returns max_slots
 * (the most units one CTA spans, <= 8; CKV_ERR_UNSUPPORTED above) and max_ctas (the most CTAs
 * one unit spans).  A warp's part of unit u is a contiguous share of the unit's tiles of each
 * kind; a unit split over several CTAs is merged by the first of its CTAs to finish its tiles
 * (bounded wait; on timeout the CTA completing the set merges).
 * Workspace: ckv_decode_wp_workspace_bytes(), zero-filled once.  Outputs as
 * ckv_decode_attention (out or partial_out). */
int64_t ckv_decode_wp_workspace_bytes(int32_t layers, int32_t batch, int32_t kv_heads, int32_t m,
                                      int32_t max_ctas);
/* Warps per CTA of the warp-plan kernel (16: one CTA per SM). */
int32_t ckv_decode_wp_cta_warps(void);
int64_t ckv_decode_wp_plan_ints(int32_t ctas);
int32_t ckv_decode_wp_plan(const int32_t* seq_host, int32_t batch, int32_t kv_heads,
                           const int32_t* unit_warps, int32_t ctas, int32_t* plan_host,
                           int32_t* max_slots, int32_t* max_ctas);
int32_t ckv_decode_attention_wp(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                                ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                                int32_t layers, int32_t batch, int32_t kv_heads, int32_t m, float scale,
                                const int32_t* plan, int32_t ctas, int32_t max_slots,
                                int32_t max_ctas, void* workspace, uint16_t* out, int64_t o_s_layer,
                                int64_t o_s_batch, float* partial_out, int32_t flags, void* stream);
/* The same over sequences [b0, b0 + n_seqs) of the cache (micro-batch chains: each range its own
 * chain of per-layer launches on its own stream): the plan is built from those rows of the seq
 * table (seq_host + 8 b0, batch n_seqs), the workspace sized for n_seqs; q / out keep the whole
 * batch's strides, rows outside the range are left untouched. */
int32_t ckv_decode_attention_wp_seqs(const uint16_t* q, int64_t q_s_layer, int64_t q_s_batch,
                                     ckv_arena k_arena, ckv_arena v_arena, const int32_t* seq,
                                     int32_t layers, int32_t batch, int32_t b0, int32_t n_seqs,
                                     int32_t kv_heads, int32_t m, float scale, const int32_t* plan,
                                     int32_t ctas, int32_t max_slots, int32_t max_ctas, void* workspace,
                                     uint16_t* out, int64_t o_s_layer, int64_t o_s_batch,
                                     float* partial_out, int32_t flags, void* stream);

/* Split-KV merge across ranks (new; the NCCL-exchanged partials of SURVEY §8e):
 * partials f32 [P][rows][128 + 2] = (acc[128] unnormalised at m, m (log2 domain), l);
 * out fp16 [rows][128].  o = sum_p acc_p 2^(m_p - m*) / sum_p l_p 2^(m_p - m*). */
int32_t ckv_lse_merge(const float* partials, int32_t n_parts, int64_t rows, uint16_t* out,
                      void* stream);
/* The same merge reading the P partial arrays through a device array of P pointers (each
 * [rows][130]): the ranks' symmetric-memory buffers, read over NVLink peer mappings after a
 * device-side barrier (distributed.P2PExchange) — no gathered copy, no NCCL collective. */
int32_t ckv_lse_merge_ptrs(const float* const* parts, int32_t n_parts, int64_t rows, uint16_t* out,
                           void* stream);

#ifdef __cplusplus
}
#endif

#endif /* CKV_H_ */
