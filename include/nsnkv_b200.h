/*
 * nsnkv_b200.h -- C ABI of the B200-native NSNQuant KV-cache hot path.
 *
 * Every entry point takes plain device pointers, element counts and an
 * explicit cudaStream_t (passed as void* so this header needs no CUDA
 * include).  Calls are stream-ordered and re-entrant; nothing blocks the host
 * except nsnkv_codebook_create (one upload).  Batch paths never fail on data:
 * clamps, zero sub-vectors and S3 fallbacks are counted, exactly like the
 * reference streaming cache (reference pkg/src/nsnkv/kvcache.py:191-194).
 *
 * Status codes mirror reference pkg/src/nsnkv/errors.py:4-29.
 *
 * Reference interfaces replaced (all paths relative to /root/reference/pkg):
 *   nsnkv_fwht_rows        -> src/nsnkv/kernels/__init__.py:31-32
 *                             (_native.pyx:16-38, _pyfallback.py:15-36)
 *   nsnkv_match_block      -> src/nsnkv/kernels/__init__.py:35-41 plus the
 *                             zero-row substitution of codebook.py:109-128
 *   nsnkv_codebook_create  -> codebook.py:71-106 (Codebook, inv_norms) and
 *                             kernels/__init__.py:44-51 (entry_inv_norms)
 *   nsnkv_rope_table       -> rope.py:29-51 (_pair_freqs, rope_rows angles)
 *   nsnkv_kmeans_assign,
 *   nsnkv_finetune_stats   -> codebook.py:175-340 (kmeans_init, finetune)
 *   nsnkv_encode_chunks    -> kvcache.py:114-154 (flush_chunk_keys/values):
 *                             nsn.py:68-85, rope.py:35-51, hadamard.py:65-83,
 *                             vq.py:211-279 in one kernel
 *   nsnkv_decode_scores    -> attention.py:83-111 (scores_quantized), batched
 *   nsnkv_decode_output    -> attention.py:114-133 (output_quantized), batched
 *   nsnkv_decode_attend    -> attention.py:136-142 (attend_quantized), fused
 *                             flash-decoding, batched over (batch, q-head)
 *   nsnkv_decode_step      -> kvcache.py:157-195 + attention.py:136-142: a
 *                             serving decode step (append without a flush,
 *                             then attend) in the attend launches
 *   nsnkv_append           -> kvcache.py:157-195 (append): residual policy,
 *                             flushes and bookkeeping of a batch of units
 *   nsnkv_pool_*, nsnkv_pages_copy -> (no reference counterpart: the
 *                             reference keeps chunks in Python lists) page
 *                             storage and kvcache.py:198-213 snapshot I/O
 */
#ifndef NSNKV_B200_H
#define NSNKV_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes (errors.py:4-29) ------------------------------------ */
#define NSNKV_OK 0
#define NSNKV_ERR_NON_POWER_OF_TWO (-1) /* NonPowerOfTwoDim   */
#define NSNKV_ERR_SHAPE (-2)            /* ShapeMismatch      */
#define NSNKV_ERR_INDEX (-3)            /* IndexOutOfRange    */
#define NSNKV_ERR_ZERO_VECTOR (-4)      /* ZeroVector         */
#define NSNKV_ERR_DEGENERATE (-5)       /* DegenerateProjection */
#define NSNKV_ERR_FORMAT (-6)           /* FormatError        */
#define NSNKV_ERR_CUDA (-7)             /* CUDA runtime error */
#define NSNKV_ERR_UNSUPPORTED (-8)      /* configuration outside the GPU path */

/* ---- fixed geometry of the GPU path ----------------------------------- */
#define NSNKV_HEAD_DIM 128   /* d (CacheConfig.d)                           */
#define NSNKV_CHUNK 64       /* residual_size R: tokens per flushed chunk   */
#define NSNKV_SUB_DIM 8      /* vq.py:25 SUB_DIM                            */
#define NSNKV_O_GROUP 32     /* vq.py:26 O_GROUP                            */

/* Packed page = one flushed chunk of one (batch, kv-head) unit.  Payload
 * bytes equal the reference bit ledger (vq.py:328-356): 2292 B (2-bit) and
 * 1268 B (1-bit); pages are padded to a multiple of 128 B.                  */
#define NSNKV_PAGE_BYTES_2B 2304
#define NSNKV_PAGE_BYTES_1B 1280
#define NSNKV_LEDGER_BYTES_2B 2292
#define NSNKV_LEDGER_BYTES_1B 1268

/* per-chunk event counters written by nsnkv_encode_chunks */
#define NSNKV_CNT_CLAMP 0      /* nsn.py:58-65 norm clamps (s1 and s2)      */
#define NSNKV_CNT_ZERO 1       /* codebook.py:118-127 zero sub-vectors      */
#define NSNKV_CNT_FALLBACK 2   /* vq.py:91-93 S3 -> norm-match fallbacks    */
#define NSNKV_CNT_NEARTIE 3    /* sub-vectors re-scored in exact fp64       */
#define NSNKV_NUM_COUNTERS 4

/* ScaleStrategy (vq.py:31-48) */
#define NSNKV_STRATEGY_NONE 0
#define NSNKV_STRATEGY_MIN_L2 1
#define NSNKV_STRATEGY_NORM_MATCH 2
#define NSNKV_STRATEGY_PARALLEL 3

int nsnkv_version(void);
/* Human-readable text of the last error raised on the calling thread. */
const char *nsnkv_last_error(void);
/* Number of kernels this library launched since load (for the bench's
 * gpu_launches evidence). */
int64_t nsnkv_launch_count(void);

/* ---- level 1: the kernel plug-in (kernels/__init__.py:31-41) ---------- */

/* Orthonormal Walsh-Hadamard transform of each row of in[n, d] (fp32,
 * row-major) into out (may alias in).  d must be a power of two, 2..4096. */
int nsnkv_fwht_rows(const float *in, float *out, int64_t n, int32_t d,
                    void *stream);

/* Cosine argmax of each 8-dim row of vecs[m, 8] against entries[256, 8],
 * scored exactly like _native.pyx:61-84 (fp64, component order, strict >).
 * fold != 0 folds |v| and writes sign bytes; signs may be NULL when
 * fold == 0.  With zero_mask == NULL this is the bare kernel
 * (_native.pyx:41-87).  With a zero_mask buffer it is codebook.match_block
 * (codebook.py:109-128): rows with fp64 |v|^2 < 1e-24 are substituted by
 * index 0 / sign 0 and flagged.  n_neartie (device int64, may be
 * NULL) receives += the number of rows that needed the exact fp64 pass. */
int nsnkv_match_block(const float *vecs, int64_t m, const float *entries,
                      const double *inv_norms, int32_t fold, uint8_t *idx,
                      uint8_t *signs, uint8_t *zero_mask, int64_t *n_neartie,
                      void *stream);

/* ---- codebook (codebook.py:71-106) ------------------------------------ */
typedef struct nsnkv_codebook nsnkv_codebook;

/* Upload one 256x8 codebook (host pointers).  inv_norms must be the fp64
 * 1/||e|| of kernels/__init__.py:44-51 (computed by the caller, or NULL to
 * compute them here in the same component order).  bit_mode 1 or 2. */
int nsnkv_codebook_create(const float *entries_host, const double *inv_norms_host,
                          int32_t bit_mode, nsnkv_codebook **out);
int nsnkv_codebook_destroy(nsnkv_codebook *cb);
int nsnkv_codebook_bit_mode(const nsnkv_codebook *cb);

/* ---- codebook build passes (codebook.py:175-340) ---------------------- */
/* One Lloyd iteration of kmeans_init (codebook.py:196-212) over data[n][8]
 * (fp32) against centroids[256][8] (fp64): assign[i] = argmax_c of
 * x.f32(c) - 0.5 f32(|c|^2) (first maximum); sums[256][8] (fp64) and
 * counts[256] (caller-zeroed) accumulate the assigned points; d2[i] (may be
 * NULL) = |x|^2 - 2 x.c + |c|^2 for the empty-cluster reseed. */
int nsnkv_kmeans_assign(const float *data, int64_t n, const double *centroids, int32_t *assign,
                        double *sums, int32_t *counts, double *d2, void *stream);
/* Statistics of one finetune step (codebook.py:300-318) for batch[n][8]
 * assigned to idx[n] (the nsnkv_match_block rule): per-entry sums of the
 * samples' unit vectors and of their cosines to entries[256][8] (fp64),
 * counts of live (non-zero) samples, and += the batch's summed cosine
 * distance.  Accumulators are caller-zeroed. */
int nsnkv_finetune_stats(const float *batch, int64_t n, const int32_t *idx,
                         const double *entries, double *sum_unit, double *sum_cos,
                         int32_t *counts, double *cosdist, void *stream);

/* ---- RoPE table (rope.py:29-51) --------------------------------------- */
/* out[n][64][2] = float32(cos/sin(float64(pos0 + i) * freqs[j])) for
 * i < n, j < 64: the exact angles of rope_rows.  freqs (device, 64 fp64) are
 * the reference _pair_freqs(d=128, base). */
int nsnkv_rope_table(const double *freqs, int64_t pos0, int64_t n, float *out,
                     void *stream);

/* ---- encode: flush full chunks into pages (kvcache.py:114-195) -------- */
/*
 * Flushes n_units * n_flush chunks.  Chunk k of unit u consists of the
 * token stream rows k*64 .. k*64+63, where stream row i is
 *     residual[u][i]            if i < n_resid
 *     fresh[u][i - n_resid]     otherwise
 * residual is fp32 [n_units][64][128]; fresh is [n_units][n_fresh][128] in
 * fp32 (fresh_bf16 == 0) or bf16 (fresh_bf16 == 1).  Keys (is_key != 0) are
 * pre-RoPE and get NSN -> RoPE(start) -> FWHT -> VQ; values are post-HT and
 * get NSN -> VQ (kvcache.py:114-154).  start_pos[u] is the absolute position
 * of chunk 0 for unit u (base_position + n_quantized); rope_cs is a table
 * built by nsnkv_rope_table covering positions [rope_pos0, rope_pos0+rope_n).
 * The page for (u, k) is pool + page_ids[u * page_id_stride + k] * page_bytes.
 * counters (device int32 [n_units * n_flush][NSNKV_NUM_COUNTERS], may be
 * NULL) receives the per-chunk event counts.
 */
int nsnkv_encode_chunks(const float *residual, int32_t n_resid,
                        const void *fresh, int32_t fresh_bf16, int64_t n_fresh,
                        int32_t n_units, int32_t n_flush, int32_t is_key,
                        const int64_t *start_pos, const float *rope_cs,
                        int64_t rope_pos0, int64_t rope_n,
                        const nsnkv_codebook *cb, int32_t strategy,
                        uint8_t *pool, const int32_t *page_ids,
                        int32_t page_id_stride, int32_t *counters,
                        void *stream);

/* ---- serving cache: one launch per append (kvcache.py:157-195) -------- */
/*
 * Appends new K/V rows to every unit of a paged cache in ONE launch: all full
 * chunks are flushed (NSN -> RoPE -> FWHT -> VQ -> pack, as
 * nsnkv_encode_chunks) into the pages the caller allocated for them, the new
 * residual rows are written, and the page table and per-unit counters are
 * updated on the device (no host synchronisation).  Unit u gains
 * new_count[u] rows (or n_new_uniform), fresh row r of unit u being row
 * fresh_off[u] + r * fresh_row_stride of fresh_k / fresh_v ([rows][128], fp32
 * or bf16; fresh_off NULL = u * n_new_uniform).  Unit u flushes
 * n_flush = (n_res_in[u] + new) / 64 chunks into new_pages[u * max_flush + k]
 * (max_flush >= every unit's n_flush), written to page_table[u][n_chunks + k].
 * Counters are double-buffered: read from *_in, written to *_out.
 * counters (may be NULL): [pages][2 (K, V)][NSNKV_NUM_COUNTERS] by page id.
 */
typedef struct nsnkv_append_args {
  int32_t n_units;
  int32_t max_flush;
  const void *fresh_k;
  const void *fresh_v;
  int32_t fresh_bf16;
  int64_t n_new_uniform;
  const int32_t *new_count;  /* device [n_units] or NULL */
  const int64_t *fresh_off;  /* device [n_units] or NULL */
  int64_t fresh_row_stride;  /* in rows (1: [units][n][128]) */
  float *k_res;              /* [n_units][64][128] fp32 */
  float *v_res;
  const int32_t *n_chunks_in;
  const int32_t *n_res_in;
  int32_t *n_chunks_out;
  int32_t *n_res_out;
  const int64_t *base_pos;   /* absolute position of each unit's token 0 */
  int32_t *page_table;
  int32_t page_table_stride;
  const int32_t *new_pages;  /* device [n_units][max_flush] */
  uint8_t *k_pool;
  uint8_t *v_pool;
  int32_t *counters;
  const float *rope_cs;
  int64_t rope_pos0;
  int64_t rope_n;
  const nsnkv_codebook *cb_k;
  const nsnkv_codebook *cb_v;
  int32_t strategy;
} nsnkv_append_args;

int nsnkv_append(const nsnkv_append_args *args, void *stream);

/* Growable page pools on CUDA virtual memory: one reserved address range,
 * physical memory mapped on demand, so growth never copies or moves a page.
 * Created on the calling thread's current device. */
typedef struct nsnkv_pool nsnkv_pool;
int nsnkv_pool_create(size_t reserve_bytes, nsnkv_pool **out);
int nsnkv_pool_reserve(nsnkv_pool *pool, size_t bytes); /* map [0, bytes) */
void *nsnkv_pool_ptr(const nsnkv_pool *pool);
size_t nsnkv_pool_mapped(const nsnkv_pool *pool);
int nsnkv_pool_destroy(nsnkv_pool *pool);
/* Copy pages ids_host[0..n) of a pool to (to_pool == 0) or from (to_pool != 0)
 * a dense buffer of n pages in host or device memory (snapshot export /
 * import of reference-serialized chunks). */
int nsnkv_pages_copy(uint8_t *pool, int32_t page_bytes, const int32_t *ids_host, int32_t n,
                     uint8_t *buf, int32_t to_pool, void *stream);

/* ---- decode over the packed cache (attention.py:83-142) --------------- */
/*
 * Cache geometry shared by the three decode entry points.  Unit u
 * (= b * n_kv_heads + h) owns n_chunks[u] pages listed in
 * page_table[u * page_table_stride + c], plus n_res[u] residual rows
 * (keys pre-RoPE in k_res, values post-HT in v_res, fp32 [units][64][128]).
 * base_pos[u] is the absolute position of the unit's first cached token.
 * q-head i of batch b reads unit b * n_kv_heads + i / (n_q_heads/n_kv_heads).
 */
typedef struct nsnkv_cache_view {
  const uint8_t *k_pool;
  const uint8_t *v_pool;
  const int32_t *page_table;
  int32_t page_table_stride;
  const int32_t *n_chunks;
  const float *k_res;
  const float *v_res;
  const int32_t *n_res;
  const int64_t *base_pos;
  int32_t batch;
  int32_t n_kv_heads;
  int32_t n_q_heads;
  int32_t max_tokens;        /* >= max over units of n_chunks*64 + n_res  */
  const float *rope_cs;      /* nsnkv_rope_table output                    */
  int64_t rope_pos0;
  int64_t rope_n;
  const nsnkv_codebook *cb_k;
  const nsnkv_codebook *cb_v;
  int64_t total_chunks;      /* sum of n_chunks (host copy), or -1 to let
                                the library read it back (synchronises)   */
  int32_t precision;         /* decode codeword precision: 0 = fp16 hi+lo
                                on scores and values (~1e-6 relative
                                output error), 1 = plain fp16 scores, hi+lo
                                values (~4e-4), 2 = plain fp16 both (~6e-4
                                on 2-bit; not for 1-bit)   */
} nsnkv_cache_view;

/* Raw q.K^T of every cached token (quantized chunks first, then residual),
 * scores[b][i][t], row stride max_tokens (attention.py:83-111).  q is
 * fp32 [batch][n_q_heads][128], already RoPE'd at its own position. */
int nsnkv_decode_scores(const nsnkv_cache_view *cv, const float *q,
                        float *scores, void *stream);

/* Weighted value sum inverse-transformed to the model basis
 * (attention.py:114-133); weights fp32 [batch][n_q_heads][max_tokens]. */
int nsnkv_decode_output(const nsnkv_cache_view *cv, const float *weights,
                        float *out, void *workspace, size_t workspace_bytes,
                        void *stream);

/* Fused softmax(q.K^T / sqrt(d)) . V over the packed cache
 * (attention.py:136-142) without materialising the weights: split-K
 * flash-decoding.  out fp32 [batch][n_q_heads][128].  lse (may be NULL)
 * receives the natural-log softmax normaliser of scores/sqrt(d). */
int nsnkv_decode_attend(const nsnkv_cache_view *cv, const float *q, float *out,
                        float *lse, void *workspace, size_t workspace_bytes,
                        void *stream);

/* Fused serving decode step = kvcache.append of n_new (1..63) rows to every
 * unit followed by nsnkv_decode_attend over the cache including them, with no
 * extra launch: the combine kernel attends the new rows as residual rows and
 * writes them into k_res / v_res.  The caller guarantees that no unit
 * flushes (n_res[u] + n_new < 64 for every unit; otherwise use nsnkv_append
 * first).  new_k / new_v: [units][n_new][128], fp32 or bf16 (new_bf16).
 * n_res_out (device int32 [units], may be cv->n_res itself) receives
 * n_res[u] + n_new. */
int nsnkv_decode_step(const nsnkv_cache_view *cv, const float *q, const void *new_k,
                      const void *new_v, int32_t new_bf16, int32_t n_new, int32_t *n_res_out,
                      float *out, float *lse, void *workspace, size_t workspace_bytes,
                      void *stream);

/* Workspace bytes nsnkv_decode_attend / nsnkv_decode_output need. */
size_t nsnkv_decode_workspace_bytes(const nsnkv_cache_view *cv);

#ifdef __cplusplus
}
#endif
#endif /* NSNKV_B200_H */
