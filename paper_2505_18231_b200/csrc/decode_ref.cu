// decode_ref.cu -- decode over the packed cache, the unfused entry points:
//   nsnkv_decode_scores  == attention.py:83-111 (scores_quantized), batched
//   nsnkv_decode_output  == attention.py:114-133 (output_quantized), batched
// Each follows the reference's own arithmetic shape (payload . HT(q) plus
// RoPE(o, pos) . q scaled by s1/s2; rows s1 * (s2 * payload + o) weighted and
// summed in the Hadamard domain, one inverse FWHT at the end), in fp32.
// The fused flash-decoding kernel lives in decode_attend.cu.
#include "common.cuh"
#include "decode_common.cuh"

namespace nsnkv {

// ---------------------------------------------------------------------------
// scores: one CTA per (unit, chunk) with 64 threads (one per token), plus one
// CTA per unit for the residual.  q and HT(q) of the G q-heads in smem.
// ---------------------------------------------------------------------------
constexpr int MAXG = 16;

__global__ void __launch_bounds__(64) scores_kernel(CacheViewDev cv, const float *__restrict__ q,
                                                    float *__restrict__ scores, int max_chunks) {
  __shared__ float s_q[MAXG][D];
  __shared__ float s_qh[MAXG][D];
  __shared__ float s_o[D];
  __shared__ float s_ent[NENT * 8];
  const int u = blockIdx.y;
  const int c = blockIdx.x;  // chunk index, or max_chunks for the residual
  const int b = u / cv.n_kv_heads, h = u - b * cv.n_kv_heads;
  const int G = cv.n_q_heads / cv.n_kv_heads;
  const int nch = cv.n_chunks[u];
  const int nres = cv.n_res[u];
  const int tid = threadIdx.x;
  if (c < max_chunks && c >= nch) return;
  if (c == max_chunks && nres == 0) return;
  const float *qb = q + ((int64_t)b * cv.n_q_heads + (int64_t)h * G) * D;
  for (int i = tid; i < G * D; i += blockDim.x) s_q[i / D][i % D] = qb[i];
  __syncthreads();
  const int64_t base = cv.base_pos[u];
  float *srow = scores + ((int64_t)b * cv.n_q_heads + (int64_t)h * G) * cv.max_tokens;
  if (c == max_chunks) {  // residual: exact RoPE(k, pos) . q (attention.py:105-108)
    const int t = tid;
    if (t < nres) {
      const int64_t pos = base + (int64_t)nch * R + t;
      const float *kr = cv.k_res + ((int64_t)u * R + t) * D;
      const float2 *cs = cv.rope_cs + (pos - cv.rope_pos0) * NPAIR;
      float acc[MAXG];
      for (int g = 0; g < G; ++g) acc[g] = 0.f;
      for (int j = 0; j < NPAIR; ++j) {
        const float2 a = cs[j];
        const float e = kr[2 * j], o = kr[2 * j + 1];
        const float re = __fsub_rn(__fmul_rn(e, a.x), __fmul_rn(o, a.y));
        const float ro = __fadd_rn(__fmul_rn(e, a.y), __fmul_rn(o, a.x));
        for (int g = 0; g < G; ++g) acc[g] = fmaf(ro, s_q[g][2 * j + 1], fmaf(re, s_q[g][2 * j], acc[g]));
      }
      for (int g = 0; g < G; ++g) srow[(int64_t)g * cv.max_tokens + (int64_t)nch * R + t] = acc[g];
    }
    return;
  }
  // HT(q) (attention.py:93) for each head: thread per (head, row) FWHT in smem
  for (int i = tid; i < G * D; i += blockDim.x) s_qh[i / D][i % D] = s_q[i / D][i % D];
  for (int i = tid; i < NENT * 8; i += blockDim.x) s_ent[i] = cv.cb_k.entries[i];
  __syncthreads();
  for (int hh = 1; hh < D; hh <<= 1) {
    for (int k = tid; k < G * (D / 2); k += blockDim.x) {
      const int g = k / (D / 2), kk = k % (D / 2);
      const int i = (kk / hh) * 2 * hh + (kk % hh);
      const float x = s_qh[g][i], y = s_qh[g][i + hh];
      s_qh[g][i] = x + y;
      s_qh[g][i + hh] = x - y;
    }
    __syncthreads();
  }
  for (int i = tid; i < G * D; i += blockDim.x) s_qh[i / D][i % D] *= 0.08838834764831845f;
  const PageLayout L = page_layout(cv.cb_k.bit_mode);
  const uint8_t *page = cv.k_pool + (int64_t)cv.page_table[(int64_t)u * cv.page_table_stride + c] * L.bytes;
  ChunkMeta m;
  load_chunk_meta(page, L, m);
  for (int i = tid; i < D; i += blockDim.x) s_o[i] = dequant_o(page, L, m, i);
  __syncthreads();
  const int t = tid;
  const float s1 = dequant_s1(page, L, m, t);
  const float s2 = f16_bits_to_f32(reinterpret_cast<const uint16_t *>(page + L.s2)[t]);
  float pd[MAXG], sd[MAXG];
  for (int g = 0; g < G; ++g) pd[g] = sd[g] = 0.f;
  for (int j = 0; j < NSUB; ++j) {  // payload . HT(q) (attention.py:102)
    const int e = page[L.idx + t * NSUB + j];
    const uint32_t sb = (L.sgn >= 0) ? sign_byte(page, L, t, j) : 0u;
    for (int k = 0; k < 8; ++k) {
      float cval = s_ent[e * 8 + k];
      if ((sb >> k) & 1u) cval = -cval;
      for (int g = 0; g < G; ++g) pd[g] = fmaf(cval, s_qh[g][8 * j + k], pd[g]);
    }
  }
  const int64_t pos = base + (int64_t)c * R + t;  // attention.py:101
  const float2 *cs = cv.rope_cs + (pos - cv.rope_pos0) * NPAIR;
  for (int j = 0; j < NPAIR; ++j) {  // rope_expand(o, pos) . q (attention.py:103)
    const float2 a = cs[j];
    const float e = s_o[2 * j], o = s_o[2 * j + 1];
    const float re = __fsub_rn(__fmul_rn(e, a.x), __fmul_rn(o, a.y));
    const float ro = __fadd_rn(__fmul_rn(e, a.y), __fmul_rn(o, a.x));
    for (int g = 0; g < G; ++g) sd[g] = fmaf(ro, s_q[g][2 * j + 1], fmaf(re, s_q[g][2 * j], sd[g]));
  }
  for (int g = 0; g < G; ++g)  // s1 * (s2 * payload_dot + shift_dot) (attention.py:104)
    srow[(int64_t)g * cv.max_tokens + (int64_t)c * R + t] = s1 * (s2 * pd[g] + sd[g]);
}

// ---------------------------------------------------------------------------
// output: CTA per (unit, split) with 128 threads (one per channel); partial
// sums in the Hadamard domain go to the workspace, then a combine kernel adds
// the splits and the residual and applies the inverse FWHT (attention.py:133).
// ---------------------------------------------------------------------------
constexpr int OUT_SPLIT_CHUNKS = 8;

__global__ void __launch_bounds__(128) output_partial_kernel(CacheViewDev cv,
                                                             const float *__restrict__ w,
                                                             float *__restrict__ part,
                                                             int n_splits) {
  __shared__ float s_ent[NENT * 8];
  const int u = blockIdx.y, sp = blockIdx.x;
  const int b = u / cv.n_kv_heads, h = u - b * cv.n_kv_heads;
  const int G = cv.n_q_heads / cv.n_kv_heads;
  const int ch = threadIdx.x;
  const int nch = cv.n_chunks[u];
  for (int i = ch; i < NENT * 8; i += blockDim.x) s_ent[i] = cv.cb_v.entries[i];
  __syncthreads();
  float acc[MAXG];
  for (int g = 0; g < G; ++g) acc[g] = 0.f;
  const PageLayout L = page_layout(cv.cb_v.bit_mode);
  const float *wb = w + ((int64_t)b * cv.n_q_heads + (int64_t)h * G) * cv.max_tokens;
  const int c0 = sp * OUT_SPLIT_CHUNKS, c1 = min(nch, c0 + OUT_SPLIT_CHUNKS);
  const int j = ch >> 3, k = ch & 7;
  for (int c = c0; c < c1; ++c) {
    const uint8_t *page = cv.v_pool + (int64_t)cv.page_table[(int64_t)u * cv.page_table_stride + c] * L.bytes;
    ChunkMeta m;
    load_chunk_meta(page, L, m);
    const float o = dequant_o(page, L, m, ch);
    for (int t = 0; t < R; ++t) {
      const int e = page[L.idx + t * NSUB + j];
      float cval = s_ent[e * 8 + k];
      if (L.sgn >= 0 && ((sign_byte_v(page, L, t, j) >> k) & 1u)) cval = -cval;
      const float s1 = dequant_s1(page, L, m, t);
      const float s2 = f16_bits_to_f32(reinterpret_cast<const uint16_t *>(page + L.s2)[t]);
      const float row = s1 * (s2 * cval + o);  // attention.py:126-128
      for (int g = 0; g < G; ++g) acc[g] = fmaf(wb[(int64_t)g * cv.max_tokens + (int64_t)c * R + t], row, acc[g]);
    }
  }
  for (int g = 0; g < G; ++g) part[(((int64_t)u * n_splits + sp) * G + g) * D + ch] = acc[g];
}

__global__ void __launch_bounds__(128) output_combine_kernel(CacheViewDev cv,
                                                             const float *__restrict__ w,
                                                             const float *__restrict__ part,
                                                             int n_splits, float *__restrict__ out) {
  __shared__ float s_acc[D];
  const int u = blockIdx.x / (cv.n_q_heads / cv.n_kv_heads);
  const int G = cv.n_q_heads / cv.n_kv_heads;
  const int g = blockIdx.x - u * G;
  const int b = u / cv.n_kv_heads, h = u - b * cv.n_kv_heads;
  const int ch = threadIdx.x;
  const int nch = cv.n_chunks[u];
  const int used = (nch + OUT_SPLIT_CHUNKS - 1) / OUT_SPLIT_CHUNKS;
  float acc = 0.f;
  for (int sp = 0; sp < used; ++sp) acc += part[(((int64_t)u * n_splits + sp) * G + g) * D + ch];
  const float *wr = w + ((int64_t)b * cv.n_q_heads + (int64_t)h * G + g) * cv.max_tokens;
  const int nres = cv.n_res[u];
  for (int t = 0; t < nres; ++t)  // attention.py:129-131
    acc = fmaf(wr[(int64_t)nch * R + t], cv.v_res[((int64_t)u * R + t) * D + ch], acc);
  s_acc[ch] = acc;
  __syncthreads();
  block_fwht128(s_acc);
  out[((int64_t)b * cv.n_q_heads + (int64_t)h * G + g) * D + ch] = s_acc[ch];
}

}  // namespace nsnkv

using namespace nsnkv;

extern "C" int nsnkv_decode_scores(const nsnkv_cache_view *cv_in, const float *q, float *scores,
                                   void *stream) {
  CacheViewDev cv;
  int rc = make_cache_view(cv_in, &cv);
  if (rc) return rc;
  if (cv.n_q_heads / cv.n_kv_heads > MAXG)
    return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "decode_scores: GQA group > 16");
  const int max_chunks = cv.max_tokens / R;
  dim3 grid(max_chunks + 1, cv.batch * cv.n_kv_heads);
  scores_kernel<<<grid, 64, 0, (cudaStream_t)stream>>>(cv, q, scores, max_chunks);
  nsnkv_internal_count_launch(1);
  return nsnkv_internal_check_launch("decode_scores");
}

static int output_splits(const CacheViewDev &cv) {
  const int max_chunks = cv.max_tokens / R;
  return max(1, (max_chunks + OUT_SPLIT_CHUNKS - 1) / OUT_SPLIT_CHUNKS);
}

size_t nsnkv_internal_output_ws(const CacheViewDev &cv) {
  const int G = cv.n_q_heads / cv.n_kv_heads;
  return (size_t)cv.batch * cv.n_kv_heads * output_splits(cv) * G * D * sizeof(float);
}

extern "C" int nsnkv_decode_output(const nsnkv_cache_view *cv_in, const float *weights, float *out,
                                   void *workspace, size_t workspace_bytes, void *stream) {
  CacheViewDev cv;
  int rc = make_cache_view(cv_in, &cv);
  if (rc) return rc;
  if (cv.n_q_heads / cv.n_kv_heads > MAXG)
    return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "decode_output: GQA group > 16");
  if (workspace_bytes < nsnkv_internal_output_ws(cv))
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "decode_output: workspace too small");
  const int ns = output_splits(cv);
  dim3 grid(ns, cv.batch * cv.n_kv_heads);
  output_partial_kernel<<<grid, 128, 0, (cudaStream_t)stream>>>(cv, weights, (float *)workspace, ns);
  output_combine_kernel<<<cv.batch * cv.n_q_heads, 128, 0, (cudaStream_t)stream>>>(
      cv, weights, (const float *)workspace, ns, out);
  nsnkv_internal_count_launch(2);
  return nsnkv_internal_check_launch("decode_output");
}
