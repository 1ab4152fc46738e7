// decode_dispatch.cu -- nsnkv_decode_attend entry point: validates the cache
// view, sizes the stream-K record workspace and dispatches to the fused
// kernel instantiation for (GQA group, bit mode, precision).  The kernel
// itself lives in decode_attend3.cu.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "decode_common.cuh"
#include "decode_att.cuh"

using namespace nsnkv;

// SM count of the calling thread's current device (one persistent CTA per SM)
static int attend_grid() {
  static int sms[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int &s = sms[dev & 63];
  if (!s) {
    cudaDeviceGetAttribute(&s, cudaDevAttrMultiProcessorCount, dev);
    if (s <= 0) s = 148;
  }
  return s;
}

// stream-K records: one per (unit + CTA, consumer group), G heads of 4 + D floats
static size_t records_bytes(const CacheViewDev &cv, int G) {
  const int units = cv.batch * cv.n_kv_heads;
  const int ngrp = 3;  // consumer groups per CTA
  return (size_t)(units + attend_grid() + 1) * ngrp * G * (4 + D) * sizeof(float);
}

extern "C" size_t nsnkv_decode_workspace_bytes(const nsnkv_cache_view *cv_in) {
  CacheViewDev cv;
  if (make_cache_view(cv_in, &cv)) return 0;
  const int G = cv.n_q_heads / cv.n_kv_heads;
  const size_t a = (records_bytes(cv, G) + 255) / 256 * 256;
  const size_t b = nsnkv_internal_output_ws(cv);
  return a > b ? a : b;
}

template <int G, bool FOLD, int PREC>
static int launch_attend(const CacheViewDev &cv, const float *q, float *out, float *lse,
                         float *recs, int64_t total, cudaStream_t st, const AppendRows &add) {
  int grid = attend_grid();
  if (total < grid) grid = (int)(total > 0 ? total : 1);
  return nsnkv_launch_attend3<G, FOLD, PREC>(cv, q, out, lse, recs, total, grid, st, add);
}

static int decode_attend(const nsnkv_cache_view *cv_in, const float *q, float *out, float *lse,
                         void *workspace, size_t workspace_bytes, void *stream,
                         const AppendRows &add) {
  CacheViewDev cv;
  int rc = make_cache_view(cv_in, &cv);
  if (rc) return rc;
  const int G = cv.n_q_heads / cv.n_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "decode_attend: GQA group must be 1, 2, 4 or 8");
  if (cv.rope_pos0 != 0)
    return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "decode_attend: RoPE table must start at position 0");
  if (cv.precision < 0 || cv.precision > 2)
    return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "decode_attend: precision must be 0, 1 or 2");
  if (workspace_bytes < records_bytes(cv, G))
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "decode_attend: workspace too small");
  const int units = cv.batch * cv.n_kv_heads;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t total = cv.total_chunks;
  if (total < 0) {  // read the counts back (synchronises the stream)
    int32_t *h = (int32_t *)malloc(sizeof(int32_t) * units);
    cudaError_t e = cudaMemcpyAsync(h, cv.n_chunks, sizeof(int32_t) * units,
                                    cudaMemcpyDeviceToHost, st);
    if (!e) e = cudaStreamSynchronize(st);
    total = 0;
    for (int u = 0; !e && u < units; ++u) total += h[u];
    free(h);
    if (e) return nsnkv_internal_set_error(NSNKV_ERR_CUDA, cudaGetErrorString(e));
  }
  float *recs = (float *)workspace;
  const bool fold = cv.cb_k.bit_mode == 2;
  const int prec = cv.precision;
#define NSNKV_ATT_P(GG, FF)                                                       \
  return prec == 0 ? launch_attend<GG, FF, 0>(cv, q, out, lse, recs, total, st, add)  \
       : prec == 1 ? launch_attend<GG, FF, 1>(cv, q, out, lse, recs, total, st, add)  \
                   : launch_attend<GG, FF, 2>(cv, q, out, lse, recs, total, st, add)
#define NSNKV_ATT(GG)         \
  if (fold) NSNKV_ATT_P(GG, true); \
  else NSNKV_ATT_P(GG, false)
  // 1-bit, G = 4, values in fp16: the key side by lookup table when the
  // CTAs' chunk ranges are long enough to amortise the per-unit table build
  if (!fold && G == 4 && prec == 1 && total >= 32 * (int64_t)attend_grid() &&
      !std::getenv("NSNKV_NO_LUT"))
    return launch_attend<4, false, 3>(cv, q, out, lse, recs, total, st, add);
  switch (G) {
    case 1: NSNKV_ATT(1);
    case 2: NSNKV_ATT(2);
    case 4: NSNKV_ATT(4);
    default: NSNKV_ATT(8);
  }
#undef NSNKV_ATT_P
#undef NSNKV_ATT
}

extern "C" int nsnkv_decode_attend(const nsnkv_cache_view *cv, const float *q, float *out,
                                   float *lse, void *workspace, size_t workspace_bytes,
                                   void *stream) {
  return decode_attend(cv, q, out, lse, workspace, workspace_bytes, stream, AppendRows{});
}

extern "C" int nsnkv_decode_step(const nsnkv_cache_view *cv, const float *q, const void *new_k,
                                 const void *new_v, int32_t new_bf16, int32_t n_new,
                                 int32_t *n_res_out, float *out, float *lse, void *workspace,
                                 size_t workspace_bytes, void *stream) {
  if (n_new < 1 || n_new >= R || !new_k || !new_v || !n_res_out)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "decode_step: need 1..63 new rows and n_res_out");
  AppendRows add;
  add.k = new_k;
  add.v = new_v;
  add.bf16 = new_bf16 ? 1 : 0;
  add.n = n_new;
  add.n_res_out = n_res_out;
  return decode_attend(cv, q, out, lse, workspace, workspace_bytes, stream, add);
}
