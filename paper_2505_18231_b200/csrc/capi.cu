// capi.cu -- C ABI glue: error state, launch accounting, codebook upload,
// cache-view validation and the fused-attend dispatch.
#include <atomic>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "decode_common.cuh"

using namespace nsnkv;

struct nsnkv_codebook {
  CodebookDev dev;
};

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

extern "C" void nsnkv_internal_count_launch(int n) { g_launches += n; }

extern "C" int nsnkv_internal_set_error(int code, const char *msg) {
  snprintf(g_err, sizeof(g_err), "%s", msg);
  return code;
}

extern "C" int nsnkv_internal_check_launch(const char *what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return NSNKV_ERR_CUDA;
  }
  return NSNKV_OK;
}

extern "C" int nsnkv_version(void) { return 1; }
extern "C" const char *nsnkv_last_error(void) { return g_err; }
extern "C" int64_t nsnkv_launch_count(void) { return (int64_t)g_launches.load(); }

// ---------------------------------------------------------------------------
// codebook upload (codebook.py:71-106; kernels/__init__.py:44-51)
// ---------------------------------------------------------------------------
static inline uint32_t pack_half2(float a, float b) {
  const __half ha = __float2half_rn(a), hb = __float2half_rn(b);
  return (uint32_t)__half_as_ushort(ha) | ((uint32_t)__half_as_ushort(hb) << 16);
}

extern "C" int nsnkv_codebook_create(const float *entries_host, const double *inv_norms_host,
                                     int32_t bit_mode, nsnkv_codebook **out) {
  if (!entries_host || !out) return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "codebook: null");
  if (bit_mode != 1 && bit_mode != 2)
    return nsnkv_internal_set_error(NSNKV_ERR_FORMAT, "codebook: bit_mode must be 1 or 2");
  std::vector<double> inv(NENT);
  for (int c = 0; c < NENT; ++c) {
    const float *e = entries_host + 8 * c;
    if (bit_mode == 2)
      for (int k = 0; k < 8; ++k)
        if (e[k] < 0.f)
          return nsnkv_internal_set_error(NSNKV_ERR_FORMAT,
                                          "two-bit codebook entries must be nonnegative");
    if (inv_norms_host) {
      inv[c] = inv_norms_host[c];
    } else {  // component-order fp64 sum, kernels/__init__.py:47-51
      double s = (double)e[0] * (double)e[0];
      for (int k = 1; k < 8; ++k) s = s + (double)e[k] * (double)e[k];
      if (s < 1e-24) return nsnkv_internal_set_error(NSNKV_ERR_FORMAT, "codebook contains a zero entry");
      inv[c] = 1.0 / std::sqrt(s);
    }
  }
  // decode gather table: row c = [hi codeword x 8 slots][lo codeword x 8 slots]
  std::vector<uint4> tw(NENT * 16);
  for (int c = 0; c < NENT; ++c) {
    const float *e = entries_host + 8 * c;
    uint32_t hw[4], lw[4];
    for (int p = 0; p < 4; ++p) {
      const float a = e[2 * p], b = e[2 * p + 1];
      const float ah = __half2float(__float2half_rn(a)), bh = __half2float(__float2half_rn(b));
      hw[p] = pack_half2(a, b);
      lw[p] = pack_half2(a - ah, b - bh);
    }
    for (int slot = 0; slot < 8; ++slot) {
      tw[c * 16 + slot] = make_uint4(hw[0], hw[1], hw[2], hw[3]);
      tw[c * 16 + 8 + slot] = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    }
  }
  // encode search B operands (tcgen05, K-major no-swizzle canonical layout):
  // matrix m (0: [e_hi | e_hi], 1: [e_lo | e_lo]) of the normalized entries
  std::vector<uint16_t> tb(2 * NENT * 16);
  for (int c = 0; c < NENT; ++c) {
    const float *e = entries_host + 8 * c;
    for (int k = 0; k < 8; ++k) {
      const float a = (float)((double)e[k] * inv[c]);
      const __half h = __float2half_rn(a);
      const __half l = __float2half_rn(a - __half2float(h));
      for (int kh = 0; kh < 2; ++kh) {
        const size_t off = (size_t)(c / 8) * 128 + kh * 64 + (c % 8) * 8 + k;  // in halves
        tb[off] = __half_as_ushort(h);
        tb[NENT * 16 + off] = __half_as_ushort(l);
      }
    }
  }
  nsnkv_codebook *cb = new nsnkv_codebook();
  cb->dev.bit_mode = bit_mode;
  for (int k = 0; k < 8; ++k) {  // mean fp16 rounding error of component k
    double acc = 0.0;
    for (int c = 0; c < NENT; ++c) {
      const float x = entries_host[8 * c + k];
      acc += (double)x - (double)__half2float(__float2half_rn(x));
    }
    cb->dev.dbar[k] = (float)(acc / NENT);
  }
  cudaError_t err = cudaSuccess;
  err = cudaMalloc(&cb->dev.entries, NENT * 8 * sizeof(float));
  if (!err) err = cudaMalloc(&cb->dev.inv, NENT * sizeof(double));
  if (!err) err = cudaMalloc(&cb->dev.tabw, NENT * 16 * sizeof(uint4));
  if (!err) err = cudaMalloc(&cb->dev.tcb, 2 * NENT * 16 * sizeof(uint16_t));
  if (!err) err = cudaMemcpy(cb->dev.entries, entries_host, NENT * 8 * sizeof(float), cudaMemcpyHostToDevice);
  if (!err) err = cudaMemcpy(cb->dev.inv, inv.data(), NENT * sizeof(double), cudaMemcpyHostToDevice);
  if (!err) err = cudaMemcpy(cb->dev.tabw, tw.data(), NENT * 16 * sizeof(uint4), cudaMemcpyHostToDevice);
  if (!err) err = cudaMemcpy(cb->dev.tcb, tb.data(), 2 * NENT * 16 * sizeof(uint16_t), cudaMemcpyHostToDevice);
  if (err) {
    nsnkv_codebook_destroy(cb);
    snprintf(g_err, sizeof(g_err), "codebook upload: %s", cudaGetErrorString(err));
    return NSNKV_ERR_CUDA;
  }
  *out = cb;
  return NSNKV_OK;
}

extern "C" int nsnkv_codebook_destroy(nsnkv_codebook *cb) {
  if (!cb) return NSNKV_OK;
  cudaFree(cb->dev.entries);
  cudaFree(cb->dev.inv);
  cudaFree(cb->dev.tabw);
  cudaFree(cb->dev.tcb);
  delete cb;
  return NSNKV_OK;
}

extern "C" int nsnkv_codebook_bit_mode(const nsnkv_codebook *cb) { return cb ? cb->dev.bit_mode : 0; }

extern "C" int nsnkv_internal_codebook_dev(const nsnkv_codebook *cb, CodebookDev *out) {
  if (!cb) return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "null codebook");
  *out = cb->dev;
  return NSNKV_OK;
}

// ---------------------------------------------------------------------------
// cache view validation
// ---------------------------------------------------------------------------
int make_cache_view(const nsnkv_cache_view *in, CacheViewDev *out) {
  if (!in) return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "null cache view");
  if (!in->cb_k || !in->cb_v) return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "cache view: null codebook");
  if (in->batch <= 0 || in->n_kv_heads <= 0 || in->n_q_heads <= 0 ||
      in->n_q_heads % in->n_kv_heads != 0)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "cache view: bad head geometry");
  if (in->max_tokens <= 0 || in->max_tokens % R != 0)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "cache view: max_tokens must be a positive multiple of 64");
  if (in->cb_k->dev.bit_mode != in->cb_v->dev.bit_mode)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "codebook bit mode does not match chunk");
  out->k_pool = in->k_pool;
  out->v_pool = in->v_pool;
  out->page_table = in->page_table;
  out->page_table_stride = in->page_table_stride;
  out->n_chunks = in->n_chunks;
  out->k_res = in->k_res;
  out->v_res = in->v_res;
  out->n_res = in->n_res;
  out->base_pos = in->base_pos;
  out->batch = in->batch;
  out->n_kv_heads = in->n_kv_heads;
  out->n_q_heads = in->n_q_heads;
  out->max_tokens = in->max_tokens;
  out->rope_cs = reinterpret_cast<const float2 *>(in->rope_cs);
  out->rope_pos0 = in->rope_pos0;
  out->rope_n = in->rope_n;
  out->cb_k = in->cb_k->dev;
  out->cb_v = in->cb_v->dev;
  out->total_chunks = in->total_chunks;
  out->precision = in->precision;
  return NSNKV_OK;
}
