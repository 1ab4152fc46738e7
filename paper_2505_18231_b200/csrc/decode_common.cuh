// decode_common.cuh -- cache view and page-field readers shared by the
// decode kernels.
#pragma once
#include "common.cuh"

namespace nsnkv {

struct CacheViewDev {
  const uint8_t *k_pool, *v_pool;
  const int32_t *page_table;
  int page_table_stride;
  const int32_t *n_chunks;
  const float *k_res, *v_res;
  const int32_t *n_res;
  const int64_t *base_pos;
  int batch, n_kv_heads, n_q_heads, max_tokens;
  const float2 *rope_cs;
  int64_t rope_pos0, rope_n;
  CodebookDev cb_k, cb_v;
  int64_t total_chunks;
  int precision;
};

struct ChunkMeta {
  float s1_scale, s1_zero;
  float o_scale[4], o_zero[4];
};

__device__ __forceinline__ void load_chunk_meta(const uint8_t *page, const PageLayout &L,
                                                ChunkMeta &m) {
  const uint16_t *par = reinterpret_cast<const uint16_t *>(page + L.par);
  m.s1_scale = f16_bits_to_f32(par[0]);
  m.s1_zero = f16_bits_to_f32(par[1]);
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    m.o_scale[g] = f16_bits_to_f32(par[2 + g]);
    m.o_zero[g] = f16_bits_to_f32(par[6 + g]);
  }
}

__device__ __forceinline__ uint32_t nibble(const uint8_t *p, int i) {
  const uint32_t b = p[i >> 1];
  return (i & 1) ? (b >> 4) : (b & 15u);
}

// rtn4_dequant (vq.py:133-136): zero + level * scale, two fp32 roundings.
__device__ __forceinline__ float dequant_s1(const uint8_t *page, const PageLayout &L,
                                            const ChunkMeta &m, int t) {
  return __fadd_rn(m.s1_zero, __fmul_rn((float)nibble(page + L.s1n, t), m.s1_scale));
}

__device__ __forceinline__ float dequant_o(const uint8_t *page, const PageLayout &L,
                                           const ChunkMeta &m, int c) {
  const int g = c >> 5;
  return __fadd_rn(m.o_zero[g], __fmul_rn((float)nibble(page + L.on, c), m.o_scale[g]));
}

// Natural sign byte of (token t, sub j) of a KEY page (decode K order: word
// q of token t covers subs 4q+m; bit 4m+p = sign of component 2p, bit
// 16+4m+p = sign of component 2p+1).
__device__ __forceinline__ uint32_t sign_byte(const uint8_t *page, const PageLayout &L, int t,
                                              int j) {
  const uint32_t w = reinterpret_cast<const uint32_t *>(page + L.sgn)[4 * t + (j >> 2)];
  const int m = j & 3;
  uint32_t b = 0;
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    b |= ((w >> (4 * m + p)) & 1u) << (2 * p);
    b |= ((w >> (16 + 4 * m + p)) & 1u) << (2 * p + 1);
  }
  return b;
}

// Natural sign byte of (token t, sub j) of a VALUE page (decode V order: word
// 8 i + c holds component c of token pair (2i, 2i+1); bit j = token 2i, sub
// j; bit 16 + j = token 2i+1).
__device__ __forceinline__ uint32_t sign_byte_v(const uint8_t *page, const PageLayout &L, int t,
                                                int j) {
  const uint32_t *w = reinterpret_cast<const uint32_t *>(page + L.sgn) + 8 * (t >> 1);
  const int sh = j + 16 * (t & 1);
  uint32_t b = 0;
#pragma unroll
  for (int c = 0; c < SUB; ++c) b |= ((w[c] >> sh) & 1u) << c;
  return b;
}

// FWHT of a 128-vector in smem, one element per thread of a 128-thread block
// (fp32 add/sub butterflies, then the orthonormal scale; _native.pyx:24-37).
__device__ __forceinline__ void block_fwht128(float *v) {
  const int i = threadIdx.x;
#pragma unroll 1
  for (int h = 1; h < D; h <<= 1) {
    const float mine = v[i], other = v[i ^ h];
    __syncthreads();
    v[i] = (i & h) ? __fsub_rn(other, mine) : __fadd_rn(mine, other);
    __syncthreads();
  }
  v[i] = __fmul_rn(v[i], 0.08838834764831845f);
  __syncthreads();
}

}  // namespace nsnkv

int make_cache_view(const nsnkv_cache_view *in, nsnkv::CacheViewDev *out);
size_t nsnkv_internal_output_ws(const nsnkv::CacheViewDev &cv);
