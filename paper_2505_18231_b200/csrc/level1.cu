// level1.cu -- drop-in replacements for the reference kernel plug-in
// (reference pkg/src/nsnkv/kernels/__init__.py:31-41): fwht_rows and
// match_block, plus the RoPE angle table (rope.py:29-51).
#include "common.cuh"
#include "match.cuh"

namespace nsnkv {

// ---------------------------------------------------------------------------
// fwht_rows: _native.pyx:16-38.  Butterflies h = 1, 2, 4, ..., d/2 in fp32,
// (x, y) -> (x + y, x - y), then one multiply by float(1/sqrt(d)).  Each
// output element depends on its pair only, so any parallel schedule of a
// stage reproduces the sequential result bit-for-bit.
// ---------------------------------------------------------------------------
__global__ void fwht_rows_kernel(const float *__restrict__ in, float *__restrict__ out,
                                 int64_t n, int d, int log_d, int rows_per_block,
                                 float scale) {
  extern __shared__ float sm[];
  const int64_t row0 = (int64_t)blockIdx.x * rows_per_block;
  const int64_t rem = n - row0;
  const int nrows = rem < rows_per_block ? (int)rem : rows_per_block;
  const int total = nrows * d;
  for (int i = threadIdx.x; i < total; i += blockDim.x) sm[i] = in[row0 * d + i];
  __syncthreads();
  const int half = d >> 1;
  const int pairs = nrows * half;
  for (int h = 1; h < d; h <<= 1) {
    for (int k = threadIdx.x; k < pairs; k += blockDim.x) {
      const int r = k / half;
      const int kk = k - r * half;
      const int i = (kk / h) * 2 * h + (kk % h);
      float *row = sm + r * d;
      const float x = row[i];
      const float y = row[i + h];
      row[i] = __fadd_rn(x, y);
      row[i + h] = __fsub_rn(x, y);
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < total; i += blockDim.x)
    out[row0 * d + i] = __fmul_rn(sm[i], scale);
}

// ---------------------------------------------------------------------------
// match_block: _native.pyx:41-87 + codebook.py:109-128 (zero rows).
// ---------------------------------------------------------------------------
constexpr int MATCH_NV = 2;  // sub-vectors per thread

__global__ void __launch_bounds__(256) match_block_kernel(
    const float *__restrict__ vecs, int64_t m, const float *__restrict__ entries,
    const double *__restrict__ inv, int fold, uint8_t *__restrict__ idx,
    uint8_t *__restrict__ signs, uint8_t *__restrict__ zero_mask,
    unsigned long long *__restrict__ n_neartie) {
  __shared__ __align__(16) float s_ent[NENT * 8];
  __shared__ double s_inv[NENT];
  __shared__ float s_inv32[NENT];
  for (int i = threadIdx.x; i < NENT * 8; i += blockDim.x) s_ent[i] = entries[i];
  for (int i = threadIdx.x; i < NENT; i += blockDim.x) {
    s_inv[i] = inv[i];
    s_inv32[i] = (float)inv[i];
  }
  __syncthreads();
  const int64_t base = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * MATCH_NV;
  if (base >= m) return;
  float u[MATCH_NV][8];
  uint32_t sb[MATCH_NV];
  bool zero[MATCH_NV];
#pragma unroll
  for (int i = 0; i < MATCH_NV; ++i) {
    float v[8];
    const int64_t r = min(base + i, m - 1);
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = vecs[r * 8 + k];
    zero[i] = sq_norm8_pairwise(v) < 1e-24;
    sb[i] = fold_signs(v, u[i], fold != 0);
  }
  int out[MATCH_NV];
  const uint32_t slow =
      match_multi<MATCH_NV>(u, reinterpret_cast<const float4 *>(s_ent), s_inv32, s_ent, s_inv, out);
  unsigned long long nslow = 0;
#pragma unroll
  for (int i = 0; i < MATCH_NV; ++i) {
    const int64_t r = base + i;
    if (r >= m) break;
    if ((slow >> i) & 1u) ++nslow;
    // zero_mask given: codebook.match_block semantics (substitute + flag);
    // NULL: the bare kernel (_native.pyx), which does not substitute
    const bool sub = zero_mask != nullptr && zero[i];
    idx[r] = sub ? 0 : (uint8_t)out[i];
    if (signs) signs[r] = sub ? 0 : (uint8_t)sb[i];
    if (zero_mask) zero_mask[r] = zero[i] ? 1 : 0;
  }
  if (n_neartie && nslow) atomicAdd(n_neartie, nslow);
}

// ---------------------------------------------------------------------------
// RoPE table: rope.py:35-51 evaluates theta = float64(pos) * freq_j in
// float64 and casts cos/sin to float32.  Same here (fp64 multiply is
// correctly rounded; fp64 cos/sin are within ~1 ulp, far below the float32
// rounding step).
// ---------------------------------------------------------------------------
__global__ void rope_table_kernel(const double *__restrict__ freqs, int64_t pos0, int64_t n,
                                  float2 *__restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n * NPAIR) return;
  const int64_t p = i / NPAIR;
  const int j = (int)(i - p * NPAIR);
  const double theta = __dmul_rn((double)(pos0 + p), freqs[j]);
  double s, c;
  sincos(theta, &s, &c);
  out[i] = make_float2(__double2float_rn(c), __double2float_rn(s));
}

}  // namespace nsnkv

using namespace nsnkv;

extern "C" int nsnkv_fwht_rows(const float *in, float *out, int64_t n, int32_t d,
                               void *stream) {
  if (d < 2 || (d & (d - 1)) != 0)
    return nsnkv_internal_set_error(NSNKV_ERR_NON_POWER_OF_TWO,
                                    "transform size must be a power of two >= 2");
  if (d > 8192) return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "fwht_rows: d > 8192");
  if (n < 0) return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "fwht_rows: n < 0");
  if (n == 0) return NSNKV_OK;
  int log_d = 0;
  while ((1 << log_d) < d) ++log_d;
  const int rows_per_block = d >= 1024 ? 1 : 1024 / d;
  const int64_t blocks = (n + rows_per_block - 1) / rows_per_block;
  const size_t smem = (size_t)rows_per_block * d * sizeof(float);
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(fwht_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const float scale = (float)(1.0 / sqrt((double)d));
  fwht_rows_kernel<<<(unsigned)blocks, 256, smem, (cudaStream_t)stream>>>(in, out, n, d, log_d,
                                                                         rows_per_block, scale);
  nsnkv_internal_count_launch(1);
  return nsnkv_internal_check_launch("fwht_rows");
}

extern "C" int nsnkv_match_block(const float *vecs, int64_t m, const float *entries,
                                 const double *inv_norms, int32_t fold, uint8_t *idx,
                                 uint8_t *signs, uint8_t *zero_mask, int64_t *n_neartie,
                                 void *stream) {
  if (m < 0) return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "match_block: m < 0");
  if (m == 0) return NSNKV_OK;
  if (fold && !signs)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "match_block: fold needs a signs buffer");
  const int64_t per_block = 256 * MATCH_NV;
  const int64_t blocks = (m + per_block - 1) / per_block;
  match_block_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(
      vecs, m, entries, inv_norms, fold, idx, fold ? signs : nullptr, zero_mask,
      reinterpret_cast<unsigned long long *>(n_neartie));
  nsnkv_internal_count_launch(1);
  return nsnkv_internal_check_launch("match_block");
}

extern "C" int nsnkv_rope_table(const double *freqs, int64_t pos0, int64_t n, float *out,
                                void *stream) {
  if (n < 0 || pos0 < 0) return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "rope_table: bad range");
  if (n == 0) return NSNKV_OK;
  const int64_t total = n * NPAIR;
  rope_table_kernel<<<(unsigned)((total + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
      freqs, pos0, n, reinterpret_cast<float2 *>(out));
  nsnkv_internal_count_launch(1);
  return nsnkv_internal_check_launch("rope_table");
}
