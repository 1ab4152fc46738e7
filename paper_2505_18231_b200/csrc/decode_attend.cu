// decode_attend.cu -- nsnkv_decode_attend (attention.py:136-142).
// v0: scores -> fp64 softmax -> weighted output, through the unfused kernels
// of decode_ref.cu.  Replaced by the split-K flash-decoding kernel.
#include "common.cuh"
#include "decode_common.cuh"

namespace nsnkv {

// softmax_rows (attention.py:46-50) on scores / sqrt(d), fp64, in place
// (fp32 result).  One CTA per (batch, q-head) row.
__global__ void __launch_bounds__(256) softmax_kernel(CacheViewDev cv, float *__restrict__ sw,
                                                      float *__restrict__ lse) {
  __shared__ double red[256];
  const int row = blockIdx.x;
  const int b = row / cv.n_q_heads, i = row - b * cv.n_q_heads;
  const int G = cv.n_q_heads / cv.n_kv_heads;
  const int u = b * cv.n_kv_heads + i / G;
  const int n = cv.n_chunks[u] * R + cv.n_res[u];
  float *s = sw + (int64_t)row * cv.max_tokens;
  const double inv_sqrt_d = 1.0 / sqrt(128.0);
  double mx = -1e300;
  for (int t = threadIdx.x; t < n; t += blockDim.x) mx = fmax(mx, (double)s[t] / sqrt(128.0));
  red[threadIdx.x] = mx;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + off]);
    __syncthreads();
  }
  mx = red[0];
  __syncthreads();
  double sum = 0.0;
  for (int t = threadIdx.x; t < n; t += blockDim.x) sum += exp((double)s[t] / sqrt(128.0) - mx);
  red[threadIdx.x] = sum;
  __syncthreads();
  for (int off = 128; off > 0; off >>= 1) {
    if (threadIdx.x < off) red[threadIdx.x] += red[threadIdx.x + off];
    __syncthreads();
  }
  sum = red[0];
  for (int t = threadIdx.x; t < n; t += blockDim.x)
    s[t] = (float)(exp((double)s[t] / sqrt(128.0) - mx) / sum);
  if (lse && threadIdx.x == 0) lse[row] = (float)(mx + log(sum));
  (void)inv_sqrt_d;
}

}  // namespace nsnkv

using namespace nsnkv;

static size_t scores_bytes(const CacheViewDev &cv) {
  return ((size_t)cv.batch * cv.n_q_heads * cv.max_tokens * sizeof(float) + 255) / 256 * 256;
}

extern "C" size_t nsnkv_decode_workspace_bytes(const nsnkv_cache_view *cv_in) {
  CacheViewDev cv;
  if (make_cache_view(cv_in, &cv)) return 0;
  return scores_bytes(cv) + nsnkv_internal_output_ws(cv);
}

extern "C" int nsnkv_decode_attend(const nsnkv_cache_view *cv_in, const float *q, float *out,
                                   float *lse, void *workspace, size_t workspace_bytes,
                                   void *stream) {
  CacheViewDev cv;
  int rc = make_cache_view(cv_in, &cv);
  if (rc) return rc;
  const size_t sb = scores_bytes(cv);
  if (workspace_bytes < sb + nsnkv_internal_output_ws(cv))
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "decode_attend: workspace too small");
  float *sw = (float *)workspace;
  rc = nsnkv_decode_scores(cv_in, q, sw, stream);
  if (rc) return rc;
  softmax_kernel<<<cv.batch * cv.n_q_heads, 256, 0, (cudaStream_t)stream>>>(cv, sw, lse);
  nsnkv_internal_count_launch(1);
  rc = nsnkv_internal_check_launch("decode_softmax");
  if (rc) return rc;
  return nsnkv_decode_output(cv_in, sw, out, (char *)workspace + sb, workspace_bytes - sb, stream);
}
