// codebook_build.cu -- the per-sample passes of the codebook build on the GPU
// (reference codebook.py:175-340): Lloyd's assignment + accumulation for
// kmeans_init, and the assignment statistics of one cosine fine-tune step.
// The random streams stay on the host (numpy PCG64, the reference's own draw
// order), and the assignment rule of the fine-tune is the exact cosine match
// (nsnkv_match_block); these kernels do the O(n * 256) and O(n) work.
#include "common.cuh"

namespace nsnkv {

// numpy pairwise sum of 8 doubles (n == 8: the 8-accumulator unrolled block)
__device__ __forceinline__ double np_sum8(const double *a) {
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

constexpr int KM_THREADS = 256;

// kmeans_init iteration (codebook.py:196-212): gram = data @ f32(centroids).T,
// assign = argmax(gram - 0.5 * f32(|c|^2)) (first maximum), then the fp64
// per-cluster sums and counts; d2 (optional) = squared distance of every
// point to its centroid, for the empty-cluster reseed.
__global__ void __launch_bounds__(KM_THREADS) kmeans_assign_kernel(
    const float *__restrict__ data, int64_t n, const double *__restrict__ centroids,
    int32_t *__restrict__ assign, double *__restrict__ sums, int32_t *__restrict__ counts,
    double *__restrict__ d2) {
  __shared__ float c32[NENT][8];
  __shared__ float hc[NENT];      // f32(0.5) * f32(|c|^2)
  __shared__ double csq[NENT];
  for (int c = threadIdx.x; c < NENT; c += KM_THREADS) {
    double sq[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double v = centroids[c * 8 + k];
      c32[c][k] = (float)v;
      sq[k] = v * v;
    }
    csq[c] = np_sum8(sq);
    hc[c] = __fmul_rn(0.5f, (float)csq[c]);
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * KM_THREADS + threadIdx.x;
  if (i >= n) return;
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = data[i * 8 + k];
  int best = 0;
  float bs = -INFINITY, bg = 0.f;
  for (int c = 0; c < NENT; ++c) {
    float g = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) g = __fmaf_rn(x[k], c32[c][k], g);
    const float s = __fsub_rn(g, hc[c]);
    if (s > bs) {  // strict: the first maximum wins (np.argmax)
      bs = s;
      best = c;
      bg = g;
    }
  }
  assign[i] = best;
  atomicAdd(&counts[best], 1);
#pragma unroll
  for (int k = 0; k < 8; ++k) atomicAdd(&sums[best * 8 + k], (double)x[k]);
  if (d2) {
    double sq[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) sq[k] = (double)x[k] * (double)x[k];
    d2[i] = np_sum8(sq) - 2.0 * (double)bg + csq[best];
  }
}

// finetune step statistics (codebook.py:300-318): unit vectors of the batch,
// cosine to the matched entry, per-entry sums of unit vectors and cosines,
// counts of live samples, and the batch's summed cosine distance.
__global__ void __launch_bounds__(KM_THREADS) finetune_stats_kernel(
    const float *__restrict__ batch, int64_t n, const int32_t *__restrict__ idx,
    const double *__restrict__ entries, double *__restrict__ sum_unit,
    double *__restrict__ sum_cos, int32_t *__restrict__ counts, double *__restrict__ cosdist) {
  __shared__ double e[NENT][8];
  __shared__ double en[NENT];
  for (int c = threadIdx.x; c < NENT; c += KM_THREADS) {
    double sq[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      e[c][k] = entries[c * 8 + k];
      sq[k] = e[c][k] * e[c][k];
    }
    en[c] = sqrt(np_sum8(sq));
  }
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * KM_THREADS + threadIdx.x;
  double dist = 0.0;
  if (i < n) {
    double u[8], sq[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      u[k] = (double)batch[i * 8 + k];
      sq[k] = u[k] * u[k];
    }
    const double un = sqrt(np_sum8(sq));
    if (un > 1e-12) {
      const int c = idx[i];
      double dot[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        u[k] /= un;
        dot[k] = u[k] * e[c][k];
      }
      const double cs = np_sum8(dot) / en[c];
#pragma unroll
      for (int k = 0; k < 8; ++k) atomicAdd(&sum_unit[c * 8 + k], u[k]);
      atomicAdd(&sum_cos[c], cs);
      atomicAdd(&counts[c], 1);
      dist = 1.0 - cs;
    }
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) dist += __shfl_xor_sync(0xffffffffu, dist, off);
  if ((threadIdx.x & 31) == 0 && dist != 0.0) atomicAdd(cosdist, dist);
}

}  // namespace nsnkv

using namespace nsnkv;

extern "C" int nsnkv_kmeans_assign(const float *data, int64_t n, const double *centroids,
                                   int32_t *assign, double *sums, int32_t *counts, double *d2,
                                   void *stream) {
  if (n < 0 || (n > 0 && (!data || !centroids || !assign || !sums || !counts)))
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "kmeans_assign: bad arguments");
  if (n == 0) return NSNKV_OK;
  kmeans_assign_kernel<<<(unsigned)((n + KM_THREADS - 1) / KM_THREADS), KM_THREADS, 0,
                         (cudaStream_t)stream>>>(data, n, centroids, assign, sums, counts, d2);
  nsnkv_internal_count_launch(1);
  return nsnkv_internal_check_launch("kmeans_assign");
}

extern "C" int nsnkv_finetune_stats(const float *batch, int64_t n, const int32_t *idx,
                                    const double *entries, double *sum_unit, double *sum_cos,
                                    int32_t *counts, double *cosdist, void *stream) {
  if (n < 0 || (n > 0 && (!batch || !idx || !entries || !sum_unit || !sum_cos || !counts || !cosdist)))
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "finetune_stats: bad arguments");
  if (n == 0) return NSNKV_OK;
  finetune_stats_kernel<<<(unsigned)((n + KM_THREADS - 1) / KM_THREADS), KM_THREADS, 0,
                          (cudaStream_t)stream>>>(batch, n, idx, entries, sum_unit, sum_cos,
                                                  counts, cosdist);
  nsnkv_internal_count_launch(1);
  return nsnkv_internal_check_launch("finetune_stats");
}
