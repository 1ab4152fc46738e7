// match.cuh -- exact cosine codebook argmax on CUDA cores.
//
// Semantics follow reference pkg/src/nsnkv/kernels/_native.pyx:61-84:
//   u_k    = fp64(|v_k|) (fold) or fp64(v_k)
//   score  = ((u0*e0 + u1*e1) + ...) + u7*e7   (fp64, component order)
//   score *= inv[c]                            (fp64 1/||e_c||)
//   strict '>' argmax starting from -1e300 -> lowest index wins ties.
// f32 x f32 products are exact in fp64, so an fp64 FMA chain reproduces the
// reference bit-for-bit.
//
// Fast path: an fp32 FMA pre-pass tracks the best and second-best cosine.
// Its error against the exact fp64 score is < 11 * 2^-24 * ||u|| (8 rounded
// FMAs, one rounded fp32 inverse norm, one rounded multiply), so when the
// runner-up trails by more than 2 * 2^-20 * ||u|| the pre-pass winner IS the
// exact argmax.  Otherwise the sub-vector is re-scored exactly in fp64 over
// all 256 entries (a "near tie", counted).
#pragma once
#include "common.cuh"

namespace nsnkv {

// fp64 squared norm in numpy's pairwise order for n == 8
// (pairwise_sum: ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))); used for the
// zero-row test of codebook.py:118-120.
__device__ __forceinline__ double sq_norm8_pairwise(const float *v) {
  double r[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    double x = (double)v[k];
    r[k] = x * x;
  }
  return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

// Exact fp64 scan of all entries (the reference loop itself).
static __device__ __noinline__ int match_exact_fp64(const float *u, const float *ent,
                                             const double *inv) {
  double ud[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) ud[k] = (double)u[k];
  int best = 0;
  double best_score = -1e300;
  for (int c = 0; c < NENT; ++c) {
    const float *e = ent + c * 8;
    double s = __dmul_rn(ud[0], (double)e[0]);
#pragma unroll
    for (int k = 1; k < 8; ++k) s = __dadd_rn(s, __dmul_rn(ud[k], (double)e[k]));
    s = __dmul_rn(s, inv[c]);
    if (s > best_score) {
      best_score = s;
      best = c;
    }
  }
  return best;
}

// Fold a raw 8-dim sub-vector: u = |v| and sign byte (bit k set iff v_k < 0;
// -0.0 counts as non-negative), _native.pyx:63-69.
__device__ __forceinline__ uint32_t fold_signs(const float *v, float *u, bool fold) {
  uint32_t sb = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    if (fold && v[k] < 0.0f) {
      u[k] = -v[k];
      sb |= 1u << k;
    } else {
      u[k] = v[k];
    }
  }
  return fold ? sb : 0u;
}

// Match NV sub-vectors at once against the smem codebook (entries as float4
// pairs: ent4[2c], ent4[2c+1]).  Returns indices and a bitmask of which
// sub-vectors needed the exact pass.
template <int NV>
__device__ __forceinline__ uint32_t match_multi(const float (&u)[NV][8],
                                                const float4 *ent4,
                                                const float *inv32,
                                                const float *ent,
                                                const double *inv, int (&out)[NV]) {
  float best[NV], second[NV];
  int bi[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    best[i] = -3.0e38f;
    second[i] = -3.0e38f;
    bi[i] = 0;
  }
#pragma unroll 2
  for (int c = 0; c < NENT; ++c) {
    const float4 a = ent4[2 * c];
    const float4 b = ent4[2 * c + 1];
    const float iv = inv32[c];
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      float s = u[i][0] * a.x;
      s = fmaf(u[i][1], a.y, s);
      s = fmaf(u[i][2], a.z, s);
      s = fmaf(u[i][3], a.w, s);
      s = fmaf(u[i][4], b.x, s);
      s = fmaf(u[i][5], b.y, s);
      s = fmaf(u[i][6], b.z, s);
      s = fmaf(u[i][7], b.w, s);
      s *= iv;
      // top-2 tracking; strict '>' keeps the lowest index on fp32 ties
      second[i] = fmaxf(second[i], fminf(best[i], s));
      if (s > best[i]) bi[i] = c;
      best[i] = fmaxf(best[i], s);
    }
  }
  uint32_t slow = 0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float n2 = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) n2 = fmaf(u[i][k], u[i][k], n2);
    const float bound = 2.0f * 9.5367431640625e-07f * sqrtf(n2);  // 2 * 2^-20 * ||u||
    // tiny or huge rows leave the relative-error regime of fp32: go exact
    const bool scaled_ok = n2 > 1e-24f && n2 < 1e30f;
    if (!scaled_ok || !(second[i] < best[i] - bound)) {
      slow |= 1u << i;
      out[i] = match_exact_fp64(u[i], ent, inv);
    } else {
      out[i] = bi[i];
    }
  }
  return slow;
}

}  // namespace nsnkv
