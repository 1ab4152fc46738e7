/*
 * nsnkv_oracle.c -- CPU restatement of the NSNQuant KV-cache hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker for the CUDA product
 * (paper_2505_18231_b200/csrc) and the CPU baseline timed by bench.py's
 * reference arm.  Nothing in the product links, loads or calls it.
 *
 * It restates the reference algorithm (reference = /root/reference/pkg,
 * package nsnkv) operation by operation:
 *   orc_fwht_rows        kernels/_native.pyx:16-38
 *   orc_match_block      kernels/_native.pyx:41-87, codebook.py:109-128
 *   orc_encode_chunk     kvcache.py:114-154 -> nsn.py:58-85, core.py:50-66,
 *                        rope.py:35-51, hadamard.py:65-83, vq.py:74-93,
 *                        vq.py:100-166, vq.py:211-279, serialize vq.py:363-380
 *   orc_attend           attention.py:83-142 (scores, fp64 softmax, output)
 * Where numpy's order is ISA-dependent (the fp32 einsum row norms,
 * core.py:53) the oracle fixes one canonical order -- the one the CUDA
 * kernel uses -- and the tests check it against the reference within 1e-5
 * (SURVEY.md Appendix A).  Everything else follows numpy's documented order
 * (pairwise 8-accumulator sums for n <= 128, sequential axis-0 means).
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off, IEEE SSE2 math).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define D 128
#define R 64
#define NSUB 16
#define NPAIR 64
#define NENT 256

/* ---------------------------------------------------------------------- */
/* f32 <-> f16, round-to-nearest-even (numpy astype(float16))              */
/* ---------------------------------------------------------------------- */
uint16_t orc_f32_to_f16(float f) {
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t e = (x >> 23) & 0xffu, m = x & 0x7fffffu;
  if (e == 0xffu) return (uint16_t)(sign | 0x7c00u | (m ? 0x200u : 0u));
  int32_t ex = (int32_t)e - 127 + 15;
  if (ex >= 31) return (uint16_t)(sign | 0x7c00u);
  if (ex <= 0) {
    if (ex < -10) return (uint16_t)sign;
    m |= 0x800000u;
    int shift = 14 - ex;
    uint32_t hm = m >> shift, rem = m & ((1u << shift) - 1u), halfway = 1u << (shift - 1);
    if (rem > halfway || (rem == halfway && (hm & 1u))) hm++;
    return (uint16_t)(sign | hm);
  }
  uint32_t h = sign | ((uint32_t)ex << 10) | (m >> 13);
  uint32_t rem = m & 0x1fffu;
  if (rem > 0x1000u || (rem == 0x1000u && (h & 1u))) h++;
  return (uint16_t)h;
}

float orc_f16_to_f32(uint16_t h) {
  uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
  uint32_t e = (h >> 10) & 0x1fu, m = h & 0x3ffu;
  uint32_t x;
  if (e == 0) {
    if (m == 0) {
      x = sign;
    } else {
      int k = 0;
      while (!(m & 0x400u)) { m <<= 1; ++k; }
      m &= 0x3ffu;
      x = sign | ((uint32_t)(113 - k) << 23) | (m << 13);
    }
  } else if (e == 31) {
    x = sign | 0x7f800000u | (m << 13);
  } else {
    x = sign | ((e + 112u) << 23) | (m << 13);
  }
  float f;
  memcpy(&f, &x, 4);
  return f;
}

/* ---------------------------------------------------------------------- */
/* fwht_rows (_native.pyx:16-38)                                            */
/* ---------------------------------------------------------------------- */
void orc_fwht_row(float *m, int d) {
  for (int h = 1; h < d; h *= 2)
    for (int i = 0; i < d; i += 2 * h)
      for (int j = i; j < i + h; ++j) {
        float x = m[j], y = m[j + h];
        m[j] = x + y;
        m[j + h] = x - y;
      }
  float scale = (float)(1.0 / sqrt((double)d));
  for (int j = 0; j < d; ++j) m[j] = m[j] * scale;
}

void orc_fwht_rows(const float *in, float *out, int64_t n, int d) {
  if (out != in) memcpy(out, in, (size_t)n * d * sizeof(float));
  for (int64_t r = 0; r < n; ++r) orc_fwht_row(out + r * d, d);
}

/* ---------------------------------------------------------------------- */
/* match (_native.pyx:41-87; zero rows codebook.py:118-127)                */
/* ---------------------------------------------------------------------- */
void orc_entry_inv_norms(const float *entries, double *inv) { /* kernels/__init__.py:44-51 */
  for (int c = 0; c < NENT; ++c) {
    const float *e = entries + 8 * c;
    double s = (double)e[0] * (double)e[0];
    for (int k = 1; k < 8; ++k) s = s + (double)e[k] * (double)e[k];
    inv[c] = 1.0 / sqrt(s);
  }
}

static double sq_norm8_pairwise(const float *v) { /* numpy pairwise_sum, n == 8 */
  double r[8];
  for (int k = 0; k < 8; ++k) r[k] = (double)v[k] * (double)v[k];
  return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

static int match_one(const float *v, const float *entries, const double *inv, int fold,
                     uint8_t *sign_out) {
  double u[8];
  int sb = 0;
  for (int k = 0; k < 8; ++k) {
    if (fold && v[k] < 0) {
      u[k] = (double)(-v[k]);
      sb |= 1 << k;
    } else {
      u[k] = (double)v[k];
    }
  }
  int best = 0;
  double best_score = -1e300;
  for (int c = 0; c < NENT; ++c) {
    const float *e = entries + 8 * c;
    double s = u[0] * (double)e[0];
    for (int k = 1; k < 8; ++k) s = s + u[k] * (double)e[k];
    s = s * inv[c];
    if (s > best_score) {
      best_score = s;
      best = c;
    }
  }
  *sign_out = (uint8_t)sb;
  return best;
}

/* zero_mask == NULL: bare kernel; otherwise codebook.match_block semantics */
void orc_match_block(const float *vecs, int64_t m, const float *entries, const double *inv,
                     int fold, uint8_t *idx, uint8_t *signs, uint8_t *zero_mask) {
  for (int64_t i = 0; i < m; ++i) {
    uint8_t sb;
    int b = match_one(vecs + 8 * i, entries, inv, fold, &sb);
    int zero = zero_mask && sq_norm8_pairwise(vecs + 8 * i) < 1e-24;
    idx[i] = zero ? 0 : (uint8_t)b;
    if (signs) signs[i] = zero ? 0 : sb;
    if (zero_mask) zero_mask[i] = (uint8_t)(sq_norm8_pairwise(vecs + 8 * i) < 1e-24);
  }
}

/* ---------------------------------------------------------------------- */
/* encode one chunk (kvcache.py:114-154) -> reference wire bytes            */
/* ---------------------------------------------------------------------- */

/* Canonical fp64 sum of squares of a 128-row: lane partials over 4
 * consecutive elements, then an xor butterfly 16..1 (matches the kernel). */
static double row_sumsq_canon(const float *x) {
  double p[32], q[32];
  for (int l = 0; l < 32; ++l) {
    double s = (double)x[4 * l] * (double)x[4 * l];
    s = s + (double)x[4 * l + 1] * (double)x[4 * l + 1];
    s = s + (double)x[4 * l + 2] * (double)x[4 * l + 2];
    s = s + (double)x[4 * l + 3] * (double)x[4 * l + 3];
    p[l] = s;
  }
  for (int off = 16; off >= 1; off >>= 1) {
    for (int l = 0; l < 32; ++l) q[l] = p[l] + p[l ^ off];
    memcpy(p, q, sizeof(p));
  }
  return p[0];
}

/* _scale_per_token (nsn.py:58-65) in place; returns clamps */
static int scale_rows(float (*x)[D], int n, float *s_out) {
  const float sqrt_d = (float)11.313708498984761;
  int clamps = 0;
  for (int t = 0; t < n; ++t) {
    float nrm = sqrtf((float)row_sumsq_canon(x[t]));
    float s = nrm / sqrt_d;
    if (s < 1e-8f) {
      s = 1e-8f;
      ++clamps;
    }
    for (int c = 0; c < D; ++c) x[t][c] = x[t][c] / s;
    s_out[t] = s;
  }
  return clamps;
}

/* numpy pairwise sum of 128 fp64 values (8 accumulators) */
static double pairwise128(const double *a) {
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  for (int i = 8; i < 128; i += 8)
    for (int j = 0; j < 8; ++j) r[j] += a[i + j];
  return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
}

static void rtn4(const float *v, int n, uint16_t *scale16, uint16_t *zero16, uint8_t *levels) {
  float lo = v[0], hi = v[0];
  for (int i = 1; i < n; ++i) {
    if (v[i] < lo) lo = v[i];
    if (v[i] > hi) hi = v[i];
  }
  float sc = (hi == lo) ? 1.0f : (hi - lo) / 15.0f; /* vq.py:109 */
  *scale16 = orc_f32_to_f16(sc);
  *zero16 = orc_f32_to_f16(lo);
  float s32 = orc_f16_to_f32(*scale16), z32 = orc_f16_to_f32(*zero16);
  for (int i = 0; i < n; ++i) { /* vq.py:113-117 */
    float lv = rintf((v[i] - z32) / s32);
    if (lv != lv) lv = 0.f;
    if (lv < 0.f) lv = 0.f;
    if (lv > 15.f) lv = 15.f;
    levels[i] = (uint8_t)lv;
  }
}

/* bytes of one wire chunk (vq.py:363-380) */
int orc_wire_bytes(int bit_mode) { return 6 + 1024 + (bit_mode == 2 ? 1024 : 0) + 36 + 80 + 128; }

/*
 * rows: [64][128] fp32 (keys pre-RoPE, or values post-HT).
 * rope_cs: [64][64][2] fp32 cos/sin for positions start .. start+63 (keys).
 * wire: orc_wire_bytes(bit_mode) bytes out.
 * nsn_out (may be NULL): s1[64], o[128], s2[64] pre-DQ byproducts, s2_adj[64].
 * counters[4]: clamps, zero sub-vectors, S3 fallbacks, 0.
 */
void orc_encode_chunk(const float *rows, int is_key, const float *rope_cs, const float *entries,
                      const double *inv, int bit_mode, int strategy, uint8_t *wire,
                      float *nsn_out, int32_t *counters) {
  static __thread float x[R][D];
  float s1[R], s2[R], o[D], s2adj[R];
  uint8_t idx[R][NSUB], sgn[R][NSUB];
  int fold = bit_mode == 2;
  memcpy(x, rows, sizeof(x));
  /* nsn_forward (nsn.py:68-85) */
  int clamps = scale_rows(x, R, s1);
  for (int c = 0; c < D; ++c) { /* col_means (core.py:56-66) */
    double acc = 0.0;
    for (int t = 0; t < R; ++t) acc = acc + (double)x[t][c];
    o[c] = (float)(acc / (double)R);
  }
  for (int t = 0; t < R; ++t)
    for (int c = 0; c < D; ++c) x[t][c] = x[t][c] - o[c];
  clamps += scale_rows(x, R, s2);
  if (is_key) { /* rope_rows (rope.py:35-51) then apply_rows (hadamard.py:65-83) */
    for (int t = 0; t < R; ++t) {
      for (int j = 0; j < NPAIR; ++j) {
        float c = rope_cs[(t * NPAIR + j) * 2], s = rope_cs[(t * NPAIR + j) * 2 + 1];
        float e = x[t][2 * j], od = x[t][2 * j + 1];
        float pe = e * c, po = od * s, qe = e * s, qo = od * c;
        x[t][2 * j] = pe - po;
        x[t][2 * j + 1] = qe + qo;
      }
      orc_fwht_row(x[t], D);
    }
  }
  /* match (codebook.match_block) */
  int zeros = 0;
  for (int t = 0; t < R; ++t)
    for (int j = 0; j < NSUB; ++j) {
      const float *v = &x[t][8 * j];
      uint8_t sb;
      int b = match_one(v, entries, inv, fold, &sb);
      if (sq_norm8_pairwise(v) < 1e-24) {
        b = 0;
        sb = 0;
        ++zeros;
      }
      idx[t][j] = (uint8_t)b;
      sgn[t][j] = fold ? sb : 0;
    }
  /* _adjust_factors (vq.py:74-93) and s2 adjustment (vq.py:254) */
  int fallbacks = 0;
  for (int t = 0; t < R; ++t) {
    double av[D], aq[D], ad[D];
    for (int c = 0; c < D; ++c) {
      int j = c >> 3, k = c & 7;
      float cv = entries[idx[t][j] * 8 + k];
      if (fold && ((sgn[t][j] >> k) & 1)) cv = -cv;
      double vd = (double)x[t][c], cd = (double)cv;
      av[c] = vd * vd;
      aq[c] = cd * cd;
      ad[c] = vd * cd;
    }
    double v2 = pairwise128(av), q2 = pairwise128(aq), dt = pairwise128(ad);
    double f = 1.0;
    if (strategy == 1) {
      f = dt / q2;
    } else if (strategy == 2) {
      f = sqrt(v2 / q2);
    } else if (strategy == 3) {
      int bad = fabs(dt) <= 1e-10 * sqrt(v2 * q2);
      f = bad ? sqrt(v2 / q2) : v2 / dt;
      fallbacks += bad;
    }
    s2adj[t] = (float)((double)s2[t] * f);
  }
  /* double quantization (vq.py:155-166) and the wire form (vq.py:363-380) */
  uint8_t *w = wire;
  w[0] = R & 0xff; w[1] = R >> 8; w[2] = D & 0xff; w[3] = D >> 8;
  w[4] = (uint8_t)bit_mode; w[5] = (uint8_t)strategy;
  w += 6;
  memcpy(w, idx, R * NSUB);
  w += R * NSUB;
  if (fold) {
    memcpy(w, sgn, R * NSUB);
    w += R * NSUB;
  }
  uint8_t lv[D];
  uint16_t sc16, z16;
  rtn4(s1, R, &sc16, &z16, lv);
  memcpy(w, &sc16, 2); memcpy(w + 2, &z16, 2);
  w += 4;
  for (int i = 0; i < R / 2; ++i) w[i] = (uint8_t)(lv[2 * i] | (lv[2 * i + 1] << 4));
  w += R / 2;
  uint8_t olv[D];
  for (int g = 0; g < 4; ++g) {
    rtn4(o + 32 * g, 32, &sc16, &z16, olv + 32 * g);
    memcpy(w, &sc16, 2); memcpy(w + 2, &z16, 2);
    w += 4;
  }
  for (int i = 0; i < D / 2; ++i) w[i] = (uint8_t)(olv[2 * i] | (olv[2 * i + 1] << 4));
  w += D / 2;
  for (int t = 0; t < R; ++t) {
    uint16_t h = orc_f32_to_f16(s2adj[t]);
    memcpy(w + 2 * t, &h, 2);
  }
  if (nsn_out) {
    memcpy(nsn_out, s1, sizeof(s1));
    memcpy(nsn_out + R, o, sizeof(o));
    memcpy(nsn_out + R + D, s2, sizeof(s2));
    memcpy(nsn_out + 2 * R + D, s2adj, sizeof(s2adj));
  }
  if (counters) {
    counters[0] = clamps;
    counters[1] = zeros;
    counters[2] = fallbacks;
    counters[3] = 0;
  }
}

/* ---------------------------------------------------------------------- */
/* decode over wire chunks (attention.py:83-142)                            */
/* ---------------------------------------------------------------------- */
typedef struct {
  const uint8_t *idx, *sgn, *s1n, *on, *s2;
  float s1_scale, s1_zero, o_scale[4], o_zero[4];
} wire_view;

static void parse_wire(const uint8_t *w, int bit_mode, wire_view *v) {
  const uint8_t *p = w + 6;
  uint16_t h;
  v->idx = p;
  p += 1024;
  v->sgn = NULL;
  if (bit_mode == 2) {
    v->sgn = p;
    p += 1024;
  }
  memcpy(&h, p, 2); v->s1_scale = orc_f16_to_f32(h);
  memcpy(&h, p + 2, 2); v->s1_zero = orc_f16_to_f32(h);
  p += 4;
  v->s1n = p;
  p += 32;
  for (int g = 0; g < 4; ++g) {
    memcpy(&h, p, 2); v->o_scale[g] = orc_f16_to_f32(h);
    memcpy(&h, p + 2, 2); v->o_zero[g] = orc_f16_to_f32(h);
    p += 4;
  }
  v->on = p;
  p += 64;
  v->s2 = p;
}

static inline float nib(const uint8_t *p, int i) { return (float)((i & 1) ? (p[i >> 1] >> 4) : (p[i >> 1] & 15)); }

/* rows s1 * (s2 * payload + o) pieces for one chunk (vq.py:193-208) */
static void chunk_pieces(const wire_view *v, const float *entries, float (*payload)[D], float *s1,
                         float *s2, float *o) {
  for (int t = 0; t < R; ++t) {
    s1[t] = v->s1_zero + nib(v->s1n, t) * v->s1_scale;
    uint16_t h;
    memcpy(&h, v->s2 + 2 * t, 2);
    s2[t] = orc_f16_to_f32(h);
    for (int j = 0; j < NSUB; ++j) {
      int e = v->idx[t * NSUB + j];
      int sb = v->sgn ? v->sgn[t * NSUB + j] : 0;
      for (int k = 0; k < 8; ++k) {
        float c = entries[e * 8 + k];
        payload[t][8 * j + k] = ((sb >> k) & 1) ? c * -1.0f : c;
      }
    }
  }
  for (int c = 0; c < D; ++c) o[c] = v->o_zero[c >> 5] + nib(v->on, c) * v->o_scale[c >> 5];
}

/*
 * One unit (one reference KvCacheState) and G queries.
 * kw, vw: n_chunks wire chunks each (stride orc_wire_bytes).
 * k_res (pre-RoPE), v_res (post-HT): n_res rows.  rope_cs: table rows for
 * absolute positions 0 .. (covering base_pos + total).  q: [G][128] RoPE'd.
 * Outputs (each may be NULL): scores[G][T], weights[G][T], out[G][128].
 */
void orc_attend(const uint8_t *kw, const uint8_t *vw, int n_chunks, const float *k_res,
                const float *v_res, int n_res, int64_t base_pos, const float *rope_cs,
                const float *ent_k, const float *ent_v, int bit_mode, const float *q, int G,
                float *scores, float *weights, float *out) {
  const int T = n_chunks * R + n_res;
  const int wb = orc_wire_bytes(bit_mode);
  float *sc = (float *)malloc(sizeof(float) * (size_t)G * (T ? T : 1));
  float (*payload)[D] = malloc(sizeof(float) * R * D);
  float s1[R], s2[R], o[D], qh[D];
  for (int g = 0; g < G; ++g) {
    const float *qg = q + g * D;
    memcpy(qh, qg, sizeof(qh));
    orc_fwht_row(qh, D); /* attention.py:93 */
    for (int ci = 0; ci < n_chunks; ++ci) {
      wire_view v;
      parse_wire(kw + (size_t)ci * wb, bit_mode, &v);
      chunk_pieces(&v, ent_k, payload, s1, s2, o);
      for (int t = 0; t < R; ++t) {
        int64_t pos = base_pos + (int64_t)ci * R + t;
        const float *cs = rope_cs + pos * NPAIR * 2;
        float pd = 0.f, sd = 0.f;
        for (int c = 0; c < D; ++c) pd += payload[t][c] * qh[c];
        for (int j = 0; j < NPAIR; ++j) { /* rope_expand(o, pos) . q */
          float e = o[2 * j], od = o[2 * j + 1], c = cs[2 * j], s = cs[2 * j + 1];
          float re = e * c - od * s, ro = e * s + od * c;
          sd += re * qg[2 * j];
          sd += ro * qg[2 * j + 1];
        }
        sc[(size_t)g * T + ci * R + t] = s1[t] * (s2[t] * pd + sd);
      }
    }
    for (int t = 0; t < n_res; ++t) { /* exact residual scores */
      int64_t pos = base_pos + (int64_t)n_chunks * R + t;
      const float *cs = rope_cs + pos * NPAIR * 2;
      const float *kr = k_res + (size_t)t * D;
      float acc = 0.f;
      for (int j = 0; j < NPAIR; ++j) {
        float e = kr[2 * j], od = kr[2 * j + 1], c = cs[2 * j], s = cs[2 * j + 1];
        float re = e * c - od * s, ro = e * s + od * c;
        acc += re * qg[2 * j];
        acc += ro * qg[2 * j + 1];
      }
      sc[(size_t)g * T + n_chunks * R + t] = acc;
    }
  }
  if (scores) memcpy(scores, sc, sizeof(float) * (size_t)G * T);
  /* softmax_rows of scores / sqrt(d) in fp64 (attention.py:46-50, 141) */
  float *w = (float *)malloc(sizeof(float) * (size_t)G * (T ? T : 1));
  const double sq = sqrt((double)D);
  for (int g = 0; g < G; ++g) {
    double mx = -1e300, sum = 0.0;
    for (int t = 0; t < T; ++t) {
      double z = (double)sc[(size_t)g * T + t] / sq;
      if (z > mx) mx = z;
    }
    for (int t = 0; t < T; ++t) sum += exp((double)sc[(size_t)g * T + t] / sq - mx);
    for (int t = 0; t < T; ++t)
      w[(size_t)g * T + t] = (float)(exp((double)sc[(size_t)g * T + t] / sq - mx) / sum);
  }
  if (weights) memcpy(weights, w, sizeof(float) * (size_t)G * T);
  if (out) { /* output_quantized (attention.py:114-133) */
    float acc[D];
    for (int g = 0; g < G; ++g) {
      memset(acc, 0, sizeof(acc));
      for (int ci = 0; ci < n_chunks; ++ci) {
        wire_view v;
        parse_wire(vw + (size_t)ci * wb, bit_mode, &v);
        chunk_pieces(&v, ent_v, payload, s1, s2, o);
        for (int t = 0; t < R; ++t) {
          float wt = w[(size_t)g * T + ci * R + t];
          for (int c = 0; c < D; ++c) acc[c] += wt * (s1[t] * (s2[t] * payload[t][c] + o[c]));
        }
      }
      for (int t = 0; t < n_res; ++t) {
        float wt = w[(size_t)g * T + n_chunks * R + t];
        for (int c = 0; c < D; ++c) acc[c] += wt * v_res[(size_t)t * D + c];
      }
      orc_fwht_row(acc, D);
      memcpy(out + g * D, acc, sizeof(acc));
    }
  }
  free(w);
  free(payload);
  free(sc);
}

/* ---------------------------------------------------------------------- */
/* multi-threaded drivers for the CPU baseline                              */
/* ---------------------------------------------------------------------- */
typedef struct {
  int kind; /* 0 encode, 1 attend */
  int64_t begin, end;
  /* encode */
  const float *rows; int is_key; const float *rope_cs; const float *entries; const double *inv;
  int bit_mode, strategy; uint8_t *wire; const int64_t *pos0;
  /* attend */
  const uint8_t *kw, *vw; int n_chunks; const float *ent_k, *ent_v; const float *q; int G;
  float *out; int64_t units_stride_k;
} job_t;

static void *worker(void *arg) {
  job_t *j = (job_t *)arg;
  int wb = orc_wire_bytes(j->bit_mode);
  for (int64_t i = j->begin; i < j->end; ++i) {
    if (j->kind == 0) {
      const float *cs = j->rope_cs && j->pos0 ? j->rope_cs + j->pos0[i] * (2 * NPAIR) : j->rope_cs;
      orc_encode_chunk(j->rows + i * R * D, j->is_key, cs, j->entries, j->inv,
                       j->bit_mode, j->strategy, j->wire + i * wb, NULL, NULL);
    } else {
      orc_attend(j->kw + i * j->units_stride_k, j->vw + i * j->units_stride_k, j->n_chunks, NULL,
                 NULL, 0, 0, j->rope_cs, j->ent_k, j->ent_v, j->bit_mode, j->q + i * j->G * D,
                 j->G, NULL, NULL, j->out + i * j->G * D);
    }
  }
  return NULL;
}

static void run_jobs(job_t *proto, int64_t n, int threads) {
  if (threads < 1) threads = 1;
  pthread_t *th = malloc(sizeof(pthread_t) * threads);
  job_t *jobs = malloc(sizeof(job_t) * threads);
  for (int i = 0; i < threads; ++i) {
    jobs[i] = *proto;
    jobs[i].begin = n * i / threads;
    jobs[i].end = n * (i + 1) / threads;
    pthread_create(&th[i], NULL, worker, &jobs[i]);
  }
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
  free(jobs);
  free(th);
}

/* n chunks of [64][128] rows, all at the same start position (rope_cs rows) */
void orc_encode_many(const float *rows, int64_t n, int is_key, const float *rope_cs,
                     const float *entries, const double *inv, int bit_mode, int strategy,
                     uint8_t *wire, int threads) {
  job_t p;
  memset(&p, 0, sizeof(p));
  p.kind = 0; p.rows = rows; p.is_key = is_key; p.rope_cs = rope_cs; p.entries = entries;
  p.inv = inv; p.bit_mode = bit_mode; p.strategy = strategy; p.wire = wire;
  run_jobs(&p, n, threads);
}

/* n chunks of [64][128] rows; chunk i's first position is row pos0[i] of the
 * rope table (keys), so whole caches encode in one call (parity tests) */
void orc_encode_many_pos(const float *rows, int64_t n, int is_key, const float *rope_table,
                         const int64_t *pos0, const float *entries, const double *inv,
                         int bit_mode, int strategy, uint8_t *wire, int threads) {
  job_t p;
  memset(&p, 0, sizeof(p));
  p.kind = 0; p.rows = rows; p.is_key = is_key; p.rope_cs = rope_table; p.pos0 = pos0;
  p.entries = entries; p.inv = inv; p.bit_mode = bit_mode; p.strategy = strategy; p.wire = wire;
  run_jobs(&p, n, threads);
}

/* n_units independent units with n_chunks wire chunks each (no residual,
 * base position 0), G queries each -> out[n_units][G][128] */
void orc_attend_many(const uint8_t *kw, const uint8_t *vw, int64_t n_units, int n_chunks,
                     const float *rope_cs, const float *ent_k, const float *ent_v, int bit_mode,
                     const float *q, int G, float *out, int threads) {
  job_t p;
  memset(&p, 0, sizeof(p));
  p.kind = 1; p.kw = kw; p.vw = vw; p.n_chunks = n_chunks; p.rope_cs = rope_cs;
  p.ent_k = ent_k; p.ent_v = ent_v; p.bit_mode = bit_mode; p.q = q; p.G = G; p.out = out;
  p.units_stride_k = (int64_t)n_chunks * orc_wire_bytes(bit_mode);
  run_jobs(&p, n_units, threads);
}
