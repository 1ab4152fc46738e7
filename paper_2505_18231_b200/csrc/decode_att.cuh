// decode_att.cuh -- PTX helpers, chunk cursor, stream-K records and the
// combine kernel shared by the decode kernels (decode_attend.cu, decode_attend3.cu).
#pragma once
#include "common.cuh"
#include "decode_common.cuh"

namespace nsnkv {

// ---------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0,%1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
// four 8x8 b16 matrices, transposed: lane l supplies the 16-byte row address
// of row l % 8 of matrix l / 8; register i receives matrix i's elements
// (row 2t, col g) and (row 2t + 1, col g) of thread (g, t)
__device__ __forceinline__ void ldsm_x4_trans(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_1d(void *dst, const void *src, uint32_t bytes,
                                            uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// x ^ (w & 0x80008000): flip the fp16 sign bits selected by bits 15 / 31 of w
// in one LOP3
__device__ __forceinline__ uint32_t xor_sign(uint32_t x, uint32_t w) {
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0x78;" : "=r"(r) : "r"(x), "r"(w), "r"(0x80008000u));
  return r;
}
__device__ __forceinline__ void named_bar(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ uint32_t pack_h2(float lo16, float hi16) {
  const __half2 h = __floats2half2_rn(lo16, hi16);
  return *reinterpret_cast<const uint32_t *>(&h);
}
// x = hi + lo with hi = fp16(x), lo = fp16(x - hi)
__device__ __forceinline__ void split_h(float x, float &hi, float &lo) {
  hi = __half2float(__float2half_rn(x));
  lo = x - hi;
}

// ---------------------------------------------------------------------------
// configuration
// ---------------------------------------------------------------------------
constexpr int ROPE_ROW_BYTES = NPAIR * 8;        // 64 x (cos, sin) fp32
constexpr int STAGE_BYTES = 2 * NSNKV_PAGE_BYTES_2B + ROPE_ROW_BYTES;
constexpr int ATT_SMEM_BYTES = 232448;           // 227 KB: two 64 KB-aligned tables + misc
constexpr int MISC_LO_MAX = 65536 - 1024;        // below the tables (1 KB is reserved)
constexpr int MISC_HI_MAX = 232448 + 1024 - 196608;  // above the tables
constexpr float LOG2E_OVER_SQRTD = 1.4426950408889634f * 0.08838834764831845f;

struct ChunkCursor {
  int u, c, n;  // unit, chunk within unit, chunks of the unit
};

__device__ __forceinline__ void cursor_advance(ChunkCursor &cur, const int32_t *n_chunks,
                                               int n_units) {
  if (++cur.c >= cur.n) {
    cur.c = 0;
    cur.n = 0;
    while (cur.n == 0 && ++cur.u < n_units) cur.n = n_chunks[cur.u];
  }
}

// Warp-parallel seek of global chunk x (all 32 lanes call; every lane gets
// the result).  Units with zero chunks are skipped.
__device__ __forceinline__ ChunkCursor cursor_seek(int64_t x, const int32_t *n_chunks,
                                                   int n_units) {
  const int lane = threadIdx.x & 31;
  int64_t acc = 0;
  for (int base = 0; base < n_units; base += 32) {
    const int u = base + lane;
    const int64_t n = u < n_units ? n_chunks[u] : 0;
    int64_t incl = n;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    const unsigned hit = __ballot_sync(0xffffffffu, n > 0 && acc + incl > x);
    if (hit) {
      const int L = __ffs(hit) - 1;
      const int64_t excl = __shfl_sync(0xffffffffu, incl - n, L);
      const int nn = (int)__shfl_sync(0xffffffffu, n, L);
      return ChunkCursor{base + L, (int)(x - acc - excl), nn};
    }
    acc += __shfl_sync(0xffffffffu, incl, 31);
  }
  return ChunkCursor{n_units, 0, 0};
}

__host__ __device__ __forceinline__ int64_t range_lo(int64_t total, int i, int grid) {
  return total * i / grid;
}

// record layout: [slot][G][4 + D]: m (log2 domain), l, -, -, acc[128] (HT
// domain); slot = (unit + cta) * NGRP + group.
template <int G>
__device__ __forceinline__ float *record_ptr(float *recs, int slot) {
  return recs + (int64_t)slot * G * (4 + D);
}

// channel of the K-side MMA k-index (thread t, k-tile kt, column group r,
// element i): thread t owns the whole sub-vectors 4t..4t+3 of each token.
__device__ __forceinline__ int k_channel(int t, int kt, int r, int i) {
  return 32 * t + 8 * (kt >> 1) + 4 * (kt & 1) + 2 * r + i;
}

// ---------------------------------------------------------------------------
// combine: merge the stream-K records of a unit with its exact residual rows,
// normalise, inverse FWHT (attention.py:105-108, 129-133, 141).
// One CTA (256 threads) per unit; warp h < G owns q-head h of the unit.
//
// Residual rows are staged once per unit: keys rotated to their positions
// (rope.py:35-51) into kr, values into vr, by all 256 threads with
// independent loads; each warp then scores its head's rows (lane = row) and
// accumulates the weighted value rows (lane = 4 channels).
//
// Fused append (nsnkv_decode_step): n_new > 0 extra rows per unit come from
// new_k / new_v ([units][n_new][128], fp32 or bf16) -- attended as residual
// rows nres .. nres + n_new - 1 and written into the residual buffer, with
// the unit's residual count published to n_res_out (which may be cv.n_res
// itself: one CTA owns the unit and reads the count before it writes it).
// ---------------------------------------------------------------------------
constexpr int COMBINE_THREADS = 256;

struct CombineSmem {
  float kr[R][D + 1];  // rotated residual keys (row stride D + 1: lane = row is conflict-free)
  __align__(16) float vr[R][D];
  __align__(16) float q[8][D];
  float w[8][R];
};

template <int G, int NGRP, bool ALLREC = false>
__global__ void __launch_bounds__(COMBINE_THREADS) combine_kernel(
    CacheViewDev cv, const float *__restrict__ qg, const float *__restrict__ recs,
    int64_t total_chunks, int grid, float *__restrict__ out, float *__restrict__ lse,
    const void *__restrict__ new_k, const void *__restrict__ new_v, int new_bf16, int n_new,
    int32_t *__restrict__ n_res_out) {
  extern __shared__ __align__(16) unsigned char combine_smem[];
  CombineSmem &S = *reinterpret_cast<CombineSmem *>(combine_smem);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int u = blockIdx.x;
  const int b = u / cv.n_kv_heads, hk = u - b * cv.n_kv_heads;
  const int nch = cv.n_chunks[u];
  const int nres = cv.n_res[u];
  const int rtot = nres + n_new;
  const int64_t pbase = cv.base_pos[u] + (int64_t)nch * R;

  // ---- stage the residual rows (old from the buffer, new from the input) --
  for (int i = threadIdx.x; i < rtot * (D / 4); i += COMBINE_THREADS) {
    const int tt = i / (D / 4), l4 = i - tt * (D / 4);
    float4 k4, v4;
    if (tt < nres) {
      k4 = *reinterpret_cast<const float4 *>(cv.k_res + ((int64_t)u * R + tt) * D + 4 * l4);
      v4 = *reinterpret_cast<const float4 *>(cv.v_res + ((int64_t)u * R + tt) * D + 4 * l4);
    } else {
      const int64_t off = ((int64_t)u * n_new + (tt - nres)) * D + 4 * l4;
      if (new_bf16) {
        const uint2 rk = *reinterpret_cast<const uint2 *>(static_cast<const uint16_t *>(new_k) + off);
        const uint2 rv = *reinterpret_cast<const uint2 *>(static_cast<const uint16_t *>(new_v) + off);
        k4 = make_float4(bf16_to_f32(rk.x & 0xffffu), bf16_to_f32(rk.x >> 16),
                         bf16_to_f32(rk.y & 0xffffu), bf16_to_f32(rk.y >> 16));
        v4 = make_float4(bf16_to_f32(rv.x & 0xffffu), bf16_to_f32(rv.x >> 16),
                         bf16_to_f32(rv.y & 0xffffu), bf16_to_f32(rv.y >> 16));
      } else {
        k4 = *reinterpret_cast<const float4 *>(static_cast<const float *>(new_k) + off);
        v4 = *reinterpret_cast<const float4 *>(static_cast<const float *>(new_v) + off);
      }
      // the new rows join the residual buffer (keys pre-RoPE, values post-HT)
      *reinterpret_cast<float4 *>(const_cast<float *>(cv.k_res) + ((int64_t)u * R + tt) * D + 4 * l4) = k4;
      *reinterpret_cast<float4 *>(const_cast<float *>(cv.v_res) + ((int64_t)u * R + tt) * D + 4 * l4) = v4;
    }
    const float4 c4 = *reinterpret_cast<const float4 *>(cv.rope_cs + (pbase + tt - cv.rope_pos0) * NPAIR + 2 * l4);
    float *kr = &S.kr[tt][4 * l4];
    kr[0] = k4.x * c4.x - k4.y * c4.y;
    kr[1] = k4.x * c4.y + k4.y * c4.x;
    kr[2] = k4.z * c4.z - k4.w * c4.w;
    kr[3] = k4.z * c4.w + k4.w * c4.z;
    *reinterpret_cast<float4 *>(&S.vr[tt][4 * l4]) = v4;
  }
  const int h = warp;
  const bool active = h < G;
  const int row = b * cv.n_q_heads + hk * G + h;
  float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
  float m = -INFINITY, l = 0.f;
  if (active) {
    *reinterpret_cast<float4 *>(&S.q[h][4 * lane]) =
        *reinterpret_cast<const float4 *>(qg + (int64_t)row * D + 4 * lane);
    // ---- stream-K records of the unit -----------------------------------
    // (launched as a programmatic dependent of the attend kernel: the staging
    // above overlaps its tail; its records are complete and visible here)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    int64_t off = 0;  // global chunk offset of unit u
    for (int uu = lane; uu < u; uu += 32) off += cv.n_chunks[uu];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) off += __shfl_xor_sync(0xffffffffu, off, o);
    if (nch > 0) {
      const int64_t x0 = off, x1 = off + nch - 1;
      int c0 = (int)(x0 * grid / total_chunks);
      while (c0 + 1 < grid && range_lo(total_chunks, c0 + 1, grid) <= x0) ++c0;
      while (c0 > 0 && range_lo(total_chunks, c0, grid) > x0) --c0;
      int c1 = (int)(x1 * grid / total_chunks);
      while (c1 + 1 < grid && range_lo(total_chunks, c1 + 1, grid) <= x1) ++c1;
      while (c1 > 0 && range_lo(total_chunks, c1, grid) > x1) --c1;
      // every (CTA, group) slot of the unit holds a record (m = -inf when
      // empty): load them in batches of 8 with independent loads, then merge
      const int nrec = (c1 - c0 + 1) * NGRP;
      for (int r0 = 0; r0 < nrec; r0 += 8) {
        float rm8 = -INFINITY, rl8 = 0.f;
        if (lane < 8 && r0 + lane < nrec) {
          const int r = r0 + lane, c = c0 + r / NGRP, gq = r % NGRP;
          const float *rec = record_ptr<G>(const_cast<float *>(recs), (u + c) * NGRP + gq) + h * (4 + D);
          rm8 = rec[0];
          rl8 = rec[1];
        }
        float4 r4[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          r4[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (r0 + i < nrec) {
            const int r = r0 + i, c = c0 + r / NGRP, gq = r % NGRP;
            const float *rec = record_ptr<G>(const_cast<float *>(recs), (u + c) * NGRP + gq) + h * (4 + D);
            r4[i] = *reinterpret_cast<const float4 *>(rec + 4 + 4 * lane);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const float rm = __shfl_sync(0xffffffffu, rm8, i);
          const float rl = __shfl_sync(0xffffffffu, rl8, i);
          if (!(rm > -INFINITY)) continue;  // the group saw no chunk of this unit
          const float mn = fmaxf(m, rm);
          const float sa = exp2f(m - mn), sb = exp2f(rm - mn);
          a.x = a.x * sa + r4[i].x * sb;
          a.y = a.y * sa + r4[i].y * sb;
          a.z = a.z * sa + r4[i].z * sb;
          a.w = a.w * sa + r4[i].w * sb;
          l = l * sa + rl * sb;
          m = mn;
        }
      }
    }
  }
  __syncthreads();  // staged rows and q visible; every thread has read n_res[u]
  if (n_new > 0 && n_res_out && threadIdx.x == 0) n_res_out[u] = rtot;  // may alias cv.n_res
  if (active && rtot > 0) {
    // ---- residual rows: exact RoPE(k, pos) . q scores (base-2 logits) ----
    for (int tt = lane; tt < rtot; tt += 32) {
      float acc[4] = {0.f, 0.f, 0.f, 0.f};  // four independent chains
#pragma unroll 8
      for (int d = 0; d < D; d += 4)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = fmaf(S.kr[tt][d + e], S.q[h][d + e], acc[e]);
      S.w[h][tt] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) * LOG2E_OVER_SQRTD;
    }
    __syncwarp();
    float rm = -INFINITY;
    for (int tt = lane; tt < rtot; tt += 32) rm = fmaxf(rm, S.w[h][tt]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rm = fmaxf(rm, __shfl_xor_sync(0xffffffffu, rm, o));
    const float mn = fmaxf(m, rm);
    const float sa = (m > -INFINITY) ? exp2f(m - mn) : 0.f;
    a.x *= sa; a.y *= sa; a.z *= sa; a.w *= sa;
    l *= sa;
#pragma unroll 4
    for (int tt = 0; tt < rtot; ++tt) {
      const float p = exp2f(S.w[h][tt] - mn);
      const float4 v4 = *reinterpret_cast<const float4 *>(&S.vr[tt][4 * lane]);
      l += p;
      a.x = fmaf(p, v4.x, a.x);
      a.y = fmaf(p, v4.y, a.y);
      a.z = fmaf(p, v4.z, a.z);
      a.w = fmaf(p, v4.w, a.w);
    }
    m = mn;
  }
  if (!active) return;
  const float inv = (l > 0.f) ? 1.f / l : 0.f;
  float4 v = make_float4(a.x * inv, a.y * inv, a.z * inv, a.w * inv);
  // inverse FWHT in the warp (stages h = 1, 2 in-lane, 4 .. 64 by shuffles)
  {
    float p0 = v.x + v.y, p1 = v.x - v.y, p2 = v.z + v.w, p3 = v.z - v.w;
    v.x = p0 + p2; v.z = p0 - p2; v.y = p1 + p3; v.w = p1 - p3;
#pragma unroll
    for (int mm = 1; mm < 32; mm <<= 1) {
      const float ox = __shfl_xor_sync(0xffffffffu, v.x, mm);
      const float oy = __shfl_xor_sync(0xffffffffu, v.y, mm);
      const float oz = __shfl_xor_sync(0xffffffffu, v.z, mm);
      const float ow = __shfl_xor_sync(0xffffffffu, v.w, mm);
      if (lane & mm) {
        v.x = ox - v.x; v.y = oy - v.y; v.z = oz - v.z; v.w = ow - v.w;
      } else {
        v.x += ox; v.y += oy; v.z += oz; v.w += ow;
      }
    }
    const float sc = 0.08838834764831845f;
    v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
  }
  *reinterpret_cast<float4 *>(out + (int64_t)row * D + 4 * lane) = v;
  if (lse && lane == 0) lse[row] = (l > 0.f) ? (m + log2f(l)) * 0.6931471805599453f : -INFINITY;
}

}  // namespace nsnkv



// rows appended to every unit's residual by the decode step itself
// (nsnkv_decode_step); n == 0 for plain attention
struct AppendRows {
  const void *k = nullptr, *v = nullptr;
  int bf16 = 0, n = 0;
  int32_t *n_res_out = nullptr;
};

// warp-specialized decode launcher (decode_attend3.cu), G = 1, 2, 4, 8
template <int G, bool FOLD, int PREC>
int nsnkv_launch_attend3(const nsnkv::CacheViewDev &cv, const float *q, float *out, float *lse,
                         float *recs, int64_t total, int grid, cudaStream_t st,
                         const AppendRows &add);
