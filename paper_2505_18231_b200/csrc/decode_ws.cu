// decode_ws.cu -- warp-specialized fused decode (GQA group G <= 4).
//
// Same algebra, page ring and stream-K split as attend_kernel
// (decode_attend.cu), but every chunk is processed by two cooperating warp
// quads of one consumer group:
//   K-warps (4): shift-term prologue, key gathers + payload MMAs, shift-term
//                MMAs, online softmax; hand p / rescale / shift weight to ...
//   V-warps (4): value gathers + token pairing (independent of the softmax,
//                so they overlap it), then P' . codewords MMAs.
// Two groups take alternate chunks: 16 warps per SM (4 per SMSP) at <= 128
// registers, the shift-term table fragments pinned in K-warp registers.
// Hand-off and stage release are mbarriers; the K-warps never run more than
// two chunks ahead of their V-warps.
#include "common.cuh"
#include "decode_common.cuh"
#include "decode_att.cuh"

namespace nsnkv {

constexpr int WS_NSTAGE = 8;
constexpr int WS_THREADS = 512;

template <int G>
struct WsGroup {
  struct Chunk {
    uint2 ab[2][8][32];  // shift-term B fragments, double-buffered per chunk
    float ov[2][D];      // dequantized value shift vector
    float4 sc[2][R];     // (s1k*s2k, s1k, s1v*s2v, s1v) per token
    float qh[G][D];      // HT(q) (unit set-up only)
  };
  struct Merge {
    float mrg[4][G][D];  // V-warp partial sums per token slice
    float ml[4][G][2];   // K-warp (max, sum) per token slice
  };
  union {
    Chunk ck;
    Merge mg;
  };
  float q[G][D];         // RoPE'd q of the group's current unit
  struct Hand {          // K-warp -> V-warp hand-off for one 16-token slice
    float p[16][4];      // softmax numerators (base 2, running max)
    float r[4];          // accumulator rescale per head
    float w[4];          // sum_t p_t * s1v_t per head (value shift weight)
  } hand[2][4];
};

struct WsLow {
  __align__(128) uint8_t st[WS_NSTAGE][STAGE_BYTES];
  uint64_t full[WS_NSTAGE];   // TMA landed (tx count)
  uint64_t vdone[WS_NSTAGE];  // the V-warps finished the chunk in this stage
  uint64_t pro[2][2];         // [group][slot]: K-warp prologue written (128)
  uint64_t hfull[2][4][2];    // [group][slice][slot]: hand-off written (1)
  uint64_t tabs;
};

template <int G>
struct WsHigh {
  WsGroup<G> grp[2];
};

template <int G, bool FOLD, int PREC>
__global__ void __launch_bounds__(WS_THREADS, 1)
    attend_ws_kernel(CacheViewDev cv, const float *__restrict__ qg, float *__restrict__ recs,
                     int64_t total_chunks) {
  static_assert(G <= 4, "warp-specialized decode handles GQA groups up to 4");
  static_assert(sizeof(WsLow) <= MISC_LO_MAX, "ring does not fit below the tables");
  static_assert(sizeof(WsHigh<G>) <= MISC_HI_MAX, "scratch does not fit above the tables");
  constexpr bool HILO_K = PREC == 0;
  constexpr bool HILO_V = PREC <= 1;
  constexpr int NGRP = 2;
  constexpr int NSTAGE = WS_NSTAGE;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n_units = cv.batch * cv.n_kv_heads;
  const PageLayout L = page_layout(FOLD ? 2 : 1);
  const uint32_t page_bytes = (uint32_t)L.bytes;

  const uint32_t base = smem_u32(smem);
  const bool aligned_window = (base & 0xffffu) == 0;
  const uint32_t tk = aligned_window ? base : ((base + 0xffffu) & ~0xffffu);
  const uint32_t tv = tk + 0x10000u;
  WsLow &M = *reinterpret_cast<WsLow *>(smem + (aligned_window ? 0x20000u : 0u));
  WsHigh<G> &GS = *reinterpret_cast<WsHigh<G> *>(
      smem + (tv + 0x10000u - base) +
      (aligned_window ? (uint32_t)((sizeof(WsLow) + 127) / 128 * 128) : 0u));

  const int grid = gridDim.x;
  const int64_t lo = range_lo(total_chunks, blockIdx.x, grid);
  const int64_t hi = range_lo(total_chunks, blockIdx.x + 1, grid);
  if (lo >= hi) return;
  const int n_local = (int)(hi - lo);

  auto load_chunk = [&](int k, const ChunkCursor &c) {
    const int s = k % NSTAGE;
    const int64_t page = cv.page_table[(int64_t)c.u * cv.page_table_stride + c.c];
    const int64_t p0 = cv.base_pos[c.u] + (int64_t)c.c * R - cv.rope_pos0;
    uint8_t *st = M.st[s];
    mbar_expect_tx(&M.full[s], 2 * page_bytes + ROPE_ROW_BYTES);
    tma_load_1d(st, cv.k_pool + page * page_bytes, page_bytes, &M.full[s]);
    tma_load_1d(st + page_bytes, cv.v_pool + page * page_bytes, page_bytes, &M.full[s]);
    tma_load_1d(st + 2 * page_bytes, cv.rope_cs + p0 * NPAIR, ROPE_ROW_BYTES, &M.full[s]);
  };

  if (warp == 0) {
    ChunkCursor c0 = cursor_seek(lo, cv.n_chunks, n_units);
    if (lane == 0) {
      for (int s = 0; s < NSTAGE; ++s) {
        mbar_init(&M.full[s], 1);
        mbar_init(&M.vdone[s], 4);
      }
      for (int q = 0; q < NGRP; ++q) {
        mbar_init(&M.pro[q][0], 128);
        mbar_init(&M.pro[q][1], 128);
        for (int w = 0; w < 4; ++w) {
          mbar_init(&M.hfull[q][w][0], 1);
          mbar_init(&M.hfull[q][w][1], 1);
        }
      }
      mbar_init(&M.tabs, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&M.tabs, 2 * 65536);
      tma_load_1d(smem + (tk - base), cv.cb_k.tabw, 65536, &M.tabs);
      tma_load_1d(smem + (tv - base), cv.cb_v.tabw, 65536, &M.tabs);
      for (int k = 0; k < NSTAGE && k < n_local; ++k) {
        load_chunk(k, c0);
        cursor_advance(c0, cv.n_chunks, n_units);
      }
    }
  }
  __syncthreads();

  const int grp = warp >> 3;          // chunks i with i % 2 == grp
  const bool kwarp = ((warp >> 2) & 1) == 0;
  const int ws = warp & 3;            // token slice [16 ws, 16 ws + 16)
  const int ci = 32 * ws + lane;      // index among the role's 128 threads
  const int gi = kwarp ? ci : 128 + ci;  // index among the group's 256 threads
  const int bar_group = 1 + grp;      // all 256 threads of the group
  const int bar_k = 3 + grp;          // the group's K-warps
  WsGroup<G> &S = GS.grp[grp];
  const uint32_t slot16 = (uint32_t)((lane & 7) * 16);

  ChunkCursor cur = cursor_seek(lo + grp, cv.n_chunks, n_units);
  int cur_unit = -1;
  bool tabs_ready = false;

  // ---- unit merge: K-warps own (max, sum), V-warps the value accumulators --
  auto merge_unit = [&](int unit) {
    named_bar(bar_group, 256);
    float *rec = record_ptr<G>(recs, (unit + blockIdx.x) * NGRP + grp);
    for (int e = gi; e < G * D; e += 256) {
      const int h = e / D, c = e - h * D;
      float mx = -INFINITY;
#pragma unroll
      for (int w2 = 0; w2 < 4; ++w2) mx = fmaxf(mx, S.mg.ml[w2][h][0]);
      float a = 0.f, l = 0.f;
      if (mx > -INFINITY) {
#pragma unroll
        for (int w2 = 0; w2 < 4; ++w2) {
          const float sc = exp2f(S.mg.ml[w2][h][0] - mx);
          a = fmaf(S.mg.mrg[w2][h][c], sc, a);
          l = fmaf(S.mg.ml[w2][h][1], sc, l);
        }
      }
      rec[h * (4 + D) + 4 + c] = a;
      if (c == 0) {
        rec[h * (4 + D) + 0] = mx;
        rec[h * (4 + D) + 1] = l;
      }
    }
    named_bar(bar_group, 256);
  };

  if (kwarp) {
    // ======================== K-warps ========================================
    uint32_t taba[8][4];  // (cos, sin)(tau f_j), tau = 16ws + g (+8), j = 8kt + t (+4)
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int tau = 16 * ws + g + ((r & 1) ? 8 : 0);
        const int j = 8 * kt + t + ((r & 2) ? 4 : 0);
        const float2 cs = cv.rope_cs[(int64_t)(tau - cv.rope_pos0) * NPAIR + j];
        taba[kt][r] = pack_h2(cs.x, cs.y);
      }
    }
    const uint32_t lbk = (tk & 0xffff0000u) | slot16;
    const bool leader = ws == 0 && lane == 0;
    ChunkCursor ahead = cursor_seek(lo + NSTAGE + grp, cv.n_chunks, n_units);
    uint32_t qB[8][2];
    float m_run = -INFINITY, l_run = 0.f;

    auto flush_k = [&](int unit) {
      float l = l_run;
      l += __shfl_xor_sync(0xffffffffu, l, 4);
      l += __shfl_xor_sync(0xffffffffu, l, 8);
      l += __shfl_xor_sync(0xffffffffu, l, 16);
      named_bar(bar_group, 256);  // the merge buffers alias the chunk buffers
      if (t < G && g == 0) {
        S.mg.ml[ws][t][0] = m_run;
        S.mg.ml[ws][t][1] = l;
      }
      merge_unit(unit);
    };
    auto setup_k = [&](int unit) {
      const int b = unit / cv.n_kv_heads, hk = unit - b * cv.n_kv_heads;
      const float *qs = qg + ((int64_t)b * cv.n_q_heads + (int64_t)hk * G) * D;
      for (int i = ci; i < G * D; i += 128) S.q[i / D][i % D] = qs[i];
      named_bar(bar_k, 128);
      if (ws < G) {  // HT(q) of head ws, 4 values per lane
        float4 v = *reinterpret_cast<float4 *>(&S.q[ws][4 * lane]);
        float a = v.x + v.y, bq = v.x - v.y, c = v.z + v.w, d = v.z - v.w;
        v.x = a + c; v.z = a - c; v.y = bq + d; v.w = bq - d;
#pragma unroll
        for (int m = 1; m < 32; m <<= 1) {
          const float ox = __shfl_xor_sync(0xffffffffu, v.x, m);
          const float oy = __shfl_xor_sync(0xffffffffu, v.y, m);
          const float oz = __shfl_xor_sync(0xffffffffu, v.z, m);
          const float ow = __shfl_xor_sync(0xffffffffu, v.w, m);
          if (lane & m) {
            v.x = ox - v.x; v.y = oy - v.y; v.z = oz - v.z; v.w = ow - v.w;
          } else {
            v.x += ox; v.y += oy; v.z += oz; v.w += ow;
          }
        }
        const float sc = 0.08838834764831845f;
        v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
        *reinterpret_cast<float4 *>(&S.ck.qh[ws][4 * lane]) = v;
      }
      named_bar(bar_k, 128);
      const int h = g >> 1;
#pragma unroll
      for (int kt = 0; kt < 8; ++kt) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          float v0 = 0.f, v1 = 0.f;
          if (h < G) {
            float h0, l0, h1, l1;
            split_h(S.ck.qh[h][k_channel(t, kt, r, 0)], h0, l0);
            split_h(S.ck.qh[h][k_channel(t, kt, r, 1)], h1, l1);
            v0 = (g & 1) ? l0 : h0;
            v1 = (g & 1) ? l1 : h1;
          }
          qB[kt][r] = pack_h2(v0, v1);
        }
      }
      m_run = -INFINITY;
      l_run = 0.f;
      named_bar(bar_k, 128);  // HT(q) aliases the per-chunk buffers
    };

    int n = 0;
    for (int i = grp; i < n_local; i += NGRP, ++n) {
      if (cur.u != cur_unit) {
        if (cur_unit >= 0) flush_k(cur_unit);
        setup_k(cur.u);
        cur_unit = cur.u;
      }
      const int s = i % NSTAGE;
      const int slot = n & 1;
      const uint32_t par = (uint32_t)(n >> 1) & 1u;
      if (n >= 2) {  // V-warps done with the group's chunk n - 2: slot and stage free
        const int i4 = i - 2 * NGRP;
        mbar_wait(&M.vdone[i4 % NSTAGE], (uint32_t)(i4 / NSTAGE) & 1u);
        if (leader && i4 + NSTAGE < n_local) load_chunk(i4 + NSTAGE, ahead);
        cursor_advance(ahead, cv.n_chunks, n_units);
        cursor_advance(ahead, cv.n_chunks, n_units);
      }
      mbar_wait(&M.full[s], (uint32_t)(i / NSTAGE) & 1u);
      if (!tabs_ready) {
        mbar_wait(&M.tabs, 0);
        tabs_ready = true;
      }
      const uint8_t *kp = M.st[s];
      const uint8_t *vp = M.st[s] + page_bytes;
      const float2 *rrow = reinterpret_cast<const float2 *>(M.st[s] + 2 * page_bytes);

      // ---- prologue: token scales, value shift vector, shift-term fragments
      {
        const int tok = ci & 63;
        const uint8_t *pg = ci < 64 ? kp : vp;
        const uint16_t *par16 = reinterpret_cast<const uint16_t *>(pg + L.par);
        const float s1sc = f16_bits_to_f32(par16[0]), s1z = f16_bits_to_f32(par16[1]);
        const uint32_t nb = pg[L.s1n + (tok >> 1)];
        const float lv = (float)((tok & 1) ? (nb >> 4) : (nb & 15u));
        const float s1 = __fadd_rn(s1z, __fmul_rn(lv, s1sc));
        const float s2 = f16_bits_to_f32(reinterpret_cast<const uint16_t *>(pg + L.s2)[tok]);
        reinterpret_cast<float2 *>(&S.ck.sc[slot][tok])[ci < 64 ? 0 : 1] = make_float2(s1 * s2, s1);
        const uint16_t *pv = reinterpret_cast<const uint16_t *>(vp + L.par);
        const int gr = ci >> 5;
        const uint32_t b = vp[L.on + (ci >> 1)];
        const float l2 = (float)((ci & 1) ? (b >> 4) : (b & 15u));
        S.ck.ov[slot][ci] = __fadd_rn(f16_bits_to_f32(pv[6 + gr]),
                                      __fmul_rn(l2, f16_bits_to_f32(pv[2 + gr])));
        const uint16_t *pk = reinterpret_cast<const uint16_t *>(kp + L.par);
        const int j = 16 * ws + (lane >> 1);
        const int gj = (2 * j) >> 5;
        const uint32_t bj = kp[L.on + j];
        const float osc = f16_bits_to_f32(pk[2 + gj]), oz = f16_bits_to_f32(pk[6 + gj]);
        const float oe = __fadd_rn(oz, __fmul_rn((float)(bj & 15u), osc));
        const float oo = __fadd_rn(oz, __fmul_rn((float)(bj >> 4), osc));
        const float2 cs = rrow[j];
        const float he = oe * cs.x - oo * cs.y;  // RoPE(o, p0)
        const float ho = oe * cs.y + oo * cs.x;
        const int kt = j >> 3, tt = j & 3, half = (j >> 2) & 1;
#pragma unroll
        for (int hh2 = 0; hh2 < 2; ++hh2) {
          const int h = 2 * hh2 + (lane & 1);
          float al = 0.f, be = 0.f;
          if (h < G) {
            const float qe = S.q[h][2 * j], qo = S.q[h][2 * j + 1];
            al = qe * he + qo * ho;
            be = qo * he - qe * ho;
          }
          float ah, alo, bh, blo;
          split_h(al, ah, alo);
          split_h(be, bh, blo);
          reinterpret_cast<uint32_t *>(&S.ck.ab[slot][kt][4 * (2 * h) + tt])[half] = pack_h2(ah, bh);
          reinterpret_cast<uint32_t *>(&S.ck.ab[slot][kt][4 * (2 * h + 1) + tt])[half] = pack_h2(alo, blo);
        }
      }
      mbar_arrive(&M.pro[grp][slot]);

      // ---- key payload on tensor cores ----------------------------------------
      const int tok0 = 16 * ws + g, tok1 = tok0 + 8;
      const uint32_t kpa = smem_u32(kp);
      const uint32_t ik0 = lds32(kpa + L.idx + tok0 * NSUB + 4 * t);
      const uint32_t ik1 = lds32(kpa + L.idx + tok1 * NSUB + 4 * t);
      uint32_t sk0 = 0, sk1 = 0;
      if (FOLD) {
        sk0 = lds32(kpa + L.sgn + tok0 * 16 + 4 * t);
        sk1 = lds32(kpa + L.sgn + tok1 * 16 + 4 * t);
      }
      float d1[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      float d2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int m = 0; m < 4; ++m) {  // item m = sub 4t + m of tokens g, g+8
        const uint32_t sel = 0x7604u | ((uint32_t)m << 4);
        const uint32_t a0 = prmt(ik0, lbk, sel), a1 = prmt(ik1, lbk, sel);
        uint4 h0 = lds128(a0), h1 = lds128(a1);
        uint4 l0 = make_uint4(0, 0, 0, 0), l1 = l0;
        if (HILO_K) {
          l0 = lds128(a0 + 128);
          l1 = lds128(a1 + 128);
        }
        if (FOLD) {
          uint32_t *ph0 = &h0.x, *ph1 = &h1.x, *pl0 = &l0.x, *pl1 = &l1.x;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const uint32_t w0 = sk0 << (15 - 4 * m - p);
            const uint32_t w1 = sk1 << (15 - 4 * m - p);
            ph0[p] = xor_sign(ph0[p], w0);
            ph1[p] = xor_sign(ph1[p], w1);
            if (HILO_K) {
              pl0[p] = xor_sign(pl0[p], w0);
              pl1[p] = xor_sign(pl1[p], w1);
            }
          }
        }
        mma16816(d1[0], h0.x, h1.x, h0.y, h1.y, qB[2 * m][0], qB[2 * m][1]);
        mma16816(d1[1], h0.z, h1.z, h0.w, h1.w, qB[2 * m + 1][0], qB[2 * m + 1][1]);
        if (HILO_K) {
          mma16816(d1[0], l0.x, l1.x, l0.y, l1.y, qB[2 * m][0], qB[2 * m][1]);
          mma16816(d1[1], l0.z, l1.z, l0.w, l1.w, qB[2 * m + 1][0], qB[2 * m + 1][1]);
        }
      }
      mbar_wait(&M.pro[grp][slot], par);  // the group's shift-term fragments and scales
#pragma unroll
      for (int kt = 0; kt < 8; ++kt) {
        const uint2 ab = *reinterpret_cast<const uint2 *>(&S.ck.ab[slot][kt][lane]);
        mma16816(d2, taba[kt][0], taba[kt][1], taba[kt][2], taba[kt][3], ab.x, ab.y);
      }

      // ---- scores, online softmax, hand-off --------------------------------
      const float4 sc0 = S.ck.sc[slot][tok0];
      const float4 sc1 = S.ck.sc[slot][tok1];
      const float pd0 = (d1[0][0] + d1[1][0]) + (d1[0][1] + d1[1][1]);
      const float pd1 = (d1[0][2] + d1[1][2]) + (d1[0][3] + d1[1][3]);
      const float x0 = (sc0.x * pd0 + sc0.y * (d2[0] + d2[1])) * LOG2E_OVER_SQRTD;
      const float x1 = (sc1.x * pd1 + sc1.y * (d2[2] + d2[3])) * LOG2E_OVER_SQRTD;
      float mx = fmaxf(x0, x1);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      const float m_new = fmaxf(m_run, mx);
      const float rs = exp2f(m_run - m_new);
      l_run *= rs;
      m_run = m_new;
      float p0 = exp2f(x0 - m_new), p1 = exp2f(x1 - m_new);
      if (t >= G) p0 = p1 = 0.f;
      l_run += p0 + p1;
      float wv = p0 * sc0.w + p1 * sc1.w;
      wv += __shfl_xor_sync(0xffffffffu, wv, 4);
      wv += __shfl_xor_sync(0xffffffffu, wv, 8);
      wv += __shfl_xor_sync(0xffffffffu, wv, 16);
      typename WsGroup<G>::Hand &H = S.hand[slot][ws];
      H.p[g][t] = p0;
      H.p[g + 8][t] = p1;
      if (g == 0) {
        H.r[t] = rs;
        H.w[t] = wv;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&M.hfull[grp][ws][slot]);
      cursor_advance(cur, cv.n_chunks, n_units);
      cursor_advance(cur, cv.n_chunks, n_units);
    }
    if (cur_unit >= 0) flush_k(cur_unit);
  } else {
    // ======================== V-warps ========================================
    const uint32_t lbv = (tv & 0xffff0000u) | slot16;
    const uint32_t vsel0 = 0x7604u | ((uint32_t)(2 * (g & 1)) << 4);
    const uint32_t vsel1 = 0x7604u | ((uint32_t)(2 * (g & 1) + 1) << 4);
    const int hs = g >> 1;                       // head of this thread's P' column
    float accV[8][4];
#pragma unroll
    for (int mt = 0; mt < 8; ++mt)
#pragma unroll
      for (int r = 0; r < 4; ++r) accV[mt][r] = 0.f;

    auto flush_v = [&](int unit) {
      named_bar(bar_group, 256);  // the merge buffers alias the chunk buffers
      if (t < G) {
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const int c = 16 * g + 8 * (mt >> 2) + 2 * (mt & 3);
          S.mg.mrg[ws][t][c] = accV[mt][0] + accV[mt][1];
          S.mg.mrg[ws][t][c + 1] = accV[mt][2] + accV[mt][3];
        }
      }
      merge_unit(unit);
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int r = 0; r < 4; ++r) accV[mt][r] = 0.f;
    };

    // gathers the 4 tokens' codewords of sub 2g + sg (signs applied)
    auto gather_v = [&](const uint32_t (&iv)[4], const uint32_t (&sv)[4], int sg, uint4 (&yh)[4],
                        uint4 (&yl)[4]) {
      const uint32_t sel = sg ? vsel1 : vsel0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t a = prmt(iv[q], lbv, sel);
        yh[q] = lds128(a);
        yl[q] = HILO_V ? lds128(a + 128) : make_uint4(0, 0, 0, 0);
        if (FOLD) {
          uint32_t *ph = &yh[q].x, *pl = &yl[q].x;
#pragma unroll
          for (int p = 0; p < 4; ++p) {
            const uint32_t wk = sv[q] << (15 - 4 * sg - p);
            ph[p] = xor_sign(ph[p], wk);
            if (HILO_V) pl[p] = xor_sign(pl[p], wk);
          }
        }
      }
    };
    auto mma_v = [&](const uint4 (&yh)[4], const uint4 (&yl)[4], int sg, uint32_t pf0,
                     uint32_t pf1) {
#pragma unroll
      for (int p = 0; p < 4; ++p) {  // m-tile 4 sg + p: channels 16g + 8sg + 2p (+1)
        const int mt = 4 * sg + p;
        const uint32_t *h0 = &yh[0].x, *h1 = &yh[1].x, *h2 = &yh[2].x, *h3 = &yh[3].x;
        mma16816(accV[mt], prmt(h0[p], h1[p], 0x5410u), prmt(h0[p], h1[p], 0x7632u),
                 prmt(h2[p], h3[p], 0x5410u), prmt(h2[p], h3[p], 0x7632u), pf0, pf1);
        if (HILO_V) {
          const uint32_t *l0 = &yl[0].x, *l1 = &yl[1].x, *l2 = &yl[2].x, *l3 = &yl[3].x;
          mma16816(accV[mt], prmt(l0[p], l1[p], 0x5410u), prmt(l0[p], l1[p], 0x7632u),
                   prmt(l2[p], l3[p], 0x5410u), prmt(l2[p], l3[p], 0x7632u), pf0, pf1);
        }
      }
    };

    int n = 0;
    for (int i = grp; i < n_local; i += NGRP, ++n) {
      if (cur.u != cur_unit) {
        if (cur_unit >= 0) flush_v(cur_unit);
        cur_unit = cur.u;
      }
      const int s = i % NSTAGE;
      const int slot = n & 1;
      const uint32_t par = (uint32_t)(n >> 1) & 1u;
      mbar_wait(&M.full[s], (uint32_t)(i / NSTAGE) & 1u);
      if (!tabs_ready) {
        mbar_wait(&M.tabs, 0);
        tabs_ready = true;
      }
      const uint32_t vpa = smem_u32(M.st[s] + page_bytes);
      const int vt0 = 16 * ws + 2 * t;  // tokens vt0, vt0+1, vt0+8, vt0+9; subs 2g, 2g+1
      uint32_t iv[4], sv[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int tok = vt0 + (q & 1) + ((q & 2) ? 8 : 0);
        iv[q] = lds32(vpa + L.idx + tok * NSUB + 4 * (g >> 1));
        sv[q] = FOLD ? (lds32(vpa + L.sgn + tok * 16 + 4 * (g >> 1)) >> (8 * (g & 1))) : 0u;
      }
      uint4 yh[4], yl[4];
      gather_v(iv, sv, 0, yh, yl);  // overlaps the K-warps' softmax

      mbar_wait(&M.pro[grp][slot], par);                // scales and o_v
      mbar_wait(&M.hfull[grp][ws][slot], par);          // p, rescale, shift weight
      const typename WsGroup<G>::Hand &H = S.hand[slot][ws];
      const float rs = H.r[t];
      const float wv = H.w[t];
      if (rs != 1.f) {
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int r = 0; r < 4; ++r) accV[mt][r] *= rs;
      }
      // B fragment of P' = p * s1v * s2v: column g = (head g/2, part g&1),
      // rows = tokens 2t, 2t+1 (reg 0) and 2t+8, 2t+9 (reg 1) of the slice
      uint32_t pf[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int ta = 2 * t + 8 * r;
        float va = 0.f, vb = 0.f;
        if (hs < G) {
          va = H.p[ta][hs] * S.ck.sc[slot][16 * ws + ta].z;
          vb = H.p[ta + 1][hs] * S.ck.sc[slot][16 * ws + ta + 1].z;
        }
        float ha, la, hb, lb;
        split_h(va, ha, la);
        split_h(vb, hb, lb);
        pf[r] = (g & 1) ? pack_h2(la, lb) : pack_h2(ha, hb);
      }
      mma_v(yh, yl, 0, pf[0], pf[1]);
      gather_v(iv, sv, 1, yh, yl);
      mma_v(yh, yl, 1, pf[0], pf[1]);
      // value shift vector: acc[c] += W * o_v[c] for the thread's 16 channels
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const float4 o4 = *reinterpret_cast<const float4 *>(&S.ck.ov[slot][16 * g + 4 * q4]);
        const int mt0 = 4 * (q4 >> 1) + 2 * (q4 & 1);
        accV[mt0][0] = fmaf(wv, o4.x, accV[mt0][0]);
        accV[mt0][2] = fmaf(wv, o4.y, accV[mt0][2]);
        accV[mt0 + 1][0] = fmaf(wv, o4.z, accV[mt0 + 1][0]);
        accV[mt0 + 1][2] = fmaf(wv, o4.w, accV[mt0 + 1][2]);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&M.vdone[s]);
      cursor_advance(cur, cv.n_chunks, n_units);
      cursor_advance(cur, cv.n_chunks, n_units);
    }
    if (cur_unit >= 0) flush_v(cur_unit);
  }
}

}  // namespace nsnkv

using namespace nsnkv;

template <int G, bool FOLD, int PREC>
int nsnkv_launch_attend_ws(const CacheViewDev &cv, const float *q, float *out, float *lse,
                           float *recs, int64_t total, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attend_ws_kernel<G, FOLD, PREC>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, ATT_SMEM_BYTES);
    attr = true;
  }
  int launches = 1;
  if (total > 0) {
    attend_ws_kernel<G, FOLD, PREC><<<grid, WS_THREADS, ATT_SMEM_BYTES, st>>>(cv, q, recs, total);
    ++launches;
  }
  combine_kernel<G, 2><<<(cv.batch * cv.n_q_heads + COMBINE_ROWS - 1) / COMBINE_ROWS, 32 * COMBINE_ROWS, 0, st>>>(cv, q, recs, total > 0 ? total : 1,
                                                                grid, out, lse);
  nsnkv_internal_count_launch(launches);
  return nsnkv_internal_check_launch("decode_attend_ws");
}

#define NSNKV_WS_INST(GG, FF, PP)                                                           \
  template int nsnkv_launch_attend_ws<GG, FF, PP>(const CacheViewDev &, const float *, float *, \
                                                  float *, float *, int64_t, int, cudaStream_t);
#define NSNKV_WS_INST_G(GG)                                                         \
  NSNKV_WS_INST(GG, true, 0) NSNKV_WS_INST(GG, true, 1) NSNKV_WS_INST(GG, true, 2)   \
  NSNKV_WS_INST(GG, false, 0) NSNKV_WS_INST(GG, false, 1) NSNKV_WS_INST(GG, false, 2)
NSNKV_WS_INST_G(1)
NSNKV_WS_INST_G(2)
NSNKV_WS_INST_G(4)
