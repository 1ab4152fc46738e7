// decode_attend.cu -- nsnkv_decode_attend: fused split-K flash-decoding over
// the packed cache (reference attention.py:83-142 in one pass).
//
// Per (unit = batch x kv-head, 64-token chunk) the kernel computes, for the G
// q-heads of the GQA group,
//   score_t = s1_t * ( s2_t * <HT(q), c_t> + <q, RoPE(o, p0 + tau)> )
//   out     = FWHT( sum_t softmax_t * s1_t * (s2_t * c'_t + o') )
// with c_t / c'_t the sign-applied codewords of the key / value payload.
//
// Engine:
//  * persistent CTAs, one per SM, stream-K split of the global chunk list;
//  * a producer warp streams each chunk's K page, V page and RoPE row p0 into
//    a 4-stage shared-memory ring with 1-D TMA bulk copies (cp.async.bulk +
//    mbarrier complete_tx);
//  * 4 consumer warps each own 16 of the chunk's 64 tokens;
//  * codewords are gathered from lane-private shared-memory tables (one
//    8-byte word per (entry, lane): the lane's component pair as fp16 hi and
//    fp16 lo halves -- conflict-free, ~22-bit precision) and fed to legacy
//    mma.sync m16n8k16 (fp16 in, fp32 accumulate):
//      K side:  D[token][head] += codewords[token][ch] . HT(q)[ch][head]
//      shift :  D[token][head] += Tab[tau][(cos,sin)_j] . AB[(cos,sin)_j][head]
//               (angle addition: <q,RoPE(o,p0+tau)> = sum_j a_j cos(tau f_j)
//                + b_j sin(tau f_j), a/b from q and RoPE(o, p0))
//      V side:  D[ch][head] += codewords^T[ch][token] . P'[token][head]
//    q and P' are split hi/lo across the two columns of each head, so every
//    product carries ~22 bits;
//  * online softmax (base-2) per warp, merged across warps / CTAs by
//    nsnkv_decode_combine together with the exact residual rows, then one
//    inverse FWHT per (batch, q-head).
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "decode_common.cuh"
#include "decode_att.cuh"

namespace nsnkv {

// ---------------------------------------------------------------------------

template <int G>
struct AttCfg {
  static constexpr int NT = (2 * G + 7) / 8;  // n-tiles of 8 (head, hi/lo) columns
  static constexpr int NGRP = G <= 4 ? 3 : 1;  // consumer groups of 4 warps
  static constexpr int THREADS = 4 * NGRP * 32;
  static constexpr int NSTAGE = NGRP == 3 ? 9 : 8;  // page ring depth
};

// Per-group prologue / merge scratch.  The unit-merge buffers alias the
// per-chunk buffers (a flush never overlaps a chunk).
template <int G>
struct AttGroup {
  static constexpr int NT = AttCfg<G>::NT;
  struct Chunk {
    uint2 ab[2][NT][8][32];   // o-term B fragments, double-buffered per chunk
    float ov[2][D];           // dequantized value shift vector
    float4 sc[2][R];          // (s1k*s2k, s1k, s1v*s2v, s1v) per token
    float qh[G][D];           // HT(q) (unit set-up only)
  };
  struct Merge {
    float mrg[4][G][D];       // per-warp partials for the unit merge
    float ml[4][G][2];
  };
  union {
    Chunk ck;
    Merge mg;
  };
  float q[G][D + 4];          // RoPE'd q of the group's current unit (padded: banks)
};

// Stage ring, constant shift-term fragments and barriers (below the 64
// KB-aligned tables); the groups' scratch lives above the tables.
template <int G>
struct AttMisc {
  static constexpr int NSTAGE = AttCfg<G>::NSTAGE;
  __align__(128) uint8_t st[NSTAGE][STAGE_BYTES];
  uint4 taba[4][8][32];               // (cos, sin)(tau f_j) A fragments per token slice
  uint64_t full[NSTAGE];
  uint64_t pro[AttCfg<G>::NGRP][2];   // per-group prologue barriers (2 slots)
  uint64_t tabs;
};
template <int G>
struct AttGroups {
  AttGroup<G> grp[AttCfg<G>::NGRP];
};


// ---------------------------------------------------------------------------
// the fused kernel
// ---------------------------------------------------------------------------
// PREC: 0 = codewords fp16 hi + lo on both sides (~1e-6 relative output
// error), 1 = scores from plain fp16 codewords, values hi + lo (~4e-4; the
// per-token score rounding is random, the value-side rounding of 1-bit
// codebooks is systematic), 2 = plain fp16 on both sides (~6e-4 on 2-bit).
template <int G, bool FOLD, int PREC>
__global__ void __launch_bounds__(AttCfg<G>::THREADS, 1)
    attend_kernel(CacheViewDev cv, const float *__restrict__ qg, float *__restrict__ recs,
                  int64_t total_chunks) {
  constexpr int NT = AttCfg<G>::NT;
  constexpr int NGRP = AttCfg<G>::NGRP;
  constexpr int NSTAGE = AttCfg<G>::NSTAGE;
  constexpr bool HILO_K = PREC == 0;
  constexpr bool HILO_V = PREC <= 1;
  static_assert(sizeof(AttMisc<G>) <= MISC_LO_MAX, "decode ring does not fit below the tables");
  static_assert(sizeof(AttGroups<G>) <= MISC_HI_MAX, "decode scratch does not fit above the tables");
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n_units = cv.batch * cv.n_kv_heads;
  const PageLayout L = page_layout(FOLD ? 2 : 1);
  const uint32_t page_bytes = (uint32_t)L.bytes;

  // ---- shared memory carve-up: tables at 64 KB-aligned shared addresses ----
  const uint32_t base = smem_u32(smem);
  const uint32_t tk = (base & 0xffffu) == 0 ? base : ((base + 0xffffu) & ~0xffffu);
  const uint32_t tv = tk + 0x10000u;
  // ring below the tables and scratch above them (both above the tables when
  // the window happens to start 64 KB-aligned)
  const bool aligned_window = (base & 0xffffu) == 0;
  AttMisc<G> &M = *reinterpret_cast<AttMisc<G> *>(smem + (aligned_window ? 0x20000u : 0u));
  AttGroups<G> &GS = *reinterpret_cast<AttGroups<G> *>(
      smem + (tv + 0x10000u - base) +
      (aligned_window ? (uint32_t)((sizeof(AttMisc<G>) + 127) / 128 * 128) : 0u));

  const int grid = gridDim.x;
  const int64_t lo = range_lo(total_chunks, blockIdx.x, grid);
  const int64_t hi = range_lo(total_chunks, blockIdx.x + 1, grid);
  if (lo >= hi) return;

  // stage loader: chunk k of the CTA range goes to stage k % NSTAGE
  // page id and RoPE row of a chunk (global loads; the refilling leader
  // fetches them one iteration ahead)
  auto chunk_src = [&](const ChunkCursor &c, int64_t &page, int64_t &p0) {
    if (c.u < n_units) {
      page = cv.page_table[(int64_t)c.u * cv.page_table_stride + c.c];
      p0 = cv.base_pos[c.u] + (int64_t)c.c * R - cv.rope_pos0;
    } else {
      page = 0;
      p0 = 0;
    }
  };
  auto load_chunk_src = [&](int k, int64_t page, int64_t p0) {
    const int s = k % NSTAGE;
    uint8_t *st = M.st[s];
    mbar_expect_tx(&M.full[s], 2 * page_bytes + ROPE_ROW_BYTES);
    tma_load_1d(st, cv.k_pool + page * page_bytes, page_bytes, &M.full[s]);
    tma_load_1d(st + page_bytes, cv.v_pool + page * page_bytes, page_bytes, &M.full[s]);
    tma_load_1d(st + 2 * page_bytes, cv.rope_cs + p0 * NPAIR, ROPE_ROW_BYTES, &M.full[s]);
  };
  auto load_chunk = [&](int k, const ChunkCursor &c) {
    int64_t page, p0;
    chunk_src(c, page, p0);
    load_chunk_src(k, page, p0);
  };
  const int n_local = (int)(hi - lo);

  if (warp == 0) {
    ChunkCursor c0 = cursor_seek(lo, cv.n_chunks, n_units);
    if (lane == 0) {
      for (int s = 0; s < NSTAGE; ++s) mbar_init(&M.full[s], 1);
      for (int q = 0; q < NGRP; ++q) {
        mbar_init(&M.pro[q][0], 128);
        mbar_init(&M.pro[q][1], 128);
      }
      mbar_init(&M.tabs, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      // codeword gather tables (2 x 64 KB) by bulk copy, overlapped with the
      // first pages and the set-up
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

  // ========================= consumer warps ==================================
  const int grp = warp >> 2;   // consumer group: chunks i with i % NGRP == grp
  const int ws = warp & 3;     // token slice [16 ws, 16 ws + 16)
  const int ci = 32 * ws + lane;
  const int bar_id = 1 + grp;
  AttGroup<G> &S = GS.grp[grp];
  const bool leader = ws == 0 && lane == 0;

  // constant o-term A fragments: (cos, sin)(tau f_j), tau = 16ws + g (+8),
  // j = 8kt + t (+4), from table rows 0..63 (positions tau); built once by
  // group 0 into shared memory (shared by all groups)
  if (grp == 0) {
#pragma unroll
    for (int kt = 0; kt < 8; ++kt) {
      uint32_t f[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const int tau = 16 * ws + g + ((r & 1) ? 8 : 0);
        const int j = 8 * kt + t + ((r & 2) ? 4 : 0);
        const float2 cs = cv.rope_cs[(int64_t)(tau - cv.rope_pos0) * NPAIR + j];
        f[r] = pack_h2(cs.x, cs.y);
      }
      M.taba[ws][kt][lane] = make_uint4(f[0], f[1], f[2], f[3]);
    }
  }
  __syncthreads();

  // gather bases: PRMT drops the index byte into bits 8..15 of
  // [table 64 KB base | idx << 8 | slot << 4]; slot = lane % 8 keeps every
  // quarter-warp of 16-byte loads on 8 distinct bank groups.
  const uint32_t slot16 = (uint32_t)((lane & 7) * 16);
  const uint32_t lbk = (tk & 0xffff0000u) | slot16;
  const uint32_t lbv = (tv & 0xffff0000u) | slot16;
  const uint32_t vsel0 = 0x7604u | ((uint32_t)(2 * (g & 1)) << 4);
  const uint32_t vsel1 = 0x7604u | ((uint32_t)(2 * (g & 1) + 1) << 4);
  const uint32_t psel = (g & 1) ? 0x7632u : 0x5410u;  // P' part (hi/lo) selector

  uint32_t qB[NT][8][2];
  float accV[NT][8][4];
  float m_run[NT], l_run[NT];

  auto flush_unit = [&](int unit) {
    named_bar(bar_id, 128);  // the merge buffers alias the per-chunk buffers
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float l = l_run[nt];
      l += __shfl_xor_sync(0xffffffffu, l, 4);
      l += __shfl_xor_sync(0xffffffffu, l, 8);
      l += __shfl_xor_sync(0xffffffffu, l, 16);
      const int h = 4 * nt + t;
      if (h < G) {
        if (g == 0) {
          S.mg.ml[ws][h][0] = m_run[nt];
          S.mg.ml[ws][h][1] = l;
        }
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const int c = 16 * g + 8 * (mt >> 2) + 2 * (mt & 3);
          S.mg.mrg[ws][h][c] = accV[nt][mt][0] + accV[nt][mt][1];
          S.mg.mrg[ws][h][c + 1] = accV[nt][mt][2] + accV[nt][mt][3];
        }
      }
    }
    named_bar(bar_id, 128);
    float *rec = record_ptr<G>(recs, (unit + blockIdx.x) * NGRP + grp);
    for (int i = ci; i < G * D; i += 128) {
      const int h = i / D, c = i - h * D;
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
    named_bar(bar_id, 128);
  };

  auto setup_unit = [&](int unit) {
    const int b = unit / cv.n_kv_heads, hk = unit - b * cv.n_kv_heads;
    const float *qs = qg + ((int64_t)b * cv.n_q_heads + (int64_t)hk * G) * D;
    for (int i = ci; i < G * D; i += 128) S.q[i / D][i % D] = qs[i];  // padded rows
    named_bar(bar_id, 128);
    for (int h = ws; h < G; h += 4) {  // HT(q), 4 values per lane
      float4 v = *reinterpret_cast<float4 *>(&S.q[h][4 * lane]);
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
      *reinterpret_cast<float4 *>(&S.ck.qh[h][4 * lane]) = v;
    }
    named_bar(bar_id, 128);
    // B fragments of HT(q) in the permuted channel order; column n = g is
    // (head 4nt + g/2, part g&1)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int h = 4 * nt + (g >> 1);
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
          qB[nt][kt][r] = pack_h2(v0, v1);
        }
      }
      m_run[nt] = -INFINITY;
      l_run[nt] = 0.f;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt)
#pragma unroll
        for (int r = 0; r < 4; ++r) accV[nt][mt][r] = 0.f;
    }
    named_bar(bar_id, 128);  // HT(q) aliases the per-chunk buffers
  };

  // the group walks its own chunks i = grp, grp + NGRP, ... of the range
  ChunkCursor cur = cursor_seek(lo + grp, cv.n_chunks, n_units);
  // the group leader refills the stage its previous chunk released: chunk
  // i - NGRP + NSTAGE, issued once the prologue barrier of chunk i shows every
  // warp of the group past chunk i - NGRP
  ChunkCursor ahead = cursor_seek(lo + NSTAGE + grp, cv.n_chunks, n_units);
  int64_t ahead_page = 0, ahead_p0 = 0;  // prefetched source of the next refill
  if (leader) chunk_src(ahead, ahead_page, ahead_p0);
  int cur_unit = -1;
  bool tabs_ready = false;
  int nloc = 0;  // chunks processed by this group (prologue slot parity)

  for (int i = grp; i < n_local; i += NGRP) {
    if (cur.u != cur_unit) {
      if (cur_unit >= 0) flush_unit(cur_unit);
      setup_unit(cur.u);
      cur_unit = cur.u;
    }
    const int s = i % NSTAGE;
    const int slot = nloc & 1;
    const uint32_t pro_parity = (uint32_t)(nloc >> 1) & 1u;
    ++nloc;
    mbar_wait(&M.full[s], (uint32_t)(i / NSTAGE) & 1u);
    if (!tabs_ready) {
      mbar_wait(&M.tabs, 0);
      tabs_ready = true;
    }
    const uint8_t *kp = M.st[s];
    const uint8_t *vp = M.st[s] + page_bytes;
    const float2 *rrow = reinterpret_cast<const float2 *>(M.st[s] + 2 * page_bytes);

    // ---- cooperative chunk prologue (group of 4 warps) ----------------------
    {
      // (a) token scales: threads 0..63 keys, 64..127 values
      const int tok = ci & 63;
      const uint8_t *pg = ci < 64 ? kp : vp;
      const uint16_t *par = reinterpret_cast<const uint16_t *>(pg + L.par);
      const float s1sc = f16_bits_to_f32(par[0]), s1z = f16_bits_to_f32(par[1]);
      const uint32_t nb = pg[L.s1n + (tok >> 1)];
      const float lv = (float)((tok & 1) ? (nb >> 4) : (nb & 15u));
      const float s1 = __fadd_rn(s1z, __fmul_rn(lv, s1sc));
      const float s2 = f16_bits_to_f32(reinterpret_cast<const uint16_t *>(pg + L.s2)[tok]);
      float2 *scp = reinterpret_cast<float2 *>(&S.ck.sc[slot][tok]);
      scp[ci < 64 ? 0 : 1] = make_float2(s1 * s2, s1);
      // (b) value shift vector, one channel per thread
      {
        const uint16_t *pv = reinterpret_cast<const uint16_t *>(vp + L.par);
        const int c = ci, gr = c >> 5;
        const uint32_t b = vp[L.on + (c >> 1)];
        const float l2 = (float)((c & 1) ? (b >> 4) : (b & 15u));
        S.ck.ov[slot][c] = __fadd_rn(f16_bits_to_f32(pv[6 + gr]),
                                  __fmul_rn(l2, f16_bits_to_f32(pv[2 + gr])));
      }
      // (c) o-term B fragments: warp ws owns pairs j in [16ws, 16ws + 16)
      {
        const uint16_t *pk = reinterpret_cast<const uint16_t *>(kp + L.par);
        const int j = 16 * ws + (lane >> 1);
        const int gr = (2 * j) >> 5;
        const uint32_t b = kp[L.on + j];
        const float osc = f16_bits_to_f32(pk[2 + gr]), oz = f16_bits_to_f32(pk[6 + gr]);
        const float oe = __fadd_rn(oz, __fmul_rn((float)(b & 15u), osc));
        const float oo = __fadd_rn(oz, __fmul_rn((float)(b >> 4), osc));
        const float2 cs = rrow[j];
        const float he = oe * cs.x - oo * cs.y;  // RoPE(o, p0)
        const float ho = oe * cs.y + oo * cs.x;
        const int kt = j >> 3, tt = j & 3, half = (j >> 2) & 1;
#pragma unroll
        for (int h = (lane & 1); h < 4 * NT; h += 2) {
          float al = 0.f, be = 0.f;
          if (h < G) {
            const float qe = S.q[h][2 * j], qo = S.q[h][2 * j + 1];
            al = qe * he + qo * ho;
            be = qo * he - qe * ho;
          }
          float ah, alo, bh, blo;
          split_h(al, ah, alo);
          split_h(be, bh, blo);
          const int nt = h >> 2, hh = h & 3;
          reinterpret_cast<uint32_t *>(&S.ck.ab[slot][nt][kt][4 * (2 * hh) + tt])[half] = pack_h2(ah, bh);
          reinterpret_cast<uint32_t *>(&S.ck.ab[slot][nt][kt][4 * (2 * hh + 1) + tt])[half] = pack_h2(alo, blo);
        }
      }
    }
    mbar_arrive(&M.pro[grp][slot]);
    if (i >= NGRP) {
      if (leader) {  // every warp of the group is past chunk i - NGRP
        mbar_wait(&M.pro[grp][slot], pro_parity);
        if (i - NGRP + NSTAGE < n_local) load_chunk_src(i - NGRP + NSTAGE, ahead_page, ahead_p0);
      }
#pragma unroll
      for (int a2 = 0; a2 < NGRP; ++a2) cursor_advance(ahead, cv.n_chunks, n_units);
      if (leader) chunk_src(ahead, ahead_page, ahead_p0);  // consumed next iteration
    }

    // ---- K side: payload dot products on tensor cores ------------------------
    const int tok0 = 16 * ws + g, tok1 = tok0 + 8;
    const uint32_t kpa = smem_u32(kp);
    const uint32_t ik0 = lds32(kpa + L.idx + tok0 * NSUB + 4 * t);
    const uint32_t ik1 = lds32(kpa + L.idx + tok1 * NSUB + 4 * t);
    uint32_t sk0 = 0, sk1 = 0;
    if (FOLD) {
      sk0 = lds32(kpa + L.sgn + tok0 * 16 + 4 * t);
      sk1 = lds32(kpa + L.sgn + tok1 * 16 + 4 * t);
    }
    float d1[NT][2][4], d2[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int r = 0; r < 4; ++r) d1[nt][0][r] = d1[nt][1][r] = d2[nt][r] = 0.f;
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
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        // k-tile 2m: pairs 0 (cols 2t..) and 1 (cols 2t+8..); k-tile 2m+1: pairs 2, 3
        mma16816(d1[nt][0], h0.x, h1.x, h0.y, h1.y, qB[nt][2 * m][0], qB[nt][2 * m][1]);
        mma16816(d1[nt][1], h0.z, h1.z, h0.w, h1.w, qB[nt][2 * m + 1][0], qB[nt][2 * m + 1][1]);
        if (HILO_K) {
          mma16816(d1[nt][0], l0.x, l1.x, l0.y, l1.y, qB[nt][2 * m][0], qB[nt][2 * m][1]);
          mma16816(d1[nt][1], l0.z, l1.z, l0.w, l1.w, qB[nt][2 * m + 1][0], qB[nt][2 * m + 1][1]);
        }
      }
    }
    mbar_wait(&M.pro[grp][slot], pro_parity);  // AB, scales, o_v of the group
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
      for (int kt = 0; kt < 8; ++kt) {
        const uint2 ab = *reinterpret_cast<const uint2 *>(&S.ck.ab[slot][nt][kt][lane]);
        const uint4 ta = M.taba[ws][kt][lane];
        mma16816(d2[nt], ta.x, ta.y, ta.z, ta.w, ab.x, ab.y);
      }
    }

    // ---- scores and online softmax (base 2) ---------------------------------
    const float4 sc0 = S.ck.sc[slot][tok0];
    const float4 sc1 = S.ck.sc[slot][tok1];
    uint32_t pf[NT][2];
    float wsum[NT];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int h = 4 * nt + t;
      const float pd0 = (d1[nt][0][0] + d1[nt][1][0]) + (d1[nt][0][1] + d1[nt][1][1]);
      const float pd1 = (d1[nt][0][2] + d1[nt][1][2]) + (d1[nt][0][3] + d1[nt][1][3]);
      const float x0 = (sc0.x * pd0 + sc0.y * (d2[nt][0] + d2[nt][1])) * LOG2E_OVER_SQRTD;
      const float x1 = (sc1.x * pd1 + sc1.y * (d2[nt][2] + d2[nt][3])) * LOG2E_OVER_SQRTD;
      float mx = fmaxf(x0, x1);
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      const float m_new = fmaxf(m_run[nt], mx);
      if (m_new > m_run[nt]) {
        const float r = exp2f(m_run[nt] - m_new);
        l_run[nt] *= r;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int q = 0; q < 4; ++q) accV[nt][mt][q] *= r;
        m_run[nt] = m_new;
      }
      float p0 = exp2f(x0 - m_new), p1 = exp2f(x1 - m_new);
      if (h >= G) p0 = p1 = 0.f;
      l_run[nt] += p0 + p1;
      // value weights: P' = p * s1v * s2v (codewords), W = sum p * s1v (shift)
      float ws2 = p0 * sc0.w + p1 * sc1.w;
      ws2 += __shfl_xor_sync(0xffffffffu, ws2, 4);
      ws2 += __shfl_xor_sync(0xffffffffu, ws2, 8);
      ws2 += __shfl_xor_sync(0xffffffffu, ws2, 16);
      wsum[nt] = ws2;
      float h0, l0, h1, l1;
      split_h(p0 * sc0.z, h0, l0);
      split_h(p1 * sc1.z, h1, l1);
      const uint32_t X0 = pack_h2(h0, l0);  // token g   (hi, lo)
      const uint32_t X1 = pack_h2(h1, l1);  // token g+8
      // B fragment of P': column g = (head 4nt + g/2, part g&1); rows are the
      // tokens 2t, 2t+1 (reg 0) and 2t+8, 2t+9 (reg 1) of the warp's slice
      const int hs = g >> 1;
      const int srcA = 8 * t + hs, srcB = 8 * t + 4 + hs;
      const uint32_t y0a = __shfl_sync(0xffffffffu, X0, srcA);
      const uint32_t y0b = __shfl_sync(0xffffffffu, X0, srcB);
      const uint32_t y1a = __shfl_sync(0xffffffffu, X1, srcA);
      const uint32_t y1b = __shfl_sync(0xffffffffu, X1, srcB);
      pf[nt][0] = prmt(y0a, y0b, psel);
      pf[nt][1] = prmt(y1a, y1b, psel);
    }

    // ---- V side: accumulate P' . codewords on tensor cores -------------------
    // thread (g, t): tokens 2t, 2t+1, 2t+8, 2t+9 of the slice; subs 2g, 2g+1
    const uint32_t vpa = smem_u32(vp);
    const int vt0 = 16 * ws + 2 * t;
    uint32_t iv[4], sv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int tok = vt0 + (q & 1) + ((q & 2) ? 8 : 0);
      iv[q] = lds32(vpa + L.idx + tok * NSUB + 4 * (g >> 1));
      sv[q] = FOLD ? (lds32(vpa + L.sgn + tok * 16 + 4 * (g >> 1)) >> (8 * (g & 1))) : 0u;
    }
#pragma unroll
    for (int sg = 0; sg < 2; ++sg) {  // sub 2g + sg
      const uint32_t sel = sg ? vsel1 : vsel0;
      uint4 yh[4], yl[4];
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
#pragma unroll
      for (int p = 0; p < 4; ++p) {  // m-tile 4 sg + p: channels 16g + 8sg + 2p (+1)
        const int mt = 4 * sg + p;
        const uint32_t *h0p = &yh[0].x, *h1p = &yh[1].x, *h2p = &yh[2].x, *h3p = &yh[3].x;
        const uint32_t a0h = prmt(h0p[p], h1p[p], 0x5410u), a1h = prmt(h0p[p], h1p[p], 0x7632u);
        const uint32_t a2h = prmt(h2p[p], h3p[p], 0x5410u), a3h = prmt(h2p[p], h3p[p], 0x7632u);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
          mma16816(accV[nt][mt], a0h, a1h, a2h, a3h, pf[nt][0], pf[nt][1]);
        if (HILO_V) {
          const uint32_t *l0p = &yl[0].x, *l1p = &yl[1].x, *l2p = &yl[2].x, *l3p = &yl[3].x;
          const uint32_t a0l = prmt(l0p[p], l1p[p], 0x5410u), a1l = prmt(l0p[p], l1p[p], 0x7632u);
          const uint32_t a2l = prmt(l2p[p], l3p[p], 0x5410u), a3l = prmt(l2p[p], l3p[p], 0x7632u);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
            mma16816(accV[nt][mt], a0l, a1l, a2l, a3l, pf[nt][0], pf[nt][1]);
        }
      }
    }
    // value shift vector: acc[c] += W * o_v[c] for the thread's 16 channels
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) {
      const float4 o4 = *reinterpret_cast<const float4 *>(&S.ck.ov[slot][16 * g + 4 * q4]);
      // channels 16g + 4q4 + {0,1,2,3}: m-tiles (sg = q4 >> 1, p = 2 (q4 & 1) + {0, 1})
      const int mt0 = 4 * (q4 >> 1) + 2 * (q4 & 1);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        accV[nt][mt0][0] = fmaf(wsum[nt], o4.x, accV[nt][mt0][0]);
        accV[nt][mt0][2] = fmaf(wsum[nt], o4.y, accV[nt][mt0][2]);
        accV[nt][mt0 + 1][0] = fmaf(wsum[nt], o4.z, accV[nt][mt0 + 1][0]);
        accV[nt][mt0 + 1][2] = fmaf(wsum[nt], o4.w, accV[nt][mt0 + 1][2]);
      }
    }
#pragma unroll
    for (int a2 = 0; a2 < NGRP; ++a2) cursor_advance(cur, cv.n_chunks, n_units);
  }
  if (cur_unit >= 0) flush_unit(cur_unit);
}

}  // namespace nsnkv

using namespace nsnkv;

static int attend_grid() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

static size_t records_bytes(const CacheViewDev &cv, int G) {
  const int units = cv.batch * cv.n_kv_heads;
  const int ngrp = 3;  // max group count over the decode kernels (v1 G<=4, v2)
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

// Kernel selection (NSNKV_DECODE_KERNEL): "v3" (default) the warp-specialized
// kernel with the shift term on tcgen05 (decode_attend3.cu); "v1" the
// first-generation grouped kernel below (kept for A/B measurements).
static int decode_kernel_choice() {
  static int v = -1;
  if (v < 0) {
    const char *e = getenv("NSNKV_DECODE_KERNEL");
    v = (e && strcmp(e, "v1") == 0) ? 1 : 3;
  }
  return v;
}

template <int G, bool FOLD, int PREC>
static int launch_attend(const CacheViewDev &cv, const float *q, float *out, float *lse,
                         float *recs, int64_t total, cudaStream_t st) {
  if (decode_kernel_choice() == 3) {
    int grid = attend_grid();
    if (total < grid) grid = (int)(total > 0 ? total : 1);
    return nsnkv_launch_attend3<G, FOLD, PREC>(cv, q, out, lse, recs, total, grid, st);
  }
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attend_kernel<G, FOLD, PREC>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, ATT_SMEM_BYTES);
    attr = true;
  }
  int grid = attend_grid();
  if (total < grid) grid = (int)(total > 0 ? total : 1);
  int launches = 1;
  if (total > 0) {
    attend_kernel<G, FOLD, PREC>
        <<<grid, AttCfg<G>::THREADS, ATT_SMEM_BYTES, st>>>(cv, q, recs, total);
    ++launches;
  }
  combine_kernel<G, AttCfg<G>::NGRP><<<(cv.batch * cv.n_q_heads + COMBINE_ROWS - 1) / COMBINE_ROWS, 32 * COMBINE_ROWS, 0, st>>>(cv, q, recs, total > 0 ? total : 1,
                                                              grid, out, lse);
  nsnkv_internal_count_launch(launches);
  return nsnkv_internal_check_launch("decode_attend");
}

extern "C" int nsnkv_decode_attend(const nsnkv_cache_view *cv_in, const float *q, float *out,
                                   float *lse, void *workspace, size_t workspace_bytes,
                                   void *stream) {
  CacheViewDev cv;
  int rc = make_cache_view(cv_in, &cv);
  if (rc) return rc;
  const int G = cv.n_q_heads / cv.n_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 8)
    return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "decode_attend: GQA group must be 1, 2, 4 or 8");
  if (cv.rope_pos0 != 0)
    return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "decode_attend: RoPE table must start at position 0");
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
  const int prec = cv.precision < 0 ? 0 : (cv.precision > 2 ? 2 : cv.precision);
#define NSNKV_ATT_P(GG, FF)                                                       \
  return prec == 0 ? launch_attend<GG, FF, 0>(cv, q, out, lse, recs, total, st)  \
       : prec == 1 ? launch_attend<GG, FF, 1>(cv, q, out, lse, recs, total, st)  \
                   : launch_attend<GG, FF, 2>(cv, q, out, lse, recs, total, st)
#define NSNKV_ATT(GG)         \
  if (fold) NSNKV_ATT_P(GG, true); \
  else NSNKV_ATT_P(GG, false)
  switch (G) {
    case 1: NSNKV_ATT(1);
    case 2: NSNKV_ATT(2);
    case 4: NSNKV_ATT(4);
    default: NSNKV_ATT(8);
  }
#undef NSNKV_ATT_P
#undef NSNKV_ATT
}
