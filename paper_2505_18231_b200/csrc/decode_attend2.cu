// decode_attend2.cu -- nsnkv_decode_attend, second-generation fused kernel:
// split-K flash-decoding over the packed cache (reference attention.py:83-142
// in one pass), organised to cut the shared-memory traffic that bounds the
// first-generation kernel (decode_attend.cu).
//
// Per (unit = batch x kv-head, 64-token chunk), for the G q-heads of the
// GQA group:
//   score_t = s1_t * ( s2_t * <HT(q), c_t> + <q, RoPE(o, p0 + tau)> )
//   out     = FWHT( sum_t softmax_t * s1_t * (s2_t * c'_t + o') )
//
// What changed against the first generation:
//  * work items are PAIRS of consecutive chunks of one unit (G <= 4): the
//    shift-term product  D[tau][(head, chunk)] = Tab[tau][(cos,sin)_j] .
//    Z[(cos,sin)_j][(head, chunk)]  covers both chunks in one n8 tile, so the
//    per-item B fragments (Z) are read once per pair instead of per chunk;
//  * the constant A operand of that product -- (cos, sin)(tau f_j) for the
//    warp's 16 token positions -- lives in 32 registers for the whole kernel
//    instead of being re-read from shared memory every chunk;
//  * Z is plain fp16 (the Tab operand it multiplies is fp16 already);
//  * every group writes a record for every unit its CTA touches (m = -inf
//    when it saw none of it), so the combine needs no ownership arithmetic.
// Codeword gathers, sign flips and the K / V tensor-core products are the
// first generation's (conflict-free LDS.128 gathers from 64 KB-aligned
// tables, channel-permuted K fragments, token-paired V fragments).
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "decode_common.cuh"
#include "decode_att.cuh"

namespace nsnkv {

template <int G>
struct A2Cfg {
  static constexpr int CP = G <= 4 ? 2 : 1;        // chunks per work item
  static constexpr int NTP = (2 * G + 7) / 8;      // payload n-tiles: (head, hi/lo) columns
  static constexpr int NGRP = G == 8 ? 2 : 3;      // consumer groups of 4 warps (G = 8: registers)
  static constexpr int THREADS = NGRP * 128;
  static constexpr int STAGE = CP * (2 * NSNKV_PAGE_BYTES_2B + ROPE_ROW_BYTES);
  static constexpr int ZF_STRIDE = 72;             // words per k-tile (64 + 8 pad: store banks)
};

template <int G>
struct A2Group {
  static constexpr int CP = A2Cfg<G>::CP;
  struct Item {
    uint32_t zf[8][A2Cfg<G>::ZF_STRIDE];  // shift-term B fragments [kt][lane][reg]
    float4 sc[CP][R];                     // (s1k*s2k, s1k, s1v*s2v, s1v) per token
    float ov[CP][D];                      // dequantized value shift vectors
  };
  struct Merge {                          // unit merge across the group's 4 warps
    float mrg[4][G][D];                   // (fixed summation order: deterministic)
    float ml[4][G][2];
  };
  struct Setup {                          // unit set-up
    float q[G][D + 4];                    // RoPE'd q (padded rows)
    float qh[G][D];                       // HT(q)
  };
  union {
    Item it[2];  // double-buffered per-item scratch
    Merge mg;    // (the group is synchronised around the merge and the set-up)
    Setup su;
  };
};

template <int G>
struct A2Bars {
  uint64_t full[16];
  uint64_t pro[A2Cfg<G>::NGRP][2];
  uint64_t tabs;
};

// Shared memory: two 64 KB-aligned codeword tables; the ring and the group
// scratch go into the two windows around them (the larger one into the
// larger window).
template <int G>
struct A2Layout {
  static constexpr int SCRATCH = A2Cfg<G>::NGRP * (int)sizeof(A2Group<G>);
  static constexpr int BARS = ((int)sizeof(A2Bars<G>) + 127) / 128 * 128;
  static constexpr int LO_WIN = MISC_LO_MAX;  // bytes below the tables
  static constexpr int HI_WIN = MISC_HI_MAX;  // bytes above the tables
  static constexpr bool RING_LO = true;       // ring below, scratch above
  static constexpr int RING_BYTES_AVAIL = LO_WIN - BARS;
  static constexpr int NSTAGE_RAW = RING_BYTES_AVAIL / A2Cfg<G>::STAGE;
  static constexpr int NSTAGE = NSTAGE_RAW > 16 ? 16 : NSTAGE_RAW;
  static_assert(SCRATCH <= HI_WIN, "group scratch does not fit above the tables");
  static_assert(NSTAGE > A2Cfg<G>::NGRP, "ring must be deeper than the group count");
};

// Work-item cursor over the CTA's chunk range [lo, hi): items are runs of up
// to CP consecutive chunks of one unit.
struct ItemCursor {
  int u, c, end;  // unit, first chunk of the item, end of the unit's run in this CTA
  int64_t x;      // global index of chunk (u, c)
};

__device__ __forceinline__ ItemCursor item_seek(int64_t lo, int64_t hi, const int32_t *n_chunks,
                                                int n_units) {
  const ChunkCursor cc = cursor_seek(lo, n_chunks, n_units);
  ItemCursor it;
  it.u = cc.u;
  it.c = cc.c;
  it.x = lo;
  const int64_t room = hi - lo;
  it.end = (int64_t)(cc.n - cc.c) < room ? cc.n : cc.c + (int)room;
  return it;
}

template <int CP>
__device__ __forceinline__ int item_count(const ItemCursor &it) {
  const int r = it.end - it.c;
  return r < CP ? r : CP;
}

template <int CP>
__device__ __forceinline__ void item_advance(ItemCursor &it, int64_t hi, const int32_t *n_chunks,
                                             int n_units) {
  const int cnt = item_count<CP>(it);
  it.x += cnt;
  it.c += cnt;
  if (it.c >= it.end) {
    if (it.x >= hi) {
      it.u = n_units;
      it.c = it.end = 0;
      return;
    }
    int n = 0;
    while (n == 0 && ++it.u < n_units) n = n_chunks[it.u];
    it.c = 0;
    const int64_t room = hi - it.x;
    it.end = (int64_t)n < room ? n : (int)room;
  }
}

template <int G, bool FOLD, int PREC>
__global__ void __launch_bounds__(A2Cfg<G>::THREADS, 1)
    attend2_kernel(CacheViewDev cv, const float *__restrict__ qg, float *__restrict__ recs,
                   int64_t total_chunks) {
  constexpr int CP = A2Cfg<G>::CP;
  constexpr int NTP = A2Cfg<G>::NTP;
  constexpr int NGRP = A2Cfg<G>::NGRP;
  constexpr int NSTAGE = A2Layout<G>::NSTAGE;
  constexpr int ZS = A2Cfg<G>::ZF_STRIDE;
  constexpr bool HILO_K = PREC == 0;
  constexpr bool HILO_V = PREC <= 1;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t = lane & 3;
  const int n_units = cv.batch * cv.n_kv_heads;
  const PageLayout L = page_layout(FOLD ? 2 : 1);
  const uint32_t page_bytes = (uint32_t)L.bytes;

  // ---- shared memory carve-up ----
  const uint32_t base = smem_u32(smem);
  const bool aligned_window = (base & 0xffffu) == 0;
  const uint32_t tk = aligned_window ? base : ((base + 0xffffu) & ~0xffffu);
  const uint32_t tv = tk + 0x10000u;
  uint8_t *lo_win = smem + (aligned_window ? 0x20000u : 0u);
  uint8_t *hi_win = smem + (tv + 0x10000u - base) +
                    (aligned_window ? (uint32_t)(A2Layout<G>::BARS +
                                                 NSTAGE * A2Cfg<G>::STAGE + 127) / 128 * 128
                                    : 0u);
  A2Bars<G> &BR = *reinterpret_cast<A2Bars<G> *>(lo_win);
  uint8_t *ring = lo_win + A2Layout<G>::BARS;
  A2Group<G> *GS = reinterpret_cast<A2Group<G> *>(hi_win);

  const int grid = gridDim.x;
  const int64_t lo = range_lo(total_chunks, blockIdx.x, grid);
  const int64_t hi = range_lo(total_chunks, blockIdx.x + 1, grid);
  if (lo >= hi) return;

  auto item_src = [&](const ItemCursor &c, int k, int64_t &page, int64_t &p0) {
    if (c.u < n_units) {
      page = cv.page_table[(int64_t)c.u * cv.page_table_stride + c.c + k];
      p0 = cv.base_pos[c.u] + (int64_t)(c.c + k) * R - cv.rope_pos0;
    } else {
      page = 0;
      p0 = 0;
    }
  };
  // issue the bulk copies of item k (stage k % NSTAGE): per chunk K page,
  // V page, RoPE row of its first position
  auto load_item = [&](int k, const ItemCursor &c, const int64_t *pages, const int64_t *p0s) {
    const int s = k % NSTAGE;
    uint8_t *st = ring + s * A2Cfg<G>::STAGE;
    const int cnt = item_count<CP>(c);
    mbar_expect_tx(&BR.full[s], (uint32_t)cnt * (2 * page_bytes + ROPE_ROW_BYTES));
    for (int q = 0; q < cnt; ++q) {
      uint8_t *sq = st + q * (2 * page_bytes);
      tma_load_1d(sq, cv.k_pool + pages[q] * page_bytes, page_bytes, &BR.full[s]);
      tma_load_1d(sq + page_bytes, cv.v_pool + pages[q] * page_bytes, page_bytes, &BR.full[s]);
      tma_load_1d(st + CP * 2 * page_bytes + q * ROPE_ROW_BYTES, cv.rope_cs + p0s[q] * NPAIR,
                  ROPE_ROW_BYTES, &BR.full[s]);
    }
  };

  const ItemCursor start = item_seek(lo, hi, cv.n_chunks, n_units);
  const int first_unit = start.u;
  const int last_unit = cursor_seek(hi - 1, cv.n_chunks, n_units).u;

  if (warp == 0) {
    ItemCursor c0 = start;
    if (lane == 0) {
      for (int s = 0; s < NSTAGE; ++s) mbar_init(&BR.full[s], 1);
      for (int q = 0; q < NGRP; ++q) {
        mbar_init(&BR.pro[q][0], 128);
        mbar_init(&BR.pro[q][1], 128);
      }
      mbar_init(&BR.tabs, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&BR.tabs, 2 * 65536);
      tma_load_1d(smem + (tk - base), cv.cb_k.tabw, 65536, &BR.tabs);
      tma_load_1d(smem + (tv - base), cv.cb_v.tabw, 65536, &BR.tabs);
      for (int k = 0; k < NSTAGE && c0.x < hi; ++k) {
        int64_t pg[CP], pp[CP];
#pragma unroll
        for (int q = 0; q < CP; ++q) item_src(c0, q < item_count<CP>(c0) ? q : 0, pg[q], pp[q]);
        load_item(k, c0, pg, pp);
        item_advance<CP>(c0, hi, cv.n_chunks, n_units);
      }
    }
  }
  __syncthreads();

  // ========================= consumer groups ===================================
  const int grp = warp >> 2;
  const int ws = warp & 3;          // token slice [16 ws, 16 ws + 16) of every chunk
  const int ci = 32 * ws + lane;    // 0..127 within the group
  const int bar_id = 1 + grp;
  A2Group<G> &S = GS[grp];
  const bool leader = ws == 0 && lane == 0;

  // constant shift-term A fragments: (cos, sin)(tau f_j), tau = 16ws + g (+8),
  // j = 8kt + t (+4)
  uint32_t taba[8][4];
#pragma unroll
  for (int kt = 0; kt < 8; ++kt)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int tau = 16 * ws + g + ((r & 1) ? 8 : 0);
      const int j = 8 * kt + t + ((r & 2) ? 4 : 0);
      const float2 cs = cv.rope_cs[(int64_t)(tau - cv.rope_pos0) * NPAIR + j];
      taba[kt][r] = pack_h2(cs.x, cs.y);
    }

  const uint32_t slot16 = (uint32_t)((lane & 7) * 16);
  const uint32_t lbk = (tk & 0xffff0000u) | slot16;
  const uint32_t lbv = (tv & 0xffff0000u) | slot16;
  const uint32_t vsel0 = 0x7604u | ((uint32_t)(2 * (g & 1)) << 4);
  const uint32_t vsel1 = 0x7604u | ((uint32_t)(2 * (g & 1) + 1) << 4);
  const uint32_t psel = (g & 1) ? 0x7632u : 0x5410u;

  uint32_t qB[NTP][8][2];
  float accV[NTP][8][4];
  // shift-term Z work of this thread: pair j = ci % 64, heads ZH0 .. ZH0+HPT-1
  // (CP = 2: every head of chunk ci / 64; CP = 1: heads 4 (ci / 64) .. +3)
  constexpr int HPT = CP == 2 ? G : 4;
  const int ZH0 = CP == 2 ? 0 : 4 * (ci >> 6);
  float2 qz[HPT];
  float m_run[NTP], l_run[NTP];

  auto write_empty = [&](int unit) {
    if (ws == 0 && lane < G) {
      float *rec = record_ptr<G>(recs, (unit + blockIdx.x) * NGRP + grp);
      rec[lane * (4 + D)] = -INFINITY;
    }
  };

  auto flush_unit = [&](int unit) {
    named_bar(bar_id, 128);  // every warp is done with the unit's last item
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt) {
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
    for (int i = ci; i < G * D; i += 128) S.su.q[i / D][i % D] = qs[i];
    named_bar(bar_id, 128);
    for (int h = ws; h < G; h += 4) {  // HT(q), 4 values per lane
      float4 v = *reinterpret_cast<float4 *>(&S.su.q[h][4 * lane]);
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
      *reinterpret_cast<float4 *>(&S.su.qh[h][4 * lane]) = v;
    }
    named_bar(bar_id, 128);
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt) {
      const int h = 4 * nt + (g >> 1);
#pragma unroll
      for (int kt = 0; kt < 8; ++kt) {
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          float v0 = 0.f, v1 = 0.f;
          if (h < G) {
            float h0, l0, h1, l1;
            split_h(S.su.qh[h][k_channel(t, kt, r, 0)], h0, l0);
            split_h(S.su.qh[h][k_channel(t, kt, r, 1)], h1, l1);
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
    // q pairs for the shift-term Z of this thread's pair j = ci % 64
#pragma unroll
    for (int hh = 0; hh < HPT; ++hh) {
      const int h = ZH0 + hh;
      qz[hh] = h < G ? *reinterpret_cast<const float2 *>(&S.su.q[h][2 * (ci & 63)])
                     : make_float2(0.f, 0.f);
    }
    named_bar(bar_id, 128);  // the set-up buffers alias the item scratch
  };

  // the group walks items k = grp, grp + NGRP, ... of the CTA's item list
  ItemCursor cur = start;
  for (int a = 0; a < grp; ++a) item_advance<CP>(cur, hi, cv.n_chunks, n_units);
  ItemCursor ahead = start;  // item k - NGRP + NSTAGE, refilled by the leader
  for (int a = 0; a < NSTAGE + grp; ++a) item_advance<CP>(ahead, hi, cv.n_chunks, n_units);
  int64_t ahead_pg[CP], ahead_p0[CP];
  if (leader) {
#pragma unroll
    for (int q = 0; q < CP; ++q) item_src(ahead, q < item_count<CP>(ahead) ? q : 0, ahead_pg[q], ahead_p0[q]);
  }
  int cur_unit = -1;
  int mark_next = first_unit;  // first unit not yet recorded by this group
  bool tabs_ready = false;
  int nloc = 0;

  for (int k = grp; cur.x < hi; k += NGRP) {
    if (cur.u != cur_unit) {
      if (cur_unit >= 0) {
        flush_unit(cur_unit);
        mark_next = cur_unit + 1;
      }
      for (int u = mark_next; u < cur.u; ++u) write_empty(u);
      mark_next = cur.u;
      setup_unit(cur.u);
      cur_unit = cur.u;
    }
    const int cnt = item_count<CP>(cur);
    const int s = k % NSTAGE;
    const int slot = nloc & 1;
    const uint32_t pro_parity = (uint32_t)(nloc >> 1) & 1u;
    ++nloc;
    mbar_wait(&BR.full[s], (uint32_t)(k / NSTAGE) & 1u);
    if (!tabs_ready) {
      mbar_wait(&BR.tabs, 0);
      tabs_ready = true;
    }
    const uint8_t *st = ring + s * A2Cfg<G>::STAGE;
    typename A2Group<G>::Item &IT = S.it[slot];

    // ---- cooperative item prologue (group of 4 warps) ------------------------
    {
      // (a) token scales: thread -> (chunk, token)
      if (CP == 2 || ci < 64) {
        const int c = CP == 2 ? (ci >> 6) : 0, tok = ci & 63;
        float4 sc4 = make_float4(0.f, 0.f, 0.f, 0.f);
        if (c < cnt) {
          const uint8_t *kp = st + c * 2 * page_bytes, *vp = kp + page_bytes;
          const uint16_t *pk = reinterpret_cast<const uint16_t *>(kp + L.par);
          const uint16_t *pv = reinterpret_cast<const uint16_t *>(vp + L.par);
          const uint32_t nk = kp[L.s1n + (tok >> 1)], nv = vp[L.s1n + (tok >> 1)];
          const float lk = (float)((tok & 1) ? (nk >> 4) : (nk & 15u));
          const float lv = (float)((tok & 1) ? (nv >> 4) : (nv & 15u));
          const float s1k = __fadd_rn(f16_bits_to_f32(pk[1]), __fmul_rn(lk, f16_bits_to_f32(pk[0])));
          const float s1v = __fadd_rn(f16_bits_to_f32(pv[1]), __fmul_rn(lv, f16_bits_to_f32(pv[0])));
          const float s2k = f16_bits_to_f32(reinterpret_cast<const uint16_t *>(kp + L.s2)[tok]);
          const float s2v = f16_bits_to_f32(reinterpret_cast<const uint16_t *>(vp + L.s2)[tok]);
          sc4 = make_float4(s1k * s2k, s1k, s1v * s2v, s1v);
        }
        IT.sc[c][tok] = sc4;
      }
      // (b) value shift vectors, one channel per thread
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        float o = 0.f;
        if (c < cnt) {
          const uint8_t *vp = st + c * 2 * page_bytes + page_bytes;
          const uint16_t *pv = reinterpret_cast<const uint16_t *>(vp + L.par);
          const int gr = ci >> 5;
          const uint32_t b = vp[L.on + (ci >> 1)];
          const float l2 = (float)((ci & 1) ? (b >> 4) : (b & 15u));
          o = __fadd_rn(f16_bits_to_f32(pv[6 + gr]), __fmul_rn(l2, f16_bits_to_f32(pv[2 + gr])));
        }
        IT.ov[c][ci] = o;
      }
      // (c) shift-term B fragments Z[(cos,sin)_j][col]: thread -> pair j and
      // (CP = 2) chunk ci / 64 for every head, or (CP = 1) heads 4 (ci/64)..+3
      {
        const int j = ci & 63;
        const int c = CP == 2 ? (ci >> 6) : 0;
        float he = 0.f, ho = 0.f;
        if (c < cnt) {
          const uint8_t *kp = st + c * 2 * page_bytes;
          const uint16_t *pk = reinterpret_cast<const uint16_t *>(kp + L.par);
          const int gr = (2 * j) >> 5;
          const uint32_t b = kp[L.on + j];
          const float osc = f16_bits_to_f32(pk[2 + gr]), oz = f16_bits_to_f32(pk[6 + gr]);
          const float oe = __fadd_rn(oz, __fmul_rn((float)(b & 15u), osc));
          const float oo = __fadd_rn(oz, __fmul_rn((float)(b >> 4), osc));
          const float2 cs =
              reinterpret_cast<const float2 *>(st + CP * 2 * page_bytes + c * ROPE_ROW_BYTES)[j];
          he = oe * cs.x - oo * cs.y;  // RoPE(o, p0)
          ho = oe * cs.y + oo * cs.x;
        }
        uint32_t *zrow = &IT.zf[j >> 3][2 * (j & 3) + ((j >> 2) & 1)];
#pragma unroll
        for (int hh = 0; hh < HPT; ++hh) {
          const int h = ZH0 + hh;
          const float2 qv = qz[hh];
          const float al = qv.x * he + qv.y * ho;
          const float be = qv.y * he - qv.x * ho;
          // column: thread t of the D fragment holds cols 2t, 2t+1 =
          // (head t, chunk 0 / 1) for CP = 2, (head t, head t + 4) for CP = 1
          const int col = CP == 2 ? (2 * h + c) : (2 * (h & 3) + (h >> 2));
          zrow[8 * col] = pack_h2(al, be);
        }
      }
    }
    mbar_arrive(&BR.pro[grp][slot]);
    if (k >= NGRP) {
      if (leader) {  // every warp of the group is past item k - NGRP
        mbar_wait(&BR.pro[grp][slot], pro_parity);
        if (ahead.x < hi) load_item(k - NGRP + NSTAGE, ahead, ahead_pg, ahead_p0);
      }
#pragma unroll 1
      for (int a2 = 0; a2 < NGRP; ++a2) item_advance<CP>(ahead, hi, cv.n_chunks, n_units);
      if (leader) {
#pragma unroll
        for (int q = 0; q < CP; ++q)
          item_src(ahead, q < item_count<CP>(ahead) ? q : 0, ahead_pg[q], ahead_p0[q]);
      }
    }

    // ---- K side: payload dot products on tensor cores ------------------------
    const int tok0 = 16 * ws + g, tok1 = tok0 + 8;
    float pd[CP][NTP][2];
#pragma unroll
    for (int c = 0; c < CP; ++c) {
#pragma unroll
      for (int nt = 0; nt < NTP; ++nt) pd[c][nt][0] = pd[c][nt][1] = 0.f;
      if (c < cnt) {
        const uint32_t kpa = smem_u32(st + c * 2 * page_bytes);
        const uint32_t ik0 = lds32(kpa + L.idx + tok0 * NSUB + 4 * t);
        const uint32_t ik1 = lds32(kpa + L.idx + tok1 * NSUB + 4 * t);
        uint32_t sk0 = 0, sk1 = 0;
        if (FOLD) {
          sk0 = lds32(kpa + L.sgn + tok0 * 16 + 4 * t);
          sk1 = lds32(kpa + L.sgn + tok1 * 16 + 4 * t);
        }
        float d1[NTP][2][4];
#pragma unroll
        for (int nt = 0; nt < NTP; ++nt)
#pragma unroll
          for (int r = 0; r < 4; ++r) d1[nt][0][r] = d1[nt][1][r] = 0.f;
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
          for (int nt = 0; nt < NTP; ++nt) {
            mma16816(d1[nt][0], h0.x, h1.x, h0.y, h1.y, qB[nt][2 * m][0], qB[nt][2 * m][1]);
            mma16816(d1[nt][1], h0.z, h1.z, h0.w, h1.w, qB[nt][2 * m + 1][0], qB[nt][2 * m + 1][1]);
            if (HILO_K) {
              mma16816(d1[nt][0], l0.x, l1.x, l0.y, l1.y, qB[nt][2 * m][0], qB[nt][2 * m][1]);
              mma16816(d1[nt][1], l0.z, l1.z, l0.w, l1.w, qB[nt][2 * m + 1][0],
                       qB[nt][2 * m + 1][1]);
            }
          }
        }
#pragma unroll
        for (int nt = 0; nt < NTP; ++nt) {
          pd[c][nt][0] = (d1[nt][0][0] + d1[nt][1][0]) + (d1[nt][0][1] + d1[nt][1][1]);
          pd[c][nt][1] = (d1[nt][0][2] + d1[nt][1][2]) + (d1[nt][0][3] + d1[nt][1][3]);
        }
      }
    }

    // ---- shift term for the whole item: D[tau][col] = Tab . Z ----------------
    mbar_wait(&BR.pro[grp][slot], pro_parity);  // Z, scales, o_v of the group
    float d2[4] = {0.f, 0.f, 0.f, 0.f};
    {
      const uint32_t zb = smem_u32(&IT.zf[0][0]) + 8u * lane;
#pragma unroll
      for (int kt = 0; kt < 8; ++kt) {
        const uint2 z = lds64(zb + 4u * ZS * kt);
        mma16816(d2, taba[kt][0], taba[kt][1], taba[kt][2], taba[kt][3], z.x, z.y);
      }
    }

    // ---- scores and online softmax (base 2) ---------------------------------
    float4 sct[CP][2];
#pragma unroll
    for (int c = 0; c < CP; ++c) {
      sct[c][0] = IT.sc[c][tok0];
      sct[c][1] = IT.sc[c][tok1];
    }
    uint32_t pf[CP][NTP][2];
    float wsum[CP][NTP];
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt) {
      const int h = 4 * nt + t;
      float x[CP][2];
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < CP; ++c)
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const float sh = d2[2 * r + (CP == 2 ? c : nt)];
          x[c][r] = (sct[c][r].x * pd[c][nt][r] + sct[c][r].y * sh) * LOG2E_OVER_SQRTD;
          if (c < cnt) mx = fmaxf(mx, x[c][r]);
        }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
      const float m_new = fmaxf(m_run[nt], mx);
      if (m_new > m_run[nt]) {
        const float rr = exp2f(m_run[nt] - m_new);
        l_run[nt] *= rr;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int q = 0; q < 4; ++q) accV[nt][mt][q] *= rr;
        m_run[nt] = m_new;
      }
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        float p0 = exp2f(x[c][0] - m_new), p1 = exp2f(x[c][1] - m_new);
        if (h >= G || c >= cnt) p0 = p1 = 0.f;
        l_run[nt] += p0 + p1;
        float ws2 = p0 * sct[c][0].w + p1 * sct[c][1].w;
        ws2 += __shfl_xor_sync(0xffffffffu, ws2, 4);
        ws2 += __shfl_xor_sync(0xffffffffu, ws2, 8);
        ws2 += __shfl_xor_sync(0xffffffffu, ws2, 16);
        wsum[c][nt] = ws2;
        float h0, l0, h1, l1;
        split_h(p0 * sct[c][0].z, h0, l0);
        split_h(p1 * sct[c][1].z, h1, l1);
        const uint32_t X0 = pack_h2(h0, l0);  // token g   (hi, lo)
        const uint32_t X1 = pack_h2(h1, l1);  // token g+8
        const int hs = g >> 1;
        const int srcA = 8 * t + hs, srcB = 8 * t + 4 + hs;
        const uint32_t y0a = __shfl_sync(0xffffffffu, X0, srcA);
        const uint32_t y0b = __shfl_sync(0xffffffffu, X0, srcB);
        const uint32_t y1a = __shfl_sync(0xffffffffu, X1, srcA);
        const uint32_t y1b = __shfl_sync(0xffffffffu, X1, srcB);
        pf[c][nt][0] = prmt(y0a, y0b, psel);
        pf[c][nt][1] = prmt(y1a, y1b, psel);
      }
    }

    // ---- V side: accumulate P' . codewords on tensor cores -------------------
    const int vt0 = 16 * ws + 2 * t;
#pragma unroll
    for (int c = 0; c < CP; ++c) {
      if (c >= cnt) break;
      const uint32_t vpa = smem_u32(st + c * 2 * page_bytes + page_bytes);
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
        for (int p = 0; p < 4; ++p) {
          const int mt = 4 * sg + p;
          const uint32_t *h0p = &yh[0].x, *h1p = &yh[1].x, *h2p = &yh[2].x, *h3p = &yh[3].x;
          const uint32_t a0h = prmt(h0p[p], h1p[p], 0x5410u), a1h = prmt(h0p[p], h1p[p], 0x7632u);
          const uint32_t a2h = prmt(h2p[p], h3p[p], 0x5410u), a3h = prmt(h2p[p], h3p[p], 0x7632u);
#pragma unroll
          for (int nt = 0; nt < NTP; ++nt)
            mma16816(accV[nt][mt], a0h, a1h, a2h, a3h, pf[c][nt][0], pf[c][nt][1]);
          if (HILO_V) {
            const uint32_t *l0p = &yl[0].x, *l1p = &yl[1].x, *l2p = &yl[2].x, *l3p = &yl[3].x;
            const uint32_t a0l = prmt(l0p[p], l1p[p], 0x5410u), a1l = prmt(l0p[p], l1p[p], 0x7632u);
            const uint32_t a2l = prmt(l2p[p], l3p[p], 0x5410u), a3l = prmt(l2p[p], l3p[p], 0x7632u);
#pragma unroll
            for (int nt = 0; nt < NTP; ++nt)
              mma16816(accV[nt][mt], a0l, a1l, a2l, a3l, pf[c][nt][0], pf[c][nt][1]);
          }
        }
      }
      // value shift vector: acc[ch] += W * o_v[ch] for the thread's 16 channels
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4) {
        const float4 o4 = *reinterpret_cast<const float4 *>(&IT.ov[c][16 * g + 4 * q4]);
        const int mt0 = 4 * (q4 >> 1) + 2 * (q4 & 1);
#pragma unroll
        for (int nt = 0; nt < NTP; ++nt) {
          accV[nt][mt0][0] = fmaf(wsum[c][nt], o4.x, accV[nt][mt0][0]);
          accV[nt][mt0][2] = fmaf(wsum[c][nt], o4.y, accV[nt][mt0][2]);
          accV[nt][mt0 + 1][0] = fmaf(wsum[c][nt], o4.z, accV[nt][mt0 + 1][0]);
          accV[nt][mt0 + 1][2] = fmaf(wsum[c][nt], o4.w, accV[nt][mt0 + 1][2]);
        }
      }
    }
#pragma unroll 1
    for (int a2 = 0; a2 < NGRP; ++a2) item_advance<CP>(cur, hi, cv.n_chunks, n_units);
  }
  if (cur_unit >= 0) {
    flush_unit(cur_unit);
    mark_next = cur_unit + 1;
  }
  for (int u = mark_next; u <= last_unit; ++u) write_empty(u);
}

}  // namespace nsnkv

using namespace nsnkv;

template <int G, bool FOLD, int PREC>
int nsnkv_launch_attend2(const CacheViewDev &cv, const float *q, float *out, float *lse,
                         float *recs, int64_t total, int grid, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(attend2_kernel<G, FOLD, PREC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         ATT_SMEM_BYTES);
    attr = true;
  }
  int launches = 0;
  if (total > 0) {
    attend2_kernel<G, FOLD, PREC><<<grid, A2Cfg<G>::THREADS, ATT_SMEM_BYTES, st>>>(cv, q, recs, total);
    ++launches;
  }
  combine_kernel<G, A2Cfg<G>::NGRP, true>
      <<<(cv.batch * cv.n_q_heads + COMBINE_ROWS - 1) / COMBINE_ROWS, 32 * COMBINE_ROWS, 0, st>>>(
          cv, q, recs, total > 0 ? total : 1, grid, out, lse);
  ++launches;
  nsnkv_internal_count_launch(launches);
  return nsnkv_internal_check_launch("decode_attend");
}

#define NSNKV_A2_INST(GG, FF, PP)                                                            \
  template int nsnkv_launch_attend2<GG, FF, PP>(const CacheViewDev &, const float *, float *, \
                                                float *, float *, int64_t, int, cudaStream_t);
#define NSNKV_A2_INST_G(GG) \
  NSNKV_A2_INST(GG, true, 0) NSNKV_A2_INST(GG, true, 1) NSNKV_A2_INST(GG, true, 2) \
  NSNKV_A2_INST(GG, false, 0) NSNKV_A2_INST(GG, false, 1) NSNKV_A2_INST(GG, false, 2)
NSNKV_A2_INST_G(1)
NSNKV_A2_INST_G(2)
NSNKV_A2_INST_G(4)
NSNKV_A2_INST_G(8)
