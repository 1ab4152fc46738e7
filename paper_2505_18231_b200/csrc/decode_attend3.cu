// decode_attend3.cu -- nsnkv_decode_attend, warp-specialized generation:
// split-K flash-decoding over the packed cache (reference
// attention.py:83-142 in one pass).
//
// Per (unit = batch x kv-head, 64-token chunk), for the G q-heads of the GQA
// group:
//   score_t = s1_t * ( s2_t * <HT(q), c_t> + <q, RoPE(o, p0 + tau)> )
//   out     = FWHT( sum_t softmax_t * s1_t * (s2_t * c'_t + o') )
//
// Roles (512 threads -- 384 for GQA-8, see A3::NGRP -- one CTA per SM,
// stream-K split of the chunk list into work items of CP consecutive chunks
// of one unit):
//  * warp 12 (TMA): streams each item's K and V page payloads, in item order,
//    into its group's shared-memory ring with 1-D bulk copies
//    (cp.async.bulk + mbarrier complete_tx);
//  * warps 13..15 (item producers, one per consumer group): per item, the
//    token scales, the value shift vectors and the shift-term B operand
//    Z[(cos,sin)_j][(chunk, head, hi/lo)] = q . RoPE(o, p0) (split hi + lo
//    fp16), then ONE thread issues the shift-term product on the 5th-gen
//    tensor cores:  D[tau][n] = Tab[tau][(cos,sin)_j] . Z  with the constant
//    Tab = (cos, sin)(tau f_j) resident in TMEM as fp16 hi + lo stacked along
//    M (8 tcgen05.mma, M = 128 = 64 positions x hi/lo, N = 16 = 2 chunks x 4
//    heads x Z hi/lo, A from TMEM, B from shared memory; `fast` chains two
//    items, N = 32), accumulator in TMEM;
//  * warps 0..11 (3 consumer groups of 4 warps; warp ws owns token positions
//    [16 ws, 16 ws + 16) of every chunk): codeword gathers from 64 KB-aligned
//    shared-memory tables, sign flips, K-side payload products and V-side
//    value products on mma.sync tensor cores, online softmax; the shift term
//    arrives by tcgen05.ld straight into the mma accumulator layout.
// Consumers never synchronise with each other inside a unit: items flow
// through full / ready / free / empty mbarriers.
#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "decode_common.cuh"
#include "decode_att.cuh"
#include "tc05.cuh"


namespace nsnkv {


template <int G, bool FOLD, int PREC>
struct A3 {
  static constexpr int CP = G <= 4 ? 2 : 1;        // chunks per work item
  static constexpr int NTP = (2 * G + 7) / 8;      // payload n-tiles: (head, hi/lo) columns
  // consumer groups of 4 warps (GQA-8: two, so the 8-head accumulators get
  // the registers of a 384-thread CTA), then the producer warpgroup: warp
  // CW streams pages, CW + 1 .. CW + NGRP produce items
  static constexpr int NGRP = G == 8 ? 2 : 3;
  static constexpr int CW = 4 * NGRP;
  static constexpr int THREADS = 32 * (CW + 4);
  static constexpr int PAGE = FOLD ? NSNKV_PAGE_BYTES_2B : NSNKV_PAGE_BYTES_1B;
  // pages split in two streams: the payload (idx [+ signs]) for the consumer
  // groups, the 256-byte tail (s2, s1 / o nibbles, RTN-4 params) for the
  // producers, each with its own ring so producers can run ahead
  static constexpr int MAIN = FOLD ? 2048 : 1024;
  static constexpr int META = 256;
  static constexpr int STAGE = CP * 2 * MAIN;
  static constexpr int TAILS = CP * 2 * META;  // producer's staged page tails per item
  static constexpr bool ONE_TABLE = PREC == 2;     // K hi | V hi interleaved per entry
  static constexpr int TBL = ONE_TABLE ? 65536 : 131072;
  static constexpr int FB = ONE_TABLE ? 2 : 1;    // items per shift-term MMA chain
  static constexpr int ZB = 4096 * FB;             // B operand: K 128 x N fp16
  static constexpr int NSLOT = ONE_TABLE ? (FB == 2 ? 4 : 3) : 2;  // producer -> consumer item slots
  static constexpr int NZB = 1;                    // shift-term B operand buffers per group
  static constexpr int BATCH = FB;                 // items per shift-term MMA chain
  static constexpr int NB = 16 * BATCH;            // MMA N: (item, chunk, head, Z hi/lo)

  struct Slot {
    float4 sc[CP][R];  // (s1k*s2k, s1k, s1v*s2v, s1v) per token
    float ov[CP][D];   // dequantized value shift vectors
  };
  struct Prod {        // written by the group's producer warp
    uint8_t zb[NZB][ZB];  // shift-term B operand (canonical no-swizzle MN-major)
    uint8_t tails[TAILS]; // page tails of the item being produced (K c0, V c0, K c1, V c1)
    Slot slot[NSLOT];
  };
  struct Cons {        // consumer-only (group-synchronised at unit changes)
    union {
      struct {
        float acc[G][D];
        float ml[G][2];
      } mg;
      struct {
        float q[G][D + 4];
        float qh[G][D];
      } su;
    };
  };
  struct Bars {
    uint64_t full[24], empty[24];
    uint64_t ready[NGRP][NSLOT], free_[NGRP][NSLOT];
    uint64_t tabs;
    uint64_t zdone[NGRP];  // the group's shift-term MMA chain finished reading Z
    uint32_t tmem_base;
  };
  static constexpr int BARS = ((int)sizeof(Bars) + 127) / 128 * 128;
  static constexpr int PROD = ((int)sizeof(Prod) + 127) / 128 * 128;
  static constexpr int CONS = ((int)sizeof(Cons) + 127) / 128 * 128;
  // windows: LO = below the 64 KB-aligned tables, HI = above them
  static constexpr int LO_WIN = MISC_LO_MAX;
  static constexpr int HI_WIN = ATT_SMEM_BYTES + 1024 - 65536 - TBL;
  // fast: bars, consumer scratch and as many producer scratch blocks as fit
  // below, the other producer blocks and the ring above; precise / balanced:
  // producer scratch above, bars + consumer scratch + ring below
  static constexpr int PLO_RAW = (LO_WIN - BARS - NGRP * CONS) / PROD;
  static constexpr int PLO = ONE_TABLE ? (PLO_RAW > NGRP ? NGRP : PLO_RAW) : 0;
  static constexpr int RING_WIN =
      ONE_TABLE ? HI_WIN - (NGRP - PLO) * PROD : LO_WIN - BARS - NGRP * CONS;
  static constexpr int NSTAGE_RAW = RING_WIN / STAGE;
  static constexpr int NS = (NSTAGE_RAW > 24 ? 24 : NSTAGE_RAW) / NGRP;  // stages per group
  static constexpr int NSTAGE = NS * NGRP;
  static_assert(!ONE_TABLE || BARS + NGRP * CONS <= LO_WIN, "scratch does not fit");
  static_assert(ONE_TABLE || NGRP * PROD <= HI_WIN, "producer scratch does not fit");
  static_assert(NS >= 2, "ring too shallow");
  // TMEM columns: Tab (hi | lo stacked in lanes) [0, 64), D[g][slot] 16 columns each
  static constexpr uint32_t D_COL0 = 64;
  static constexpr uint32_t TMEM_COLS = D_COL0 + 16 * NGRP * NSLOT <= 256 ? 256 : 512;
};

// ---------------------------------------------------------------------------
// Work items: runs of up to CP consecutive chunks of one unit inside the
// CTA's chunk range [lo, hi).
struct Item3 {
  int u, c, end;
  int64_t x;
};

__device__ __forceinline__ Item3 item3_seek(int64_t lo, int64_t hi, const int32_t *n_chunks,
                                            int n_units) {
  const ChunkCursor cc = cursor_seek(lo, n_chunks, n_units);
  Item3 it;
  it.u = cc.u;
  it.c = cc.c;
  it.x = lo;
  const int64_t room = hi - lo;
  it.end = (int64_t)(cc.n - cc.c) < room ? cc.n : cc.c + (int)room;
  return it;
}
template <int CP>
__device__ __forceinline__ int item3_count(const Item3 &it) {
  const int r = it.end - it.c;
  return r < CP ? r : CP;
}
template <int CP>
__device__ __forceinline__ void item3_next(Item3 &it, int64_t hi, const int32_t *n_chunks,
                                           int n_units) {
  const int cnt = item3_count<CP>(it);
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

// rtn4_dequant (vq.py:133-136): zero + level * scale, two fp32 roundings
__device__ __forceinline__ float rtn4(uint32_t level, float zero, float scale) {
  return __fadd_rn(zero, __fmul_rn((float)level, scale));
}

template <int G, bool FOLD, int PREC>
__global__ void __launch_bounds__(A3<G, FOLD, PREC>::THREADS, 1)
    attend3_kernel(CacheViewDev cv, const float *__restrict__ qg, float *__restrict__ recs,
                   int64_t total_chunks) {
  using C = A3<G, FOLD, PREC>;
  constexpr int CP = C::CP, NTP = C::NTP, NGRP = C::NGRP, NSTAGE = C::NSTAGE;
  constexpr bool HILO_K = PREC <= 1;  // precise (0) and vfast (1): fp16 hi + lo key codewords
  // 3 (1-bit, G = 4): key side by a per-unit lookup table in shared memory,
  // LUT[c][j] = (<HT(q_h)_j, e_c>, h = 0..3) in fp32, built by the consumers
  // at every unit change of the CTA's range (all groups step through the
  // units together); values as in vfast
  constexpr bool LUTK = PREC == 3;
  static_assert(!LUTK || (G == 4 && !FOLD), "the key lookup table is built for 1-bit, G = 4");
  constexpr bool HILO_V = PREC == 0;  // precise only: fp16 hi + lo value codewords
  // plain-fp16 unsigned (1-bit) value codewords: add (sum of P') x dbar per
  // sub-vector at the end of a unit (the codebook's mean rounding error)
  constexpr bool VBIAS = !FOLD && !HILO_V;
  constexpr PageLayout L = page_layout(FOLD ? 2 : 1);
  constexpr uint32_t PB = (uint32_t)C::PAGE;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int n_units = cv.batch * cv.n_kv_heads;

  const int grid = gridDim.x;
  const int64_t lo = range_lo(total_chunks, blockIdx.x, grid);
  const int64_t hi = range_lo(total_chunks, blockIdx.x + 1, grid);
  if (lo >= hi) return;

  // ---- shared memory carve-up ----
  const uint32_t base = smem_u32(smem);
  const uint32_t tk = (base + 0xffffu) & ~0xffffu;  // tables, 64 KB aligned
  if (tk - base < (uint32_t)C::BARS) __trap();       // (the window is never 64 KB aligned)
  uint8_t *lo_win = smem;
  uint8_t *hi_win = smem + (tk - base) + C::TBL;
  typename C::Bars &BR = *reinterpret_cast<typename C::Bars *>(lo_win);
  typename C::Cons *CS = reinterpret_cast<typename C::Cons *>(lo_win + C::BARS);
  // producer scratch of group g
  auto prod_of = [&](int g) -> typename C::Prod & {
    uint8_t *p = g < C::PLO ? lo_win + C::BARS + NGRP * C::CONS + g * C::PROD
                            : hi_win + (g - C::PLO) * C::PROD;
    return *reinterpret_cast<typename C::Prod *>(p);
  };
  uint8_t *ring = C::ONE_TABLE ? hi_win + (NGRP - C::PLO) * C::PROD
                               : lo_win + C::BARS + NGRP * C::CONS;
  const uint32_t tab_k = tk;                                  // K table (or K|V interleaved)
  const uint32_t tab_v = C::ONE_TABLE ? tk + 128u : tk + 0x10000u;

  const Item3 start = item3_seek(lo, hi, cv.n_chunks, n_units);
  const int first_unit = start.u;
  const int last_unit = cursor_seek(hi - 1, cv.n_chunks, n_units).u;

  // ---- set-up: barriers, TMEM, tables --------------------------------------
  if (warp == C::CW) {
    tc05::alloc(smem_u32(&BR.tmem_base), C::TMEM_COLS);
    tc05::relinquish();
    if (lane == 0) {
      for (int s = 0; s < NSTAGE; ++s) {
        mbar_init(&BR.full[s], 1);  // the streaming thread's expect_tx arrive
        mbar_init(&BR.empty[s], 128);  // every thread of the group's 4 consumer warps
      }
      for (int q = 0; q < NGRP; ++q)
        for (int s = 0; s < C::NSLOT; ++s) {
          mbar_init(&BR.ready[q][s], 33);  // the producer warp's lanes + the MMA commit
          mbar_init(&BR.free_[q][s], 128);  // every consumer thread of the group
        }
      mbar_init(&BR.tabs, C::ONE_TABLE ? 128 : 1);
      for (int q = 0; q < NGRP; ++q) mbar_init(&BR.zdone[q], 1);  // one commit per chain
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      if (!C::ONE_TABLE) {
        mbar_expect_tx(&BR.tabs, LUTK ? 65536 : 2 * 65536);
        if (!LUTK) tma_load_1d(smem + (tab_k - base), cv.cb_k.tabw, 65536, &BR.tabs);
        tma_load_1d(smem + (tab_v - base), cv.cb_v.tabw, 65536, &BR.tabs);
      }
    }
  }
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  const uint32_t tmem = BR.tmem_base;
  // the combine kernel (programmatic dependent) may be scheduled as SMs free
  // up; it waits for this grid's completion before it reads the records
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp >= C::CW) {
    // ======================= producer warpgroup ================================
    const int pq = warp - C::CW;  // TMEM lane quarter of this warp (CW is a multiple of 4)
    if (C::ONE_TABLE) {        // interleave the K and V hi gather tables
      const int t128 = tid - 32 * C::CW;
      const uint4 *sk = reinterpret_cast<const uint4 *>(cv.cb_k.tabw);
      const uint4 *sv = reinterpret_cast<const uint4 *>(cv.cb_v.tabw);
      uint4 *dst = reinterpret_cast<uint4 *>(smem + (tab_k - base));
      for (int i = t128; i < NENT * 8; i += 128) {
        const int e = i >> 3, s = i & 7;
        dst[e * 16 + s] = sk[e * 16 + s];
        dst[e * 16 + 8 + s] = sv[e * 16 + s];
      }
      mbar_arrive(&BR.tabs);
    }
    // constant shift-term A operand into TMEM, fp16 hi and lo parts stacked
    // along M: lane L = 32 q + 16 p + i holds position tau = 16 q + i, part p
    // (0 = hi, 1 = lo); column j = (cos, sin)(tau f_j)
    {
      const int L = 32 * pq + lane;
      const int tau = 16 * (L >> 5) + (L & 15);
      const bool lo_part = (L >> 4) & 1;
      const float2 *row = cv.rope_cs + (int64_t)(tau - cv.rope_pos0) * NPAIR;
#pragma unroll 1
      for (int c0 = 0; c0 < 64; c0 += 16) {
        uint32_t rv[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) {
          const float2 cs = row[c0 + c];
          float ch, cl, sh, sl;
          split_h(cs.x, ch, cl);
          split_h(cs.y, sh, sl);
          rv[c] = lo_part ? pack_h2(cl, sl) : pack_h2(ch, sh);
        }
        tc05::st_32x32b_x16(tmem + ((uint32_t)(32 * pq) << 16) + c0, rv);
      }
      tc05::wait_st();
      tc05::fence_before();
    }
    named_bar(5, 128);  // Tab in TMEM before the first MMA
    tc05::fence_after();

    constexpr int NSLOT = C::NSLOT, NZB = C::NZB;
    if (warp == C::CW) {
      // ---------------- warp CW: page streaming ---------------------------------
      // payload (idx [+ signs]) of every item, in item order, into its group's
      // ring (NS stages per group) with 1-D bulk copies (TMA engine).  Page ids
      // come from 32-entry windows of the page table loaded by all lanes at
      // once (one load latency per 32 chunks).
      {
        constexpr uint32_t MB = (uint32_t)C::MAIN;
        int wu = -1, wc0 = 0;
        int32_t wv = 0;
        Item3 tit = start;
        for (int k = 0; tit.x < hi; ++k) {
          const int gk = k % NGRP, nk = k / NGRP;
          const int s2 = gk * C::NS + nk % C::NS;
          const int cnt2 = item3_count<CP>(tit);
          int64_t pg[CP];
#pragma unroll
          for (int q = 0; q < CP; ++q) {
            const int c = tit.c + (q < cnt2 ? q : 0);
            if (tit.u != wu || c < wc0 || c >= wc0 + 32) {
              wu = tit.u;
              wc0 = c;
              const int cc = c + lane;
              wv = cc < tit.end ? cv.page_table[(int64_t)tit.u * cv.page_table_stride + cc] : 0;
            }
            pg[q] = (int64_t)__shfl_sync(0xffffffffu, wv, c - wc0);
          }
          if (nk >= C::NS) mbar_wait(&BR.empty[s2], (uint32_t)((nk / C::NS) - 1) & 1u);
          if (lane == 0) {
            uint8_t *st2 = ring + s2 * C::STAGE;
            mbar_expect_tx(&BR.full[s2], (uint32_t)cnt2 * 2u * MB);
            for (int q = 0; q < cnt2; ++q) {
              tma_load_1d(st2 + q * 2 * MB, cv.k_pool + pg[q] * PB, MB, &BR.full[s2]);
              tma_load_1d(st2 + q * 2 * MB + MB, cv.v_pool + pg[q] * PB, MB, &BR.full[s2]);
            }
          }
          __syncwarp();
          item3_next<CP>(tit, hi, cv.n_chunks, n_units);
        }
      }
    } else if (warp - C::CW - 1 < NGRP) {
      // ---------------- item producer of group gp ------------------------------
      const int gp = warp - C::CW - 1;
      typename C::Prod &P = prod_of(gp);
      constexpr int HPR = CP == 2 ? G : 8;  // heads per Z row pair (CP = 1: two 4-head rows)
      Item3 it = start;
      for (int a = 0; a < gp; ++a) item3_next<CP>(it, hi, cv.n_chunks, n_units);
      int cur_unit = -1;
      float2 qz[2][HPR];  // q pairs (2j, 2j+1) of this lane's j = lane, lane + 32
      // RoPE rows of the chunks' first positions, prefetched one item ahead
      auto rope_rows = [&](const Item3 &x, float2 (&r)[CP][2]) {
        if (x.x >= hi) return;
        const int cnt = item3_count<CP>(x);
        const int64_t pb = cv.base_pos[x.u] - cv.rope_pos0;
#pragma unroll
        for (int c = 0; c < CP; ++c) {
          const int64_t p0 = pb + (int64_t)(x.c + (c < cnt ? c : 0)) * R;
          r[c][0] = __ldg(cv.rope_cs + p0 * NPAIR + lane);
          r[c][1] = __ldg(cv.rope_cs + p0 * NPAIR + lane + 32);
        }
      };
      float2 rcs[CP][2];
      rope_rows(it, rcs);
      // page tails (last 256 bytes of the K and V page of each chunk), two
      // items ahead: lane l loads 32 bytes of tail l / 8 (K c0, V c0, K c1, V c1)
      auto tail_load = [&](const Item3 &x, uint4 (&r)[2]) {
        r[0] = r[1] = make_uint4(0, 0, 0, 0);
        if (x.x >= hi) return;
        const int t = lane >> 3, c = t >> 1;
        if (c >= item3_count<CP>(x)) return;
        const int64_t page = cv.page_table[(int64_t)x.u * cv.page_table_stride + x.c + c];
        const uint8_t *src = ((t & 1) ? cv.v_pool : cv.k_pool) + page * PB + C::MAIN + 32 * (lane & 7);
        r[0] = __ldg(reinterpret_cast<const uint4 *>(src));
        r[1] = __ldg(reinterpret_cast<const uint4 *>(src + 16));
      };
      Item3 it1 = it;
      for (int a = 0; a < NGRP; ++a) item3_next<CP>(it1, hi, cv.n_chunks, n_units);
      uint4 tl0[2], tl1[2];  // tails of items n and n + 1
      tail_load(it, tl0);
      tail_load(it1, tl1);
      // the address operands of those prefetches (page id of this lane's tail,
      // the unit's base position) are loaded one item earlier still, so no
      // prefetch waits on a dependent load inside the loop
      auto pid_load = [&](const Item3 &x) -> int32_t {
        const int c = lane >> 4;
        if (x.x >= hi || c >= item3_count<CP>(x)) return 0;
        return cv.page_table[(int64_t)x.u * cv.page_table_stride + x.c + c];
      };
      auto tail_load_p = [&](const Item3 &x, int32_t page, uint4 (&r)[2]) {
        r[0] = r[1] = make_uint4(0, 0, 0, 0);
        if (x.x >= hi) return;
        const int t = lane >> 3, c = t >> 1;
        if (c >= item3_count<CP>(x)) return;
        const uint8_t *src = ((t & 1) ? cv.v_pool : cv.k_pool) + (int64_t)page * PB + C::MAIN + 32 * (lane & 7);
        r[0] = __ldg(reinterpret_cast<const uint4 *>(src));
        r[1] = __ldg(reinterpret_cast<const uint4 *>(src + 16));
      };
      auto rope_rows_p = [&](const Item3 &x, int64_t bp, float2 (&r)[CP][2]) {
        if (x.x >= hi) return;
        const int cnt = item3_count<CP>(x);
        const int64_t pb = bp - cv.rope_pos0;
#pragma unroll
        for (int c = 0; c < CP; ++c) {
          const int64_t p0 = pb + (int64_t)(x.c + (c < cnt ? c : 0)) * R;
          r[c][0] = __ldg(cv.rope_cs + p0 * NPAIR + lane);
          r[c][1] = __ldg(cv.rope_cs + p0 * NPAIR + lane + 32);
        }
      };
      Item3 it2 = it1;
      for (int a = 0; a < NGRP; ++a) item3_next<CP>(it2, hi, cv.n_chunks, n_units);
      int32_t pid2 = pid_load(it2);
      int64_t bp1 = it1.x < hi ? cv.base_pos[it1.u] : 0;
      int n = 0;
      for (int k = gp; it.x < hi; k += NGRP, ++n) {
        const int cnt = item3_count<CP>(it);
        const int slot = n % NSLOT;
        if (it.u != cur_unit) {
          cur_unit = it.u;
          const int qb = it.u / cv.n_kv_heads, qhk = it.u - qb * cv.n_kv_heads;
          const float *qs = qg + ((int64_t)qb * cv.n_q_heads + (int64_t)qhk * G) * D;
#pragma unroll
          for (int jj = 0; jj < 2; ++jj)
#pragma unroll
            for (int h = 0; h < HPR; ++h)
              qz[jj][h] = h < G ? __ldg(reinterpret_cast<const float2 *>(qs + h * D + 2 * (lane + 32 * jj)))
                                : make_float2(0.f, 0.f);
        }
        Item3 nx = it1;  // next item of this producer: prefetch its RoPE rows
        Item3 it3 = it2;  // three items ahead: its tail's page id
        for (int a = 0; a < NGRP; ++a) item3_next<CP>(it3, hi, cv.n_chunks, n_units);
        const int32_t pid3 = pid_load(it3);
        const int64_t bp2 = it2.x < hi ? cv.base_pos[it2.u] : 0;
        float2 rcs_next[CP][2];
        rope_rows_p(nx, bp1, rcs_next);
        uint4 tl2[2];  // two items ahead: its page tails
        tail_load_p(it2, pid2, tl2);
        if (n >= NSLOT) mbar_wait(&BR.free_[gp][slot], (uint32_t)((n / NSLOT) - 1) & 1u);
        // stage the item's page tails; field offsets are relative to the tail
        __syncwarp();
        if (lane < 16 * CP) {  // 8 lanes per tail, K and V tail per chunk (TAILS bytes)
          *reinterpret_cast<uint4 *>(P.tails + 32 * lane) = tl0[0];
          *reinterpret_cast<uint4 *>(P.tails + 32 * lane + 16) = tl0[1];
        }
        __syncwarp();
        const uint8_t *st = P.tails;
        // tail field offsets (the page layout's minus the payload size)
        constexpr PageLayout LT{L.idx, L.sgn, L.s2 - C::MAIN, L.s1n - C::MAIN, L.on - C::MAIN,
                                L.par - C::MAIN, L.ledger - C::MAIN, L.bytes - C::MAIN};
        constexpr uint32_t TP = 2u * C::META;  // chunk stride in the staged tails
        typename C::Slot &SL = P.slot[slot];
        {
        // token scales (rtn4 s1, f16 s2) of tokens 2 lane, 2 lane + 1, keys and values
#pragma unroll
        for (int c = 0; c < CP; ++c) {
          float4 v0 = make_float4(0.f, 0.f, 0.f, 0.f), v1 = v0;
          float4 o4 = v0;
          if (c < cnt) {
            const uint8_t *kp = st + c * TP, *vp = kp + C::META;
            const uint32_t pk01 = *reinterpret_cast<const uint32_t *>(kp + LT.par);  // s1 scale, zero
            const uint32_t pv01 = *reinterpret_cast<const uint32_t *>(vp + LT.par);
            const uint32_t nk = kp[LT.s1n + lane], nv = vp[LT.s1n + lane];
            const uint32_t s2k = *reinterpret_cast<const uint32_t *>(kp + LT.s2 + 4 * lane);
            const uint32_t s2v = *reinterpret_cast<const uint32_t *>(vp + LT.s2 + 4 * lane);
            const float ksc = f16_bits_to_f32(pk01 & 0xffffu), kz = f16_bits_to_f32(pk01 >> 16);
            const float vsc = f16_bits_to_f32(pv01 & 0xffffu), vz = f16_bits_to_f32(pv01 >> 16);
            const float s1k0 = rtn4(nk & 15u, kz, ksc), s1k1 = rtn4(nk >> 4, kz, ksc);
            const float s1v0 = rtn4(nv & 15u, vz, vsc), s1v1 = rtn4(nv >> 4, vz, vsc);
            const float k20 = f16_bits_to_f32(s2k & 0xffffu), k21 = f16_bits_to_f32(s2k >> 16);
            const float v20 = f16_bits_to_f32(s2v & 0xffffu), v21 = f16_bits_to_f32(s2v >> 16);
            v0 = make_float4(s1k0 * k20, s1k0, s1v0 * v20, s1v0);
            v1 = make_float4(s1k1 * k21, s1k1, s1v1 * v21, s1v1);
            // value shift vector: channels 4 lane .. 4 lane + 3 (group lane / 8)
            const int gr = lane >> 3;
            const float zs = f16_bits_to_f32(reinterpret_cast<const uint16_t *>(vp + LT.par)[6 + gr]);
            const float ss = f16_bits_to_f32(reinterpret_cast<const uint16_t *>(vp + LT.par)[2 + gr]);
            const uint32_t b2 = *reinterpret_cast<const uint16_t *>(vp + LT.on + 2 * lane);
            o4 = make_float4(rtn4(b2 & 15u, zs, ss), rtn4((b2 >> 4) & 15u, zs, ss),
                             rtn4((b2 >> 8) & 15u, zs, ss), rtn4((b2 >> 12) & 15u, zs, ss));
          }
          SL.sc[c][2 * lane] = v0;
          SL.sc[c][2 * lane + 1] = v1;
          // value shift channel ch = 16 mt + 8 h + g stored at 16 g + 2 mt + h:
          // a consumer lane reads its 16 accumulator rows as four float4
          {
            const float ov4[4] = {o4.x, o4.y, o4.z, o4.w};
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int ch = 4 * lane + e;
              SL.ov[c][16 * (ch & 7) + 2 * (ch >> 4) + ((ch >> 3) & 1)] = ov4[e];
            }
          }
        }
        }
        // the MMA chain that last used this Z buffer (batch m - NZB) is done
        constexpr int BATCH = C::BATCH, NB = C::NB;
        const int m = n / BATCH, e = n % BATCH;
        if (m >= NZB) {
          const int n0 = (m - NZB) * BATCH;
          (void)n0;
          mbar_wait(&BR.zdone[gp], (uint32_t)((m - NZB) & 1));
        }
        const uint32_t zb_s = smem_u32(P.zb[m % NZB]);
        // Z (MN-major B operand): element (k, n) at (k/8)*256 + (n/8)*128 +
        // (k%8)*16 + (n%8)*2 with k = 2j (cos coefficient a_j) / 2j + 1 (sin
        // coefficient b_j) and n = 8 (chunk | head group) + 2 head + (hi | lo):
        // each (j, chunk) writes two 16-byte rows (a_j and b_j for 4 heads x hi/lo);
        // lanes 4..7 of every 8 store the b row first (conflict-free phases)
#pragma unroll
        for (int c = 0; c < CP; ++c) {
          float osc = 0.f, oz = 0.f, osc2 = 0.f, oz2 = 0.f;
          uint32_t ob0 = 0, ob1 = 0;
          if (c < cnt) {
            const uint8_t *kp = st + c * TP;
            const uint16_t *pk = reinterpret_cast<const uint16_t *>(kp + LT.par);
            osc = f16_bits_to_f32(pk[2 + (lane >> 4)]);      // group of channels 2 lane
            oz = f16_bits_to_f32(pk[6 + (lane >> 4)]);
            osc2 = f16_bits_to_f32(pk[2 + 2 + (lane >> 4)]); // channels 2 (lane + 32)
            oz2 = f16_bits_to_f32(pk[6 + 2 + (lane >> 4)]);
            ob0 = kp[LT.on + lane];
            ob1 = kp[LT.on + lane + 32];
          }
#pragma unroll
          for (int jj = 0; jj < 2; ++jj) {
            const int j = lane + 32 * jj;
            const uint32_t b = jj ? ob1 : ob0;
            const float sc_ = jj ? osc2 : osc, z_ = jj ? oz2 : oz;
            const float oe = rtn4(b & 15u, z_, sc_), oo = rtn4(b >> 4, z_, sc_);
            const float2 cs = rcs[c][jj];
            const float he = c < cnt ? oe * cs.x - oo * cs.y : 0.f;  // RoPE(o, p0)
            const float ho = c < cnt ? oe * cs.y + oo * cs.x : 0.f;
#pragma unroll
            for (int hg = 0; hg < (HPR + 3) / 4; ++hg) {
              uint32_t ra[4], rb[4];
#pragma unroll
              for (int hh = 0; hh < 4; ++hh) {
                const int h = 4 * hg + hh;
                float al = 0.f, be = 0.f;
                if (h < HPR) {
                  const float2 qv = qz[jj][h < HPR ? h : 0];
                  al = qv.x * he + qv.y * ho;
                  be = qv.y * he - qv.x * ho;
                }
                // hi = the top 11 significant bits (exact in fp16), lo = the
                // exact fp32 remainder rounded to fp16: |error| < 2^-21 |x|
                const float ah = __uint_as_float(__float_as_uint(al) & 0xffffe000u);
                const float bh = __uint_as_float(__float_as_uint(be) & 0xffffe000u);
                const __half2 pa = __floats2half2_rn(ah, al - ah);
                const __half2 pb = __floats2half2_rn(bh, be - bh);
                ra[hh] = *reinterpret_cast<const uint32_t *>(&pa);  // (a hi, a lo)
                rb[hh] = *reinterpret_cast<const uint32_t *>(&pb);  // (b hi, b lo)
              }
              const int n1 = (CP == 2 ? c : hg) + 2 * e;
              const uint32_t row = zb_s + (uint32_t)((j >> 2) * (NB * 16) + n1 * 128 + (j & 3) * 32);
              const bool bfirst = (lane >> 2) & 1;
              const uint32_t a0 = bfirst ? row + 16 : row, a1 = bfirst ? row : row + 16;
              const uint4 v0 = bfirst ? make_uint4(rb[0], rb[1], rb[2], rb[3]) : make_uint4(ra[0], ra[1], ra[2], ra[3]);
              const uint4 v1 = bfirst ? make_uint4(ra[0], ra[1], ra[2], ra[3]) : make_uint4(rb[0], rb[1], rb[2], rb[3]);
              asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a0), "r"(v0.x), "r"(v0.y), "r"(v0.z), "r"(v0.w));
              asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a1), "r"(v1.x), "r"(v1.y), "r"(v1.z), "r"(v1.w));
            }
          }
        }
        // Z stores become visible to the tensor core (async proxy) before the
        // batch's MMA chain; one fence per batch covers both items' stores
        const bool issue = e == BATCH - 1 || nx.x >= hi;
        if (issue) tc05::fence_proxy_async();
        __syncwarp();
        mbar_arrive(&BR.ready[gp][slot]);  // every lane: its scales and value shift vectors
        if (lane == 0) {
          if (issue) {  // issue the batch's shift-term MMA chain
            tc05::fence_after();
            const int nf = m * BATCH;          // first item of the batch
            const uint32_t dcol = tmem + C::D_COL0 + (uint32_t)(16 * (NSLOT * gp + nf % NSLOT));
            constexpr uint32_t idesc = tc05::idesc_f16(128, NB) | (1u << 16);  // B MN-major
#pragma unroll
            for (int kt = 0; kt < 8; ++kt)
              tc05::mma_f16_ts(dcol, tmem + 8 * kt,
                               tc05::smem_desc(zb_s + (uint32_t)(kt * NB * 32), NB * 16, 128), idesc,
                               kt > 0);
            for (int q = nf; q <= n; ++q) tc05::commit(smem_u32(&BR.ready[gp][q % NSLOT]));
            tc05::commit(smem_u32(&BR.zdone[gp]));
          }
        }
        __syncwarp();
        it = nx;
        it1 = it2;
        it2 = it3;
        pid2 = pid3;
        bp1 = bp2;
        tl0[0] = tl1[0], tl0[1] = tl1[1];
        tl1[0] = tl2[0], tl1[1] = tl2[1];
#pragma unroll
        for (int c = 0; c < CP; ++c) rcs[c][0] = rcs_next[c][0], rcs[c][1] = rcs_next[c][1];
      }
    }
  } else {
    // ======================= consumer groups ===================================
    const int g = lane >> 2, t = lane & 3;
    const int grp = warp >> 2;
    const int ws = warp & 3;
    const int ci = 32 * ws + lane;
    const int bar_id = 1 + grp;
    typename C::Cons &S = CS[grp];
    typename C::Prod &P = prod_of(grp);

    const uint32_t slot16 = (uint32_t)((lane & 7) * 16);
    const uint32_t lbk = (tab_k & 0xffff0000u) | (tab_k & 0xffu) | slot16;
    const uint32_t lbv = (tab_v & 0xffff0000u) | (tab_v & 0xffu) | slot16;
    constexpr uint32_t LO_OFS = C::ONE_TABLE ? 0u : 128u;  // hi -> lo half of an entry
    // V side (ldmatrix.x4.trans): lane supplies the row address of token
    // vT (of the warp's 16) for sub 2 mt + vodd; the index byte sits in word
    // mt / 2 at byte 2 (mt & 1) + vodd
    const int vT = (lane & 7) + 8 * (lane >> 4), vodd = (lane >> 3) & 1;
    const uint32_t vselA = 0x7604u | ((uint32_t)vodd << 4);
    const uint32_t vselB = 0x7604u | ((uint32_t)(2 + vodd) << 4);
    const uint32_t psel = (g & 1) ? 0x7632u : 0x5410u;

    uint32_t qB[NTP][8][2];
    float accV[NTP][8][4];
    float m_run[NTP], l_run[NTP];
    float pv_run[NTP];  // VBIAS: running sum of P' = p s1 s2 (this lane's tokens)
    const float dbar_g = VBIAS ? cv.cb_v.dbar[g] : 0.f;  // channels 16 mt + g (+ 8)

    // LUTK: entry c, sub j at byte c * 256 + lut_slot(j) * 16 of the K table
    // region: the 8 lanes of a quarter-warp (g = 2q, 2q + 1; t = 0..3) read
    // subs 4 t + m and 4 t + (m ^ 2), whose slots fall in 8 different bank
    // groups, so every LDS.128 phase is conflict-free
    auto lut_slot = [](int j) -> uint32_t { return (uint32_t)((j & 8) | ((j + (j >> 3)) & 7)); };
    uint32_t lutb[4], lsel[4];
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const int mm = (g & 1) ? (m ^ 2) : m;
      lutb[m] = tab_k | (lut_slot(4 * t + mm) << 4);
      lsel[m] = 0x7604u | ((uint32_t)mm << 4);
    }
    auto lut_transition = [&](int U) {
      __syncwarp();       // converged warps at the (aligned) named barrier
      named_bar(4, 32 * C::CW);  // every consumer is done with the previous unit's table
      if (grp == 0) {     // HT(q_h) of the unit's G = 4 q-heads (warp ws: head ws)
        const int b = U / cv.n_kv_heads, hk = U - b * cv.n_kv_heads;
        const float *qs = qg + ((int64_t)b * cv.n_q_heads + (int64_t)hk * G + ws) * D;
        float4 v = *reinterpret_cast<const float4 *>(qs + 4 * lane);
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
        *reinterpret_cast<float4 *>(&CS[0].su.qh[ws][4 * lane]) = v;
      }
      named_bar(4, 32 * C::CW);
      {  // thread i: sub j = i % 16, entries c = i / 16 + 24 k
        const int i = 128 * grp + ci, j = i & 15;
        float qv[4][8];
#pragma unroll
        for (int h = 0; h < 4; ++h)
#pragma unroll
          for (int k = 0; k < 8; ++k) qv[h][k] = CS[0].su.qh[h][8 * j + k];
        const uint32_t sl = lut_slot(j) << 4;
        const float4 *ent = reinterpret_cast<const float4 *>(cv.cb_k.entries);
        for (int c = i >> 4; c < NENT; c += 2 * C::CW) {
          const float4 e0 = __ldg(ent + 2 * c), e1 = __ldg(ent + 2 * c + 1);
          float r[4];
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            float x = qv[h][0] * e0.x;
            x = fmaf(qv[h][1], e0.y, x); x = fmaf(qv[h][2], e0.z, x); x = fmaf(qv[h][3], e0.w, x);
            x = fmaf(qv[h][4], e1.x, x); x = fmaf(qv[h][5], e1.y, x); x = fmaf(qv[h][6], e1.z, x);
            r[h] = fmaf(qv[h][7], e1.w, x);
          }
          asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(tab_k + (uint32_t)c * 256u + sl),
                       "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]));
        }
      }
      named_bar(4, 32 * C::CW);  // table complete
    };

    auto write_empty = [&](int unit) {
      if (ws == 0 && lane < G) {
        float *rec = record_ptr<G>(recs, (unit + blockIdx.x) * NGRP + grp);
        rec[lane * (4 + D)] = -INFINITY;
      }
    };

    // merge the 4 warps' partials in a fixed order (3, 2, 1, 0) through one
    // [G][D] buffer; warp 0 writes the record
    auto flush_unit = [&](int unit) {
      float lw[NTP], cor[NTP];
#pragma unroll
      for (int nt = 0; nt < NTP; ++nt) {
        float l = l_run[nt];
        l += __shfl_xor_sync(0xffffffffu, l, 4);
        l += __shfl_xor_sync(0xffffffffu, l, 8);
        l += __shfl_xor_sync(0xffffffffu, l, 16);
        lw[nt] = l;
        cor[nt] = 0.f;
        if (VBIAS) {
          float pv = pv_run[nt];
          pv += __shfl_xor_sync(0xffffffffu, pv, 4);
          pv += __shfl_xor_sync(0xffffffffu, pv, 8);
          pv += __shfl_xor_sync(0xffffffffu, pv, 16);
          cor[nt] = pv * dbar_g;
        }
      }
      named_bar(bar_id, 128);
      for (int r = 3; r >= 0; --r) {
        if (ws == r) {
          float mnew[NTP], lnew[NTP];
#pragma unroll
          for (int nt = 0; nt < NTP; ++nt) {
            const int h = 4 * nt + t;
            mnew[nt] = -INFINITY;
            lnew[nt] = 0.f;
            if (h >= G) continue;
            float sa = 1.f, sb = 0.f, m = m_run[nt], l = lw[nt];
            if (r < 3) {
              const float mb = S.mg.ml[h][0], lb = S.mg.ml[h][1];
              const float mx = fmaxf(m, mb);
              sa = mx > -INFINITY ? exp2f(m - mx) : 0.f;
              sb = mx > -INFINITY ? exp2f(mb - mx) : 0.f;
              l = l * sa + lb * sb;
              m = mx;
            }
            if (r > 0) {
#pragma unroll
              for (int mt = 0; mt < 8; ++mt) {
                const int c = 16 * mt + g;  // accumulator rows g / g + 8 of m-tile mt
                float a0 = (accV[nt][mt][0] + accV[nt][mt][1] + cor[nt]) * sa;
                float a1 = (accV[nt][mt][2] + accV[nt][mt][3] + cor[nt]) * sa;
                if (r < 3) {
                  a0 = fmaf(S.mg.acc[h][c], sb, a0);
                  a1 = fmaf(S.mg.acc[h][c + 8], sb, a1);
                }
                S.mg.acc[h][c] = a0;
                S.mg.acc[h][c + 8] = a1;
              }
              mnew[nt] = m;
              lnew[nt] = l;
            } else {
              float *rec = record_ptr<G>(recs, (unit + blockIdx.x) * NGRP + grp) + h * (4 + D);
#pragma unroll
              for (int mt = 0; mt < 8; ++mt) {
                const int c = 16 * mt + g;
                rec[4 + c] = fmaf(S.mg.acc[h][c], sb, (accV[nt][mt][0] + accV[nt][mt][1] + cor[nt]) * sa);
                rec[4 + c + 8] = fmaf(S.mg.acc[h][c + 8], sb, (accV[nt][mt][2] + accV[nt][mt][3] + cor[nt]) * sa);
              }
              if (g == 0) {
                rec[0] = m;
                rec[1] = l;
              }
            }
          }
          if (r > 0) {
            __syncwarp();  // every lane read ml before it is overwritten
#pragma unroll
            for (int nt = 0; nt < NTP; ++nt) {
              const int h = 4 * nt + t;
              if (h < G && g == 0) {
                S.mg.ml[h][0] = mnew[nt];
                S.mg.ml[h][1] = lnew[nt];
              }
            }
          }
        }
        named_bar(bar_id, 128);
      }
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
        pv_run[nt] = 0.f;
#pragma unroll
        for (int mt = 0; mt < 8; ++mt)
#pragma unroll
          for (int r = 0; r < 4; ++r) accV[nt][mt][r] = 0.f;
      }
      named_bar(bar_id, 128);  // the set-up buffer aliases the merge buffer
    };

    Item3 cur = start;
    for (int a = 0; a < grp; ++a) item3_next<CP>(cur, hi, cv.n_chunks, n_units);
    int cur_unit = -1;
    int mark_next = first_unit;
    int n = 0;
    mbar_wait(&BR.tabs, 0);
    // units of the CTA's range in order; with the key table every group runs
    // every unit's transition from this one call site (named barriers)
    // with the key table, the units of the CTA's range are walked in order
    // and every group runs each unit's table transition from this one call
    // site (named barriers), flushing its own partials of a unit first;
    // otherwise one pass over the group's items
    // one work item (CP chunks of unit cur.u) of this consumer group
    auto process_item = [&]() {
      const int cnt = item3_count<CP>(cur);
      const int s = grp * C::NS + n % C::NS, slot = n % C::NSLOT;
      mbar_wait(&BR.full[s], (uint32_t)(n / C::NS) & 1u);
      const uint8_t *st = ring + s * C::STAGE;

      // ---- K side: payload dot products on tensor cores ----------------------
      const int tok0 = 16 * ws + g, tok1 = tok0 + 8;
      float pd[CP][NTP][2];
#pragma unroll
      for (int c = 0; c < CP; ++c) {
#pragma unroll
        for (int nt = 0; nt < NTP; ++nt) pd[c][nt][0] = pd[c][nt][1] = 0.f;
        // fast mode computes a missing second chunk on stale stage bytes
        // (gathers only ever return finite table entries; its weights are
        // masked to zero) so both chunks' gathers can interleave
        if (LUTK) {
          if (c < cnt) {
            const uint32_t kpa = smem_u32(st + c * 2 * C::MAIN);
            const uint32_t ik0 = lds32(kpa + L.idx + tok0 * NSUB + 4 * t);
            const uint32_t ik1 = lds32(kpa + L.idx + tok1 * NSUB + 4 * t);
            float a0[4] = {0.f, 0.f, 0.f, 0.f}, a1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int m = 0; m < 4; ++m) {
              const uint4 w0 = lds128(prmt(ik0, lutb[m], lsel[m]));
              const uint4 w1 = lds128(prmt(ik1, lutb[m], lsel[m]));
              a0[0] += __uint_as_float(w0.x); a0[1] += __uint_as_float(w0.y);
              a0[2] += __uint_as_float(w0.z); a0[3] += __uint_as_float(w0.w);
              a1[0] += __uint_as_float(w1.x); a1[1] += __uint_as_float(w1.y);
              a1[2] += __uint_as_float(w1.z); a1[3] += __uint_as_float(w1.w);
            }
            // sum the 4 lanes t of a token, lane t keeping head t: heads
            // (t & 2, +1) over xor 2, then head t over xor 1
            const bool hb = t & 2, lb = t & 1;
            float k0 = hb ? a0[2] : a0[0], k1 = hb ? a0[3] : a0[1];
            float k2 = hb ? a1[2] : a1[0], k3 = hb ? a1[3] : a1[1];
            k0 += __shfl_xor_sync(0xffffffffu, hb ? a0[0] : a0[2], 2);
            k1 += __shfl_xor_sync(0xffffffffu, hb ? a0[1] : a0[3], 2);
            k2 += __shfl_xor_sync(0xffffffffu, hb ? a1[0] : a1[2], 2);
            k3 += __shfl_xor_sync(0xffffffffu, hb ? a1[1] : a1[3], 2);
            float v0 = lb ? k1 : k0, v1 = lb ? k3 : k2;
            v0 += __shfl_xor_sync(0xffffffffu, lb ? k0 : k1, 1);
            v1 += __shfl_xor_sync(0xffffffffu, lb ? k2 : k3, 1);
            pd[c][0][0] = v0;
            pd[c][0][1] = v1;
          }
        } else if (C::ONE_TABLE || c < cnt) {
          const uint32_t kpa = smem_u32(st + c * 2 * C::MAIN);
          const uint32_t ik0 = lds32(kpa + L.idx + tok0 * NSUB + 4 * t);
          const uint32_t ik1 = lds32(kpa + L.idx + tok1 * NSUB + 4 * t);
          uint32_t sk0 = 0, sk1 = 0;
          if (FOLD) {
            sk0 = lds32(kpa + (FOLD ? L.sgn : 0) + tok0 * 16 + 4 * t);
            sk1 = lds32(kpa + (FOLD ? L.sgn : 0) + tok1 * 16 + 4 * t);
          }
          float d1[NTP][2][4];
#pragma unroll
          for (int nt = 0; nt < NTP; ++nt)
#pragma unroll
            for (int r = 0; r < 4; ++r) d1[nt][0][r] = d1[nt][1][r] = 0.f;
#pragma unroll
          for (int m = 0; m < 4; ++m) {
            const uint32_t sel = 0x7604u | ((uint32_t)m << 4);
            const uint32_t a0 = prmt(ik0, lbk, sel), a1 = prmt(ik1, lbk, sel);
            uint4 h0 = lds128(a0), h1 = lds128(a1);
            uint4 l0 = make_uint4(0, 0, 0, 0), l1 = l0;
            if (HILO_K) {
              l0 = lds128(a0 + LO_OFS);
              l1 = lds128(a1 + LO_OFS);
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

      // ---- shift term (tensor memory) and token scales from the producer -----
      mbar_wait(&BR.ready[grp][slot], (uint32_t)(n / C::NSLOT) & 1u);
      tc05::fence_after();
      const typename C::Slot &SL = P.slot[slot];
      float sh[CP][NTP][2];
      {
        const uint32_t dcol = tmem + C::D_COL0 + (uint32_t)(16 * (C::NSLOT * grp + slot));
        float r4[CP][NTP][2][4];
#pragma unroll
        for (int c = 0; c < CP; ++c)
#pragma unroll
          for (int nt = 0; nt < NTP; ++nt)
#pragma unroll
            for (int p = 0; p < 2; ++p)
              // lanes 32 ws + 16 p (+g, +8+g): Tab hi / lo rows of the slice;
              // columns (chunk c | head group nt) x 8: (head, Z hi / lo)
              tc05::ld_16x256b(tmem + ((uint32_t)(32 * ws + 16 * p) << 16) +
                                   (dcol - tmem) + (uint32_t)(8 * (CP == 2 ? c : nt)),
                               r4[c][nt][p]);
        tc05::wait_ld();
#pragma unroll
        for (int c = 0; c < CP; ++c)
#pragma unroll
          for (int nt = 0; nt < NTP; ++nt) {
            sh[c][nt][0] = (r4[c][nt][0][0] + r4[c][nt][0][1]) + (r4[c][nt][1][0] + r4[c][nt][1][1]);
            sh[c][nt][1] = (r4[c][nt][0][2] + r4[c][nt][0][3]) + (r4[c][nt][1][2] + r4[c][nt][1][3]);
          }
      }
      float4 sct[CP][2];
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        sct[c][0] = SL.sc[c][tok0];
        sct[c][1] = SL.sc[c][tok1];
      }

      // ---- scores and online softmax (base 2) -------------------------------
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
            x[c][r] = (sct[c][r].x * pd[c][nt][r] + sct[c][r].y * sh[c][nt][r]) * LOG2E_OVER_SQRTD;
            if (c < cnt) mx = fmaxf(mx, x[c][r]);
          }
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const float m_new = fmaxf(m_run[nt], mx);
        if (m_new > m_run[nt]) {
          const float rr = exp2f(m_run[nt] - m_new);
          l_run[nt] *= rr;
          if (VBIAS) pv_run[nt] *= rr;
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
          if (VBIAS) pv_run[nt] = fmaf(p1, sct[c][1].z, fmaf(p0, sct[c][0].z, pv_run[nt]));
          float ws2 = p0 * sct[c][0].w + p1 * sct[c][1].w;
          ws2 += __shfl_xor_sync(0xffffffffu, ws2, 4);
          ws2 += __shfl_xor_sync(0xffffffffu, ws2, 8);
          ws2 += __shfl_xor_sync(0xffffffffu, ws2, 16);
          wsum[c][nt] = ws2;
          float h0, l0, h1, l1;
          split_h(p0 * sct[c][0].z, h0, l0);
          split_h(p1 * sct[c][1].z, h1, l1);
          const uint32_t X0 = pack_h2(h0, l0);
          const uint32_t X1 = pack_h2(h1, l1);
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

      // ---- V side: accumulate P' . codewords on tensor cores -----------------
      // A = codewords^T [channel][token] straight from the gather table with
      // ldmatrix.trans (each lane one 16-byte codeword row; replica slot =
      // row in the 8x8 matrix, so every phase is conflict-free); m-tile mt =
      // channels 16 mt .. 16 mt + 15 (subs 2 mt, 2 mt + 1), k = the warp's
      // 16 tokens.  Value-page sign words are stored in this fragment order
      // (encode.cu): word 8 i + c = component c of token pair (2i, 2i+1).
#pragma unroll
      for (int c = 0; c < CP; ++c) {
        if (!C::ONE_TABLE && c >= cnt) break;
        const uint32_t vpa = smem_u32(st + c * 2 * C::MAIN + C::MAIN);
        const uint4 iw = lds128(vpa + L.idx + (16 * ws + vT) * NSUB);
        uint32_t sw0 = 0, sw1 = 0;
        if (FOLD) {
          sw0 = lds32(vpa + (FOLD ? L.sgn : 0) + ((8 * ws + t) * 8 + g) * 4);
          sw1 = lds32(vpa + (FOLD ? L.sgn : 0) + ((8 * ws + 4 + t) * 8 + g) * 4);
        }
        const uint32_t iwv[4] = {iw.x, iw.y, iw.z, iw.w};
#pragma unroll
        for (int mt = 0; mt < 8; ++mt) {
          const uint32_t a = prmt(iwv[mt >> 1], lbv, (mt & 1) ? vselB : vselA);
          uint32_t x[4], y[4] = {0u, 0u, 0u, 0u};
          ldsm_x4_trans(a, x);
          if (HILO_V) ldsm_x4_trans(a + LO_OFS, y);
          if (FOLD) {
            const uint32_t m0 = sw0 << (15 - 2 * mt), m1 = sw0 << (14 - 2 * mt);
            const uint32_t m2 = sw1 << (15 - 2 * mt), m3 = sw1 << (14 - 2 * mt);
            x[0] = xor_sign(x[0], m0); x[1] = xor_sign(x[1], m1);
            x[2] = xor_sign(x[2], m2); x[3] = xor_sign(x[3], m3);
            if (HILO_V) {
              y[0] = xor_sign(y[0], m0); y[1] = xor_sign(y[1], m1);
              y[2] = xor_sign(y[2], m2); y[3] = xor_sign(y[3], m3);
            }
          }
#pragma unroll
          for (int nt = 0; nt < NTP; ++nt) {
            mma16816(accV[nt][mt], x[0], x[1], x[2], x[3], pf[c][nt][0], pf[c][nt][1]);
            if (HILO_V) mma16816(accV[nt][mt], y[0], y[1], y[2], y[3], pf[c][nt][0], pf[c][nt][1]);
          }
        }
        // value shift o' of the chunk: rows 16 mt + g, 16 mt + 8 + g
        const float *ovp = &SL.ov[c][16 * g];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 o4 = *reinterpret_cast<const float4 *>(ovp + 4 * q4);
#pragma unroll
          for (int nt = 0; nt < NTP; ++nt) {
            accV[nt][2 * q4][0] = fmaf(wsum[c][nt], o4.x, accV[nt][2 * q4][0]);
            accV[nt][2 * q4][2] = fmaf(wsum[c][nt], o4.y, accV[nt][2 * q4][2]);
            accV[nt][2 * q4 + 1][0] = fmaf(wsum[c][nt], o4.z, accV[nt][2 * q4 + 1][0]);
            accV[nt][2 * q4 + 1][2] = fmaf(wsum[c][nt], o4.w, accV[nt][2 * q4 + 1][2]);
          }
        }
      }
      // release the stage and the producer slot (scales, value shifts, TMEM D)
      tc05::fence_before();
      mbar_arrive(&BR.empty[s]);
      mbar_arrive(&BR.free_[grp][slot]);
    };

    if constexpr (!LUTK) {
    for (;; ++n) {
      if (!(cur.x < hi)) break;
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
      process_item();
      for (int a = 0; a < NGRP; ++a) item3_next<CP>(cur, hi, cv.n_chunks, n_units);
    }
    if (cur_unit >= 0) {
      flush_unit(cur_unit);
      mark_next = cur_unit + 1;
    }
    for (int u = mark_next; u <= last_unit; ++u) write_empty(u);
    } else {
    int lut_unit = first_unit - 1;  // last unit whose table transition this group ran
    for (;; ++n) {
      const bool have = cur.x < hi;
      const int next_u = have ? cur.u : last_unit + 1;
      if (next_u != cur_unit) {  // unit change (or the end of the range)
        if (cur_unit >= 0) {
          flush_unit(cur_unit);
          mark_next = cur_unit + 1;
        }
        for (int u = mark_next; u < next_u && u <= last_unit; ++u) write_empty(u);
        mark_next = next_u;
        // every group runs every unit's table transition, from this one call
        // site (named barriers), the skipped and the trailing units included
        if (LUTK)
          while (lut_unit < (next_u <= last_unit ? next_u : last_unit)) lut_transition(++lut_unit);
        if (!have) break;
        setup_unit(cur.u);
        cur_unit = cur.u;
      }
      process_item();
      for (int a = 0; a < NGRP; ++a) item3_next<CP>(cur, hi, cv.n_chunks, n_units);
    }
    }
  }

  tc05::fence_before();
  __syncthreads();
  if (warp == C::CW) {
    tc05::fence_after();
    tc05::dealloc(tmem, C::TMEM_COLS);
  }
}

}  // namespace nsnkv

using namespace nsnkv;


template <int G, bool FOLD, int PREC>
int nsnkv_launch_attend3(const CacheViewDev &cv, const float *q, float *out, float *lse,
                         float *recs, int64_t total, int grid, cudaStream_t st,
                         const AppendRows &add) {
  static unsigned long long attr = 0, attr_c = 0;
  set_smem_attr_once(attend3_kernel<G, FOLD, PREC>, ATT_SMEM_BYTES, attr);
  using C = A3<G, FOLD, PREC>;
  set_smem_attr_once(combine_kernel<G, C::NGRP, true>, (int)sizeof(CombineSmem), attr_c);
  int launches = 0;
  if (total > 0) {
    attend3_kernel<G, FOLD, PREC><<<grid, C::THREADS, ATT_SMEM_BYTES, st>>>(cv, q, recs, total);
    ++launches;
  }
  {  // programmatic dependent launch: the combine CTAs start (residual rows,
     // RoPE) while the attend kernel drains, then wait for its records
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(cv.batch * cv.n_kv_heads));
    lc.blockDim = dim3(COMBINE_THREADS);
    lc.dynamicSmemBytes = sizeof(CombineSmem);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = total > 0 ? 1 : 0;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, combine_kernel<G, C::NGRP, true>, cv, q, (const float *)recs,
                       (int64_t)(total > 0 ? total : 1), grid, out, lse, add.k, add.v, add.bf16,
                       add.n, add.n_res_out);
  }
  ++launches;
  nsnkv_internal_count_launch(launches);
  return nsnkv_internal_check_launch("decode_attend");
}

#define NSNKV_A3_INST(GG, FF, PP)                                                            \
  template int nsnkv_launch_attend3<GG, FF, PP>(const CacheViewDev &, const float *, float *, \
                                                float *, float *, int64_t, int, cudaStream_t,    \
                                                const AppendRows &);
#define NSNKV_A3_INST_G(GG) \
  NSNKV_A3_INST(GG, true, 0) NSNKV_A3_INST(GG, true, 1) NSNKV_A3_INST(GG, true, 2) \
  NSNKV_A3_INST(GG, false, 0) NSNKV_A3_INST(GG, false, 1) NSNKV_A3_INST(GG, false, 2)
NSNKV_A3_INST_G(1)
NSNKV_A3_INST_G(2)
NSNKV_A3_INST_G(4)
NSNKV_A3_INST_G(8)
NSNKV_A3_INST(4, false, 3)
