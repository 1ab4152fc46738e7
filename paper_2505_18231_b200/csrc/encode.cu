// encode.cu -- fused chunk flush: Normalize -> Shift -> Normalize, RoPE at
// absolute positions (keys), fast Walsh-Hadamard transform (keys), exact
// codebook search with the codebook in shared memory, scale adjustment,
// 4-bit double quantization of s1 / o and bit-packing into one page.
//
// Reference (pkg/src/nsnkv): kvcache.py:114-154 (flush_chunk_keys/values),
// nsn.py:58-85, core.py:50-66, rope.py:35-51, _native.pyx:16-38,
// codebook.py:109-128, vq.py:74-93, vq.py:100-166, vq.py:211-279.
//
// One CTA (256 threads) per 64-token chunk.  All arithmetic that defines the
// reference's outputs is reproduced operation by operation (IEEE fp32
// divides, no FMA contraction where the reference rounds products, fp64 sums
// in numpy's pairwise order), so pages are bit-identical to the oracle's.
#include "common.cuh"
#include "decode_att.cuh"
#include "match.cuh"
#include "tc05.cuh"

namespace nsnkv {

constexpr int ENC_THREADS = 256;
// TMEM columns per CTA for the codebook search: one round of the search
// scores 128 sub-vectors against ENC_NCOL entries (tcgen05.mma M = 128,
// N = ENC_NCOL), so 256 / ENC_NCOL rounds cover the codebook; at most
// 512 / ENC_NCOL CTAs share an SM's tensor memory.
#ifndef ENC_NCOL
#define ENC_NCOL 128
#endif
// resident CTAs per SM the register budget is sized for: the phases of a
// chunk are separated by block barriers, so more CTAs keep the SM busy while
// others wait (bounded by shared memory and the TMEM budget above)
#ifndef ENC_MIN_BLOCKS
#define ENC_MIN_BLOCKS 3
#endif
static_assert(ENC_MIN_BLOCKS * ENC_NCOL <= 512, "TMEM oversubscribed");
constexpr int XS = D + 4;  // padded smem row stride (floats)

struct EncodeSmem {
  float x[R][XS];                 // working rows
  __align__(128) uint16_t tcb[2 * NENT * 16];  // search B operands (CodebookDev::tcb image)
  __align__(128) uint16_t atile[2][128 * 16];  // search A operands (double-buffered): 128 sub-vectors [u_hi | u_lo]
  __align__(16) float ent[NENT * 8];
  double inv[NENT];
  float2 rec[2][128];             // per column half: best score, index | near-tie flag
  float s1[R], s2[R];
  __align__(16) float o[D];
  uint16_t zmask[R];              // zero sub-vectors per token (bit j)
  float s2adj[R];
  __align__(16) uint8_t idx[R][NSUB];
  __align__(16) uint8_t sgn[R][NSUB];
  int cnt[NSNKV_NUM_COUNTERS];
  uint64_t mbar;                  // tcgen05.commit -> search rounds
  uint64_t tbar;                  // bulk copies of the codebook tables
  uint32_t tmem_base;
};

// _scale_per_token (nsn.py:58-65) on every row of s.x (minus `shift` per
// column when given); returns clamps.
// Warp w owns rows w + 8 i (i = 0..7), lane l elements 4l..4l+3 of each.
// The fp64 sum of squares follows exactly the order of warp_row_sumsq (lane
// partial, then the xor tree 16, 8, 4, 2, 1; the oracle restates it), but
// the eight rows are reduced together by recursive halving: at each level a
// lane keeps half of its rows and adds the partner's partials of them (the
// same pairwise sums as the butterfly), so after three levels lane l holds
// row (l >> 2)'s tree and the norm, scale and clamp are computed once per
// row.  The division v / sc is exact: RN32((double)v * RN64(1 / sc)) is
// RN32(v / sc) because the fp64 product is within 2^-52 of the quotient and a
// quotient of two binary32 numbers is never closer than 2^-49 (relative) to a
// binary32 rounding boundary.
__device__ int scale_rows(EncodeSmem &s, float *scale_out, const float *shift = nullptr) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float sqrt_d = 11.313708498984761f;  // float32(sqrt(128))
  constexpr int NR = R / (ENC_THREADS / 32);  // 8 rows per warp
  float4 v[NR];
  double p[NR];
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    v[i] = *reinterpret_cast<float4 *>(&s.x[warp + 8 * i][4 * lane]);
    if (shift) {  // column shift first (the rows are rewritten below)
      const float4 o4 = *reinterpret_cast<const float4 *>(shift + 4 * lane);
      v[i].x = __fsub_rn(v[i].x, o4.x);
      v[i].y = __fsub_rn(v[i].y, o4.y);
      v[i].z = __fsub_rn(v[i].z, o4.z);
      v[i].w = __fsub_rn(v[i].w, o4.w);
    }
    const double a = v[i].x, b = v[i].y, c = v[i].z, d = v[i].w;
    double q = a * a;  // products of binary32 values are exact in fp64
    q = __fma_rn(b, b, q);
    q = __fma_rn(c, c, q);
    p[i] = __fma_rn(d, d, q);
  }
  const int bA = (lane >> 4) & 1, bB = (lane >> 3) & 1, bC = (lane >> 2) & 1;
  double q4[4], q2[2];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const double keep = bA ? p[4 + k] : p[k], send = bA ? p[k] : p[4 + k];
    q4[k] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 16));
  }
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const double keep = bB ? q4[2 + k] : q4[k], send = bB ? q4[k] : q4[2 + k];
    q2[k] = __dadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, 8));
  }
  double ss = __dadd_rn(bC ? q2[1] : q2[0], __shfl_xor_sync(0xffffffffu, bC ? q2[0] : q2[1], 4));
  ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, 2));
  ss = __dadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, 1));
  // this lane's row: i* = 4 bA + 2 bB + bC (= lane >> 2)
  const float nrm = __fsqrt_rn(__double2float_rn(ss));  // row_norms, core.py:50-53
  float sc = __fdiv_rn(nrm, sqrt_d);
  int clamps = 0;
  if (sc < 1e-8f) {  // NORM_EPS clamp, nsn.py:61-64
    sc = 1e-8f;
    clamps = (lane & 3) == 0 ? 1 : 0;
  }
  if ((lane & 3) == 0) scale_out[warp + 8 * (lane >> 2)] = sc;
  const double y = __drcp_rn((double)sc);
#pragma unroll
  for (int i = 0; i < NR; ++i) {
    const double yi = __shfl_sync(0xffffffffu, y, 4 * i);
    float4 w = v[i];
    w.x = __double2float_rn(__dmul_rn((double)w.x, yi));
    w.y = __double2float_rn(__dmul_rn((double)w.y, yi));
    w.z = __double2float_rn(__dmul_rn((double)w.z, yi));
    w.w = __double2float_rn(__dmul_rn((double)w.w, yi));
    *reinterpret_cast<float4 *>(&s.x[warp + 8 * i][4 * lane]) = w;
  }
  return clamps;
}

// In-warp FWHT of one 128-row held 4-per-lane (fp32 add/sub only), then the
// single orthonormal scale multiply (_native.pyx:24-37).
__device__ __forceinline__ float4 warp_fwht128(float4 v) {
  const int lane = threadIdx.x & 31;
  // h = 1
  float a = __fadd_rn(v.x, v.y), b = __fsub_rn(v.x, v.y);
  float c = __fadd_rn(v.z, v.w), d = __fsub_rn(v.z, v.w);
  // h = 2
  v.x = __fadd_rn(a, c);
  v.z = __fsub_rn(a, c);
  v.y = __fadd_rn(b, d);
  v.w = __fsub_rn(b, d);
#pragma unroll
  for (int m = 1; m < 32; m <<= 1) {  // h = 4m
    const float ox = __shfl_xor_sync(0xffffffffu, v.x, m);
    const float oy = __shfl_xor_sync(0xffffffffu, v.y, m);
    const float oz = __shfl_xor_sync(0xffffffffu, v.z, m);
    const float ow = __shfl_xor_sync(0xffffffffu, v.w, m);
    // the "y" half (lane & m) takes o - v, the "x" half v + o: one FMA with
    // an exact +-1 product is the same single rounding as the add / sub
    const float sg = (lane & m) ? -1.0f : 1.0f;
    v.x = __fmaf_rn(sg, v.x, ox);
    v.y = __fmaf_rn(sg, v.y, oy);
    v.z = __fmaf_rn(sg, v.z, oz);
    v.w = __fmaf_rn(sg, v.w, ow);
  }
  const float sc = 0.08838834764831845f;  // float32(1/sqrt(128))
  v.x = __fmul_rn(v.x, sc);
  v.y = __fmul_rn(v.y, sc);
  v.z = __fmul_rn(v.z, sc);
  v.w = __fmul_rn(v.w, sc);
  return v;
}

// RTN-4 with f16 parameters (vq.py:100-117, 155-166) on n values held one
// per thread of the first n threads of a group; lo/hi come in exact.
__device__ __forceinline__ void rtn4_params(float lo, float hi, uint16_t &scale16,
                                            uint16_t &zero16, float &scale32f, float &zero32f) {
  const float sc = (hi == lo) ? 1.0f : __fdiv_rn(__fsub_rn(hi, lo), 15.0f);
  scale16 = f32_to_f16_bits(sc);
  zero16 = f32_to_f16_bits(lo);
  scale32f = f16_bits_to_f32(scale16);
  zero32f = f16_bits_to_f32(zero16);
}

__device__ __forceinline__ uint32_t rtn4_level(float v, float zero32f, float scale32f) {
  float lv = rintf(__fdiv_rn(__fsub_rn(v, zero32f), scale32f));  // np.rint: half-even
  if (!(lv == lv)) lv = 0.f;  // NaN (scale16 == 0): the reference leaves this undefined
  lv = fminf(fmaxf(lv, 0.f), 15.f);
  return (uint32_t)lv;
}

// 4 consecutive elements of a fp32 or bf16 row buffer as fp32 (bf16 -> fp32
// is exact)
__device__ __forceinline__ float4 load_row4(const void *base, int64_t off, int bf16) {
  if (bf16) {
    const uint2 raw = *reinterpret_cast<const uint2 *>(static_cast<const uint16_t *>(base) + off);
    return make_float4(bf16_to_f32((uint16_t)(raw.x & 0xffffu)), bf16_to_f32((uint16_t)(raw.x >> 16)),
                       bf16_to_f32((uint16_t)(raw.y & 0xffffu)), bf16_to_f32((uint16_t)(raw.y >> 16)));
  }
  return *reinterpret_cast<const float4 *>(static_cast<const float *>(base) + off);
}

// Where one chunk's 64 stream rows come from (kvcache.py:179-186): stream row
// i of the unit is res[i] for i < n_resid, else fresh row i - n_resid, the
// fresh rows of the unit being fresh[r * fresh_stride] (fp32 or bf16).
struct ChunkSrc {
  const float *res;      // the unit's residual rows [64][128] (fp32)
  int n_resid;
  const void *fresh;     // the unit's first fresh row
  int64_t fresh_stride;  // elements between consecutive fresh rows
  int fresh_bf16;
  int k;                 // chunk index within this flush (stream rows 64 k ..)
  int64_t pos_base;      // absolute position of the chunk's first token
  uint8_t *page;         // destination page
  int32_t *cnt_out;      // NSNKV_NUM_COUNTERS event counts, or nullptr
  // after the rows are gathered (so the old residual is no longer read):
  // copy res_n fresh rows starting at fresh row res_from into res_dst
  float *res_dst;
  int res_from, res_n;
};

template <bool FOLD>
__device__ __forceinline__ void encode_chunk(EncodeSmem &s, const ChunkSrc &J, int is_key,
                                             const float2 *__restrict__ rope_cs, int64_t rope_pos0,
                                             int64_t rope_n, const CodebookDev &cb, int strategy) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const PageLayout L = page_layout(FOLD ? 2 : 1);
  constexpr bool fold = FOLD;
  const int k = J.k;

  if (tid < NSNKV_NUM_COUNTERS) s.cnt[tid] = 0;
  // codebook tables by bulk copy (TMA engine), overlapping the row gather;
  // TMEM for the search scores
  if (warp == 0) {
    tc05::alloc(smem_u32(&s.tmem_base), ENC_NCOL);
    tc05::relinquish();
    if (lane == 0) {
      mbar_init(&s.mbar, 1);
      mbar_init(&s.tbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&s.tbar, (uint32_t)(sizeof(s.tcb) + sizeof(s.ent) + sizeof(s.inv)));
      tma_load_1d(s.tcb, cb.tcb, sizeof(s.tcb), &s.tbar);
      tma_load_1d(s.ent, cb.entries, sizeof(s.ent), &s.tbar);
      tma_load_1d(s.inv, cb.inv, sizeof(s.inv), &s.tbar);
    }
  }
  // ---- 1. gather the chunk's 64 stream rows (kvcache.py:179-186) ----------
  // (every load of the thread issued before the first store: one exposed
  // memory latency per chunk)
  {
    const int c4 = tid & 31;
    float4 v[R * (D / 4) / ENC_THREADS];
#pragma unroll
    for (int n = 0; n < R * (D / 4) / ENC_THREADS; ++n) {
      const int t = (tid >> 5) + (ENC_THREADS / 32) * n;
      const int64_t srow = (int64_t)k * R + t;
      v[n] = srow < J.n_resid ? *reinterpret_cast<const float4 *>(J.res + srow * D + 4 * c4)
                              : load_row4(J.fresh, (srow - J.n_resid) * J.fresh_stride + 4 * c4,
                                          J.fresh_bf16);
    }
#pragma unroll
    for (int n = 0; n < R * (D / 4) / ENC_THREADS; ++n)
      *reinterpret_cast<float4 *>(&s.x[(tid >> 5) + (ENC_THREADS / 32) * n][4 * c4]) = v[n];
  }
  __syncthreads();
  if (J.res_dst) {  // the unit's new residual rows (its old ones are in s.x now)
    for (int i = tid; i < J.res_n * (D / 4); i += ENC_THREADS) {
      const int t = i / (D / 4), c4 = i - t * (D / 4);
      *reinterpret_cast<float4 *>(J.res_dst + (int64_t)t * D + 4 * c4) =
          load_row4(J.fresh, (int64_t)(J.res_from + t) * J.fresh_stride + 4 * c4, J.fresh_bf16);
    }
  }

  // ---- 2. nsn_forward (nsn.py:68-85) --------------------------------------
  int clamps = scale_rows(s, s.s1);
  __syncthreads();
  if (tid < D) {  // col_means: fp64 sequential sum over tokens / n (core.py:56-66)
    double acc = 0.0;
    for (int t = 0; t < R; ++t) acc = __dadd_rn(acc, (double)s.x[t][tid]);
    s.o[tid] = __double2float_rn(__ddiv_rn(acc, (double)R));
  }
  __syncthreads();
  clamps += scale_rows(s, s.s2, s.o);  // v_ns = v_n - o (nsn.py:80), then s2
  __syncthreads();

  // ---- 3. keys: RoPE at absolute positions, then FWHT (kvcache.py:121-123)
  if (is_key) {
    const int64_t pos_base = J.pos_base;
    for (int t = warp; t < R; t += ENC_THREADS / 32) {
      int64_t row = pos_base + t - rope_pos0;
      row = row < 0 ? 0 : (row >= rope_n ? rope_n - 1 : row);
      float4 v = *reinterpret_cast<float4 *>(&s.x[t][4 * lane]);
      const float4 cs = *reinterpret_cast<const float4 *>(&rope_cs[row * NPAIR + 2 * lane]);
      // pair j = 2*lane: (v.x, v.y) ; pair j+1: (v.z, v.w); rope.py:49-50
      float4 r;
      r.x = __fsub_rn(__fmul_rn(v.x, cs.x), __fmul_rn(v.y, cs.y));
      r.y = __fadd_rn(__fmul_rn(v.x, cs.y), __fmul_rn(v.y, cs.x));
      r.z = __fsub_rn(__fmul_rn(v.z, cs.z), __fmul_rn(v.w, cs.w));
      r.w = __fadd_rn(__fmul_rn(v.z, cs.w), __fmul_rn(v.w, cs.z));
      r = warp_fwht128(r);
      *reinterpret_cast<float4 *>(&s.x[t][4 * lane]) = r;
    }
    __syncthreads();
  }

  // ---- 4. codebook match (codebook.py:109-128, _native.pyx:41-87) -------
  // (a) sign bytes and zero rows, one thread per (token, 4 sub-vectors)
  {
    const int tt = tid >> 2, j0 = (tid & 3) * 4;
    uint32_t zm = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      float v[8], u[8];
      const float4 a = *reinterpret_cast<float4 *>(&s.x[tt][8 * (j0 + i)]);
      const float4 b = *reinterpret_cast<float4 *>(&s.x[tt][8 * (j0 + i) + 4]);
      v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
      v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
      // codebook.py:118-120 zero test; a component of magnitude >= 1e-11 puts
      // the (nonnegative, monotonically rounded) fp64 sum of squares above
      // 1e-22, so the exact pairwise sum is only needed below that
      float mx = fmaxf(fmaxf(fabsf(v[0]), fabsf(v[1])), fmaxf(fabsf(v[2]), fabsf(v[3])));
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v[4]), fabsf(v[5])), fmaxf(fabsf(v[6]), fabsf(v[7]))));
      const bool zero = !(mx >= 1e-11f) && sq_norm8_pairwise(v) < 1e-24;
      const uint32_t sb = fold_signs(v, u, FOLD);
      s.sgn[tt][j0 + i] = zero ? 0 : (uint8_t)sb;
      zm |= (zero ? 1u : 0u) << (j0 + i);
    }
    // the four threads of a token combine their zero bits
    zm |= __shfl_xor_sync(0xffffffffu, zm, 1);
    zm |= __shfl_xor_sync(0xffffffffu, zm, 2);
    if ((tid & 3) == 0) {
      s.zmask[tt] = (uint16_t)zm;
      if (zm) atomicAdd(&s.cnt[NSNKV_CNT_ZERO], __popc(zm));
    }
    // token tt belongs to warp tt / 8, which also decides its sub-vectors below
    __syncwarp();
  }
  // (b) codebook search on the 5th-gen tensor cores.  A tile = the 128
  // sub-vectors of 8 tokens (row r = token 8 tile + r / 16, sub r % 16).
  // Thread r (and r + 128) writes row r of the A operand [u_hi | u_lo] (fp16
  // split of u = |v| or v) to shared memory; one thread issues, per round,
  //   D[r][j] = [u_hi | u_lo] . [e_hi | e_hi]_c + [u_hi | u_lo] . [e_lo | e_lo]_c
  // (two tcgen05.mma, M = 128, N = ENC_NCOL, K = 16; c = ENC_NCOL round + j)
  // into TMEM, i.e. u . e_c / ||e_c|| with an error below 2^-19 ||u||
  // (fp16 hi + lo operands, fp32 accumulation).  Thread r (TMEM lane r)
  // then scans its half of the columns in 32-column segments, two passes
  // over the registers of one tcgen05.ld: the segment maximum m, then
  // the count and position of the entries >= m - bound.  Segments merge by
  // their maxima; a sub-vector whose best entry is not alone within `bound`
  // (4 x 2^-17 ||u||, twice the pair error) is a near tie and is re-scored
  // exactly in fp64 (the reference loop).  No top-2 tracking and no index
  // packing: about 2.5 instructions per (sub-vector, entry).
  mbar_wait(&s.tbar, 0);
  int slow = 0;
  {
    constexpr int ROUNDS = NENT / ENC_NCOL;
    constexpr int NTILE = R / 8;
    constexpr uint32_t IDESC = tc05::idesc_f16(128, ENC_NCOL);  // A, B K-major
    const int r_row = tid & 127;   // A row written and TMEM lane read by this thread
    const int chalf = tid >> 7;    // components 4 chalf.. of the A row / column half scanned
    const uint32_t b_s = smem_u32(s.tcb);
    const uint32_t t_lane = s.tmem_base + ((uint32_t)(32 * (warp & 3)) << 16);
    uint32_t mma_phase = 0;
    // A operand of tile `tile` into buffer `buf`: this thread converts
    // components 4 chalf .. 4 chalf + 3 of row r_row into fp16 hi (K 0..7)
    // and lo (K 8..15) halves; returns ||v||^2 of the row (fp32)
    auto build_a = [&](int tile, int buf) -> float {
      const int tau = 8 * tile + (r_row >> 4), sub = r_row & 15;
      const float4 a = *reinterpret_cast<const float4 *>(&s.x[tau][8 * sub]);
      const float4 b = *reinterpret_cast<const float4 *>(&s.x[tau][8 * sub + 4]);
      float n2 = 0.f;
      n2 = fmaf(a.x, a.x, n2); n2 = fmaf(a.y, a.y, n2); n2 = fmaf(a.z, a.z, n2); n2 = fmaf(a.w, a.w, n2);
      n2 = fmaf(b.x, b.x, n2); n2 = fmaf(b.y, b.y, n2); n2 = fmaf(b.z, b.z, n2); n2 = fmaf(b.w, b.w, n2);
      const float4 m = chalf ? b : a;
      const float u0 = FOLD ? fabsf(m.x) : m.x, u1 = FOLD ? fabsf(m.y) : m.y;
      const float u2 = FOLD ? fabsf(m.z) : m.z, u3 = FOLD ? fabsf(m.w) : m.w;
      const __half2 h01 = __floats2half2_rn(u0, u1), h23 = __floats2half2_rn(u2, u3);
      const float2 f01 = __half22float2(h01), f23 = __half22float2(h23);
      const __half2 l01 = __floats2half2_rn(u0 - f01.x, u1 - f01.y);
      const __half2 l23 = __floats2half2_rn(u2 - f23.x, u3 - f23.y);
      const uint32_t dst = smem_u32(s.atile[buf]) +
                           (uint32_t)((r_row >> 3) * 256 + (r_row & 7) * 16 + chalf * 8);
      asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(dst),
                   "r"(*reinterpret_cast<const uint32_t *>(&h01)),
                   "r"(*reinterpret_cast<const uint32_t *>(&h23)));
      asm volatile("st.shared.v2.u32 [%0], {%1,%2};" ::"r"(dst + 128u),
                   "r"(*reinterpret_cast<const uint32_t *>(&l01)),
                   "r"(*reinterpret_cast<const uint32_t *>(&l23)));
      return n2;
    };
    auto issue = [&](int buf, int rnd) {
      if (tid == 0) {
        tc05::fence_after();
        const uint64_t ad = tc05::smem_desc(smem_u32(s.atile[buf]), 128, 256);
        const uint32_t bo = (uint32_t)rnd * (ENC_NCOL * 32);
        tc05::mma_f16_ss(s.tmem_base, ad, tc05::smem_desc(b_s + bo, 128, 256), IDESC, 0);
        tc05::mma_f16_ss(s.tmem_base, ad, tc05::smem_desc(b_s + NENT * 32 + bo, 128, 256), IDESC, 1);
        tc05::commit(smem_u32(&s.mbar));
      }
    };
    // scan this thread's columns of round `rnd` in 32-column segments
    auto scan = [&](int rnd, float bound, float &M, int &bidx, bool &near) {
      mbar_wait(&s.mbar, mma_phase);
      mma_phase ^= 1u;
      tc05::fence_after();
#pragma unroll 1
      for (int sg = 0; sg < ENC_NCOL / 64; ++sg) {
        const int col0 = (ENC_NCOL / 2) * chalf + 32 * sg;
        uint32_t xv[32];
        tc05::ld_32x32b_x32(t_lane + (uint32_t)col0, xv);
        tc05::wait_ld();
        float mq[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          mq[q] = fmaxf(__uint_as_float(xv[q]), __uint_as_float(xv[q + 4]));
#pragma unroll
          for (int j = q + 8; j < 32; j += 8)
            mq[q] = fmaxf(mq[q], fmaxf(__uint_as_float(xv[j]), __uint_as_float(xv[j + 4])));
        }
        const float m = fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3]));
        const float thr = m - bound;
        int ac2[4] = {0, 0, 0, 0};  // four chains: count << 8 | sum of positions
#pragma unroll
        for (int j = 0; j < 32; ++j)  // one compare + one predicated add per entry
          asm("{\n\t.reg .pred p;\n\tsetp.ge.f32 p, %1, %2;\n\t@p add.s32 %0, %0, %3;\n\t}"
              : "+r"(ac2[j & 3])
              : "f"(__uint_as_float(xv[j])), "f"(thr), "r"(256 + j));
        const int acc = (ac2[0] + ac2[1]) + (ac2[2] + ac2[3]);
        const bool nr = (acc >> 8) != 1;
        const int ix = rnd * ENC_NCOL + col0 + (acc & 255);
        if (m > M) {
          near = nr || M >= m - bound;
          M = m;
          bidx = ix;
        } else {
          near = near || m >= M - bound;
        }
      }
    };

    float n2 = build_a(0, 0);
    tc05::fence_proxy_async();
    __syncthreads();
    issue(0, 0);
#pragma unroll 1
    for (int tile = 0; tile < NTILE; ++tile) {
      const int buf = tile & 1;
      const int tau = 8 * tile + (r_row >> 4), sub = r_row & 15;
      const float bound = 3.0517578e-05f * sqrtf(n2);  // 4 x 2^-17 ||u||
      float M = -INFINITY;
      int bidx = 0;
      bool near = false;
      float n2_next = 0.f;
#pragma unroll 1
      for (int rnd = 0; rnd < ROUNDS; ++rnd) {
        if (rnd) {
          tc05::fence_before();
          __syncthreads();  // every thread read the previous round's scores
          issue(buf, rnd);
        }
        if (rnd == ROUNDS - 1 && tile + 1 < NTILE) {  // next tile's A while the MMA runs
          n2_next = build_a(tile + 1, buf ^ 1);
          tc05::fence_proxy_async();
        }
        scan(rnd, bound, M, bidx, near);
      }
      s.rec[chalf][r_row] = make_float2(M, __int_as_float(bidx | (near ? 0x10000 : 0)));
      tc05::fence_before();
      __syncthreads();  // records complete; scores read; next A complete
      if (tile + 1 < NTILE) issue(buf ^ 1, 0);  // next tile's first round under the merge
      uint32_t need = 0;
      if (tid < 128) {
        const float2 A = s.rec[0][r_row], B = s.rec[1][r_row];
        const int ia = __float_as_int(A.y), ib = __float_as_int(B.y);
        bool nr;
        int ix;
        float best;
        if (B.x > A.x) {
          nr = (ib >> 16) || A.x >= B.x - bound;
          ix = ib & 0xffff;
          best = B.x;
        } else {
          nr = (ia >> 16) || B.x >= A.x - bound;
          ix = ia & 0xffff;
          best = A.x;
        }
        uint8_t res = 0;
        if (!((s.zmask[tau] >> sub) & 1u)) {
          if (n2 > 1e-24f && n2 < 1e30f && !nr && fabsf(best) > 1e-30f)
            res = (uint8_t)ix;
          else
            need = 1;
        }
        s.idx[tau][sub] = res;
      }
      // near ties: the whole warp re-scores one sub-vector at a time exactly
      // in fp64 (the reference loop: component-order sum, times inv[c],
      // strict '>' from -1e300 so the lowest index wins ties); lane l scores
      // entries l, l + 32, ..., then an argmax butterfly, lower index on ties
      if (warp < 4) {
        for (uint32_t pend = __ballot_sync(0xffffffffu, need != 0); pend; pend &= pend - 1) {
          const int src = __ffs(pend) - 1;
          const int rr = 32 * warp + src;
          const int tau2 = 8 * tile + (rr >> 4), sub2 = rr & 15;
          double ud[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const float v = s.x[tau2][8 * sub2 + k];
            ud[k] = (double)((FOLD && v < 0.f) ? -v : v);
          }
          double bs = -1e300;
          int bc = 0;
#pragma unroll 2
          for (int i = 0; i < NENT / 32; ++i) {
            const int c = 32 * i + lane;
            const float4 e0 = *reinterpret_cast<const float4 *>(&s.ent[8 * c]);
            const float4 e1 = *reinterpret_cast<const float4 *>(&s.ent[8 * c + 4]);
            double sc = __dmul_rn(ud[0], (double)e0.x);
            sc = __dadd_rn(sc, __dmul_rn(ud[1], (double)e0.y));
            sc = __dadd_rn(sc, __dmul_rn(ud[2], (double)e0.z));
            sc = __dadd_rn(sc, __dmul_rn(ud[3], (double)e0.w));
            sc = __dadd_rn(sc, __dmul_rn(ud[4], (double)e1.x));
            sc = __dadd_rn(sc, __dmul_rn(ud[5], (double)e1.y));
            sc = __dadd_rn(sc, __dmul_rn(ud[6], (double)e1.z));
            sc = __dadd_rn(sc, __dmul_rn(ud[7], (double)e1.w));
            sc = __dmul_rn(sc, s.inv[c]);
            if (sc > bs) {
              bs = sc;
              bc = c;
            }
          }
#pragma unroll
          for (int off = 16; off >= 1; off >>= 1) {
            const double os = __shfl_xor_sync(0xffffffffu, bs, off);
            const int oc = __shfl_xor_sync(0xffffffffu, bc, off);
            if (os > bs || (os == bs && oc < bc)) {
              bs = os;
              bc = oc;
            }
          }
          if (lane == src) {
            s.idx[tau2][sub2] = (uint8_t)bc;
            ++slow;
          }
        }
      }
      n2 = n2_next;
    }
  }
  if (slow) atomicAdd(&s.cnt[NSNKV_CNT_NEARTIE], slow);
  if (clamps) atomicAdd(&s.cnt[NSNKV_CNT_CLAMP], clamps);
  tc05::fence_before();
  __syncthreads();
  if (warp == 0) {
    tc05::fence_after();
    tc05::dealloc(s.tmem_base, ENC_NCOL);
  }

  // ---- 5. scale adjustment (vq.py:74-93, 249-254) --------------------------
  {
    // 4 tokens per warp pass; lane = 8 * token_slot + accumulator j.
    const int slot = lane >> 3, j = lane & 7;
    for (int t0 = warp * 4; t0 < R; t0 += (ENC_THREADS / 32) * 4) {
      const int t = t0 + slot;
      double v2 = 0.0, q2 = 0.0, dt = 0.0;
      const uint4 iw = *reinterpret_cast<const uint4 *>(&s.idx[t][0]);
      const uint4 sw = *reinterpret_cast<const uint4 *>(&s.sgn[t][0]);
      const uint32_t iws[4] = {iw.x, iw.y, iw.z, iw.w}, sws[4] = {sw.x, sw.y, sw.z, sw.w};
#pragma unroll
      for (int i = 0; i < NSUB; ++i) {  // element 8i + j; numpy pairwise_sum order
        const float v = s.x[t][8 * i + j];
        const uint32_t ci = (iws[i >> 2] >> (8 * (i & 3))) & 0xffu;
        float c = s.ent[ci * 8 + j];
        if (fold)  // _SIGN_LUT, codebook.py:49: flip where sign bit j of the byte is set
          c = __uint_as_float(__float_as_uint(c) ^ (((sws[i >> 2] >> (8 * (i & 3) + j)) & 1u) << 31));
        const double vd = (double)v, cd = (double)c;
        if (i == 0) {  // products of binary32 values are exact in fp64: fma == mul + add
          v2 = vd * vd; q2 = cd * cd; dt = vd * cd;
        } else {
          v2 = __fma_rn(vd, vd, v2);
          q2 = __fma_rn(cd, cd, q2);
          dt = __fma_rn(vd, cd, dt);
        }
      }
#pragma unroll
      for (int off = 1; off <= 4; off <<= 1) {
        v2 = __dadd_rn(v2, __shfl_xor_sync(0xffffffffu, v2, off));
        q2 = __dadd_rn(q2, __shfl_xor_sync(0xffffffffu, q2, off));
        dt = __dadd_rn(dt, __shfl_xor_sync(0xffffffffu, dt, off));
      }
      if (j == 0) {
        double f = 1.0;
        int fb = 0;
        if (strategy == NSNKV_STRATEGY_MIN_L2) {
          f = __ddiv_rn(dt, q2);
        } else if (strategy == NSNKV_STRATEGY_NORM_MATCH) {
          f = __dsqrt_rn(__ddiv_rn(v2, q2));
        } else if (strategy == NSNKV_STRATEGY_PARALLEL) {
          const bool bad = fabs(dt) <= __dmul_rn(1e-10, __dsqrt_rn(__dmul_rn(v2, q2)));
          f = bad ? __dsqrt_rn(__ddiv_rn(v2, q2)) : __ddiv_rn(v2, dt);
          fb = bad ? 1 : 0;
        }
        s.s2adj[t] = __double2float_rn(__dmul_rn((double)s.s2[t], f));
        if (fb) atomicAdd(&s.cnt[NSNKV_CNT_FALLBACK], 1);
      }
    }
  }
  __syncthreads();

  // ---- 6. pack the page ----------------------------------------------------
  uint8_t *page = J.page;
  // indices: 1024 bytes, 4 per thread
  {
    const uint32_t w = *reinterpret_cast<const uint32_t *>(&s.idx[0][0] + 4 * tid);
    *reinterpret_cast<uint32_t *>(page + L.idx + 4 * tid) = w;
  }
  if (fold && is_key) {  // key signs, decode K order: word q of token t covers subs 4q..4q+3
    const int t = tid >> 2, q = tid & 3;
    uint32_t w = 0;
#pragma unroll
    for (int m = 0; m < 4; ++m) {
      const uint32_t b = s.sgn[t][4 * q + m];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        w |= ((b >> (2 * p)) & 1u) << (4 * m + p);
        w |= ((b >> (2 * p + 1)) & 1u) << (16 + 4 * m + p);
      }
    }
    *reinterpret_cast<uint32_t *>(page + L.sgn + 4 * tid) = w;
  } else if (fold) {  // value signs, decode V order: word 8 i + c = component c of
    // token pair (2i, 2i+1); bit j = token 2i, sub j; bit 16 + j = token 2i+1
    const int i = tid >> 3, c = tid & 7;
    uint32_t w = 0;
#pragma unroll
    for (int j = 0; j < NSUB; ++j) {
      w |= ((uint32_t)(s.sgn[2 * i][j] >> c) & 1u) << j;
      w |= ((uint32_t)(s.sgn[2 * i + 1][j] >> c) & 1u) << (16 + j);
    }
    *reinterpret_cast<uint32_t *>(page + L.sgn + 4 * tid) = w;
  }
  // s2 (f16, vq.py:259), s1 and o double quantization (vq.py:257-258)
  if (warp == 0) {
    // s1: one group of 64 values; lane holds tokens lane and lane + 32
    const float a = s.s1[lane], b = s.s1[lane + 32];
    float lo = fminf(a, b), hi = fmaxf(a, b);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    uint16_t sc16, z16;
    float sc32, z32;
    rtn4_params(lo, hi, sc16, z16, sc32, z32);
    const uint32_t la = rtn4_level(a, z32, sc32), lb = rtn4_level(b, z32, sc32);
    // nibble pairs: byte i = level[2i] | level[2i+1] << 4
    const uint32_t la_next = __shfl_down_sync(0xffffffffu, la, 1);
    const uint32_t lb_next = __shfl_down_sync(0xffffffffu, lb, 1);
    if ((lane & 1) == 0) {
      page[L.s1n + lane / 2] = (uint8_t)(la | (la_next << 4));
      page[L.s1n + 16 + lane / 2] = (uint8_t)(lb | (lb_next << 4));
    }
    if (lane == 0) {
      uint16_t *par = reinterpret_cast<uint16_t *>(page + L.par);
      par[0] = sc16;
      par[1] = z16;
    }
  } else if (warp >= 1 && warp <= 4) {
    // o: group g = warp - 1 covers channels 32g .. 32g+31
    const int g = warp - 1;
    const float v = s.o[32 * g + lane];
    float lo = v, hi = v;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, off));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, off));
    }
    uint16_t sc16, z16;
    float sc32, z32;
    rtn4_params(lo, hi, sc16, z16, sc32, z32);
    const uint32_t lv = rtn4_level(v, z32, sc32);
    const uint32_t lv_next = __shfl_down_sync(0xffffffffu, lv, 1);
    if ((lane & 1) == 0) page[L.on + 16 * g + lane / 2] = (uint8_t)(lv | (lv_next << 4));
    if (lane == 0) {
      uint16_t *par = reinterpret_cast<uint16_t *>(page + L.par);
      par[2 + g] = sc16;
      par[6 + g] = z16;
    }
  } else if (warp == 5) {
    uint16_t *s2p = reinterpret_cast<uint16_t *>(page + L.s2);
    s2p[lane] = f32_to_f16_bits(s.s2adj[lane]);
    s2p[lane + 32] = f32_to_f16_bits(s.s2adj[lane + 32]);
  } else if (warp == 6) {
    // zero the page padding so pages are deterministic byte images
    for (int i = L.ledger + lane; i < L.bytes; i += 32) page[i] = 0;
  }
  if (J.cnt_out && tid < NSNKV_NUM_COUNTERS) J.cnt_out[tid] = s.cnt[tid];
}

// nsnkv_encode_chunks: chunk k of unit u per CTA, every unit flushing n_flush
template <bool FOLD>
__global__ void __launch_bounds__(ENC_THREADS, ENC_MIN_BLOCKS) encode_chunks_kernel(
    const float *__restrict__ residual, int n_resid, const void *__restrict__ fresh, int fresh_bf16,
    int64_t n_fresh, int n_flush, int is_key, const int64_t *__restrict__ start_pos,
    const float2 *__restrict__ rope_cs, int64_t rope_pos0, int64_t rope_n, CodebookDev cb,
    int strategy, uint8_t *__restrict__ pool, const int32_t *__restrict__ page_ids,
    int page_id_stride, int32_t *__restrict__ counters) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EncodeSmem &s = *reinterpret_cast<EncodeSmem *>(smem_raw);
  const int u = blockIdx.x / n_flush;
  const int k = blockIdx.x - u * n_flush;
  const PageLayout L = page_layout(FOLD ? 2 : 1);
  ChunkSrc J;
  J.res = residual + (int64_t)u * R * D;
  J.n_resid = n_resid;
  J.fresh_bf16 = fresh_bf16;
  J.fresh = fresh_bf16 ? (const void *)(static_cast<const uint16_t *>(fresh) + (int64_t)u * n_fresh * D)
                       : (const void *)(static_cast<const float *>(fresh) + (int64_t)u * n_fresh * D);
  J.fresh_stride = D;
  J.k = k;
  J.pos_base = is_key ? start_pos[u] + (int64_t)k * R : 0;
  J.page = pool + (int64_t)page_ids[(int64_t)u * page_id_stride + k] * L.bytes;
  J.cnt_out = counters ? counters + (int64_t)blockIdx.x * NSNKV_NUM_COUNTERS : nullptr;
  J.res_dst = nullptr;
  J.res_from = J.res_n = 0;
  encode_chunk<FOLD>(s, J, is_key, rope_cs, rope_pos0, rope_n, cb, strategy);
}

}  // namespace nsnkv

using namespace nsnkv;

extern "C" int nsnkv_internal_codebook_dev(const nsnkv_codebook *cb, CodebookDev *out);

extern "C" int nsnkv_encode_chunks(const float *residual, int32_t n_resid, const void *fresh,
                                   int32_t fresh_bf16, int64_t n_fresh, int32_t n_units,
                                   int32_t n_flush, int32_t is_key, const int64_t *start_pos,
                                   const float *rope_cs, int64_t rope_pos0, int64_t rope_n,
                                   const nsnkv_codebook *cb, int32_t strategy, uint8_t *pool,
                                   const int32_t *page_ids, int32_t page_id_stride,
                                   int32_t *counters, void *stream) {
  if (n_units < 0 || n_flush < 0 || n_resid < 0 || n_resid > R || n_fresh < 0)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "encode_chunks: bad sizes");
  if ((int64_t)n_flush * R > (int64_t)n_resid + n_fresh)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "encode_chunks: not enough rows to flush");
  if (strategy < 0 || strategy > 3)
    return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "encode_chunks: unknown strategy");
  if ((int64_t)n_units * n_flush == 0) return NSNKV_OK;
  if (is_key && (!rope_cs || rope_n <= 0))
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "encode_chunks: keys need a RoPE table");
  CodebookDev dev;
  int rc = nsnkv_internal_codebook_dev(cb, &dev);
  if (rc) return rc;
  const size_t smem = sizeof(EncodeSmem);
  static unsigned long long attr_k = 0, attr_v = 0;
  set_smem_attr_once(encode_chunks_kernel<true>, (int)smem, attr_k, 100);
  set_smem_attr_once(encode_chunks_kernel<false>, (int)smem, attr_v, 100);
  const int64_t blocks = (int64_t)n_units * n_flush;
  auto kern = dev.bit_mode == 2 ? encode_chunks_kernel<true> : encode_chunks_kernel<false>;
  kern<<<(unsigned)blocks, ENC_THREADS, smem, (cudaStream_t)stream>>>(
      residual, n_resid, fresh, fresh_bf16, n_fresh, n_flush, is_key, start_pos,
      reinterpret_cast<const float2 *>(rope_cs), rope_pos0, rope_n, dev, strategy, pool, page_ids,
      page_id_stride, counters);
  nsnkv_internal_count_launch(1);
  return nsnkv_internal_check_launch("encode_chunks");
}

// ---------------------------------------------------------------------------
// nsnkv_append: one launch per append of any shape (uniform or per-unit
// token counts): every full chunk of every unit is flushed into the page the
// caller allocated for it, the new residual rows are written, and the page
// table and per-unit counters are updated on the device (kvcache.py:157-195).
// two launches (keys, then values), grid n_units * max(max_flush, 1); CTA (u, k):
//   k < n_flush[u]          encode chunk k of the unit's stream into
//                           new_pages[u][k]; k == 0 also writes the new
//                           residual rows (after gathering the old ones)
//   k == 0, n_flush[u] == 0 append the fresh rows to the residual
// Counters are double-buffered (in -> out) so no CTA reads a value another
// CTA of the same launch writes; the kind-0 CTA with k == 0 owns them.
// ---------------------------------------------------------------------------
template <bool FOLD, int KIND>
__global__ void __launch_bounds__(ENC_THREADS, ENC_MIN_BLOCKS)
    append_kernel(nsnkv_append_args a, CodebookDev cb) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  EncodeSmem &s = *reinterpret_cast<EncodeSmem *>(smem_raw);
  const int fmax = a.max_flush > 0 ? a.max_flush : 1;
  const int u = blockIdx.x / fmax, k = blockIdx.x - u * fmax;
  constexpr int kind = KIND;  // 0 keys, 1 values
  const int n_res = a.n_res_in[u], n_ch = a.n_chunks_in[u];
  const int64_t n_new = a.new_count ? (int64_t)a.new_count[u] : a.n_new_uniform;
  const int64_t off = a.fresh_off ? a.fresh_off[u] : (int64_t)u * a.n_new_uniform;
  const int n_flush = (int)((n_res + n_new) / R);
  const int64_t stride = a.fresh_row_stride * D;  // elements between a unit's fresh rows
  const void *fresh = kind ? a.fresh_v : a.fresh_k;
  const void *fresh_u = a.fresh_bf16 ? (const void *)(static_cast<const uint16_t *>(fresh) + off * D)
                                     : (const void *)(static_cast<const float *>(fresh) + off * D);
  float *res = (kind ? a.v_res : a.k_res) + (int64_t)u * R * D;
  const int new_res = (int)(n_res + n_new - (int64_t)n_flush * R);
  if (k < n_flush) {
    const PageLayout L = page_layout(FOLD ? 2 : 1);
    const int32_t pid = a.new_pages[(int64_t)u * a.max_flush + k];
    ChunkSrc J;
    J.res = res;
    J.n_resid = n_res;
    J.fresh = fresh_u;
    J.fresh_stride = stride;
    J.fresh_bf16 = a.fresh_bf16;
    J.k = k;
    J.pos_base = a.base_pos[u] + (int64_t)(n_ch + k) * R;
    J.page = (kind ? a.v_pool : a.k_pool) + (int64_t)pid * L.bytes;
    J.cnt_out = a.counters ? a.counters + ((int64_t)pid * 2 + kind) * NSNKV_NUM_COUNTERS : nullptr;
    J.res_dst = k == 0 ? res : nullptr;
    J.res_from = (int)((int64_t)n_flush * R - n_res);
    J.res_n = new_res;
    encode_chunk<FOLD>(s, J, kind == 0, reinterpret_cast<const float2 *>(a.rope_cs), a.rope_pos0,
                       a.rope_n, cb, a.strategy);
    if (kind == 0 && threadIdx.x == 0) a.page_table[(int64_t)u * a.page_table_stride + n_ch + k] = pid;
  } else if (k == 0) {  // no flush: the fresh rows join the residual
    for (int i = threadIdx.x; i < (int)n_new * (D / 4); i += ENC_THREADS) {
      const int t = i / (D / 4), c4 = i - t * (D / 4);
      *reinterpret_cast<float4 *>(res + (int64_t)(n_res + t) * D + 4 * c4) =
          load_row4(fresh_u, (int64_t)t * stride + 4 * c4, a.fresh_bf16);
    }
  }
  if (kind == 0 && k == 0 && threadIdx.x == 0) {
    a.n_chunks_out[u] = n_ch + n_flush;
    a.n_res_out[u] = new_res;
  }
}

extern "C" int nsnkv_append(const nsnkv_append_args *a, void *stream) {
  if (!a || a->n_units < 0 || a->max_flush < 0 || a->fresh_row_stride < 1)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "append: bad sizes");
  if (!a->n_res_in || !a->n_chunks_in || !a->n_res_out || !a->n_chunks_out || !a->k_res ||
      !a->v_res || !a->base_pos || (a->max_flush > 0 && (!a->new_pages || !a->page_table)))
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "append: null cache buffers");
  if (a->strategy < 0 || a->strategy > 3)
    return nsnkv_internal_set_error(NSNKV_ERR_UNSUPPORTED, "append: unknown strategy");
  if (a->max_flush > 0 && (!a->rope_cs || a->rope_n <= 0))
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "append: keys need a RoPE table");
  if (a->n_units == 0) return NSNKV_OK;
  CodebookDev ck, cv;
  int rc = nsnkv_internal_codebook_dev(a->cb_k, &ck);
  if (!rc) rc = nsnkv_internal_codebook_dev(a->cb_v, &cv);
  if (rc) return rc;
  if (ck.bit_mode != cv.bit_mode)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "append: codebook bit modes differ");
  const size_t smem = sizeof(EncodeSmem);
  static unsigned long long attr[4] = {0, 0, 0, 0};
  set_smem_attr_once(append_kernel<true, 0>, (int)smem, attr[0], 100);
  set_smem_attr_once(append_kernel<true, 1>, (int)smem, attr[1], 100);
  set_smem_attr_once(append_kernel<false, 0>, (int)smem, attr[2], 100);
  set_smem_attr_once(append_kernel<false, 1>, (int)smem, attr[3], 100);
  const int fmax = a->max_flush > 0 ? a->max_flush : 1;
  const unsigned grid = (unsigned)((int64_t)a->n_units * fmax);
  cudaStream_t st = (cudaStream_t)stream;
  // values first: the key launch owns the counters (double-buffered, so the
  // order does not matter for correctness)
  if (ck.bit_mode == 2) {
    append_kernel<true, 1><<<grid, ENC_THREADS, smem, st>>>(*a, cv);
    append_kernel<true, 0><<<grid, ENC_THREADS, smem, st>>>(*a, ck);
  } else {
    append_kernel<false, 1><<<grid, ENC_THREADS, smem, st>>>(*a, cv);
    append_kernel<false, 0><<<grid, ENC_THREADS, smem, st>>>(*a, ck);
  }
  nsnkv_internal_count_launch(2);
  return nsnkv_internal_check_launch("append");
}
