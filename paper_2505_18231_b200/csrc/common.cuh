// common.cuh -- shared constants, page layout and helpers for the sm_100a
// NSNQuant KV-cache kernels.  See DESIGN.md for the HBM layout rationale.
#pragma once

#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nsnkv_b200.h"

namespace nsnkv {

constexpr int D = NSNKV_HEAD_DIM;       // 128
constexpr int R = NSNKV_CHUNK;          // 64 tokens per chunk
constexpr int SUB = NSNKV_SUB_DIM;      // 8
constexpr int NSUB = D / SUB;           // 16 sub-vectors per token
constexpr int NPAIR = D / 2;            // 64 RoPE pairs
constexpr int NENT = 256;               // codebook entries

// ---------------------------------------------------------------------------
// Page layout (one 64-token chunk of one (batch, kv-head) unit).
//
//   [IDX]   u8  idx[64][16]          payload index per (token, sub-vector)
//   [SGN]   u32 sgn[64][4]           2-bit mode only; 128 sign bits per token,
//                                    bit-permuted for the decode fragments:
//                                    word q covers subs 4q+m (m = 0..3);
//                                    bit 4m+p      = sign bit 2p   of sub 4q+m
//                                    bit 16+4m+p   = sign bit 2p+1 of sub 4q+m
//   [S2]    f16 s2[64]               adjusted second scale (vq.py:254-259)
//   [S1N]   u8  s1 nibbles[32]       RTN-4 levels of s1, low nibble first
//   [ON]    u8  o nibbles[64]        RTN-4 levels of o, low nibble first
//   [PAR]   f16 s1_scale, s1_zero, o_scale[4], o_zero[4]
//
// Payload bytes = reference bit ledger (vq.py:328-356): 2292 / 1268.
// ---------------------------------------------------------------------------
struct PageLayout {
  int idx, sgn, s2, s1n, on, par, ledger, bytes;
};

__host__ __device__ constexpr PageLayout page_layout(int bit_mode) {
  return bit_mode == 2
             ? PageLayout{0, 1024, 2048, 2176, 2208, 2272, 2292, NSNKV_PAGE_BYTES_2B}
             : PageLayout{0, -1, 1024, 1152, 1184, 1248, 1268, NSNKV_PAGE_BYTES_1B};
}

// Device-side codebook tables (built once by nsnkv_codebook_create).
struct CodebookDev {
  float *entries;      // [256][8] fp32 (codebook.py active_entries)
  double *inv;         // [256] fp64 1/||e|| (kernels/__init__.py:44-51)
  // decode gather table (64 KB): row c = 256 bytes = [hi x 8 slots][lo x 8
  // slots], each slot the whole codeword as 8 fp16 (hi = fp16(e),
  // lo = fp16(e - hi)); 8 replicas so a quarter-warp of 16-byte loads with
  // slot = lane % 8 never bank-conflicts.
  uint4 *tabw;
  // encode search B operands for tcgen05.mma (16 KB, the shared-memory
  // image): normalized entries e_c / ||e_c|| split into fp16 hi + lo, two
  // K = 16 matrices [e_hi | e_hi] and [e_lo | e_lo] (row c), each in the
  // no-swizzle K-major canonical layout: byte (c / 8) * 256 + khalf * 128 +
  // (c % 8) * 16.
  uint4 *tcb;
  // mean over the 256 entries of the fp16 rounding error e - fp16(e), per
  // component: decode with plain-fp16 value codewords adds
  // (sum of the chunk weights) x dbar to every sub-vector of the output, so
  // the unsigned (1-bit) codewords' rounding leaves no bias that grows with
  // the context
  float dbar[8];
  int bit_mode;
};

// Small helpers -------------------------------------------------------------
__device__ __forceinline__ float bf16_to_f32(uint16_t h) {
  return __uint_as_float(uint32_t(h) << 16);
}

__device__ __forceinline__ float f16_bits_to_f32(uint16_t h) {
  return __half2float(__ushort_as_half(h));
}

__device__ __forceinline__ uint16_t f32_to_f16_bits(float x) {
  return __half_as_ushort(__float2half_rn(x));
}

// Set a kernel's dynamic shared-memory attributes once per DEVICE (not once
// per process: a process driving two GPUs must set it on each).  `done` is a
// per-kernel bitmask of device ordinals.
template <typename K>
inline void set_smem_attr_once(K kern, int bytes, unsigned long long &done, int carveout = -1) {
  int dev = 0;
  cudaGetDevice(&dev);
  const unsigned long long bit = 1ull << (dev & 63);
  if (__atomic_load_n(&done, __ATOMIC_ACQUIRE) & bit) return;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (carveout >= 0) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, carveout);
  __atomic_fetch_or(&done, bit, __ATOMIC_ACQ_REL);
}

}  // namespace nsnkv

// Launch bookkeeping shared by all translation units (capi.cu owns it).
extern "C" void nsnkv_internal_count_launch(int n);
extern "C" int nsnkv_internal_set_error(int code, const char *msg);
extern "C" int nsnkv_internal_check_launch(const char *what);
