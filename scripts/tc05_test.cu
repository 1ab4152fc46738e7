// tc05_test.cu -- checks the tcgen05 conventions the decode kernel relies on:
// A operand in TMEM (fp16 pairs packed along K per column), B in shared
// memory in the SWIZZLE_NONE K-major canonical layout, M=128 N=16 K=128 as 8
// MMAs, D read back with 32x32b and 16x256b loads.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I.. -o tc05_test tc05_test.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_fp16.h>
#include "../paper_2505_18231_b200/csrc/tc05.cuh"

using namespace nsnkv;
constexpr int M = 128, N = 16, K = 128;

__device__ long long g_cyc[4];
template <bool MN>
__global__ void k(const __half *A, const __half *B, float *out1, float *out2, uint32_t p_sb) {
  __shared__ __align__(1024) uint8_t bsm[K * N * 2];
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // B (K x N) into the canonical layout: element (n, k) at
  // kt*512 + (n/8)*256 + ((k%16)/8)*128 + (n%8)*16 + (k%8)*2
  for (int i = tid; i < K * N; i += blockDim.x) {
    const int kk = i / N, n = i % N;
    const int kt = kk / 16, kh = (kk % 16) / 8, k0 = kk % 8;
    if (MN)  // MN-major: element (k, n) at (k/8)*256 + (n/8)*128 + (k%8)*16 + (n%8)*2
      *reinterpret_cast<__half *>(bsm + (kk / 8) * 256 + (n / 8) * 128 + k0 * 16 + (n % 8) * 2) = B[i];
    else
      *reinterpret_cast<__half *>(bsm + kt * 512 + (n / 8) * 256 + kh * 128 + (n % 8) * 16 + k0 * 2) = B[i];
  }
  if (warp == 0) {
    tc05::alloc((uint32_t)__cvta_generic_to_shared(&tbase), 128);
    tc05::relinquish();
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc05::fence_proxy_async();
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  const uint32_t tb = tbase;
  // A rows into TMEM: lane = row, column c = (A[row][2c], A[row][2c+1])
  {
    const int row = 32 * warp + lane;
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t r[16];
      for (int c = 0; c < 16; ++c) {
        __half2 h = __halves2half2(A[row * K + 2 * (c0 + c)], A[row * K + 2 * (c0 + c) + 1]);
        r[c] = *reinterpret_cast<uint32_t *>(&h);
      }
      tc05::st_32x32b_x16(tb + ((uint32_t)(32 * warp) << 16) + 16 + c0, r);
    }
    tc05::wait_st();
  }
  tc05::fence_before();
  __syncthreads();
  tc05::fence_after();
  if (tid == 0) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(bsm);
    // issue cost of 16 back-to-back MMAs (accumulating into column 64.. so
    // the checked result below is unaffected), then time to completion
    {
      const long long c0 = clock64();
      for (int kt = 0; kt < 16; ++kt)
        tc05::mma_f16_ts(tb + 96, tb + 16 + 8 * (kt & 7),
                         MN ? tc05::smem_desc(sb + 512 * (kt & 7), 256, 128) : tc05::smem_desc(sb + 512 * (kt & 7), 128, 256),
                         tc05::idesc_f16(M, N) | (MN ? (1u << 16) : 0u), kt > 0);
      const long long c1 = clock64();
      tc05::commit((uint32_t)__cvta_generic_to_shared(&bar));
      asm volatile(
          "{\n\t.reg .pred p;\n\tW0:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, 1000000;\n\t"
          "@!p bra W0;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar))
          : "memory");
      const long long c2 = clock64();
      g_cyc[0] = c1 - c0;
      g_cyc[1] = c2 - c0;
    }
    if (sb == p_sb && tb == 0) {  // operands provably uniform: kernel parameter + constants
      const long long c0 = clock64();
#pragma unroll
      for (int kt = 0; kt < 16; ++kt)
        tc05::mma_f16_ts(96, 16 + 8 * (kt & 7),
                         MN ? tc05::smem_desc(p_sb + 512 * (kt & 7), 256, 128) : tc05::smem_desc(p_sb + 512 * (kt & 7), 128, 256),
                         tc05::idesc_f16(M, N) | (MN ? (1u << 16) : 0u), kt > 0);
      const long long c1 = clock64();
      tc05::commit((uint32_t)__cvta_generic_to_shared(&bar));
      asm volatile(
          "{\n\t.reg .pred p;\n\tW1:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 1, 1000000;\n\t"
          "@!p bra W1;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar))
          : "memory");
      const long long c2 = clock64();
      g_cyc[2] = c1 - c0;
      g_cyc[3] = c2 - c0;
    } else {
      g_cyc[2] = -1; g_cyc[3] = (long long)sb * 1000000 + tb;
    }
    for (int kt = 0; kt < 8; ++kt)
      tc05::mma_f16_ts(tb + 0, tb + 16 + 8 * kt,
                       MN ? tc05::smem_desc(sb + 512 * kt, 256, 128) : tc05::smem_desc(sb + 512 * kt, 128, 256),
                       tc05::idesc_f16(M, N) | (MN ? (1u << 16) : 0u), kt > 0);
    tc05::commit((uint32_t)__cvta_generic_to_shared(&bar));
  }
  asm volatile(
      "{\n\t.reg .pred p;\n\tW:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0, 1000000;\n\t"
      "@!p bra W;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar))
      : "memory");
  tc05::fence_after();
  {
    uint32_t r[16];
    tc05::ld_32x32b_x16(tb + ((uint32_t)(32 * warp) << 16), r);
    tc05::wait_ld();
    for (int c = 0; c < 16; ++c) out1[(32 * warp + lane) * N + c] = __uint_as_float(r[c]);
  }
  {
    const int g = lane >> 2, t = lane & 3;
    for (int half = 0; half < 2; ++half)
      for (int cb = 0; cb < 2; ++cb) {
        float r[4];
        tc05::ld_16x256b(tb + ((uint32_t)(32 * warp + 16 * half) << 16) + 8 * cb, r);
        tc05::wait_ld();
        const int row0 = 32 * warp + 16 * half + g;
        out2[row0 * N + 8 * cb + 2 * t] = r[0];
        out2[row0 * N + 8 * cb + 2 * t + 1] = r[1];
        out2[(row0 + 8) * N + 8 * cb + 2 * t] = r[2];
        out2[(row0 + 8) * N + 8 * cb + 2 * t + 1] = r[3];
      }
  }
  tc05::fence_before();
  __syncthreads();
  if (warp == 0) tc05::dealloc(tb, 128);
}

int main() {
  __half *hA = (__half *)malloc(M * K * 2), *hB = (__half *)malloc(K * N * 2);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = __float2half((rand() % 2001 - 1000) / 1000.f);
  for (int i = 0; i < K * N; ++i) hB[i] = __float2half((rand() % 2001 - 1000) / 1000.f);
  __half *dA, *dB;
  float *d1, *d2;
  cudaMalloc(&dA, M * K * 2);
  cudaMalloc(&dB, K * N * 2);
  cudaMalloc(&d1, M * N * 4);
  cudaMalloc(&d2, M * N * 4);
  cudaMemcpy(dA, hA, M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, K * N * 2, cudaMemcpyHostToDevice);
  for (int mn = 0; mn < 2; ++mn) {
  cudaMemset(d2, 0xff, M * N * 4);
  unsigned sbh = (unsigned)atoi(getenv("SB") ? getenv("SB") : "1024");
  if (mn) k<true><<<1, 128>>>(dA, dB, d1, d2, sbh); else k<false><<<1, 128>>>(dA, dB, d1, d2, sbh);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  float o1[M * N], o2[M * N];
  cudaMemcpy(o1, d1, sizeof(o1), cudaMemcpyDeviceToHost);
  cudaMemcpy(o2, d2, sizeof(o2), cudaMemcpyDeviceToHost);
  double e1 = 0, e2 = 0, mx = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int kk = 0; kk < K; ++kk) ref += (double)__half2float(hA[m * K + kk]) * __half2float(hB[kk * N + n]);
      e1 = fmax(e1, fabs(ref - o1[m * N + n]));
      e2 = fmax(e2, fabs(ref - o2[m * N + n]));
      mx = fmax(mx, fabs(ref));
    }
  long long cyc[4];
  cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(cyc));
  printf("16 MMA (M128 N16 K16, A tmem): issue %lld cycles, issue+complete %lld cycles; uniform operands: issue %lld, +complete %lld\n", cyc[0], cyc[1], cyc[2], cyc[3]);
  printf("%s max|ref| %.3f  err(32x32b) %.3e  err(16x256b) %.3e  %s\n", mn ? "MN-major" : "K-major", mx, e1, e2,
         (e1 < 1e-3 && e2 < 1e-3) ? "PASS" : "FAIL");
  }
  return 0;
}
