// V-side design microbenchmark (evidence for DESIGN.md §3.2 / §6): the cost per
// 64-token chunk, per SM, of accumulating softmax-weighted value codewords for
// the G = 4 q-heads of a unit, three ways:
//   hist_f32  north_star's codeword histogram: per (token, sub-vector, head) one
//             shared-memory fp32 atomicAdd into H[head][sub][entry] (4096 per
//             chunk), then the histogram x codebook product is off the hot path
//   hist_i32  the same with 32-bit fixed-point integer atomics (native ATOMS.ADD)
//   gather    the shipped kernel's way: ldmatrix.x4.trans gathers of fp16
//             codeword rows straight into mma.sync A fragments (8 per warp per
//             chunk for its 16 tokens) and one m16n8k16 per gather
// Each CTA (512 threads, 16 warps) processes `chunks` chunks with random
// codeword indices; 4 warps share a chunk like the decode consumers.  Times are
// CUDA-event totals over all SMs, reported as SM cycles per chunk.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/vside scripts/vside_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>

constexpr int NENT = 256, NSUB = 16, G = 4;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// 16 warps = 4 chunk-groups of 4 warps; warp w of a group owns tokens 16w..16w+15
__global__ void __launch_bounds__(512, 1) hist_f32(int chunks, float *sink) {
  extern __shared__ float H[];  // [G][NSUB][NENT] = 64 KB
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < G * NSUB * NENT; i += 512) H[i] = 0.f;
  __syncthreads();
  const int grp = warp >> 2, ws = warp & 3;
  for (int c = grp; c < chunks; c += 4) {
    // lane = (token 16 ws + lane / 2, subs 8 (lane & 1) .. +7)
    const int tok = 16 * ws + (lane >> 1);
    const uint32_t seed = hash32((uint32_t)(blockIdx.x * 7919 + c) * 131u + tok);
    const float w = 1.0f + (float)(seed & 255) * (1.0f / 256.0f);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int sub = 8 * (lane & 1) + s;
      const int e = (int)(hash32(seed + s) & 255u);
#pragma unroll
      for (int h = 0; h < G; ++h) atomicAdd(&H[(h * NSUB + sub) * NENT + e], w * (float)(h + 1));
    }
  }
  __syncthreads();
  if (tid == 0) sink[blockIdx.x] = H[blockIdx.x % (G * NSUB * NENT)];
}

__global__ void __launch_bounds__(512, 1) hist_i32(int chunks, float *sink) {
  extern __shared__ int Hi[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < G * NSUB * NENT; i += 512) Hi[i] = 0;
  __syncthreads();
  const int grp = warp >> 2, ws = warp & 3;
  for (int c = grp; c < chunks; c += 4) {
    const int tok = 16 * ws + (lane >> 1);
    const uint32_t seed = hash32((uint32_t)(blockIdx.x * 7919 + c) * 131u + tok);
    const int w = 65536 + (int)(seed & 255);
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      const int sub = 8 * (lane & 1) + s;
      const int e = (int)(hash32(seed + s) & 255u);
#pragma unroll
      for (int h = 0; h < G; ++h) atomicAdd(&Hi[(h * NSUB + sub) * NENT + e], w * (h + 1));
    }
  }
  __syncthreads();
  if (tid == 0) sink[blockIdx.x] = (float)Hi[blockIdx.x % (G * NSUB * NENT)];
}

__device__ __forceinline__ void ldsm_x4_trans(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// the shipped gather: table row c = 8 replicas of the 16-byte fp16 codeword
// (32 KB); lane supplies the row address of its (token, sub) for ldmatrix
__global__ void __launch_bounds__(512, 1) gather_mma(int chunks, float *sink) {
  extern __shared__ __align__(16) uint8_t T[];  // [NENT][8 slots][16 B]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < NENT * 8 * 4; i += 512)
    reinterpret_cast<uint32_t *>(T)[i] = 0x3c003c00u ^ (uint32_t)(i * 2654435761u & 0x00ff00ffu);
  __syncthreads();
  const uint32_t tb = (uint32_t)__cvta_generic_to_shared(T);
  const int grp = warp >> 2, ws = warp & 3;
  float acc[8][4] = {};
  const uint32_t pf0 = 0x3c003c00u, pf1 = 0x38003800u;  // weights (B operand)
  const int vT = (lane & 7) + 8 * (lane >> 4), vodd = (lane >> 3) & 1;
  for (int c = grp; c < chunks; c += 4) {
    const int tok = 16 * ws + vT;
    const uint32_t seed = hash32((uint32_t)(blockIdx.x * 7919 + c) * 131u + tok);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      const uint32_t e = hash32(seed + 2 * mt + vodd) & 255u;
      uint32_t x[4];
      ldsm_x4_trans(tb + e * 128u + (uint32_t)(lane & 7) * 16u, x);
      mma16816(acc[mt], x[0], x[1], x[2], x[3], pf0, pf1);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) s += acc[mt][0] + acc[mt][1] + acc[mt][2] + acc[mt][3];
  if (s == 12345.f) sink[blockIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  float *sink;
  cudaMalloc(&sink, sms * sizeof(float));
  const int chunks = 4096;  // per CTA
  cudaFuncSetAttribute(hist_f32, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(hist_i32, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  cudaFuncSetAttribute(gather_mma, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char *names[3] = {"hist_f32", "hist_i32", "gather"};
  for (int k = 0; k < 3; ++k) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (k == 0) hist_f32<<<sms, 512, 65536>>>(chunks, sink);
      if (k == 1) hist_i32<<<sms, 512, 65536>>>(chunks, sink);
      if (k == 2) gather_mma<<<sms, 512, 32768>>>(chunks, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 1)
        printf("%-9s %8.3f ms  %7.1f SM cycles per chunk (at %d MHz)\n", names[k], ms,
               ms * 1e-3 * clk_khz * 1e3 / chunks, clk_khz / 1000);
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
