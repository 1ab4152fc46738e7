// microbench.cu -- B200 pipe rates that shape the decode kernel design:
// legacy mma.sync m16n8k16 (fp16 -> fp32) and m16n8k32 (e4m3, s8) issue
// rates per SM, conflict-free LDS.128 gathers, SHFL.  One CTA per SM,
// clock64() around an unrolled loop; prints cycles per instruction per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void hmma(float *d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void imma(int *d, uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                     uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int MODE>
__global__ void bench(long long *out, uint32_t seed, int iters) {
  extern __shared__ __align__(16) uint4 sm[];
  const int lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < 65536 / 16; i += blockDim.x) sm[i] = make_uint4(i, i * 3, i * 5, i * 7);
  __syncthreads();
  float acc[8][4] = {};
  int iacc[8][4] = {};
  uint32_t a = seed ^ lane, b = seed * 3 + lane;
  uint32_t x = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) {  // 8 independent HMMA chains
#pragma unroll
      for (int k = 0; k < 8; ++k) hmma(acc[k], a, b, a ^ k, b ^ k, a, b);
    } else if (MODE == 1) {  // IMMA
#pragma unroll
      for (int k = 0; k < 8; ++k) imma(iacc[k], a, b, a ^ k, b ^ k, a, b);
    } else if (MODE == 2) {  // conflict-free LDS.128 gathers (slot = lane % 8)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t idx = (a >> (k * 4)) & 255u;
        const uint4 v = sm[(idx * 16 + (lane & 7)) & 4095];
        x += v.x ^ v.y ^ v.z ^ v.w;
        a = a * 1664525u + v.x;
      }
    } else if (MODE == 3) {  // SHFL
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        x += __shfl_sync(0xffffffffu, a + k, (lane + k) & 31);
      }
      a += x;
    }
  }
  long long t1 = clock64();
  float s = 0.f;
  for (int k = 0; k < 8; ++k) s += acc[k][0] + acc[k][1] + acc[k][2] + acc[k][3] + iacc[k][0];
  if (s == 1.2345f || x == 7u) out[1] = 1;
  if (threadIdx.x == 0) out[blockIdx.x * 2] = t1 - t0;
}

int main() {
  long long *d;
  cudaMalloc(&d, 2 * 1024 * sizeof(long long));
  const char *names[] = {"HMMA.16816.F32 (per SM)", "IMMA.16832.S32 (per SM)",
                         "LDS.128 gather slot=lane%8 (per SM)", "SHFL (per SM)"};
  const int iters = 4096;
  for (int mode = 0; mode < 4; ++mode) {
    for (int warps : {4, 8, 12, 16}) {
      void (*k)(long long *, uint32_t, int) =
          mode == 0 ? bench<0> : mode == 1 ? bench<1> : mode == 2 ? bench<2> : bench<3>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
      k<<<148, warps * 32, 65536>>>(d, 12345u, 16);
      k<<<148, warps * 32, 65536>>>(d, 12345u, iters);
      cudaDeviceSynchronize();
      long long h[2];
      cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
      const double per = (double)h[0] / ((double)iters * 8 * warps);
      printf("%-40s warps=%2d  %.3f cycles/instr/SM\n", names[mode], warps, per);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
