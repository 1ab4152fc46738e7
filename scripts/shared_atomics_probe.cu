// atomicAdd on shared memory: u32, u64, f16x2, f32 (and red.shared forms).
#include <cuda_fp16.h>
__global__ void probe(unsigned *out, const int *idx, const unsigned *w, const float *wf) {
  __shared__ unsigned long long h64[2048];
  __shared__ unsigned h32[2048];
  __shared__ __half2 hh[2048];
  __shared__ float hf[2048];
  const int a = idx[threadIdx.x];
  const unsigned v = w[threadIdx.x];
  atomicAdd(&h32[a & 2047], v);                          // u32
  atomicAdd(&h64[a & 2047], (unsigned long long)v);      // u64
  atomicAdd(&hh[(a >> 3) & 2047], __halves2half2(__float2half(1.f), __float2half(2.f)));  // f16x2
  atomicAdd(&hf[(a >> 5) & 2047], wf[threadIdx.x]);      // f32
  __syncthreads();
  out[threadIdx.x] = h32[threadIdx.x] + (unsigned)h64[threadIdx.x] + *(unsigned *)&hh[threadIdx.x] +
                     __float_as_uint(hf[threadIdx.x]);
}
