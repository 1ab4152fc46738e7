// tma_rate.cu -- issue cost of 1-D bulk copies (cp.async.bulk global ->
// shared, mbarrier complete_tx) from one thread: 64 copies of S bytes,
// clock64 around the issue loop and to completion.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tma_rate tma_rate.cu
#include <cstdio>
#include <cstdint>

__device__ long long g_cyc[8][2];

__global__ void k(const uint8_t *src) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint32_t phase = 0;
    int slot = 0;
    for (int S = 256; S <= 4096; S *= 2, ++slot) {
      const int n = 64;
      const long long c0 = clock64();
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(n * S) : "memory");
      for (int i = 0; i < n; ++i) {
        const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + (i % 16) * 4096);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
            "l"(src + (size_t)(i * 7919 % 4096) * 8192), "r"(S), "r"(b)
            : "memory");
      }
      const long long c1 = clock64();
      asm volatile(
          "{\n\t.reg .pred p;\n\tW:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
          "@!p bra W;\n\t}" ::"r"(b), "r"(phase)
          : "memory");
      phase ^= 1;
      const long long c2 = clock64();
      g_cyc[slot][0] = c1 - c0;
      g_cyc[slot][1] = c2 - c0;
    }
  }
}

int main() {
  uint8_t *src;
  cudaMalloc(&src, (size_t)4096 * 8192);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
  k<<<1, 32, 65536>>>(src);
  k<<<1, 32, 65536>>>(src);
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  long long c[8][2];
  cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
  int s = 0;
  for (int S = 256; S <= 4096; S *= 2, ++s)
    printf("64 bulk copies of %4d B: issue %6lld cycles (%.1f per copy), complete %6lld\n", S, c[s][0],
           c[s][0] / 64.0, c[s][1]);
  return 0;
}
