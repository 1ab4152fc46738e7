// tc05_rate.cu -- issue-to-completion time of 16 back-to-back tcgen05.mma
// kind::f16 (M = 128, K = 16 each) for several N, A from TMEM vs A from
// shared memory; one CTA, one issuing thread.  Decides how much shift-term
// work to batch per MMA instruction in the decode kernel.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tc05_rate tc05_rate.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2505_18231_b200/csrc/tc05.cuh"
using namespace nsnkv;

__device__ long long g_cyc[16];

__global__ void k() {
  extern __shared__ __align__(1024) uint8_t sm[];  // A (128 x 128 fp16) and B (up to 256 x 128)
  __shared__ uint32_t tbase;
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < (32768 + 65536) / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3c003c00u;
  if (warp == 0) {
    tc05::alloc((uint32_t)__cvta_generic_to_shared(&tbase), 512);
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
  if (tid == 0) {
    const uint32_t sa = (uint32_t)__cvta_generic_to_shared(sm), sbm = sa + 32768;
    uint32_t phase = 0;
    int slot = 0;
    for (int mode = 0; mode < 2; ++mode)
      for (int N = 16; N <= 256; N *= 2) {
        const uint32_t idesc = tc05::idesc_f16(128, N);
        const long long c0 = clock64();
        for (int kt = 0; kt < 16; ++kt) {
          const uint64_t bd = tc05::smem_desc(sbm + 256 * (kt & 7), 128, 256 * 8);
          if (mode == 0)
            tc05::mma_f16_ts(tb + 256, tb + 8 * (kt & 7), bd, idesc, kt > 0);
          else {
            const uint64_t ad = tc05::smem_desc(sa + 256 * (kt & 7), 128, 256 * 8);
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tb + 256),
                "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(kt > 0))
                : "memory");
          }
        }
        const long long c1 = clock64();
        tc05::commit((uint32_t)__cvta_generic_to_shared(&bar));
        asm volatile(
            "{\n\t.reg .pred p;\n\tW:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, 1000000;\n\t"
            "@!p bra W;\n\t}" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(phase)
            : "memory");
        phase ^= 1;
        const long long c2 = clock64();
        g_cyc[slot++] = (c1 - c0) * 100000 + (c2 - c0);
      }
  }
  tc05::fence_before();
  __syncthreads();
  if (warp == 0) tc05::dealloc(tb, 512);
}

int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 65536);
  k<<<1, 128, 32768 + 65536>>>();
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  long long c[16];
  cudaMemcpyFromSymbol(c, g_cyc, sizeof(c));
  int s = 0;
  for (int mode = 0; mode < 2; ++mode)
    for (int N = 16; N <= 256; N *= 2, ++s)
      printf("%s N=%3d: 16 MMA issue %5lld cycles, complete %5lld cycles (%.1f per MMA)\n",
             mode ? "A smem" : "A tmem", N, c[s] / 100000, c[s] % 100000, (c[s] % 100000) / 16.0);
  return 0;
}
