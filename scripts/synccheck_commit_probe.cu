// Does compute-sanitizer synccheck model tcgen05.commit's mbarrier arrive?
// One CTA: init an mbarrier (count 1), allocate TMEM, issue tcgen05.commit
// onto the barrier (no MMA outstanding: it arrives at once), wait on it.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/probe scripts/synccheck_commit_probe.cu
// Run:   compute-sanitizer --tool synccheck /tmp/probe
#include <cstdio>
#include <cstdint>
__global__ void probe(int *out) {
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b)
                 : "memory");
  asm volatile(
      "{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(b)
      : "memory");
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tbase));
  if (threadIdx.x == 0) *out = 1;
}
int main() {
  int *d, h = 0;
  cudaMalloc(&d, 4);
  probe<<<1, 64>>>(d);
  cudaMemcpy(&h, d, 4, cudaMemcpyDeviceToHost);
  printf("probe %s (%d)\n", h == 1 ? "ok" : "FAILED", h);
  return 0;
}
