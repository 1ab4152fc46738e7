// pool.cu -- growable page pools on CUDA virtual memory, and page copies.
//
// A pool reserves one large virtual address range up front and maps physical
// memory into it on demand (cuMemCreate + cuMemMap), so the page pools of a
// serving cache grow without copying a single page and every page keeps its
// device address (the page table indexes one base pointer).  The driver entry
// points are fetched through the runtime (cudaGetDriverEntryPoint), so the
// library has no link-time dependency on libcuda.
#include <cuda.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace {

struct Drv {
  CUresult (*reserve)(CUdeviceptr *, size_t, size_t, CUdeviceptr, unsigned long long) = nullptr;
  CUresult (*free_va)(CUdeviceptr, size_t) = nullptr;
  CUresult (*create)(CUmemGenericAllocationHandle *, size_t, const CUmemAllocationProp *,
                     unsigned long long) = nullptr;
  CUresult (*release)(CUmemGenericAllocationHandle) = nullptr;
  CUresult (*map)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle,
                  unsigned long long) = nullptr;
  CUresult (*unmap)(CUdeviceptr, size_t) = nullptr;
  CUresult (*set_access)(CUdeviceptr, size_t, const CUmemAccessDesc *, size_t) = nullptr;
  CUresult (*granularity)(size_t *, const CUmemAllocationProp *,
                          CUmemAllocationGranularity_flags) = nullptr;
  bool ok = false;
};

template <typename F>
bool entry(const char *name, F &fn) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !p)
    return false;
  fn = reinterpret_cast<F>(p);
  return true;
}

const Drv &drv() {
  static Drv d = [] {
    Drv x;
    x.ok = entry("cuMemAddressReserve", x.reserve) && entry("cuMemAddressFree", x.free_va) &&
           entry("cuMemCreate", x.create) && entry("cuMemRelease", x.release) &&
           entry("cuMemMap", x.map) && entry("cuMemUnmap", x.unmap) &&
           entry("cuMemSetAccess", x.set_access) &&
           entry("cuMemGetAllocationGranularity", x.granularity);
    return x;
  }();
  return d;
}

}  // namespace

struct nsnkv_pool {
  int device;
  CUdeviceptr base;
  size_t reserved, mapped, gran;
  std::vector<std::pair<CUmemGenericAllocationHandle, size_t>> chunks;  // (handle, bytes)
};

static int drv_err(const char *what, CUresult r) {
  char msg[160];
  snprintf(msg, sizeof(msg), "%s failed (CUresult %d)", what, (int)r);
  return nsnkv_internal_set_error(NSNKV_ERR_CUDA, msg);
}

extern "C" int nsnkv_pool_create(size_t reserve_bytes, nsnkv_pool **out) {
  if (!out || reserve_bytes == 0) return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "pool: bad size");
  const Drv &d = drv();
  if (!d.ok) return nsnkv_internal_set_error(NSNKV_ERR_CUDA, "pool: CUDA virtual memory API unavailable");
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nsnkv_internal_check_launch("pool: cudaGetDevice");
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = dev;
  size_t gran = 0;
  CUresult r = d.granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
  if (r != CUDA_SUCCESS || gran == 0) return drv_err("cuMemGetAllocationGranularity", r);
  const size_t res = (reserve_bytes + gran - 1) / gran * gran;
  CUdeviceptr base = 0;
  r = d.reserve(&base, res, gran, 0, 0);
  if (r != CUDA_SUCCESS) return drv_err("cuMemAddressReserve", r);
  nsnkv_pool *p = new nsnkv_pool{dev, base, res, 0, gran, {}};
  *out = p;
  return NSNKV_OK;
}

// map physical memory so that [0, bytes) of the pool is usable (grow-only;
// pages already mapped keep their addresses and contents)
extern "C" int nsnkv_pool_reserve(nsnkv_pool *p, size_t bytes) {
  if (!p) return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "pool: null");
  if (bytes <= p->mapped) return NSNKV_OK;
  if (bytes > p->reserved)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "pool: request exceeds the reserved address range");
  const Drv &d = drv();
  // grow by at least 1/8 of what is mapped, in whole granules
  size_t want = bytes - p->mapped;
  if (want < p->mapped / 8) want = p->mapped / 8;
  want = (want + p->gran - 1) / p->gran * p->gran;
  if (p->mapped + want > p->reserved) want = p->reserved - p->mapped;
  CUmemAllocationProp prop;
  memset(&prop, 0, sizeof(prop));
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  prop.location.id = p->device;
  CUmemGenericAllocationHandle h;
  CUresult r = d.create(&h, want, &prop, 0);
  if (r != CUDA_SUCCESS) return drv_err("cuMemCreate", r);
  r = d.map(p->base + p->mapped, want, 0, h, 0);
  if (r != CUDA_SUCCESS) {
    d.release(h);
    return drv_err("cuMemMap", r);
  }
  CUmemAccessDesc acc;
  memset(&acc, 0, sizeof(acc));
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = p->device;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  r = d.set_access(p->base + p->mapped, want, &acc, 1);
  if (r != CUDA_SUCCESS) {
    d.unmap(p->base + p->mapped, want);
    d.release(h);
    return drv_err("cuMemSetAccess", r);
  }
  p->chunks.emplace_back(h, want);
  p->mapped += want;
  return NSNKV_OK;
}

extern "C" void *nsnkv_pool_ptr(const nsnkv_pool *p) { return p ? (void *)p->base : nullptr; }
extern "C" size_t nsnkv_pool_mapped(const nsnkv_pool *p) { return p ? p->mapped : 0; }

extern "C" int nsnkv_pool_destroy(nsnkv_pool *p) {
  if (!p) return NSNKV_OK;
  const Drv &d = drv();
  cudaDeviceSynchronize();
  size_t off = 0;
  for (auto &c : p->chunks) {
    d.unmap(p->base + off, c.second);
    d.release(c.first);
    off += c.second;
  }
  d.free_va(p->base, p->reserved);
  delete p;
  return NSNKV_OK;
}

// pages ids[0..n) of a pool <-> a dense buffer of n pages (host or device):
// to_pool == 0 gathers pool pages into dst, to_pool != 0 scatters src into them
extern "C" int nsnkv_pages_copy(uint8_t *pool, int32_t page_bytes, const int32_t *ids_host,
                                int32_t n, uint8_t *buf, int32_t to_pool, void *stream) {
  if ((n > 0 && (!pool || !ids_host || !buf)) || page_bytes <= 0 || n < 0)
    return nsnkv_internal_set_error(NSNKV_ERR_SHAPE, "pages_copy: bad arguments");
  cudaStream_t st = (cudaStream_t)stream;
  for (int32_t i = 0; i < n;) {
    int32_t j = i + 1;  // coalesce runs of consecutive page ids
    while (j < n && ids_host[j] == ids_host[j - 1] + 1) ++j;
    uint8_t *pp = pool + (int64_t)ids_host[i] * page_bytes;
    uint8_t *bp = buf + (int64_t)i * page_bytes;
    const size_t bytes = (size_t)(j - i) * page_bytes;
    cudaError_t e = to_pool ? cudaMemcpyAsync(pp, bp, bytes, cudaMemcpyDefault, st)
                            : cudaMemcpyAsync(bp, pp, bytes, cudaMemcpyDefault, st);
    if (e != cudaSuccess) return nsnkv_internal_check_launch("pages_copy");
    i = j;
  }
  return NSNKV_OK;
}
