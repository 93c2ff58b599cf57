// Library-level entry points: version, status strings, pinned host registration,
// and the shared host helpers (tensor-map encoding, SM count).
#include <sys/mman.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstring>
#include <map>
#include <mutex>
#include <type_traits>
#include <algorithm>
#include <utility>

#include "common.cuh"

namespace {
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}
}  // namespace

bool ess_make_tmap_2d(CUtensorMap *m, CUtensorMapDataType dtype, const void *base,
                      uint64_t inner, uint64_t rows, uint64_t row_stride_bytes,
                      uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle swizzle) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {box_inner, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(m, dtype, 2, const_cast<void *>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Per-device state (a process may drive several GPUs, one stream per caller thread):
// the SM count and each kernel's dynamic shared-memory opt-in are per device.
int ess_sm_count() {
  constexpr int MAXDEV = 64;
  static int n[MAXDEV] = {};  // benign race: every writer stores the same value
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= MAXDEV) dev = 0;
  if (!n[dev]) {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
    n[dev] = v > 0 ? v : 148;
  }
  return n[dev];
}

int ess_smem_optin(const void *func, size_t bytes) {
  // no shortcut below 48 KB: the default dynamic limit is 48 KB minus the kernel's
  // static shared memory, so a kernel with large static storage needs the opt-in too
  if (bytes == 0) return ESS_OK;
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> done;  // (kernel, device) -> bytes
  int dev = 0;
  ESS_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  size_t &have = done[{func, dev}];
  if (have >= bytes) return ESS_OK;
  ESS_CUDA_TRY(cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  have = bytes;
  return ESS_OK;
}

int ess_preload_indexer();
int ess_preload_topk();
int ess_preload_pool();
int ess_preload_mla();
int ess_preload_mla2();

extern "C" {

const char *ess_version(void) { return "ess_b200 0.1 sm_100a"; }

// the host latent store row pitch this library was compiled with (the Python side
// lays the store out with its own constant and must agree)
int ess_host_row_pitch(void) { return ESS_HOST_ROW_PITCH; }

const char *ess_status_string(int status) {
  switch (status) {
    case ESS_OK: return "ok";
    case ESS_ERR_CAPACITY: return "capacity must be >= 1 and <= cap_max";
    case ESS_ERR_SHRINK: return "capacity may only grow";
    case ESS_ERR_DUPLICATE: return "duplicate generated entry id";
    case ESS_ERR_NOMEM: return "out of device memory";
    case ESS_ERR_RATIO: return "sparse_ratio must be in (0, 1]";
    case ESS_ERR_ARG: return "invalid argument (id out of range, request too long, bad size)";
    case ESS_ERR_CUDA: return "CUDA error";
    case ESS_ERR_CLOCK: return "recency clock exhausted";
    case ESS_ERR_RANGE: return "attention operand outside the f16 range (|x| >= 65520)";
    default: return "unknown status";
  }
}

// The host latent store: page-locked, mapped into the device address space so
// the gather kernel reads it with plain 16-B loads over PCIe (zero copy, UVA).
int ess_host_register(void *host_ptr, size_t bytes, void **d_alias) {
  if (!host_ptr || !bytes || !d_alias) return ESS_ERR_ARG;
  ESS_CUDA_TRY(cudaHostRegister(host_ptr, bytes, cudaHostRegisterMapped | cudaHostRegisterPortable));
  ESS_CUDA_TRY(cudaHostGetDevicePointer(d_alias, host_ptr, 0));
  return ESS_OK;
}

// Diagnostic: one thread writes the device's global nanosecond timer to *d_dst, in
// stream order (usable inside captured CUDA graphs, where events cannot be timed).
// Input staging: up to ESS_COPY_MAX device-to-device copies (16-B aligned, multiples of
// 16 B) in one grid-stride SM kernel.  The decode step's per-step inputs (q, q_idx, the
// generated rows) land in the captured graph's static buffers this way: as separate
// cudaMemcpyAsync copies they ran on the copy engine at ~0.4 TB/s plus a few us of
// latency each, serialised in front of every step (24 us of a 211-us C2 step).
struct CopyArgs {
  uint4 *dst[ESS_COPY_MAX];
  const uint4 *src[ESS_COPY_MAX];
  int64_t pref[ESS_COPY_MAX + 1];  // 16-B units before copy i
  int n;
};

__global__ void __launch_bounds__(256) copy_many_kernel(const __grid_constant__ CopyArgs a) {
  const int64_t total = a.pref[a.n];
  int c = 0;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < total;
       u += (int64_t)gridDim.x * blockDim.x) {
    while (u >= a.pref[c + 1]) c++;  // units are visited in increasing order per thread
    const int64_t o = u - a.pref[c];
    a.dst[c][o] = __ldg(a.src[c] + o);
  }
}

__global__ void timestamp_kernel(uint64_t *dst) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

int ess_copy_many(int32_t n, void *const *d_dst, const void *const *d_src, const int64_t *bytes,
                  void *stream) {
  if (n < 0 || n > ESS_COPY_MAX || (n && (!d_dst || !d_src || !bytes))) return ESS_ERR_ARG;
  CopyArgs a;
  a.n = n;
  a.pref[0] = 0;
  for (int i = 0; i < n; i++) {
    if (!d_dst[i] || !d_src[i] || bytes[i] < 0 || (bytes[i] & 15) ||
        (reinterpret_cast<uintptr_t>(d_dst[i]) & 15) || (reinterpret_cast<uintptr_t>(d_src[i]) & 15))
      return ESS_ERR_ARG;
    a.dst[i] = static_cast<uint4 *>(d_dst[i]);
    a.src[i] = static_cast<const uint4 *>(d_src[i]);
    a.pref[i + 1] = a.pref[i] + bytes[i] / 16;
  }
  if (n == 0 || a.pref[n] == 0) return ESS_OK;
  const int64_t want = (a.pref[n] + 255) / 256;
  const int grid = (int)(want < 4 * (int64_t)ess_sm_count() ? want : 4 * (int64_t)ess_sm_count());
  copy_many_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(a);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_timestamp(uint64_t *d_dst, void *stream) {
  if (!d_dst) return ESS_ERR_ARG;
  timestamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d_dst);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

// The host latent store, allocated here rather than by the caller: 2-MB aligned anonymous
// memory, transparent huge pages requested (madvise) so the GPU's zero-copy row reads
// walk few IOMMU / page-table entries across a multi-GB store, optionally bound to the
// GPU's NUMA node (mbind; one NUMA-local host pool per GPU), then
// page-locked and mapped into the device address space.
namespace {
constexpr size_t kHugePage = 2u << 20;
size_t host_span(size_t bytes) { return (bytes + kHugePage - 1) / kHugePage * kHugePage; }
}  // namespace

// ESS_HOST_VMM: the store as ONE host-located VMM allocation (cuMemCreate with a
// CU_MEM_LOCATION_TYPE_HOST_NUMA location, mapped at one VA for the device and the CPU).
// A cudaHostRegister'd store is mapped into the GPU's page tables in small pages, THP or
// not: random row reads across a multi-GB store then miss the SMs' translation caches,
// and the gather needs >= 48 SMs at 5.5 GiB (C4) to reach the rate 20 SMs reach at
// 1.4 GiB (scripts/gather_tlb.py).  The VMM allocation is mapped at its allocation
// granularity.
namespace {
struct VmmFns {
  decltype(&cuMemGetAllocationGranularity) gran = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) vfree = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) access = nullptr;
  bool ok = false;
};
const VmmFns &vmm_fns() {
  static VmmFns f;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char *name, auto &out) {
      void *p = nullptr;
      cudaDriverEntryPointQueryResult q;
      if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
          q == cudaDriverEntryPointSuccess)
        out = reinterpret_cast<std::remove_reference_t<decltype(out)>>(p);
      return out != nullptr;
    };
    f.ok = get("cuMemGetAllocationGranularity", f.gran) & get("cuMemCreate", f.create) &
           get("cuMemRelease", f.release) & get("cuMemAddressReserve", f.reserve) &
           get("cuMemAddressFree", f.vfree) & get("cuMemMap", f.map) & get("cuMemUnmap", f.unmap) &
           get("cuMemSetAccess", f.access);
  });
  return f;
}
struct VmmAlloc {
  CUmemGenericAllocationHandle h;
  size_t size;
};
std::mutex g_vmm_mu;
std::map<uintptr_t, VmmAlloc> g_vmm;  // VA -> allocation (ess_host_free tells the two kinds apart)

int vmm_alloc(size_t bytes, int32_t numa_node, void **ptr, size_t *mapped) {
  const VmmFns &f = vmm_fns();
  if (!f.ok) return ESS_ERR_CUDA;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return ESS_ERR_CUDA;
  cudaFree(nullptr);  // the runtime's primary context is current for the driver calls
  CUmemAllocationProp prop = {};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  prop.location.id = numa_node >= 0 ? numa_node : 0;
  size_t g = 0;
  if (f.gran(&g, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !g) return ESS_ERR_CUDA;
  const size_t size = (bytes + g - 1) / g * g;
  CUmemGenericAllocationHandle h;
  if (f.create(&h, size, &prop, 0) != CUDA_SUCCESS) return ESS_ERR_NOMEM;
  CUdeviceptr va = 0;
  if (f.reserve(&va, size, std::max<size_t>(g, kHugePage), 0, 0) != CUDA_SUCCESS) {
    f.release(h);
    return ESS_ERR_CUDA;
  }
  CUmemAccessDesc acc[2] = {};
  acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc[0].location.id = dev;
  acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  acc[1].location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;  // the CPU fills / writes back rows
  acc[1].location.id = prop.location.id;
  acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (f.map(va, size, 0, h, 0) != CUDA_SUCCESS) {
    f.vfree(va, size);
    f.release(h);
    return ESS_ERR_CUDA;
  }
  if (f.access(va, size, acc, 2) != CUDA_SUCCESS) {
    f.unmap(va, size);
    f.vfree(va, size);
    f.release(h);
    return ESS_ERR_CUDA;
  }
  {
    std::lock_guard<std::mutex> l(g_vmm_mu);
    g_vmm[(uintptr_t)va] = {h, size};
  }
  *ptr = reinterpret_cast<void *>(va);
  *mapped = size;
  return ESS_OK;
}

bool vmm_free(void *p) {
  VmmAlloc a;
  {
    std::lock_guard<std::mutex> l(g_vmm_mu);
    auto it = g_vmm.find((uintptr_t)p);
    if (it == g_vmm.end()) return false;
    a = it->second;
    g_vmm.erase(it);
  }
  const VmmFns &f = vmm_fns();
  f.unmap((CUdeviceptr)p, a.size);
  f.vfree((CUdeviceptr)p, a.size);
  f.release(a.h);
  return true;
}
}  // namespace

int ess_host_alloc(size_t bytes, int32_t flags, int32_t numa_node, void **host_ptr, void **d_alias,
                   int32_t *placed) {
  if (!bytes || !host_ptr || !d_alias) return ESS_ERR_ARG;
  if (flags & ESS_HOST_VMM) {
    void *p = nullptr;
    size_t mapped = 0;
    if (vmm_alloc(bytes, numa_node, &p, &mapped) == ESS_OK) {
      memset(p, 0, bytes);  // CPU access check + first touch (as the register path)
      *host_ptr = p;
      *d_alias = p;
      if (placed) *placed = ESS_HOST_VMM | (numa_node >= 0 ? ESS_HOST_NUMA_BOUND : 0);
      return ESS_OK;
    }
    // no host VMM on this driver / platform: the registered store below
  }
  const size_t span = host_span(bytes);
  void *raw = mmap(nullptr, span + kHugePage, PROT_READ | PROT_WRITE,
                   MAP_PRIVATE | MAP_ANONYMOUS | MAP_NORESERVE, -1, 0);
  if (raw == MAP_FAILED) return ESS_ERR_NOMEM;
  uintptr_t a = (reinterpret_cast<uintptr_t>(raw) + kHugePage - 1) & ~(uintptr_t)(kHugePage - 1);
  uint8_t *p = reinterpret_cast<uint8_t *>(a);
  const size_t head = a - reinterpret_cast<uintptr_t>(raw);
  if (head) munmap(raw, head);
  const size_t tail = kHugePage - head;
  if (tail) munmap(p + span, tail);
  int got = 0;
  if ((flags & ESS_HOST_HUGEPAGES) && madvise(p, span, MADV_HUGEPAGE) == 0) got |= ESS_HOST_HUGEPAGES;
  if (numa_node >= 0 && numa_node < 64) {
    unsigned long mask = 1ul << numa_node;
    // MPOL_BIND = 2; the pages are first touched by cudaHostRegister below
    if (syscall(SYS_mbind, p, span, 2, &mask, 64, 0) == 0) got |= ESS_HOST_NUMA_BOUND;
  }
  cudaError_t e = cudaHostRegister(p, span, cudaHostRegisterMapped | cudaHostRegisterPortable);
  if (e != cudaSuccess) {
    munmap(p, span);
    return e == cudaErrorMemoryAllocation ? ESS_ERR_NOMEM : ESS_ERR_CUDA;
  }
  if (cudaHostGetDevicePointer(d_alias, p, 0) != cudaSuccess) {
    cudaHostUnregister(p);
    munmap(p, span);
    return ESS_ERR_CUDA;
  }
  *host_ptr = p;
  if (placed) *placed = got;
  return ESS_OK;
}

int ess_host_free(void *host_ptr, size_t bytes) {
  if (!host_ptr || !bytes) return ESS_ERR_ARG;
  if (vmm_free(host_ptr)) return ESS_OK;
  const cudaError_t e = cudaHostUnregister(host_ptr);
  munmap(host_ptr, host_span(bytes));
  return e == cudaSuccess ? ESS_OK : ESS_ERR_CUDA;
}

int ess_host_unregister(void *host_ptr) {
  if (!host_ptr) return ESS_ERR_ARG;
  ESS_CUDA_TRY(cudaHostUnregister(host_ptr));
  return ESS_OK;
}

int ess_preload(void) {
  static std::mutex mu;
  static int done[64] = {};
  int dev = 0;
  ESS_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (dev >= 0 && dev < 64 && done[dev]) return ESS_OK;
  cudaFuncAttributes a;
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)timestamp_kernel));
  ESS_CUDA_TRY(cudaFuncGetAttributes(&a, (const void *)copy_many_kernel));
  if (int rc = ess_preload_indexer()) return rc;
  if (int rc = ess_preload_topk()) return rc;
  if (int rc = ess_preload_pool()) return rc;
  if (int rc = ess_preload_mla()) return rc;
  if (int rc = ess_preload_mla2()) return rc;
  if (dev >= 0 && dev < 64) done[dev] = 1;
  return ESS_OK;
}

}  // extern "C"
