// Library-level entry points: version, status strings, pinned host registration,
// and the shared host helpers (tensor-map encoding, SM count).
#include <cstring>
#include <mutex>

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

int ess_sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

extern "C" {

const char *ess_version(void) { return "ess_b200 0.1 sm_100a"; }

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
__global__ void timestamp_kernel(uint64_t *dst) {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *dst = t;
}

int ess_timestamp(uint64_t *d_dst, void *stream) {
  if (!d_dst) return ESS_ERR_ARG;
  timestamp_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(d_dst);
  ESS_CUDA_TRY(cudaGetLastError());
  return ESS_OK;
}

int ess_host_unregister(void *host_ptr) {
  if (!host_ptr) return ESS_ERR_ARG;
  ESS_CUDA_TRY(cudaHostUnregister(host_ptr));
  return ESS_OK;
}

}  // extern "C"
