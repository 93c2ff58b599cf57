// Library-level entry points: version, status strings, pinned host registration.
#include <cstring>

#include "common.cuh"

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

int ess_host_unregister(void *host_ptr) {
  if (!host_ptr) return ESS_ERR_ARG;
  ESS_CUDA_TRY(cudaHostUnregister(host_ptr));
  return ESS_OK;
}

}  // extern "C"
