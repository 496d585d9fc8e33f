// Result rows written straight into one rank's device buffer:
// the owner allocates the B x k result buffer and exports a CUDA IPC
// handle; every other process on the node maps it, and its transform
// kernel's epilogue stores its row shard there over NVLink / NVSwitch peer
// memory.  The final gather of the reference's per-signal outputs (each
// rank's coefficients on one rank) then needs no separate collective and
// no extra copy.  Host-side plumbing only: the stores are the transform's
// own (sfft_hidft / sfft_hidft_to_dft_fused with the mapped pointer as
// their output).

#include <cstring>

#include "sfft_common.cuh"
#include "structfft_b200.h"

using namespace sfft;

extern "C" int sfft_peer_alloc(int64_t bytes, void** dptr, unsigned char* handle) {
  if (!dptr || !handle) return fail(SFFT_ERR_INVALID, "null pointer");
  if (bytes <= 0) return fail(SFFT_ERR_INVALID, "peer buffer size must be positive");
  *dptr = nullptr;
  void* p = nullptr;
  SFFT_CUDA(cudaMalloc(&p, (size_t)bytes));  // its own allocation: the IPC handle covers exactly it
  cudaIpcMemHandle_t h;
  const cudaError_t e = cudaIpcGetMemHandle(&h, p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_fail(e, "cudaIpcGetMemHandle");
  }
  static_assert(sizeof(h) == SFFT_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(handle, &h, sizeof(h));
  *dptr = p;
  return SFFT_OK;
}

extern "C" int sfft_peer_free(void* dptr) {
  if (!dptr) return SFFT_OK;
  SFFT_CUDA(cudaFree(dptr));
  return SFFT_OK;
}

extern "C" int sfft_peer_open(const unsigned char* handle, void** dptr) {
  if (!dptr || !handle) return fail(SFFT_ERR_INVALID, "null pointer");
  *dptr = nullptr;
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle, sizeof(h));
  SFFT_CUDA(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess));
  return SFFT_OK;
}

extern "C" int sfft_peer_close(void* dptr) {
  if (!dptr) return SFFT_OK;
  SFFT_CUDA(cudaIpcCloseMemHandle(dptr));
  return SFFT_OK;
}
