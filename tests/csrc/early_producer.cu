// Test-only foreign producer (tests/test_gpu_parity.py::test_foreign_producer_early_trigger):
// a kernel that lets its dependents launch at entry (griddepcontrol.launch_dependents, as
// CUTLASS-style kernels do), then spins and only afterwards writes its output.  A consumer
// launched as a programmatic dependent launch that read the output before griddepcontrol.wait
// would see the old contents.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_early_producer(float2* __restrict__ dst, const float2* __restrict__ src, int64_t n, int64_t spin) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const long long t0 = clock64();
  while (clock64() - t0 < spin) {
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

extern "C" __attribute__((visibility("default"))) int sfft_test_early_producer(void* dst, const void* src,
                                                                                int64_t n, int64_t spin_cycles,
                                                                                void* stream) {
  k_early_producer<<<148, 256, 0, (cudaStream_t)stream>>>((float2*)dst, (const float2*)src, n, spin_cycles);
  return cudaGetLastError() == cudaSuccess ? 0 : 5;
}
