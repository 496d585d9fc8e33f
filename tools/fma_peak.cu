// Non-tensor FP32 / FP64 FMA peaks (SURVEY 8(d) asks for them: the roofline
// denominators for flops, not in MEASURED_PEAKS.json).  Independent FMA
// chains per thread, full grid, timed with events.
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void k_fma(T* out, int iters, T a, T b) {
  T x[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += x[c];
  if (s == (T)12345) out[0] = s;
}

template <typename T>
double run(const char* name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  T* out;
  cudaMalloc(&out, sizeof(T));
  const int grid = sms * 8, nt = 256, iters = 4096;
  constexpr int CH = 8;
  k_fma<T, CH><<<grid, nt>>>(out, 16, (T)0.999, (T)0.001);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k_fma<T, CH><<<grid, nt>>>(out, iters, (T)0.999, (T)0.001);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double flops = 2.0 * grid * nt * (double)iters * CH;
  const double tf = flops / (ms * 1e-3) / 1e12;
  printf("%s FMA: %.1f TFLOP/s (%.3f ms)\n", name, tf, ms);
  return tf;
}

int main() {
  run<float>("fp32");
  run<double>("fp64");
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
