// FP64 FMA peak of the device (the FP64 roofline denominator of bench.py):
// every thread runs 8 independent DFMA chains; 2 flops per FMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak tools/fp64_peak.cu && ./fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_fma(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-9 + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains live
}

int main() {
  int dev = 0, sms = 0, mhz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 1 << 20);
  const int threads = 256, blocks = sms * 8, iters = 1 << 14;
  k_fma<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    k_fma<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8.0 * iters * static_cast<double>(blocks) * threads;
  std::printf("{\"fp64_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %d, \"how\": \"8 independent DFMA chains per thread, %d x %d threads, best of 5\"}\n",
              flops / (best * 1e-3) / 1e12, sms, mhz / 1000, blocks, threads);
  return 0;
}
