// Measured FP64 / FP32 FMA throughput of this GPU (the LiDAR kernel's FP64
// roofline and the radial kernel's FP32 roofline denominators).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp_peak tools/fp_peak.cu
//   /tmp/fp_peak  ->  {"fp64_tflops": ..., "fp32_tflops": ..., ...}
// Every thread runs kChains independent FMA chains (enough ILP to saturate
// the pipes), grid = 4 CTAs of 256 threads per SM; best of 5 launches,
// CUDA events.  2 FLOP per FMA.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kChains = 8;
constexpr int kIters = 4096;

template <typename T>
__global__ void fma_kernel(T *out, T a, T b) {
  T v[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) v[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < kIters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) v[c] = fma(v[c], a, b);
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += v[c];
  if (s == (T)-1.2345) out[threadIdx.x] = s;   // never true: keeps the work
}

template <typename T>
double tflops(int sms) {
  T *out;
  cudaMalloc(&out, 1024 * sizeof(T));
  const int blocks = sms * 4, threads = 256;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_kernel<T><<<blocks, threads>>>(out, (T)0.999999, (T)1e-7);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_kernel<T><<<blocks, threads>>>(out, (T)0.999999, (T)1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaFree(out);
  const double flop = 2.0 * kChains * (double)kIters * blocks * threads;
  return flop / (best * 1e-3) / 1e12;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double f64 = tflops<double>(p.multiProcessorCount);
  const double f32 = tflops<float>(p.multiProcessorCount);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_mhz_attr\": %.0f, \"fp64_tflops\": %.2f, "
         "\"fp32_tflops\": %.2f, \"how\": \"FMA chains, %d per thread, %d CTAs x 256 threads, best of 5\"}\n",
         p.name, p.multiProcessorCount, clk_khz / 1e3, f64, f32, kChains, p.multiProcessorCount * 4);
  return 0;
}
