// FP32 (FFMA) and FP64 (DFMA) issue-rate microbenchmark for the roofline
// denominators ("Measure an FFMA microbenchmark, and a DFMA one").
#include <cstdio>
#include <cuda_runtime.h>
template <typename T, int ILP>
__global__ void fma_loop(T* out, int iters, T a, T b) {
  T x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = (T)(threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = x[k] * a + b;
  }
  T s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  if (s == (T)-1.2345) out[threadIdx.x] = s;
}
template <typename T>
double run(int blocks, int threads, int iters) {
  T* out; cudaMalloc(&out, 4096 * sizeof(T));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) fma_loop<T, 8><<<blocks, threads>>>(out, iters, (T)0.9999, (T)0.0001);
  cudaEventRecord(e0);
  fma_loop<T, 8><<<blocks, threads>>>(out, iters, (T)0.9999, (T)0.0001);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * 8 * (double)iters * blocks * threads;
  cudaFree(out);
  return flops / (ms * 1e-3) / 1e12;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"gpu\": \"%s\", \"sm_count\": %d, \"l2_bytes\": %d, \"smem_per_sm\": %zu, \"regs_per_sm\": %d, \"clock_khz_attr\": %d,", p.name, p.multiProcessorCount, p.l2CacheSize, p.sharedMemPerMultiprocessor, p.regsPerMultiprocessor, clk);
  double f32 = run<float>(p.multiProcessorCount * 8, 256, 1 << 16);
  double f64 = run<double>(p.multiProcessorCount * 8, 256, 1 << 14);
  printf(" \"fp32_ffma_tflops\": %.2f, \"fp64_dfma_tflops\": %.2f}\n", f32, f64);
  return 0;
}
