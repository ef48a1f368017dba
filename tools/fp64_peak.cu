// FP64 DFMA throughput microbenchmark (the roofline denominator missing from
// MEASURED_PEAKS.json).  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 256, iters = 4096;
  const int blocks = sms * 8;
  constexpr int CH = 8;
  dfma_loop<CH><<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    dfma_loop<CH><<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * (double)blocks * threads * iters * CH;
  const double tf = flops / (best * 1e-3) / 1e12;
  printf("{\"fp64_fma_tflops\": %.3f, \"sms\": %d, \"clock_mhz_attr\": %d, \"ms\": %.4f, "
         "\"per_sm_per_clk_at_attr\": %.2f}\n",
         tf, sms, clk / 1000, best, flops / (best * 1e-3) / sms / (clk * 1e3) / 2.0);
  return 0;
}
