// peak.cu -- FP64-pipe roofline denominator: a DFMA throughput microbenchmark.
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the AM solver is bound
// by the FP64 pipe, so the achieved fraction is
// reported against this measured DFMA rate (2 flops per DFMA).
#include <cuda_runtime.h>

namespace bmpc {

constexpr int kChains = 8;

__global__ void __launch_bounds__(256) k_dfma_peak(int iters, double seed, double* out) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = seed + threadIdx.x * 1e-9 + c;
  const double m1 = 0.9999999, a1 = 1e-7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int c = 0; c < kChains; ++c) acc[c] = fma(acc[c], m1, a1);
  }
  double s = 0.0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;  // keep the chains live
}

// Returns achieved fp64 TFLOP/s (best of `reps`) for a full-chip launch.
cudaError_t dfma_peak_tflops(int reps, double* tflops, cudaStream_t st) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = 256, blocks = sms * 8, iters = 4096;
  double* out = nullptr;
  cudaError_t e = cudaMalloc(&out, sizeof(double));
  if (e != cudaSuccess) return e;
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0);
  cudaEventCreate(&t1);
  k_dfma_peak<<<blocks, threads, 0, st>>>(iters / 8, 1.0, out);  // warm-up
  double best = 0.0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(t0, st);
    k_dfma_peak<<<blocks, threads, 0, st>>>(iters, 1.0, out);
    cudaEventRecord(t1, st);
    cudaEventSynchronize(t1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t0, t1);
    const double flops = 2.0 * kChains * 8.0 * iters * (double)threads * blocks;
    const double tf = flops / (ms * 1e-3) / 1e12;
    if (tf > best) best = tf;
  }
  e = cudaGetLastError();
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  cudaFree(out);
  *tflops = best;
  return e;
}

}  // namespace bmpc
