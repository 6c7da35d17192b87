// peak.cu -- FP64-pipe roofline denominator: a DFMA throughput microbenchmark.
//
// MEASURED_PEAKS.json carries HBM and bf16 peaks only; the AM solver is bound
// by the FP64 pipe, so the achieved fraction is
// reported against this measured DFMA rate (2 flops per DFMA).
#include <cuda_runtime.h>

#include "common.cuh"

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

// ------------------------------------------------------ latency probes --
// Dependent-chain latency (SM cycles per instruction, one thread):
// 0 DFMA, 1 DADD, 2 DMUL, 3 MUFU.RSQ64H (+ 0 ALU, via rsqrt.approx), 4 FFMA,
// 5 LDS.64 (pointer chase in shared memory), 6 SHFL (64-bit), 7 fp64 rsqrt_nb.
namespace bmpc {
template <int WHICH>
__global__ void k_latency(int iters, double seed, long long* cycles, double* sink) {
  __shared__ long long chase[64];
  if (threadIdx.x == 0)
    for (int i = 0; i < 64; ++i) chase[i] = (i + 1) & 63;
  __syncwarp();
  double x = seed, y = 1.0000001, z = 1e-9;
  float xf = (float)seed;
  long long p = 0;
  const long long t0 = clock64();
#pragma unroll 8
  for (int i = 0; i < iters; ++i) {
    if (WHICH == 0) x = fma(x, y, z);
    if (WHICH == 1) x = x + z;
    if (WHICH == 2) x = x * y;
    if (WHICH == 3) asm volatile("rsqrt.approx.ftz.f64 %0, %0;" : "+d"(x));
    if (WHICH == 4) xf = fmaf(xf, 1.0000001f, 1e-9f);
    if (WHICH == 5) p = chase[p];
    if (WHICH == 6) x = __shfl_xor_sync(0xffffffffu, x, 1);
    if (WHICH == 7) x = rsqrt_nb(x) + 0.5;
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    cycles[0] = t1 - t0;
    sink[0] = x + xf + (double)p;
  }
}

cudaError_t latency_probe(int which, double* cyc_per_op, cudaStream_t st) {
  long long* c = nullptr;
  double* s = nullptr;
  cudaMalloc(&c, sizeof(long long));
  cudaMalloc(&s, sizeof(double));
  const int iters = 4096;
  void (*fns[8])(int, double, long long*, double*) = {
      k_latency<0>, k_latency<1>, k_latency<2>, k_latency<3>,
      k_latency<4>, k_latency<5>, k_latency<6>, k_latency<7>};
  if (which < 0 || which > 7) return cudaErrorInvalidValue;
  fns[which]<<<1, 32, 0, st>>>(64, 1.5, c, s);
  fns[which]<<<1, 32, 0, st>>>(iters, 1.5, c, s);
  long long h = 0;
  cudaMemcpyAsync(&h, c, sizeof(long long), cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  cudaFree(c);
  cudaFree(s);
  *cyc_per_op = (double)h / iters;
  return cudaGetLastError();
}
}  // namespace bmpc
