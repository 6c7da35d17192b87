// dmma_probe.cu -- does fp64 mma.sync (DMMA) on sm_100a run beside the DFMA
// pipe?  Times DFMA-only, DMMA-only and interleaved loops on every SM.
// Build + run (GPU box): nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
//   -o /tmp/dmma_probe tools/dmma_probe.cu && /tmp/dmma_probe
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void probe(int iters, double seed, double* out) {
  double a0 = seed + threadIdx.x, a1 = a0 * 0.5, a2 = a0 * 0.25, a3 = a0 * 0.125;
  double f[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = seed * (i + 1);
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  const double b = 1.0000001, a = 0.9999999;
  for (int it = 0; it < iters; ++it) {
    if (MODE != 1) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = fma(f[i], b, 1e-9);
    }
    if (MODE != 0) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                     : "+d"(c[i][0]), "+d"(c[i][1])
                     : "d"(a0 + i), "d"(a));
    }
  }
  double s = a1 + a2 + a3;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += f[i] + c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  double* out;
  cudaMalloc(&out, 8);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    const int grid = sms, block = 32 * warps;
    auto run = [&](auto kern, const char* name, double flop_per_iter_thread) {
      kern<<<grid, block>>>(10, 1.0, out);
      cudaEventRecord(e0);
      kern<<<grid, block>>>(iters, 1.0, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * flop_per_iter_thread * iters * (double)grid * block;
      printf("warps/SM %2d %-10s %8.3f ms  %7.2f TFLOP/s\n", warps, name, ms, flops / ms / 1e9);
    };
    // DFMA: 32 per thread per iter; DMMA: 8 mma x 256 FMA / 32 threads = 64 per thread per iter
    run(probe<0>, "dfma", 32.0);
    run(probe<1>, "dmma", 64.0);
    run(probe<2>, "both", 96.0);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
