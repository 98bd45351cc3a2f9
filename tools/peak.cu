// FP64 roofline denominator, measured live by bench.py (MEASURED_PEAKS.json
// has no FP64 figure).  Not part of the hot path.  Returns DFMA thread-
// instructions per second of an independent-chain DFMA kernel on all SMs.
#include <cuda_runtime.h>

__global__ void dfma_peak_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6,
         x7 = x0 + 7;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

extern "C" double tool_dfma_rate(int reps) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  double* d = nullptr;
  if (cudaMalloc(&d, 64) != cudaSuccess) return -1.0;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int blocks = sms * 8, thr = 256, iters = 4000;
  dfma_peak_kernel<<<blocks, thr>>>(d, iters, 0.999999, 1e-7);
  double best = 0.0;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a);
    dfma_peak_kernel<<<blocks, thr>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    double rate = (double)blocks * thr * iters * 64 / (ms * 1e-3);
    if (rate > best) best = rate;
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(d);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}
