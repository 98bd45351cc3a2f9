// Microbenchmarks used to pick the nonbonded force-scatter design and to
// measure the FP64 roofline denominator (MEASURED_PEAKS.json has none).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
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
// scattered RED.F64: each warp takes a "row": 32 distinct j inside a window of W atoms
__global__ void red_kernel(double* F, int n, int rows, int W, unsigned seed) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  int nw = (gridDim.x * blockDim.x) >> 5;
  for (int r = warp; r < rows; r += nw) {
    unsigned h = (r * 2654435761u) ^ seed;
    int base = (h % (unsigned)(n - W));
    int j = base + ((lane * 7 + (h >> 7)) % W);
    atomicAdd(&F[j], 1.0); atomicAdd(&F[j + n], 1.0); atomicAdd(&F[j + 2 * n], 1.0);
  }
}
__global__ void cas_kernel(double* out, int iters) {
  __shared__ double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    int j = (w * 256 + ((lane * 7 + it) & 255)) & 2047;
    atomicAdd(&s[j], 1.0);
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}
__global__ void rmw_kernel(double* out, int iters) {
  __shared__ double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = 0;
  __syncthreads();
  int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int it = 0; it < iters; ++it) {
    int j = (w * 256 + ((lane * 7 + it) & 255)) & 2047;
    s[j] += 1.0;
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = s[0];
}
// pair-like transcendental chain: 2 log, 3 exp, rcbrt, sqrt, div per element
__global__ void pair_kernel(const double* r2in, double* out, int n, int reps) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0;
  double r2 = r2in[i % n];
  for (int k = 0; k < reps; ++k) {
    double r = sqrt(r2);
    double lr = log(r);
    double rp = exp(1.55 * lr);
    double sv = rp + 0.3;
    double f13 = exp(log(sv) * (1.0 / 1.55));
    double u = 1.0 - f13 * 0.3;
    double e = exp(5.0 * u);
    double s = r * r2 + 0.5;
    double c = rcbrt(s);
    acc += e * e - 2 * e + c / s + rp / r;
    r2 += 1e-3;
  }
  out[i] = acc;
}
int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  double* d; CK(cudaMalloc(&d, 1 << 20));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  int sms = p.multiProcessorCount;
  // DFMA: blocks = sms*8, 256 thr
  for (int rep = 0; rep < 3; ++rep) {
    int iters = 20000, blocks = sms * 8, thr = 256;
    cudaEventRecord(a); dfma_kernel<<<blocks, thr>>>(d, iters, 0.999999, 1e-7); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double inst = (double)blocks * thr * iters * 64;
    printf("DFMA: %.3f ms  %.3e DP inst/s  %.2f TFLOP/s\n", ms, inst / (ms * 1e-3), 2 * inst / (ms * 1e-3) / 1e12);
  }
  // RED scatter
  for (int n : {1 << 20, 1 << 24}) for (int W : {128, 1024}) {
    double* F; CK(cudaMalloc(&F, sizeof(double) * 3 * (size_t)n)); cudaMemset(F, 0, sizeof(double) * 3 * (size_t)n);
    int rows = 1 << 22;
    red_kernel<<<sms * 16, 256>>>(F, n, rows, W, 1);
    cudaEventRecord(a); red_kernel<<<sms * 16, 256>>>(F, n, rows, W, 7); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double nred = (double)rows * 32 * 3;
    printf("RED.F64 n=%d W=%d: %.3f ms %.3e lane-REDs/s  (%.2f per SM-cycle @1.9GHz)\n", n, W, ms, nred / (ms * 1e-3), nred / (ms * 1e-3) / sms / 1.9e9);
    cudaFree(F);
  }
  {
    int iters = 4096;
    cas_kernel<<<sms * 4, 256>>>(d, iters);
    cudaEventRecord(a); cas_kernel<<<sms * 4, 256>>>(d, iters); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double n = (double)sms * 4 * 256 * iters;
    printf("smem CAS f64 add: %.3f ms %.3e lane-ops/s (%.2f per SM-cycle @1.9GHz)\n", ms, n / (ms * 1e-3), n / (ms * 1e-3) / sms / 1.9e9);
    rmw_kernel<<<sms * 4, 256>>>(d, iters);
    cudaEventRecord(a); rmw_kernel<<<sms * 4, 256>>>(d, iters); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    printf("smem plain RMW f64: %.3f ms %.3e lane-ops/s (%.2f per SM-cycle @1.9GHz)\n", ms, n / (ms * 1e-3), n / (ms * 1e-3) / sms / 1.9e9);
  }
  {
    int n = 1 << 20; double* r2; double* o; CK(cudaMalloc(&r2, n * 8)); CK(cudaMalloc(&o, (size_t)sms * 2048 * 8 * 4));
    double* h = (double*)malloc(n * 8); for (int i = 0; i < n; ++i) h[i] = 1.0 + 99.0 * (i % 1000) / 1000.0;
    cudaMemcpy(r2, h, n * 8, cudaMemcpyHostToDevice);
    int reps = 200, blocks = sms * 16, thr = 256;
    pair_kernel<<<blocks, thr>>>(r2, o, n, reps);
    cudaEventRecord(a); pair_kernel<<<blocks, thr>>>(r2, o, n, reps); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double ev = (double)blocks * thr * reps;
    printf("pair chain: %.3f ms %.3e evals/s\n", ms, ev / (ms * 1e-3));
  }
  return 0;
}
