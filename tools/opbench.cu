// Per-instruction-class throughput probes on sm_100a, used to balance the
// nonbonded pair evaluation across the FP64, XU (MUFU/conversions), ALU/FMA
// and shared-memory pipes.  Each kernel runs 8 independent chains per thread
// (enough ILP that latency is hidden) and reports warp-instructions per SM-cycle.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o opbench opbench.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

#define CHAINS 8
template <int OP>
__device__ __forceinline__ double step(double x, double a, int& iacc) {
  if (OP == 0) return fma(x, a, 1e-7);                                   // DFMA
  if (OP == 1) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }   // MUFU.RCP64H
  if (OP == 2) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; } // MUFU.RSQ64H
  if (OP == 3) { float f = (float)x; return (double)f + a; }              // F2F pair + DADD
  if (OP == 4) { int k = __double2int_rn(x); iacc += k; return x + a; }   // F2I + DADD
  if (OP == 5) { return (double)(iacc += 3) * a + x; }                    // I2F + DFMA
  if (OP == 6) { float f = __int_as_float(__double2hiint(x)); float e = __expf(f); iacc ^= __float_as_int(e); return x + a; }  // MUFU.EX2 f32 + DADD
  if (OP == 7) {   // DFMA + 2 int ops (mix)
    int h = __double2hiint(x); iacc = (iacc + h) ^ (h >> 3); return fma(x, a, 1e-7);
  }
  if (OP == 8) {   // DFMA + 4 fp32 ops (mix)
    float f = __int_as_float(__double2hiint(x) | 0x3f000000); float g = fmaf(f, f, 1.0f); g = fmaf(g, f, 0.5f); iacc += __float_as_int(g * f); return fma(x, a, 1e-7);
  }
  return x;
}
template <int OP>
__global__ void opk(double* out, int iters, double a) {
  double x[CHAINS];
  int iacc = threadIdx.x;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = 1.0 + threadIdx.x * 1e-6 + c * 1e-3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = step<OP>(x[c], a, iacc);
  }
  double s = iacc;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;
}
// shared-memory random ops: per iteration one op per lane at a hashed address in [0, 2048)
template <int OP>
__global__ void smk(double* out, int iters) {
  __shared__ double s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = 1.0;
  __syncthreads();
  unsigned h = threadIdx.x * 2654435761u;
  double acc = 0;
  int* si = reinterpret_cast<int*>(s);
  for (int it = 0; it < iters; ++it) {
    h = h * 1664525u + 1013904223u;
    int j = (h >> 10) & 2047;
    if (OP == 0) acc += s[j];                               // LDS.64 random
    if (OP == 1) atomicAdd(&si[2 * j], 1);                  // ATOMS.ADD (int32, no return)
    if (OP == 2) atomicAdd(&s[j], 1.0);                     // ATOMS.CAS.64 loop
    if (OP == 3) { acc += s[j]; s[(j + 17) & 2047] = acc; } // plain LDS/STS
  }
  __syncthreads();
  if (acc == 12345.678 || s[threadIdx.x] == 1e300) out[blockIdx.x] = acc;
}

// dependent-chain latency: one warp per SM, one chain
template <int OP>
__global__ void latk(double* out, int iters, double a) {
  double x = 1.0 + threadIdx.x * 1e-9;
  int ix = threadIdx.x;
  __shared__ double tbl[64];
  if (threadIdx.x < 64) tbl[threadIdx.x] = 1.0 + threadIdx.x * 1e-9;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (OP == 0) x = fma(x, a, 1e-9);
    if (OP == 1) x = x * a;
    if (OP == 2) x = x + a;
    if (OP == 3) { asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(x) : "d"(x)); }
    if (OP == 4) { x = tbl[(__double2loint(x) + it) & 63]; }              // LDS + int op
    if (OP == 5) { ix = ix * 3 + 1; ix ^= ix >> 3; }                       // 2 int ops
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (double)(t1 - t0) / iters;
  if (x == 12345.678 || ix == 7) out[1000 + blockIdx.x] = x + ix;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int sms = p.multiProcessorCount;
  printf("device %s SMs %d\n", p.name, sms);
  double* d; CK(cudaMalloc(&d, 1 << 20));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  const double clk = 1.965e9;
  auto run = [&](const char* name, void (*k)(double*, int, double), int per) {
    int iters = 4000, blocks = sms * 8, thr = 256;
    k<<<blocks, thr>>>(d, iters, 0.9999999);
    cudaEventRecord(a); k<<<blocks, thr>>>(d, iters, 0.9999999); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double warp_steps = (double)blocks * thr / 32 * iters * CHAINS;
    printf("%-34s %.3f ms  %.3f steps/SM-cycle (x32 lanes = %.1f lane-ops/SM-clk)\n", name, ms,
           warp_steps / (ms * 1e-3) / sms / clk, 32 * warp_steps / (ms * 1e-3) / sms / clk);
  };
  run("DFMA", opk<0>, 1);
  run("MUFU.RCP64H", opk<1>, 1);
  run("MUFU.RSQ64H", opk<2>, 1);
  run("F2F.F32.F64+F2F.F64.F32+DADD", opk<3>, 1);
  run("F2I.F64+DADD+IADD", opk<4>, 1);
  run("I2F.F64+DFMA", opk<5>, 1);
  run("MUFU.EX2(f32)+DADD", opk<6>, 1);
  run("DFMA+2 int", opk<7>, 1);
  run("DFMA+4 fp32", opk<8>, 1);
  auto runs = [&](const char* name, void (*k)(double*, int)) {
    int iters = 4096, blocks = sms * 4, thr = 256;
    k<<<blocks, thr>>>(d, iters);
    cudaEventRecord(a); k<<<blocks, thr>>>(d, iters); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    double n = (double)blocks * thr * iters;
    printf("%-34s %.3f ms  %.2f lane-ops/SM-cycle\n", name, ms, n / (ms * 1e-3) / sms / clk);
  };
  auto lat = [&](const char* name, void (*k)(double*, int, double)) {
    double* o; CK(cudaMalloc(&o, 4096 * 8));
    k<<<sms, 32>>>(o, 10000, 0.9999999);
    CK(cudaDeviceSynchronize());
    double h; CK(cudaMemcpy(&h, o, 8, cudaMemcpyDeviceToHost));
    printf("latency %-24s %.1f cycles/op\n", name, h);
    cudaFree(o);
  };
  lat("DFMA", latk<0>);
  lat("DMUL", latk<1>);
  lat("DADD", latk<2>);
  lat("MUFU.RSQ64H", latk<3>);
  lat("LDS.64 (+int)", latk<4>);
  lat("2 int ops", latk<5>);
  runs("smem LDS.64 random", smk<0>);
  runs("smem ATOMS.ADD int32 random", smk<1>);
  runs("smem atomicAdd f64 (CAS) random", smk<2>);
  runs("smem LDS.64+STS.64 random", smk<3>);
  return 0;
}
