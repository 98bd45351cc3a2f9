// Throughput probes of the warp-collective and bit-manipulation instructions
// the list build leans on (POPC, VOTE, REDUX, SHFL, FLO, __fns), to find which
// of them issue to the narrow XU pipe on sm_100a.  8 independent chains per
// thread; reports warp-instructions per SM-cycle of the probed op (1 op per
// chain step plus one cheap ALU op that keeps the chain dependent).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o warpops warpops.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); exit(1);}}while(0)

#define CHAINS 8
template <int OP>
__device__ __forceinline__ unsigned step(unsigned x, unsigned k) {
  if (OP == 0) return x + k;                                           // IADD (baseline)
  if (OP == 1) return __popc(x) + x + k;                               // POPC
  if (OP == 2) return __ballot_sync(0xffffffffu, x & 1u) ^ (x + k);    // VOTE.ANY (ballot)
  if (OP == 3) return __reduce_or_sync(0xffffffffu, x) + k;            // REDUX.OR
  if (OP == 4) return __shfl_sync(0xffffffffu, x, (x + k) & 31) + k;   // SHFL.IDX
  if (OP == 5) return __clz(x | 1u) + x + k;                           // FLO
  if (OP == 6) return __fns(x | 1u, 0, 1) + x + k;                     // __fns
  if (OP == 7) return __popc(x & ((1u << (k & 31)) - 1u)) + x;         // POPC of a masked word
  if (OP == 8) return (unsigned)__float2int_rd(__uint_as_float((x & 0x007fffffu) | 0x3f800000u) * 3.f) + x + k;  // F2I.FLOOR
  if (OP == 9) return __any_sync(0xffffffffu, (x & 7u) == 0u) + x + k;  // VOTE.ANY (predicate)
  return x;
}
template <int OP>
__global__ void wk(unsigned* out, int iters, unsigned k) {
  unsigned x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 7919u + c * 104729u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = step<OP>(x[c], k + c);
  }
  unsigned s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s ^= x[c];
  if (s == 0x12345678u) out[0] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  const int sms = p.multiProcessorCount;
  int clk_khz = 0; CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const double clk = clk_khz * 1e3;
  printf("device %s SMs %d clock %.0f MHz\n", p.name, sms, clk / 1e6);
  unsigned* d; CK(cudaMalloc(&d, 1 << 20));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); float ms;
  auto run = [&](const char* name, void (*k)(unsigned*, int, unsigned)) {
    const int iters = 4000, blocks = sms * 8, thr = 256;
    k<<<blocks, thr>>>(d, iters, 3u);
    cudaEventRecord(a); k<<<blocks, thr>>>(d, iters, 3u); cudaEventRecord(b);
    CK(cudaEventSynchronize(b)); cudaEventElapsedTime(&ms, a, b);
    const double warp_steps = (double)blocks * thr / 32 * iters * CHAINS;
    printf("%-28s %.3f ms  %.3f steps/SM-cycle  (%.1f lane-ops/SM-clk)\n", name, ms,
           warp_steps / (ms * 1e-3) / sms / clk, 32 * warp_steps / (ms * 1e-3) / sms / clk);
  };
  run("IADD (baseline)", wk<0>);
  run("POPC+2 IADD", wk<1>);
  run("VOTE.ballot+LOP+IADD", wk<2>);
  run("REDUX.OR+IADD", wk<3>);
  run("SHFL.IDX+2 IADD", wk<4>);
  run("FLO+2 IADD", wk<5>);
  run("__fns+2 IADD", wk<6>);
  run("POPC(masked)+IADD", wk<7>);
  run("F2I.FLOOR+FMUL+LOP", wk<8>);
  run("VOTE.ANY+IADD", wk<9>);
  return 0;
}
