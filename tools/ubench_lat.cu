// Dependent-chain latency (cycles per op) of the FP64 ops on the Jacobi critical path.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsq(double x) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__device__ __forceinline__ double rcp(double x) { double y; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
#define N 256
__global__ void lat(double x0, double* out, long long* cyc) {
  double x = x0 + threadIdx.x * 1e-20;
  long long t0, t1;
  // DFMA
  t0 = clock64(); for (int i = 0; i < N; ++i) x = fma(x, 0.9999999, 1e-9); t1 = clock64(); cyc[0] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = x * 0.99999999; t1 = clock64(); cyc[1] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = x + 1e-12; t1 = clock64(); cyc[2] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = rsq(x) + 0.5; t1 = clock64(); cyc[3] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x = rcp(x) + 0.5; t1 = clock64(); cyc[4] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1) * 1e-30; t1 = clock64(); cyc[5] = t1 - t0;
  float f = (float)x;
  t0 = clock64(); for (int i = 0; i < N; ++i) f = fmaf(f, 0.9999f, 1e-5f); t1 = clock64(); cyc[6] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) f += __shfl_xor_sync(0xffffffffu, f, 1) * 1e-30f; t1 = clock64(); cyc[7] = t1 - t0;
  __shared__ double sh[64];
  sh[threadIdx.x] = x;
  __syncthreads();
  int idx = threadIdx.x;
  t0 = clock64(); for (int i = 0; i < N; ++i) { idx = (int)sh[idx & 31] & 31; } t1 = clock64(); cyc[8] = t1 - t0;
  t0 = clock64(); for (int i = 0; i < N; ++i) { sh[threadIdx.x] = x + i; __syncthreads(); x = sh[(threadIdx.x + 1) & 31]; } t1 = clock64(); cyc[9] = t1 - t0;
  out[threadIdx.x] = x + f + idx;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 4096); cudaMallocManaged(&c, 128);
  const char* names[] = {"DFMA", "DMUL", "DADD", "MUFU.RSQ64H+DADD", "MUFU.RCP64H+DADD", "SHFL f64 + DFMA", "FFMA", "SHFL f32 + FFMA", "LDS f64->idx chain", "STS+BAR+LDS (1 warp)"};
  for (int rep = 0; rep < 2; ++rep) { lat<<<1, 32>>>(1.5, o, c); cudaDeviceSynchronize(); }
  for (int i = 0; i < 10; ++i) printf("%-24s %.1f cycles\n", names[i], (double)c[i] / N);
  lat<<<1, 128>>>(1.5, o, c); cudaDeviceSynchronize();
  printf("%-24s %.1f cycles (4 warps)\n", names[9], (double)c[9] / N);
  return 0;
}
