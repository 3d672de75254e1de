#include <cstdio>
constexpr int D = 50, NP = 135;
__global__ void cal(const long long* g, long long* out, long long* cyc, int n) {
  extern __shared__ long long vp[];
  __shared__ int order[NP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < NP * D; e += blockDim.x) vp[e] = g[e];
  for (int p = tid; p < NP; p += blockDim.x) order[p] = (p * 37) % NP;
  __syncthreads();
  long long s = 0, t0, t1;
  // A: 17 independent LDS.64 (addresses from the loop counter)
  t0 = clock64();
  for (int q = 0; q < n; ++q) s += vp[((q * 8 + warp) % NP) * D + lane];
  t1 = clock64();
  if (lane == 0) cyc[warp] = t1 - t0;
  // B: indirect through order[]
  t0 = clock64();
  for (int q = 0; q < n; ++q) s += vp[order[(q * 8 + warp) % NP] * D + lane];
  t1 = clock64();
  if (lane == 0) cyc[8 + warp] = t1 - t0;
  // C: batches of 4, indirect
  t0 = clock64();
  for (int q = 0; q < n; q += 4) {
    int p4[4]; long long a4[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) p4[u] = order[((q + u) * 8 + warp) % NP];
#pragma unroll
    for (int u = 0; u < 4; ++u) a4[u] = vp[p4[u] * D + lane];
#pragma unroll
    for (int u = 0; u < 4; ++u) s += a4[u];
  }
  t1 = clock64();
  if (lane == 0) cyc[16 + warp] = t1 - t0;
  out[tid] = s;
}
int main() {
  long long *g, *o, *c; cudaMalloc(&g, 8 * NP * D); cudaMemset(g, 0, 8 * NP * D); cudaMalloc(&o, 8 * 1024); cudaMallocManaged(&c, 8 * 64);
  cudaFuncSetAttribute(cal, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int nw : {1, 8}) {
    for (int r = 0; r < 2; ++r) { cal<<<1, 32 * nw, 8 * NP * D>>>(g, o, c, 16); cudaDeviceSynchronize(); }
    printf("%d warps, 16 rows: A direct %lld  B indirect %lld  C batch4 %lld cycles (warp 0)\n", nw, c[0], c[8], c[16]);
  }
  return 0;
}
