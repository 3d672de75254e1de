// ubench_jacobi.cu -- dissect the per-round latency of the one-sided Jacobi round
// (development tool).  Each variant removes one stage of the round; k = 50, LP = 8, E = 8.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_jacobi tools/ubench_jacobi.cu
#include <cfloat>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ int rr_player(int j, int r, int np) {
  int x = j - 1 + r;
  if (x >= np - 1) x -= np - 1;
  return j == 0 ? 0 : 1 + x;
}

// MODE bits: 1 = loads, 2 = dots+shuffles, 4 = angle, 8 = stores, 16 = barrier
template <int MODE, int LP, int E>
__global__ void rounds(double* out, int k, int nrounds, long long* cyc) {
  extern __shared__ double A[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int e = tid; e < k * k; e += blockDim.x) A[e] = 1.0 + (e % 7) * 0.1;
  __syncthreads();
  constexpr int kGroups = 32 / LP;
  const int grp = lane / LP, gl = lane % LP;
  const int np = (k + 1) & ~1, npairs = np / 2;
  double acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < nrounds; ++it) {
    const int rnd = it % (np - 1);
    for (int base = warp * kGroups; base < npairs; base += nwarps * kGroups) {
      const int pr = base + grp;
      const int prc = pr < npairs ? pr : 0;
      int p = rr_player(prc, rnd, np), q = rr_player(np - 1 - prc, rnd, np);
      const int lo = p < q ? p : q, hi = p < q ? q : p;
      const bool real = pr < npairs && hi < k;
      double* ap = A + (size_t)(real ? lo : 0) * k;
      double* aq = A + (size_t)(real ? hi : 0) * k;
      double x[E], y[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = gl + LP * e;
        if (MODE & 1) {
          x[e] = (real && i < k) ? ap[i] : 0.0;
          y[e] = (real && i < k) ? aq[i] : 0.0;
        } else {
          x[e] = 1.0 + e + it;
          y[e] = 2.0 + e;
        }
      }
      double al = 1, be = 2, ga = 0.5;
      if (MODE & 2) {
        double al0 = 0, be0 = 0, ga0 = 0, al1 = 0, be1 = 0, ga1 = 0;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
          al0 = fma(x[e], x[e], al0); be0 = fma(y[e], y[e], be0); ga0 = fma(x[e], y[e], ga0);
          al1 = fma(x[e + 1], x[e + 1], al1); be1 = fma(y[e + 1], y[e + 1], be1); ga1 = fma(x[e + 1], y[e + 1], ga1);
        }
        al = al0 + al1; be = be0 + be1; ga = ga0 + ga1;
#pragma unroll
        for (int o = LP / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
      }
      double c = 1, sn = 0;
      if (MODE & 4) {
        const double dx = be - al, dy = 2.0 * ga;
        const double mx = fmax(fabs(dx), fabs(dy));
        const int ex = static_cast<int>((__double_as_longlong(mx) >> 52) & 0x7ff);
        const double scl = __longlong_as_double(static_cast<long long>(2046 - ex) << 52);
        const float xf = static_cast<float>(dx * scl), yf = static_cast<float>(dy * scl);
        const float hyp = fmaf(xf, xf, yf * yf);
        const float den = fabsf(xf) + hyp * __frsqrt_rn(hyp);
        float tf = copysignf(1.f, xf) * __fdividef(yf, den);
        tf = (ga * ga > 1e-30 * al * be) ? tf : 0.f;
        const double t = static_cast<double>(tf);
        const double q1 = fma(t, t, 1.0);
        c = static_cast<double>(__frsqrt_rn(static_cast<float>(q1)));
        c = c * fma(-0.5 * q1, c * c, 1.5);
        c = c * fma(-0.5 * q1, c * c, 1.5);
        sn = c * t * 1e-3;
      }
      if (MODE & 8) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = gl + LP * e;
          if (real && i < k) {
            ap[i] = c * x[e] - sn * y[e];
            aq[i] = sn * x[e] + c * y[e];
          }
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) acc += c * x[e] - sn * y[e];
      }
    }
    if (MODE & 16) __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) *cyc = (t1 - t0) / nrounds;
  if (acc == 12345.0) out[0] = acc;
}

template <int MODE, int LP = 8, int E = 8>
void run(const char* name, double* d, long long* c, int threads, int k = 50) {
  const int nr = 441;
  rounds<MODE, LP, E><<<1, threads, 2 * k * k * 8>>>(d, k, nr, c);
  long long h;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %6lld cycles/round\n", name, h);
}

int main() {
  double* d;
  long long* c;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&c, 64);
  const int T = 256;
  run<31>("full (loads dots angle stores barrier)", d, c, T);
  run<31 - 16>("no barrier", d, c, T);
  run<31 - 8>("no stores", d, c, T);
  run<31 - 4>("no angle", d, c, T);
  run<31 - 2>("no dots/shuffles", d, c, T);
  run<31 - 1>("no loads", d, c, T);
  run<16>("barrier only", d, c, T);
  run<1 | 16>("loads + barrier", d, c, T);
  run<2 | 16>("dots + barrier", d, c, T);
  run<4 | 16>("angle + barrier", d, c, T);
  run<1 | 8 | 16>("loads + stores + barrier", d, c, T);
  run<31>("full, 1024 threads", d, c, 1024);
  run<31, 16, 4>("LP16 E4 full", d, c, 512);
  run<1 | 16, 16, 4>("LP16 E4 loads + barrier", d, c, 512);
  run<1 | 8 | 16, 16, 4>("LP16 E4 loads + stores + barrier", d, c, 512);
  run<31, 32, 2>("LP32 E2 full", d, c, 1024);
  run<1 | 8 | 16, 32, 2>("LP32 E2 loads + stores + barrier", d, c, 1024);
  run<31, 4, 16>("LP4 E16 full", d, c, 256);
  run<31, 16, 2>("LP16 E2 k=20 full", d, c, 512, 20);
  run<31, 4, 8>("LP4 E8 k=20 full", d, c, 256, 20);
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
