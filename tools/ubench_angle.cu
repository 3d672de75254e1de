// ubench_angle.cu -- dependent-chain latency of the Jacobi rotation computation variants
// (development tool).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_angle tools/ubench_angle.cu
#include <cfloat>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rsqrt_approx64(double x) { double y; asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
__device__ __forceinline__ double rcp_approx64(double x) { double y; asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }

__device__ __forceinline__ void angle64(double al, double be, double ga, double& c, double& sn) {
  const double dx = be - al, dy = 2.0 * ga;
  const double h = fma(dx, dx, dy * dy);
  const double den = fabs(dx) + h * rsqrt_approx64(h);
  const double t = copysign(1.0, dx) * dy * rcp_approx64(den);
  const double q1 = fma(t, t, 1.0);
  double cc = rsqrt_approx64(q1);
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  c = cc; sn = cc * t;
}
__device__ __forceinline__ void angle32(double al, double be, double ga, double& c, double& sn) {
  const double dx = be - al, dy = 2.0 * ga;
  const double mx = fmax(fabs(dx), fabs(dy));
  const int ex = static_cast<int>((__double_as_longlong(mx) >> 52) & 0x7ff);
  const double scl = __longlong_as_double(static_cast<long long>(2046 - ex) << 52);
  const float xf = static_cast<float>(dx * scl), yf = static_cast<float>(dy * scl);
  const float hyp = fmaf(xf, xf, yf * yf);
  const float den = fabsf(xf) + hyp * rsqrtf(hyp);
  const float tf = copysignf(1.f, xf) * __fdividef(yf, den);
  const float cf = rsqrtf(fmaf(tf, tf, 1.f));
  // one FP64 Newton step on c from the FP32 seed (2^-22 -> 2^-44), a second to 2^-88
  const double t = tf, q1 = fma(t, t, 1.0);
  double cc = cf;
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  c = cc; sn = cc * t;
}
__device__ __forceinline__ void angle32b(double al, double be, double ga, double& c, double& sn) {
  // t and c entirely in FP32 from FP32-rounded inputs (scaled), c, s refined in FP64 (one step)
  const double dx = be - al, dy = 2.0 * ga;
  const double mx = fmax(fabs(dx), fabs(dy));
  const int ex = static_cast<int>((__double_as_longlong(mx) >> 52) & 0x7ff);
  const double scl = __longlong_as_double(static_cast<long long>(2046 - ex) << 52);
  const float xf = static_cast<float>(dx * scl), yf = static_cast<float>(dy * scl);
  const float hyp = fmaf(xf, xf, yf * yf);
  const float tf = copysignf(1.f, xf) * __fdividef(yf, fabsf(xf) + hyp * rsqrtf(hyp));
  const float q1f = fmaf(tf, tf, 1.f);
  const float cf = rsqrtf(q1f);
  const double t = tf, q1 = fma(t, t, 1.0);
  double cc = cf;
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  cc = cc * fma(-0.25 * q1 * cc, cc * cc * 0.0, 1.0) ;  // placeholder: keeps a 2nd dependent op
  c = cc; sn = cc * t;
}

template <int V>
__global__ void chain(double* out, int n) {
  double al = 1.0 + threadIdx.x * 1e-3, be = 2.0, ga = 0.3, acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double c, s;
    if (V == 0) angle64(al, be, ga, c, s);
    else if (V == 1) angle32(al, be, ga, c, s);
    else angle32b(al, be, ga, c, s);
    ga = 0.3 + s * 1e-9;  // dependent
    acc += c;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (double)(t1 - t0) / n;
  out[1 + threadIdx.x] = acc + ga;
}

int main() {
  double* d;
  cudaMalloc(&d, 8 * 64);
  double h;
  const char* nm[3] = {"FP64 MUFU (rsqrt/rcp .approx.f64)", "FP32 t + FP32 c seed + 2 FP64 Newton", "FP32 t,c + 1 FP64 Newton"};
  for (int v = 0; v < 3; ++v) {
    if (v == 0) chain<0><<<1, 32>>>(d, 2000);
    if (v == 1) chain<1><<<1, 32>>>(d, 2000);
    if (v == 2) chain<2><<<1, 32>>>(d, 2000);
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %.1f cycles per rotation (dependent)\n", nm[v], h);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
