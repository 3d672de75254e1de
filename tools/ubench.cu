// ubench.cu -- B200 microbenchmarks the roofline denominators need:
// dependent-latency of the FP64/FP32 ops the Jacobi SVD chains, FFMA and DFMA peak
// throughput, and the random 4-byte-in-32-byte-sector gather bandwidth.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench tools/ubench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void lat_dfma(double* out, int n, double a, double b) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
__global__ void lat_ffma(float* out, int n, float a, float b) {
  float x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fmaf(x, a, b);
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1000] = (float)(t1 - t0) / n;
}
__global__ void lat_shfl_dadd(double* out, int n) {
  double x = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x += __shfl_xor_sync(0xffffffffu, x, 1) * 1e-9;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
__global__ void lat_lds64(double* out, int n) {
  __shared__ double s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = (double)(i + 1) * 0;  // zeros
  __syncthreads();
  int idx = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) idx = (int)s[idx] + threadIdx.x;  // dependent chain
  long long t1 = clock64();
  out[threadIdx.x] = idx;
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
__global__ void lat_rsqrt64(double* out, int n) {
  double x = out[threadIdx.x] + 2.0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + 1.5;
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
__global__ void lat_f2f(double* out, int n) {
  double x = out[threadIdx.x] + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    float f = static_cast<float>(x);
    x = static_cast<double>(f * 1.0000001f);
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
__global__ void lat_dsetp(double* out, int n) {
  double x = out[threadIdx.x] + 1.5;
  int c = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (x * x > 2.0) c++;
    x = x * 1.0000001 + (double)(c & 1) * 1e-30;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x + c;
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
__global__ void lat_atoms(double* out, int n) {
  __shared__ int cnt;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if ((threadIdx.x & 7) == 0) atomicAdd(&cnt, 1);
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
__global__ void lat_syncthreads(double* out, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
// throughput: 8 independent chains per thread, many warps
__global__ void thr_ffma(float* out, int n) {
  float a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = out[(threadIdx.x + j) & 1023];
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], 0.999f, 0.001f);
  float s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.f) out[0] = s;
}
__global__ void thr_dfma(double* out, int n) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = out[(threadIdx.x + j) & 1023];
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], 0.999, 0.001);
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.0) out[0] = s;
}
// random-sector gather: each thread reads one float per row at column cols[t % k]
__global__ void gather_sector(const float* __restrict__ A, long long lda, long long m, const int* __restrict__ cols,
                              int k, float* __restrict__ C) {
  long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long total = m * k;
  for (long long e = tid; e < total; e += (long long)gridDim.x * blockDim.x) {
    long long r = e / k;
    int b = (int)(e % k);
    C[e] = __ldg(A + r * lda + cols[b]);
  }
}

// conversion / packed-FP32 latencies and throughputs used by the Lloyd accumulation
__global__ void lat_cvt_f32_f64(double* out, int n) {
  float f = (float)out[threadIdx.x] + 1.5f;
  double acc = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    double d = static_cast<double>(f);  // F2F.F64.F32
    acc = fma(d, 1.0000001, acc);
    f = __uint_as_float(__float_as_uint(f) ^ (static_cast<unsigned>(__double_as_longlong(acc)) & 1u));
  }
  long long t1 = clock64();
  out[threadIdx.x] = acc + f;
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
__global__ void lat_f2i64(double* out, int n) {
  double x = out[threadIdx.x] + 1.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    long long v = llrint(x);  // F2I.S64.F64
    x = static_cast<double>(v & 7) + 1.25;
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) out[1000] = (double)(t1 - t0) / n;
}
__global__ void thr_cvt(double* out, int n, int kind) {
  float f[8];
  double a[8];
  long long q[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) { f[j] = (float)out[(threadIdx.x + j) & 1023] + j; a[j] = 0; q[j] = 0; }
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (kind == 0) { a[j] += static_cast<double>(f[j]); f[j] += 1.0f; }
      else if (kind == 1) { q[j] += llrint(a[j]); a[j] += 1.0; }
      else { a[j] = fma(a[j], 0.999, 0.001); }
    }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j] + f[j] + q[j];
  if (s == 12345.0) out[0] = s;
}
__global__ void thr_ffma2(float* out, int n) {
  unsigned long long a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = __double_as_longlong((double)out[(threadIdx.x + j) & 1023]);
  const unsigned long long m = 0x3f7ff9723f7ff972ull, c = 0x3a83126f3a83126full;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(m), "l"(c));
  unsigned long long s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s ^= a[j];
  if (s == 12345) out[0] = 1.f;
}

int main() {
  double* d;
  float* f;
  CK(cudaMalloc(&d, 8 * 4096));
  CK(cudaMalloc(&f, 4 * 4096));
  CK(cudaMemset(d, 0, 8 * 4096));
  CK(cudaMemset(f, 0, 4 * 4096));
  double h;
  float hf;
  const int n = 4096;
  lat_dfma<<<1, 32>>>(d, n, 1.0000001, 1e-9);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("dependent DFMA latency      %.1f cycles\n", h);
  lat_ffma<<<1, 32>>>(f, n, 1.0000001f, 1e-9f);
  CK(cudaMemcpy(&hf, f + 1000, 4, cudaMemcpyDeviceToHost)); printf("dependent FFMA latency      %.1f cycles\n", hf);
  lat_shfl_dadd<<<1, 32>>>(d, n);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("dependent SHFL64+DFMA       %.1f cycles\n", h);
  lat_lds64<<<1, 32>>>(d, n);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("dependent LDS.64 (+cvt)     %.1f cycles\n", h);
  lat_rsqrt64<<<1, 32>>>(d, n);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("dependent rsqrt(double)+add %.1f cycles\n", h);
  lat_f2f<<<1, 32>>>(d, n);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("dependent F2F f64->f32->f64 + FMUL %.1f cycles\n", h);
  lat_dsetp<<<1, 32>>>(d, n);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("dependent DMUL+DSETP+branch %.1f cycles\n", h);
  lat_atoms<<<1, 256>>>(d, n);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("smem atomic (32 lanes) + sync %.1f cycles\n", h);
  lat_syncthreads<<<1, 1024>>>(d, n);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("__syncthreads (1024 thr)    %.1f cycles\n", h);
  CK(cudaDeviceSynchronize());
  int dev = 0, nsm = 0, clk = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int it = 20000;
  thr_ffma<<<nsm * 4, 512>>>(f, it);
  cudaEventRecord(e0);
  thr_ffma<<<nsm * 4, 512>>>(f, it);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  double fl = 2.0 * 8 * it * (double)nsm * 4 * 512;
  printf("FFMA peak                   %.1f TFLOP/s\n", fl / ms / 1e9);
  thr_dfma<<<nsm * 4, 512>>>(d, it / 4);
  cudaEventRecord(e0);
  thr_dfma<<<nsm * 4, 512>>>(d, it / 4);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  fl = 2.0 * 8 * (it / 4) * (double)nsm * 4 * 512;
  printf("DFMA peak                   %.1f TFLOP/s\n", fl / ms / 1e9);
  // random-sector gather: A 4e5 x 1e5 would be 160 GB; use 2e5 x 25000 (20 GB), k = 200 sorted random cols
  long long m = 200000, ncol = 25000, k = 200;
  float* A;
  float* Cm;
  int* cols;
  CK(cudaMalloc(&A, sizeof(float) * m * ncol));
  CK(cudaMalloc(&Cm, sizeof(float) * m * k));
  CK(cudaMalloc(&cols, sizeof(int) * k));
  int hc[200];
  for (int b = 0; b < k; ++b) hc[b] = (int)((b * 124.9) + (b * 7919) % 97);
  CK(cudaMemcpy(cols, hc, sizeof(int) * k, cudaMemcpyHostToDevice));
  CK(cudaMemset(A, 0, sizeof(float) * m * ncol));
  gather_sector<<<nsm * 8, 256>>>(A, ncol, m, cols, (int)k, Cm);
  cudaEventRecord(e0);
  gather_sector<<<nsm * 8, 256>>>(A, ncol, m, cols, (int)k, Cm);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  printf("random-sector gather        %.1f GB/s sectors (%.1f GB/s useful)\n", 32.0 * m * k / ms / 1e6,
         4.0 * m * k / ms / 1e6);
  printf("SMs %d, clock %d kHz\n", nsm, clk);
  lat_cvt_f32_f64<<<1, 32>>>(d, n);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("dependent F2F.F64.F32+DFMA+LOP %.1f cycles\n", h);
  lat_f2i64<<<1, 32>>>(d, n);
  CK(cudaMemcpy(&h, d + 1000, 8, cudaMemcpyDeviceToHost)); printf("dependent F2I.S64.F64+I2F+DADD %.1f cycles\n", h);
  const char* kn[3] = {"F2F.F64.F32 (+DADD)", "F2I.S64.F64 (+DADD,IADD)", "DFMA"};
  for (int kind = 0; kind < 3; ++kind) {
    thr_cvt<<<nsm * 4, 512>>>(d, 1000, kind);
    cudaEventRecord(e0);
    thr_cvt<<<nsm * 4, 512>>>(d, 4000, kind);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 8.0 * 4000 * nsm * 4 * 512;
    printf("throughput %-26s %.1f G ops/s = %.1f per SM per clock\n", kn[kind], ops / ms / 1e6,
           ops / ms / 1e6 / nsm / (clk / 1e6));
  }
  thr_ffma2<<<nsm * 4, 512>>>(f, 1000);
  cudaEventRecord(e0);
  thr_ffma2<<<nsm * 4, 512>>>(f, 10000);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  printf("FFMA2 peak                  %.1f TFLOP/s\n", 4.0 * 8 * 10000 * (double)nsm * 4 * 512 / ms / 1e9);
  return 0;
}
