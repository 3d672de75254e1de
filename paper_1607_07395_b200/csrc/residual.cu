// residual.cu -- S10: the evaluation ||A - F diag(s) G^T||_F, fused.
//
// Each CTA forms 128 x 128 tiles of F diag(s) G^T in registers (FP32 FFMA, K =
// ncomp ascending), streams the matching tile of A, and accumulates (a - a~)^2 and
// a^2; the reconstruction is never written.  Persistent grid with a static
// tile -> CTA map, FP64 per-thread accumulators and fixed-order block / grid
// reductions, so the result is bit-reproducible run to run.
#include "common.cuh"
#include "kernels.cuh"

namespace cabsk {

constexpr int kRBM = 128, kRBN = 128, kRBK = 8;

__global__ void __launch_bounds__(256) residual_ffma_kernel(const float* __restrict__ A, int64_t lda, int64_t m,
                                                            int64_t n, const float* __restrict__ F, int64_t ldf,
                                                            const float* __restrict__ s, const float* __restrict__ G,
                                                            int64_t ldg, int K, double* __restrict__ part) {
  __shared__ __align__(16) float Fs[kRBK][kRBM];
  __shared__ __align__(16) float Gs[kRBK][kRBN];
  __shared__ double red[2][8];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t ntr = ceil_div(m, kRBM), ntc = ceil_div(n, kRBN);
  const int64_t ntiles = ntr * ntc;
  double r2 = 0.0, a2 = 0.0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t r0 = (t / ntc) * kRBM, c0 = (t % ntc) * kRBN;
    float acc[8][8] = {};
    for (int k0 = 0; k0 < K; k0 += kRBK) {
      {  // 128 rows x 8 k of F and of G (scaled by s): 4 elements per thread each
        const int row = tid >> 1, kk = (tid & 1) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int kc = k0 + kk + q;
          const int64_t gr = r0 + row, gc = c0 + row;
          Fs[kk + q][row] = (gr < m && kc < K) ? __ldg(F + gr * ldf + kc) : 0.f;
          const float sk = (kc < K) ? (s ? __ldg(s + kc) : 1.f) : 0.f;
          Gs[kk + q][row] = (gc < n && kc < K) ? __ldg(G + gc * ldg + kc) * sk : 0.f;
        }
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < kRBK; ++kk) {
        float a[8], b[8];
        const float4 a0 = *reinterpret_cast<const float4*>(&Fs[kk][ty * 4]);
        const float4 a1 = *reinterpret_cast<const float4*>(&Fs[kk][64 + ty * 4]);
        const float4 b0 = *reinterpret_cast<const float4*>(&Gs[kk][tx * 4]);
        const float4 b1 = *reinterpret_cast<const float4*>(&Gs[kk][64 + tx * 4]);
        a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
        a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
        b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
        b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
          for (int v = 0; v < 8; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
      }
      __syncthreads();
    }
    float tr = 0.f, ta = 0.f;
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t gr = r0 + (u < 4 ? ty * 4 + u : 64 + ty * 4 + (u - 4));
      if (gr >= m) continue;
      const float* arow = A + gr * lda;
#pragma unroll
      for (int v = 0; v < 8; ++v) {
        const int64_t gc = c0 + (v < 4 ? tx * 4 + v : 64 + tx * 4 + (v - 4));
        if (gc < n) {
          const float av = __ldg(arow + gc);
          const float e = av - acc[u][v];
          tr = fmaf(e, e, tr);
          ta = fmaf(av, av, ta);
        }
      }
    }
    r2 += static_cast<double>(tr);
    a2 += static_cast<double>(ta);
  }
  r2 = warp_sum_d(r2);
  a2 = warp_sum_d(a2);
  if ((tid & 31) == 0) {
    red[0][tid >> 5] = r2;
    red[1][tid >> 5] = a2;
  }
  __syncthreads();
  if (tid == 0) {
    double x = 0, y = 0;
    for (int q = 0; q < 8; ++q) { x += red[0][q]; y += red[1][q]; }
    part[2 * blockIdx.x] = x;
    part[2 * blockIdx.x + 1] = y;
  }
}

__global__ void __launch_bounds__(256) residual_final_kernel(const double* __restrict__ part, int G, double* out) {
  __shared__ double s0[256], s1[256];
  double x = 0, y = 0;
  for (int b = threadIdx.x; b < G; b += blockDim.x) { x += part[2 * b]; y += part[2 * b + 1]; }
  s0[threadIdx.x] = x;
  s1[threadIdx.x] = y;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) { s0[threadIdx.x] += s0[threadIdx.x + w]; s1[threadIdx.x] += s1[threadIdx.x + w]; }
    __syncthreads();
  }
  if (threadIdx.x == 0) { out[0] = s0[0]; out[1] = s1[0]; }
}

void launch_residual_final(const double* part, int G, double* out, cudaStream_t st) {
  note_launch();
  residual_final_kernel<<<1, 256, 0, st>>>(part, G, out);
}

int launch_residual(const float* A, int64_t lda, int64_t m_loc, int64_t n, const float* F, int64_t ldf, const float* s,
                    const float* G, int64_t ldg, int ncomp, double* part, double* out, cudaStream_t st) {
  const int64_t ntiles = ceil_div(m_loc, kRBM) * ceil_div(n, kRBN);
  int64_t g = ntiles < kResGrid ? ntiles : kResGrid;
  if (g < 1) g = 1;
  if (m_loc > 0 && n > 0) {
    note_launch();
    residual_ffma_kernel<<<static_cast<unsigned>(g), 256, 0, st>>>(A, lda, m_loc, n, F, ldf, s, G, ldg, ncomp, part);
  } else {
    cudaMemsetAsync(part, 0, sizeof(double) * 2 * g, st);
  }
  launch_residual_final(part, static_cast<int>(g), out, st);
  return 0;
}

}  // namespace cabsk
