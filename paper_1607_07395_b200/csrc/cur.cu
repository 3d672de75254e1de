// cur.cu -- SURVEY NEXT-4 on the same kernels: the middle matrix of BR-CUR (Algorithm 1,
// PAPER.md P:83-103; Sketch-CUR P:115 is BR-CUR with independent uniform targets), and the
// rank sweep on a validation block.
//
// BR-CUR: U* = C_bar^+ M R_bar^+ (step 4's minimum-norm least-squares solution).  C_bar
// (k2 x k1) and R_bar (k1 x k2) are zero-padded to k2 x k2 so that the FP64 Jacobi SVD of
// svd.cu / svd_cluster.cu serves them: the padding adds zero singular values only (dropped by
// the tol rule), so pinv(pad) restricted to the first k1 rows / columns is the pseudo-inverse.
// The products run in FP64 (small_gemm_kernel); F = C U* (FP32, the tiled apply of orth.cu)
// and G = R^T give A ~ F G^T for cabs_residual.
//
// Rank sweep: e[rho] = ||B - U_H[:, :rho] S V_H[:, :rho]^T||^2, rho = 0..r, on B = A(Hr, Hc),
// through the expansion ||B||^2 - 2 sum_{t<rho} s_t u_t^T B v_t + sum_{t,t'<rho} s_t s_t'
// (U_H^T U_H)_{tt'} (V_H^T V_H)_{tt'} (FP64; the Gram products from orth.cu's Gram kernels),
// accumulated over rho in a fixed order.
#include <float.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cabsk {

constexpr int kCurT = 256;

// C[i, j] = sum_q A(i, q) d(q) B(q, j), A(i, q) = A[i * a_rs + q * a_cs], B(q, j) = B[q * b_rs + j * b_cs]
// (any transposition by the strides), d = NULL -> 1; FP64, one thread per output, q in order.
__global__ void __launch_bounds__(kCurT) small_gemm_kernel(int M, int N, int K, const double* __restrict__ A,
                                                           int64_t a_rs, int64_t a_cs, const double* __restrict__ d,
                                                           const double* __restrict__ B, int64_t b_rs, int64_t b_cs,
                                                           double* __restrict__ Cm, int64_t ldc) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * kCurT + threadIdx.x;
  if (e >= static_cast<int64_t>(M) * N) return;
  const int i = static_cast<int>(e / N), j = static_cast<int>(e % N);
  double s = 0.0;
  for (int q = 0; q < K; ++q) s = fma(A[i * a_rs + q * a_cs] * (d ? d[q] : 1.0), B[q * b_rs + j * b_cs], s);
  Cm[static_cast<int64_t>(i) * ldc + j] = s;
}

static void small_gemm(int M, int N, int K, const double* A, int64_t a_rs, int64_t a_cs, const double* d,
                       const double* B, int64_t b_rs, int64_t b_cs, double* Cm, int64_t ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return;
  note_launch();
  small_gemm_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(M) * N, kCurT)), kCurT, 0, st>>>(
      M, N, K, A, a_rs, a_cs, d, B, b_rs, b_cs, Cm, ldc);
}

// out[i, c] = src[i, cols[c]] (c < nc) as FP32 (ld ldo), columns [nc, pad) zero; rows < nr; FP64
// copy to out64 (ld nc) when given
__global__ void __launch_bounds__(kCurT) pick_cols_kernel(const float* __restrict__ src, int64_t lds, int nr,
                                                          const int64_t* __restrict__ cols, int nc, int pad,
                                                          float* out, int64_t ldo, double* out64) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * kCurT + threadIdx.x;
  if (e >= static_cast<int64_t>(nr) * pad) return;
  const int i = static_cast<int>(e / pad), c = static_cast<int>(e % pad);
  const float v = c < nc ? src[static_cast<int64_t>(i) * lds + cols[c]] : 0.f;
  if (out) out[static_cast<int64_t>(i) * ldo + c] = v;
  if (out64 && c < nc) out64[static_cast<int64_t>(i) * nc + c] = static_cast<double>(v);
}

// out[a, c] = X[rows[a], c] for c < ncol (FP32, ld ldo, zero to pad) and / or FP64 (ld ncol)
__global__ void __launch_bounds__(kCurT) pick_rows_kernel(const float* __restrict__ X, int64_t ldx,
                                                          const int64_t* __restrict__ rows, int nr, int ncol, int pad,
                                                          float* out, int64_t ldo, double* out64) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * kCurT + threadIdx.x;
  if (e >= static_cast<int64_t>(nr) * pad) return;
  const int a = static_cast<int>(e / pad), c = static_cast<int>(e % pad);
  const float v = c < ncol ? X[rows[a] * ldx + c] : 0.f;
  if (out) out[static_cast<int64_t>(a) * ldo + c] = v;
  if (out64 && c < ncol) out64[static_cast<int64_t>(a) * ncol + c] = static_cast<double>(v);
}

void launch_pick_rows(const float* X, int64_t ldx, const int64_t* rows, int nr, int ncol, int pad, float* out,
                      int64_t ldo, double* out64, cudaStream_t st) {
  if (nr <= 0 || pad <= 0) return;
  note_launch();
  pick_rows_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(nr) * pad, kCurT)), kCurT, 0, st>>>(
      X, ldx, rows, nr, ncol, pad, out, ldo, out64);
}

// rows [nr, npad) of a FP32 matrix zeroed (columns < ncol)
__global__ void __launch_bounds__(kCurT) zero_rows_kernel(float* X, int64_t ldx, int nr, int npad, int ncol) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * kCurT + threadIdx.x;
  if (e >= static_cast<int64_t>(npad - nr) * ncol) return;
  X[(nr + e / ncol) * ldx + e % ncol] = 0.f;
}

// G[j, c] = R[c, j] (n x k, ld ldg) from R (k x n, ld ldr); 32 x 32 tiles through shared memory
__global__ void __launch_bounds__(kCurT) transpose_kernel(const float* __restrict__ R, int64_t ldr, int k, int64_t n,
                                                          float* G, int64_t ldg) {
  __shared__ float t[32][33];
  const int64_t j0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int c0 = blockIdx.y * 32;
  for (int y = threadIdx.x >> 5; y < 32; y += kCurT / 32) {
    const int c = c0 + y;
    const int64_t j = j0 + (threadIdx.x & 31);
    t[y][threadIdx.x & 31] = (c < k && j < n) ? R[c * ldr + j] : 0.f;
  }
  __syncthreads();
  for (int y = threadIdx.x >> 5; y < 32; y += kCurT / 32) {
    const int64_t j = j0 + y;
    const int c = c0 + (threadIdx.x & 31);
    if (j < n && c < k) G[j * ldg + c] = t[threadIdx.x & 31][y];
  }
}

// d[q] = 1 / sigma_q for sigma_q > tol sigma_0, else 0 (the pseudo-inverse's truncation)
__global__ void pinv_diag_kernel(const double* __restrict__ sig, int k, double tol, double* d) {
  for (int q = threadIdx.x; q < k; q += blockDim.x) d[q] = (sig[0] > 0 && sig[q] > tol * sig[0]) ? 1.0 / sig[q] : 0.0;
}

__global__ void to_f32_kernel(const double* __restrict__ X, int rows, int cols, float* Y, int64_t ldy, int pad) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * kCurT + threadIdx.x;
  if (e >= static_cast<int64_t>(rows) * pad) return;
  const int i = static_cast<int>(e / pad), c = static_cast<int>(e % pad);
  Y[i * ldy + c] = c < cols ? static_cast<float>(X[static_cast<int64_t>(i) * cols + c]) : 0.f;
}

void launch_pick_cols(const float* src, int64_t lds, int nr, const int64_t* cols, int nc, int pad, float* out,
                      int64_t ldo, double* out64, cudaStream_t st) {
  if (nr <= 0 || pad <= 0) return;
  note_launch();
  pick_cols_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(nr) * pad, kCurT)), kCurT, 0, st>>>(
      src, lds, nr, cols, nc, pad, out, ldo, out64);
}

void launch_transpose(const float* R, int64_t ldr, int k, int64_t n, float* G, int64_t ldg, cudaStream_t st) {
  if (k <= 0 || n <= 0) return;
  note_launch();
  transpose_kernel<<<dim3(static_cast<unsigned>(ceil_div(n, 32)), static_cast<unsigned>(ceil_div(k, 32))), kCurT, 0,
                     st>>>(R, ldr, k, n, G, ldg);
}

// U* (k1 x k1, FP64 row-major) from the SVDs of the padded C_bar (U1, V1, sig1) and R_bar (U2, V2,
// sig2), all k2 x k2 (ld k2), and M (k2 x k2 FP64): X1 = V1[:k1] diag(d1) U1^T (k1 x k2),
// Y = X1 M, X2 = V2 diag(d2) U2[:k1]^T (k2 x k1), U* = Y X2.
void launch_cur_middle(int k1, int k2, const double* U1, const double* V1, const double* sig1, const double* U2,
                       const double* V2, const double* sig2, double tol, const double* M, double* d1, double* d2,
                       double* X1, double* Y, double* X2, double* Ustar, cudaStream_t st) {
  note_launch();
  pinv_diag_kernel<<<1, 256, 0, st>>>(sig1, k2, tol, d1);
  note_launch();
  pinv_diag_kernel<<<1, 256, 0, st>>>(sig2, k2, tol, d2);
  small_gemm(k1, k2, k2, V1, k2, 1, d1, U1, 1, k2, X1, k2, st);  // X1[i,t] = sum_q V1[i,q] d1 U1[t,q]
  small_gemm(k1, k2, k2, X1, k2, 1, nullptr, M, k2, 1, Y, k2, st);
  small_gemm(k2, k1, k2, V2, k2, 1, d2, U2, 1, k2, X2, k1, st);  // X2[t,j] = sum_q V2[t,q] d2 U2[j,q]
  small_gemm(k1, k1, k2, Y, k2, 1, nullptr, X2, k1, 1, Ustar, k1, st);
}

void launch_f32_of(const double* X, int rows, int cols, float* Y, int64_t ldy, int pad, cudaStream_t st) {
  note_launch();
  to_f32_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(rows) * pad, kCurT)), kCurT, 0, st>>>(
      X, rows, cols, Y, ldy, pad);
}

void launch_zero_rows(float* X, int64_t ldx, int nr, int npad, int ncol, cudaStream_t st) {
  if (npad <= nr || ncol <= 0) return;
  note_launch();
  zero_rows_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(npad - nr) * ncol, kCurT)), kCurT, 0, st>>>(
      X, ldx, nr, npad, ncol);
}

// ---------------------------------------------------------------- rank sweep
// a_t = sum_i U_H[i, t] (B V_H)[i, t]; inc[rho] (rho = 1..r) = e[rho] - e[rho - 1]; then the prefix in order
__global__ void __launch_bounds__(kCurT) sweep_kernel(const double* __restrict__ B, int hr, int hc,
                                                      const double* __restrict__ W1, const double* __restrict__ UH,
                                                      const float* __restrict__ s, const double* __restrict__ gram,
                                                      int r, double* err) {
  extern __shared__ double inc[];  // [r + 1]
  __shared__ double s_b2[kCurT];
  const double* Gu = gram;
  const double* Gv = gram + static_cast<int64_t>(r) * r;
  double b2 = 0.0;
  for (int64_t e = threadIdx.x; e < static_cast<int64_t>(hr) * hc; e += kCurT) b2 = fma(B[e], B[e], b2);
  s_b2[threadIdx.x] = b2;
  for (int t = threadIdx.x; t < r; t += kCurT) {
    double at = 0.0;
    for (int i = 0; i < hr; ++i) at = fma(UH[static_cast<int64_t>(i) * r + t], W1[static_cast<int64_t>(i) * r + t], at);
    const double st = static_cast<double>(s[t]);
    double cross = 0.0;
    for (int u = 0; u < t; ++u) cross = fma(static_cast<double>(s[u]) * Gu[u * r + t], Gv[u * r + t], cross);
    inc[t + 1] = -2.0 * st * at + st * st * Gu[t * r + t] * Gv[t * r + t] + 2.0 * st * cross;
  }
  __syncthreads();
  for (int w = kCurT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s_b2[threadIdx.x] += s_b2[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double e = s_b2[0];
    err[0] = e;
    for (int rho = 1; rho <= r; ++rho) {
      e += inc[rho];
      err[rho] = e;
    }
  }
}

void launch_sweep(const double* B, int hr, int hc, const double* VH, const double* UH, const float* s,
                  const double* gram, int r, double* W1, double* err, cudaStream_t st) {
  small_gemm(hr, r, hc, B, hc, 1, nullptr, VH, r, 1, W1, r, st);  // W1 = B V_H
  note_launch();
  sweep_kernel<<<1, kCurT, sizeof(double) * (r + 1), st>>>(B, hr, hc, W1, UH, s, gram, r, err);
}

}  // namespace cabsk
