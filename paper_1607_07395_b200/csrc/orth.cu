// Orthogonalization of a sketch (Supp. section 3).
//
// The paper's recipe -- U = U0 S0 V0^T, then S0 V0^T diag(s) V^T = U1 S1 V1^T, result
// (U0 U1, S1, V1) -- is the thin SVD of U diag(s) V^T.  The B200 path reaches the same unique
// factors through r x r work only (O((m + n) r^2) in total, the paper's cost):
//   orth_gram_kernel    G_U = U^T U and G_V = V^T V, FP64 (products of FP32 entries are
//                       exact), per-CTA partials over a fixed row partition
//   orth_reduce_kernel  fixed-order sum of the partials (deterministic; then an allreduce
//                       across ranks)
//   orth_core_kernel    Cholesky G_U = R_U^T R_U, G_V = R_V^T R_V (FP64, one CTA), core
//                       K = R_U diag(s) R_V^T -> FP32 for the Jacobi SVD K = U_K S_K V_K^T
//   orth_solve_kernel   T_U = R_U^-1 U_K, T_V = R_V^-1 V_K (back substitution, FP64)
//   orth_apply_kernel   U_o = U T_U, V_o = V T_V (FP32, T staged in shared memory)
// so U diag(s) V^T = (U R_U^-1) K (V R_V^-1)^T = (U T_U) S_K (V T_V)^T with orthonormal
// U R_U^-1, V R_V^-1.  r <= 64 (the two-SM Jacobi SVD).
#include "common.cuh"
#include "kernels.cuh"

namespace cabsk {

constexpr int kOrthThreads = 256;
constexpr int kOrthRows = 32;  // rows staged per step of the Gram kernel

// Problem q of CTA b: rows [b * chunk, ...) of X_q, partial Gram to part + (q * nblk + b) * r * r.
__global__ void __launch_bounds__(kOrthThreads) orth_gram_kernel(OrthArgs a) {
  __shared__ float xs[kOrthRows][65];
  const int q = static_cast<int>(blockIdx.x) >= a.nblk;
  const int b = q ? blockIdx.x - a.nblk : blockIdx.x;
  const float* __restrict__ X = q ? a.V : a.U;
  const int64_t ld = q ? a.ldv : a.ldu, N = q ? a.nv : a.nu;
  const int r = a.r, rr = r * r;
  double acc[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = 0.0;
  const int64_t per = (N + a.nblk - 1) / a.nblk;
  const int64_t lo = b * per, hi = lo + per < N ? lo + per : N;
  for (int64_t r0 = lo; r0 < hi; r0 += kOrthRows) {
    const int nr = hi - r0 < kOrthRows ? static_cast<int>(hi - r0) : kOrthRows;
    __syncthreads();
    for (int e = threadIdx.x; e < kOrthRows * r; e += kOrthThreads) {
      const int i = e / r, c = e % r;
      xs[i][c] = i < nr ? X[(r0 + i) * ld + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int e = threadIdx.x + kOrthThreads * j;
      if (e < rr) {
        const int ca = e / r, cb = e % r;
        double s = acc[j];
        for (int i = 0; i < nr; ++i) s = fma(static_cast<double>(xs[i][ca]), static_cast<double>(xs[i][cb]), s);
        acc[j] = s;
      }
    }
  }
  double* out = a.part + (static_cast<int64_t>(q) * a.nblk + b) * rr;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int e = threadIdx.x + kOrthThreads * j;
    if (e < rr) out[e] = acc[j];
  }
}

__global__ void __launch_bounds__(kOrthThreads) orth_reduce_kernel(OrthArgs a) {
  const int q = blockIdx.x, rr = a.r * a.r;
  const double* p = a.part + static_cast<int64_t>(q) * a.nblk * rr;
  for (int e = threadIdx.x; e < rr; e += kOrthThreads) {
    double s = 0.0;
    for (int b = 0; b < a.nblk; ++b) s += p[static_cast<int64_t>(b) * rr + e];
    a.gram[q * 64 * 64 + (e / a.r) * 64 + e % a.r] = s;
  }
}

// In-place right-looking Cholesky of the r x r matrix A (row-major, ld 64) into its upper
// factor R (A = R^T R); entries below the diagonal are zeroed.  A zero pivot (an all-zero
// column) leaves a zero row of R, whose component then drops out; returns false on a negative
// or NaN pivot (a numerically rank-deficient factor).
__device__ bool orth_cholesky(double* A, int r, double* s_piv) {
  bool ok = true;
  for (int j = 0; j < r; ++j) {
    if (threadIdx.x == 0) {
      const double d = A[j * 64 + j];
      *s_piv = d > 0.0 ? sqrt(d) : (d == 0.0 ? 0.0 : -1.0);
    }
    __syncthreads();
    double p = *s_piv;
    ok = ok && p >= 0.0;  // an exactly-zero column (zero padding of a truncated factor) is dropped
    p = p > 0.0 ? p : 0.0;
    const double ip = p > 0.0 ? 1.0 / p : 0.0;
    for (int c = j + threadIdx.x; c < r; c += kOrthThreads) A[j * 64 + c] = c == j ? p : A[j * 64 + c] * ip;
    __syncthreads();
    const int t = r - j - 1;  // trailing (a, b), j < a <= b
    for (int e = threadIdx.x; e < t * t; e += kOrthThreads) {
      const int ia = j + 1 + e / t, ib = j + 1 + e % t;
      if (ia <= ib) A[ia * 64 + ib] -= A[j * 64 + ia] * A[j * 64 + ib];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < r * r; e += kOrthThreads)
    if (e / r > e % r) A[(e / r) * 64 + e % r] = 0.0;
  __syncthreads();
  return ok;
}

// One CTA: R_U, R_V (to ws), K = R_U diag(s) R_V^T as FP32 (ld kp) for the Jacobi SVD.
__global__ void __launch_bounds__(kOrthThreads) orth_core_kernel(OrthArgs a, void* ws) {
  __shared__ double s_piv;
  const int r = a.r;
  double* RU = a.gram;            // in place: G_U -> R_U
  double* RV = a.gram + 64 * 64;  // G_V -> R_V
  const bool ok1 = orth_cholesky(RU, r, &s_piv);
  const bool ok2 = orth_cholesky(RV, r, &s_piv);
  if (threadIdx.x == 0 && !(ok1 && ok2)) set_status(ws, CABS_DEV_ORTH_RANK);
  for (int e = threadIdx.x; e < r * r; e += kOrthThreads) {
    const int i = e / r, j = e % r;
    double sum = 0.0;  // sum_l R_U[i][l] s_l R_V[j][l], l >= max(i, j)
    for (int l = i > j ? i : j; l < r; ++l)
      sum = fma(RU[i * 64 + l] * (a.s ? static_cast<double>(a.s[l]) : 1.0), RV[j * 64 + l], sum);
    a.K[static_cast<int64_t>(i) * a.kp + j] = static_cast<float>(sum);
  }
}

// One CTA per side: T = R^-1 M (R upper triangular, M = U_K or V_K, k x k row-major FP64)
// by back substitution, row by row from the bottom; 4 threads per right-hand side column.
// Side 0 also writes s_out (FP32) and r_out from the SVD.
__global__ void __launch_bounds__(kOrthThreads) orth_solve_kernel(OrthArgs a) {
  __shared__ double T[64][65];
  const int q = blockIdx.x, r = a.r;
  const double* R = a.gram + q * 64 * 64;
  const double* M = q ? a.VK : a.UK;
  float* out = q ? a.TV : a.TU;
  const int c = threadIdx.x >> 2, part = threadIdx.x & 3;
  for (int i = r - 1; i >= 0; --i) {
    double sum = 0.0;
    if (c < r)
      for (int l = i + 1 + part; l < r; l += 4) sum = fma(R[i * 64 + l], T[l][c], sum);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (c < r && part == 0) {
      const double d = R[i * 64 + i];
      T[i][c] = d > 0.0 ? (M[static_cast<int64_t>(i) * r + c] - sum) / d : 0.0;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < r * a.kp; e += kOrthThreads) {
    const int i = e / a.kp, j = e % a.kp;
    out[e] = j < r ? static_cast<float>(T[i][j]) : 0.f;
  }
  if (q == 0) {
    const int rk = *a.r_svd;
    for (int j = threadIdx.x; j < r; j += kOrthThreads) a.s_out[j] = j < rk ? static_cast<float>(a.sig[j]) : 0.f;
    if (threadIdx.x == 0 && a.r_out) *a.r_out = rk;
  }
}

// Out[l][:] = X[l][:r] T (T r x kp FP32 in shared memory), columns [r, ldo) zero.  Grid:
// blocks of 64 rows, first the U side (nbu blocks), then the V side.
__global__ void __launch_bounds__(kOrthThreads) orth_apply_kernel(OrthArgs a, int nbu) {
  __shared__ float Ts[64][64];
  __shared__ float xs[64][65];
  const int q = static_cast<int>(blockIdx.x) >= nbu;
  const int64_t b = q ? blockIdx.x - nbu : blockIdx.x;
  const float* __restrict__ X = q ? a.V : a.U;
  const int64_t ldx = q ? a.ldv : a.ldu, N = q ? a.nv : a.nu;
  float* __restrict__ O = q ? a.Vo : a.Uo;
  const int64_t ldo = q ? a.ldvo : a.lduo;
  const float* T = q ? a.TV : a.TU;
  const int r = a.r;
  for (int e = threadIdx.x; e < 64 * 64; e += kOrthThreads) {
    const int i = e / 64, j = e % 64;
    Ts[i][j] = (i < r && j < r) ? T[static_cast<int64_t>(i) * a.kp + j] : 0.f;
  }
  const int64_t r0 = b * 64;
  const int nr = N - r0 < 64 ? static_cast<int>(N - r0) : 64;
  for (int e = threadIdx.x; e < 64 * 64; e += kOrthThreads) {
    const int i = e / 64, c = e % 64;
    xs[i][c] = (i < nr && c < r) ? X[(r0 + i) * ldx + c] : 0.f;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < nr * ldo; e += kOrthThreads) {
    const int i = static_cast<int>(e / ldo), j = static_cast<int>(e % ldo);
    float sum = 0.f;
    if (j < r)
      for (int l = 0; l < r; ++l) sum = fmaf(xs[i][l], Ts[l][j], sum);
    O[(r0 + i) * ldo + j] = sum;
  }
}

int orth_gram_blocks(int64_t nu, int64_t nv) {
  const int64_t n = nu > nv ? nu : nv;
  const int64_t b = ceil_div(n > 0 ? n : 1, 512);
  return static_cast<int>(b < kOrthMaxBlocks ? b : kOrthMaxBlocks);
}

void launch_orth_gram(OrthArgs& a, cudaStream_t st) {
  note_launch();
  orth_gram_kernel<<<2 * a.nblk, kOrthThreads, 0, st>>>(a);
  note_launch();
  orth_reduce_kernel<<<2, kOrthThreads, 0, st>>>(a);
}

void launch_orth_core(const OrthArgs& a, void* ws, cudaStream_t st) {
  note_launch();
  orth_core_kernel<<<1, kOrthThreads, 0, st>>>(a, ws);
}

void launch_orth_finish(const OrthArgs& a, cudaStream_t st) {
  note_launch();
  orth_solve_kernel<<<2, kOrthThreads, 0, st>>>(a);
  const int64_t nbu = ceil_div(a.nu, 64), nbv = ceil_div(a.nv, 64);
  if (nbu + nbv == 0) return;
  note_launch();
  orth_apply_kernel<<<static_cast<unsigned>(nbu + nbv), kOrthThreads, 0, st>>>(a, static_cast<int>(nbu));
}

}  // namespace cabsk
