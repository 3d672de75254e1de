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
  __shared__ __align__(16) double xs[kOrthRows][64];  // converted once per element, zero-padded to 64 columns
  const int q = static_cast<int>(blockIdx.x) >= a.nblk;
  const int b = q ? blockIdx.x - a.nblk : blockIdx.x;
  const float* __restrict__ X = q ? a.V : a.U;
  const int64_t ld = q ? a.ldv : a.ldu, N = q ? a.nv : a.nu;
  const int r = a.r, rr = r * r;
  // thread t owns the 4 x 4 block of entries (4 (t / 16) + i, 4 (t % 16) + j)
  const int A0 = 4 * (threadIdx.x >> 4), B0 = 4 * (threadIdx.x & 15);
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  const int64_t per = (N + a.nblk - 1) / a.nblk;
  const int64_t lo = b * per, hi = lo + per < N ? lo + per : N;
  for (int64_t r0 = lo; r0 < hi; r0 += kOrthRows) {
    const int nr = hi - r0 < kOrthRows ? static_cast<int>(hi - r0) : kOrthRows;
    __syncthreads();
    for (int e = threadIdx.x; e < kOrthRows * 64; e += kOrthThreads) {
      const int i = e >> 6, c = e & 63;
      xs[i][c] = (i < nr && c < r) ? static_cast<double>(X[(r0 + i) * ld + c]) : 0.0;
    }
    __syncthreads();
    for (int i = 0; i < nr; ++i) {
      const double2 a01 = *reinterpret_cast<const double2*>(&xs[i][A0]);
      const double2 a23 = *reinterpret_cast<const double2*>(&xs[i][A0 + 2]);
      const double2 b01 = *reinterpret_cast<const double2*>(&xs[i][B0]);
      const double2 b23 = *reinterpret_cast<const double2*>(&xs[i][B0 + 2]);
      const double xa[4] = {a01.x, a01.y, a23.x, a23.y}, xb[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(xa[u], xb[v], acc[u][v]);  // exact products
    }
  }
  double* out = a.part + (static_cast<int64_t>(q) * a.nblk + b) * rr;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v)
      if (A0 + u < r && B0 + v < r) out[(A0 + u) * r + B0 + v] = acc[u][v];
}

// one thread per (side, entry); the partials are added in CTA order (deterministic)
__global__ void __launch_bounds__(kOrthThreads) orth_reduce_kernel(OrthArgs a) {
  const int rr = a.r * a.r;
  const int t = blockIdx.x * kOrthThreads + threadIdx.x;
  if (t >= 2 * rr) return;
  const int q = t >= rr, e = q ? t - rr : t;
  const double* p = a.part + static_cast<int64_t>(q) * a.nblk * rr + e;
  double s = 0.0;
  int b = 0;
  for (; b + 8 <= a.nblk; b += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = p[static_cast<int64_t>(b + j) * rr];
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  for (; b < a.nblk; ++b) s += p[static_cast<int64_t>(b) * rr];
  a.gram[q * 64 * 64 + (e / a.r) * 64 + e % a.r] = s;
}

// In-place right-looking Cholesky of the two r x r matrices A[0], A[1] (row-major, ld 64,
// consecutive) into their upper factors R (A = R^T R) in one loop; entries below the diagonal
// are zeroed.  A zero pivot (an all-zero column) leaves a zero row of R, whose component then
// drops out; returns false on a negative or NaN pivot (a numerically rank-deficient factor).
__device__ bool orth_cholesky2(double* A, int r, double* s_piv) {
  bool ok = true;
  for (int j = 0; j < r; ++j) {
    if (threadIdx.x < 2) {
      const double d = A[threadIdx.x * 4096 + j * 64 + j];
      s_piv[threadIdx.x] = d > 0.0 ? sqrt(d) : (d == 0.0 ? 0.0 : -1.0);
    }
    __syncthreads();
    const double p0 = s_piv[0], p1 = s_piv[1];
    ok = ok && p0 >= 0.0 && p1 >= 0.0;
    const int w = r - j;
    for (int e = threadIdx.x; e < 2 * w; e += kOrthThreads) {
      const int q = e >= w, c = j + (q ? e - w : e);
      const double p = q ? p1 : p0;
      double* row = A + q * 4096 + j * 64;
      row[c] = c == j ? (p > 0.0 ? p : 0.0) : (p > 0.0 ? row[c] / p : 0.0);
    }
    __syncthreads();
    // trailing update (ia, ib), j < ia <= ib, both matrices: threads as 2 x 8 x 16
    {
      const int q = threadIdx.x >> 7, ty = (threadIdx.x >> 4) & 7, tx = threadIdx.x & 15;
      double* M = A + q * 4096;
      for (int ia = j + 1 + ty; ia < r; ia += 8) {
        const double ra = M[j * 64 + ia];
        for (int ib = ia + tx; ib < r; ib += 16) M[ia * 64 + ib] -= ra * M[j * 64 + ib];
      }
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < 2 * r * r; e += kOrthThreads) {
    const int q = e >= r * r, f = q ? e - r * r : e;
    if (f / r > f % r) A[q * 4096 + (f / r) * 64 + f % r] = 0.0;
  }
  __syncthreads();
  return ok;
}

// One CTA: R_U, R_V (to ws), K = R_U diag(s) R_V^T as FP32 (ld kp) for the Jacobi SVD.
__global__ void __launch_bounds__(kOrthThreads) orth_core_kernel(OrthArgs a, void* ws) {
  extern __shared__ double oc_smem[];  // R_U | R_V (ld 64) during the factorisation
  __shared__ double s_piv[2], s_s[64];
  const int r = a.r;
  double* RU = oc_smem;
  double* RV = oc_smem + 64 * 64;
  for (int e = threadIdx.x; e < 2 * 64 * 64; e += kOrthThreads) oc_smem[e] = a.gram[e];
  for (int l = threadIdx.x; l < 64; l += kOrthThreads) s_s[l] = l < r ? (a.s ? static_cast<double>(a.s[l]) : 1.0) : 0.0;
  __syncthreads();
  const bool ok = orth_cholesky2(oc_smem, r, s_piv);
  if (threadIdx.x == 0 && !ok) set_status(ws, CABS_DEV_ORTH_RANK);
  for (int e = threadIdx.x; e < 2 * 64 * 64; e += kOrthThreads) a.gram[e] = oc_smem[e];
  for (int e = threadIdx.x; e < r * r; e += kOrthThreads) {
    const int i = e / r, j = e % r;
    double sum = 0.0;  // sum_l R_U[i][l] s_l R_V[j][l], l >= max(i, j)
    for (int l = i > j ? i : j; l < r; ++l)
      sum = fma(RU[i * 64 + l] * s_s[l], RV[j * 64 + l], sum);
    a.K[static_cast<int64_t>(i) * a.kp + j] = static_cast<float>(sum);
  }
}

// One CTA per side: T = R^-1 M (R upper triangular, M = U_K or V_K, k x k row-major FP64)
// by back substitution, row by row from the bottom; 4 threads per right-hand side column.
// Side 0 also writes s_out (FP32) and r_out from the SVD.
__global__ void __launch_bounds__(kOrthThreads) orth_solve_kernel(OrthArgs a) {
  __shared__ double T[64][65];
  extern __shared__ double R[];  // [64 * 64]
  const int q = blockIdx.x, r = a.r;
  for (int e = threadIdx.x; e < 64 * 64; e += kOrthThreads) R[e] = a.gram[q * 64 * 64 + e];
  __syncthreads();
  __shared__ double s_inv[64];
  const double* M = q ? a.VK : a.UK;
  float* out = q ? a.TV : a.TU;
  for (int e = threadIdx.x; e < r * r; e += kOrthThreads) T[e / r][e % r] = M[e];
  for (int i = threadIdx.x; i < r; i += kOrthThreads) {
    const double d = R[i * 64 + i];
    s_inv[i] = d > 0.0 ? 1.0 / d : 0.0;
  }
  __syncthreads();
  const int c = threadIdx.x >> 2, part = threadIdx.x & 3;
  for (int i = r - 1; i >= 0; --i) {
    double sum = 0.0;
    if (c < r)
      for (int l = i + 1 + part; l < r; l += 4) sum = fma(R[i * 64 + l], T[l][c], sum);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (c < r && part == 0) T[i][c] = (T[i][c] - sum) * s_inv[i];
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
  const int j = threadIdx.x & 63, g = threadIdx.x >> 6;  // column j of rows 16g .. 16g + 15
  float acc[16];
#pragma unroll
  for (int ii = 0; ii < 16; ++ii) acc[ii] = 0.f;
  for (int l = 0; l < r; ++l) {
    const float tv = Ts[l][j];
#pragma unroll
    for (int ii = 0; ii < 16; ++ii) acc[ii] = fmaf(xs[16 * g + ii][l], tv, acc[ii]);
  }
#pragma unroll
  for (int ii = 0; ii < 16; ++ii) {
    const int i = 16 * g + ii;
    if (i < nr && j < ldo) O[(r0 + i) * ldo + j] = acc[ii];
  }
  for (int e = threadIdx.x; e < nr * (ldo > 64 ? ldo - 64 : 0); e += kOrthThreads) {  // columns >= 64: zero
    const int64_t w = ldo - 64;
    O[(r0 + e / w) * ldo + 64 + e % w] = 0.f;
  }
}

int orth_gram_blocks(int64_t nu, int64_t nv) {
  const int64_t n = nu > nv ? nu : nv;
  const int64_t b = ceil_div(n > 0 ? n : 1, 256);
  return static_cast<int>(b < kOrthMaxBlocks ? b : kOrthMaxBlocks);
}

void launch_orth_gram(OrthArgs& a, cudaStream_t st) {
  note_launch();
  orth_gram_kernel<<<2 * a.nblk, kOrthThreads, 0, st>>>(a);
  note_launch();
  orth_reduce_kernel<<<static_cast<unsigned>(ceil_div(2 * a.r * a.r, kOrthThreads)), kOrthThreads, 0, st>>>(a);
}

void launch_orth_core(const OrthArgs& a, void* ws, cudaStream_t st) {
  note_launch();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(orth_core_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 64 * 64 * 8);
    attr = true;
  }
  orth_core_kernel<<<1, kOrthThreads, 2 * 64 * 64 * sizeof(double), st>>>(a, ws);
}

void launch_orth_finish(const OrthArgs& a, cudaStream_t st) {
  note_launch();
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(orth_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 64 * 8);
    attr = true;
  }
  orth_solve_kernel<<<2, kOrthThreads, 64 * 64 * sizeof(double), st>>>(a);
  const int64_t nbu = ceil_div(a.nu, 64), nbv = ceil_div(a.nv, 64);
  if (nbu + nbv == 0) return;
  note_launch();
  orth_apply_kernel<<<static_cast<unsigned>(nbu + nbv), kOrthThreads, 0, st>>>(a, static_cast<int>(nbu));
}

}  // namespace cabsk
