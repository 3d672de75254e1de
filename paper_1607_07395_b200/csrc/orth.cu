// Orthogonalization of a sketch (Supp. section 3).
//
// The paper's recipe -- U = U0 S0 V0^T, then S0 V0^T diag(s) V^T = U1 S1 V1^T, result
// (U0 U1, S1, V1) -- is the thin SVD of U diag(s) V^T.  The B200 path reaches the same unique
// factors through r x r work only (O((m + n) r^2) in total, the paper's cost):
//   orth_gram_kernel    G_U = U^T U and G_V = V^T V, FP64 (products of FP32 entries are
//                       exact): 64 x 64 tiles of the upper triangle, per-CTA partials over a
//                       fixed row partition
//   orth_reduce_kernel  fixed-order sum of the partials, mirrored to a dense r x r (ld r)
//                       matrix (deterministic; then an allreduce across ranks)
//   orth_chol_kernel    Cholesky G_U = R_U^T R_U, G_V = R_V^T R_V (FP64, one CTA per side; the
//                       packed upper triangle in shared memory for r <= 221, else in place in
//                       global memory)
//   orth_kcore_kernel   core K = R_U diag(s) R_V^T -> FP32 for the Jacobi SVD K = U_K S_K V_K^T
//   orth_solve_kernel   T_U = R_U^-1 U_K, T_V = R_V^-1 V_K (back substitution in place, FP64;
//                       one warp per 8 right-hand-side columns)
//   orth_apply_kernel   U_o = U T_U, V_o = V T_V (FP32, 64 x 64 output tiles, K in 64-chunks)
// so U diag(s) V^T = (U R_U^-1) K (V R_V^-1)^T = (U T_U) S_K (V T_V)^T with orthonormal
// U R_U^-1, V R_V^-1.  r <= CABS_KMAX (the Jacobi SVD's range).
#include "common.cuh"
#include "kernels.cuh"

namespace cabsk {

constexpr int kOrthThreads = 256;
constexpr int kOrthRows = 32;     // rows staged per step of the Gram kernel
constexpr int kOrthCholT = 1024;  // Cholesky CTA
constexpr int kOrthPackedMax = 221;  // r (r + 1) / 2 doubles <= 196 KB of shared memory

__host__ __device__ inline int orth_tiles(int r) { return (r + 63) / 64; }
__host__ __device__ inline int orth_pairs(int r) { const int t = orth_tiles(r); return t * (t + 1) / 2; }

// CTA = (side q, row block b, tile pair tp): the 64 x 64 block (ti, tj), ti <= tj, of X_q^T X_q
// over rows [b * per, ...), partial to part + ((q * nblk + b) * npair + tp) * 4096.
__global__ void __launch_bounds__(kOrthThreads) orth_gram_kernel(OrthArgs a) {
  __shared__ __align__(16) double xa[kOrthRows][64];
  __shared__ __align__(16) double xb[kOrthRows][64];
  const int npair = orth_pairs(a.r), nt = orth_tiles(a.r);
  const int per_side = a.nblk * npair;
  const int q = static_cast<int>(blockIdx.x) >= per_side;
  const int rem = q ? blockIdx.x - per_side : blockIdx.x;
  const int b = rem / npair, tp = rem % npair;
  int ti = 0, tj = 0;
  for (int t = tp, w = nt; ; ++ti, --w) {  // tp -> (ti, tj) in row-major order of the upper triangle
    if (t < w) { tj = ti + t; break; }
    t -= w;
  }
  const float* __restrict__ X = q ? a.V : a.U;
  const int64_t ld = q ? a.ldv : a.ldu, N = q ? a.nv : a.nu;
  const int r = a.r, ca = 64 * ti, cb = 64 * tj;
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
      xa[i][c] = (i < nr && ca + c < r) ? static_cast<double>(X[(r0 + i) * ld + ca + c]) : 0.0;
      xb[i][c] = (i < nr && cb + c < r) ? static_cast<double>(X[(r0 + i) * ld + cb + c]) : 0.0;
    }
    __syncthreads();
    for (int i = 0; i < nr; ++i) {
      const double2 a01 = *reinterpret_cast<const double2*>(&xa[i][A0]);
      const double2 a23 = *reinterpret_cast<const double2*>(&xa[i][A0 + 2]);
      const double2 b01 = *reinterpret_cast<const double2*>(&xb[i][B0]);
      const double2 b23 = *reinterpret_cast<const double2*>(&xb[i][B0 + 2]);
      const double va[4] = {a01.x, a01.y, a23.x, a23.y}, vb[4] = {b01.x, b01.y, b23.x, b23.y};
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(va[u], vb[v], acc[u][v]);  // exact products
    }
  }
  double* out = a.part + ((static_cast<int64_t>(q) * a.nblk + b) * npair + tp) * 4096;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) out[(A0 + u) * 64 + B0 + v] = acc[u][v];
}

// one thread per (side, tile pair, tile entry); the partials are added in CTA order
// (deterministic) and written to both mirrored positions of the dense r x r Gram
__global__ void __launch_bounds__(kOrthThreads) orth_reduce_kernel(OrthArgs a) {
  const int npair = orth_pairs(a.r), nt = orth_tiles(a.r), r = a.r;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * kOrthThreads + threadIdx.x;
  if (t >= 2LL * npair * 4096) return;
  const int q = static_cast<int>(t / (npair * 4096));
  const int tp = static_cast<int>((t / 4096) % npair), e = static_cast<int>(t & 4095);
  int ti = 0, tj = 0;
  for (int u = tp, w = nt; ; ++ti, --w) {
    if (u < w) { tj = ti + u; break; }
    u -= w;
  }
  const int i = 64 * ti + (e >> 6), j = 64 * tj + (e & 63);
  if (i >= r || j >= r) return;
  const double* p = a.part + (static_cast<int64_t>(q) * a.nblk * npair + tp) * 4096 + e;
  const int64_t stride = static_cast<int64_t>(npair) * 4096;
  double s = 0.0;
  int b = 0;
  for (; b + 8 <= a.nblk; b += 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = p[static_cast<int64_t>(b + k) * stride];
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
  }
  for (; b < a.nblk; ++b) s += p[static_cast<int64_t>(b) * stride];
  double* G = a.gram + static_cast<int64_t>(q) * r * r;
  G[static_cast<int64_t>(i) * r + j] = s;
  G[static_cast<int64_t>(j) * r + i] = s;
}

// In-place right-looking Cholesky of one r x r matrix into its upper factor R (A = R^T R).
// M(i, j), i <= j, addresses the upper triangle (packed in shared memory or dense in global
// memory).  A zero pivot (an all-zero column) leaves a zero row of R, whose component then drops
// out; returns false on a negative or NaN pivot (a numerically rank-deficient factor).
template <typename Addr>
__device__ bool orth_cholesky(double* M, int r, Addr at, double* s_piv) {
  bool ok = true;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = kOrthCholT / 32;
  for (int j = 0; j < r; ++j) {
    if (threadIdx.x == 0) {
      const double d = M[at(j, j)];
      *s_piv = d > 0.0 ? sqrt(d) : (d == 0.0 ? 0.0 : -1.0);
    }
    __syncthreads();
    const double p = *s_piv;
    ok = ok && p >= 0.0;
    for (int c = j + threadIdx.x; c < r; c += kOrthCholT) {
      double& x = M[at(j, c)];
      x = c == j ? (p > 0.0 ? p : 0.0) : (p > 0.0 ? x / p : 0.0);
    }
    __syncthreads();
    // trailing update (ia, ib), j < ia <= ib: warps over rows, lanes over columns
    for (int ia = j + 1 + warp; ia < r; ia += nw) {
      const double ra = M[at(j, ia)];
      for (int ib = ia + lane; ib < r; ib += 32) M[at(ia, ib)] -= ra * M[at(j, ib)];
    }
    __syncthreads();
  }
  return ok;
}

struct PackedAt {
  int r;
  __device__ int operator()(int i, int j) const { return i * r - (i * (i - 1)) / 2 + (j - i); }
};
struct DenseAt {
  int r;
  __device__ int64_t operator()(int i, int j) const { return static_cast<int64_t>(i) * r + j; }
};

// One CTA per side: R_q in place of G_q (dense, ld r, zeros below the diagonal).
__global__ void __launch_bounds__(kOrthCholT) orth_chol_kernel(OrthArgs a, void* ws) {
  extern __shared__ double pk[];  // packed upper triangle (r <= kOrthPackedMax)
  __shared__ double s_piv;
  const int q = blockIdx.x, r = a.r;
  double* G = a.gram + static_cast<int64_t>(q) * r * r;
  bool ok;
  if (r <= kOrthPackedMax) {
    const PackedAt at{r};
    for (int e = threadIdx.x; e < r * r; e += kOrthCholT) {
      const int i = e / r, j = e % r;
      if (j >= i) pk[at(i, j)] = G[e];
    }
    __syncthreads();
    ok = orth_cholesky(pk, r, at, &s_piv);
    for (int e = threadIdx.x; e < r * r; e += kOrthCholT) {
      const int i = e / r, j = e % r;
      G[e] = j >= i ? pk[at(i, j)] : 0.0;
    }
  } else {
    ok = orth_cholesky(G, r, DenseAt{r}, &s_piv);
    for (int e = threadIdx.x; e < r * r; e += kOrthCholT)
      if (e / r > e % r) G[e] = 0.0;
  }
  if (threadIdx.x == 0 && !ok) set_status(ws, CABS_DEV_ORTH_RANK);
}

// K[i][j] = sum_{l >= max(i, j)} R_U[i][l] s_l R_V[j][l] (FP64) -> FP32, ld kp; one thread per entry
__global__ void __launch_bounds__(kOrthThreads) orth_kcore_kernel(OrthArgs a) {
  const int r = a.r;
  const int64_t e = static_cast<int64_t>(blockIdx.x) * kOrthThreads + threadIdx.x;
  if (e >= static_cast<int64_t>(r) * r) return;
  const int i = static_cast<int>(e / r), j = static_cast<int>(e % r);
  const double* RU = a.gram;
  const double* RV = a.gram + static_cast<int64_t>(r) * r;
  double sum = 0.0;
  for (int l = i > j ? i : j; l < r; ++l) {
    const double sl = a.s ? static_cast<double>(__ldg(a.s + l)) : 1.0;
    sum = fma(__ldg(RU + static_cast<int64_t>(i) * r + l) * sl, __ldg(RV + static_cast<int64_t>(j) * r + l), sum);
  }
  a.K[static_cast<int64_t>(i) * a.kp + j] = static_cast<float>(sum);
}

// T = R^-1 M in place of M (R upper triangular r x r, M = U_K or V_K, r x r row-major FP64) by
// back substitution from the bottom row; 4 lanes per right-hand-side column, so a column's rows
// depend only on its own warp.  Then T -> FP32 (ld kp, zero past r).  Grid: (side, 32-column
// group); side 0's first CTA also writes s_out and r_out.
__global__ void __launch_bounds__(128) orth_solve_kernel(OrthArgs a) {
  const int r = a.r, ng = (r + 31) / 32;
  const int q = static_cast<int>(blockIdx.x) / ng, grp = static_cast<int>(blockIdx.x) % ng;
  const double* R = a.gram + static_cast<int64_t>(q) * r * r;
  double* T = q ? a.VK : a.UK;
  float* out = q ? a.TV : a.TU;
  const int c = 32 * grp + (threadIdx.x >> 2), part = threadIdx.x & 3;
  for (int i = r - 1; i >= 0; --i) {
    double sum = 0.0;
    if (c < r)
      for (int l = i + 1 + part; l < r; l += 4)
        sum = fma(__ldg(R + static_cast<int64_t>(i) * r + l), T[static_cast<int64_t>(l) * r + c], sum);
    sum += __shfl_xor_sync(0xffffffffu, sum, 1);
    sum += __shfl_xor_sync(0xffffffffu, sum, 2);
    if (c < r && part == 0) {
      const double d = __ldg(R + static_cast<int64_t>(i) * r + i);
      double& t = T[static_cast<int64_t>(i) * r + c];
      t = d > 0.0 ? (t - sum) * (1.0 / d) : 0.0;
    }
    __syncwarp();
  }
  if (c < r && part == 0)
    for (int i = 0; i < r; ++i) out[static_cast<int64_t>(i) * a.kp + c] = static_cast<float>(T[static_cast<int64_t>(i) * r + c]);
  for (int cc = 32 * grp + (threadIdx.x >> 2); cc < a.kp && grp == ng - 1; cc += 32)  // padding columns
    if (cc >= r && part == 0)
      for (int i = 0; i < r; ++i) out[static_cast<int64_t>(i) * a.kp + cc] = 0.f;
  if (q == 0 && grp == 0) {
    const int rk = *a.r_svd;
    for (int j = threadIdx.x; j < r; j += 128) a.s_out[j] = j < rk ? static_cast<float>(a.sig[j]) : 0.f;
    if (threadIdx.x == 0 && a.r_out) *a.r_out = rk;
  }
}

// Out[l][c] = sum_k X[l][k] T[k][c] for c < r, 0 for r <= c < ldo.  CTA = (side, 64-row block,
// 64-column block); K in chunks of 64 staged in shared memory.
__global__ void __launch_bounds__(kOrthThreads) orth_apply_kernel(OrthArgs a, int nbu, int ncb) {
  __shared__ float Ts[64][64];
  __shared__ float xs[64][65];
  const int rb = static_cast<int>(blockIdx.x) / ncb, cbk = static_cast<int>(blockIdx.x) % ncb;
  const int q = rb >= nbu;
  const int64_t b = q ? rb - nbu : rb;
  const float* __restrict__ X = q ? a.V : a.U;
  const int64_t ldx = q ? a.ldv : a.ldu, N = q ? a.nv : a.nu;
  float* __restrict__ O = q ? a.Vo : a.Uo;
  const int64_t ldo = q ? a.ldvo : a.lduo;
  const float* T = q ? a.TV : a.TU;
  const int r = a.r, c0 = 64 * cbk;
  if (c0 >= ldo) return;
  const int64_t r0 = b * 64;
  const int nr = N - r0 < 64 ? static_cast<int>(N - r0) : 64;
  const int j = threadIdx.x & 63, g = threadIdx.x >> 6;  // column c0 + j of rows 16 g .. 16 g + 15
  float acc[16];
#pragma unroll
  for (int ii = 0; ii < 16; ++ii) acc[ii] = 0.f;
  if (c0 < r) {
    for (int k0 = 0; k0 < r; k0 += 64) {
      __syncthreads();
      for (int e = threadIdx.x; e < 64 * 64; e += kOrthThreads) {
        const int i = e / 64, cc = e % 64;
        Ts[i][cc] = (k0 + i < r && c0 + cc < r) ? T[static_cast<int64_t>(k0 + i) * a.kp + c0 + cc] : 0.f;
        xs[i][cc] = (i < nr && k0 + cc < r) ? X[(r0 + i) * ldx + k0 + cc] : 0.f;
      }
      __syncthreads();
      const int kn = r - k0 < 64 ? r - k0 : 64;
      for (int l = 0; l < kn; ++l) {
        const float tv = Ts[l][j];
#pragma unroll
        for (int ii = 0; ii < 16; ++ii) acc[ii] = fmaf(xs[16 * g + ii][l], tv, acc[ii]);
      }
    }
  }
#pragma unroll
  for (int ii = 0; ii < 16; ++ii) {
    const int i = 16 * g + ii;
    if (i < nr && c0 + j < ldo) O[(r0 + i) * ldo + c0 + j] = c0 + j < r ? acc[ii] : 0.f;
  }
}

int orth_gram_blocks(int64_t nu, int64_t nv, int r) {
  const int64_t n = nu > nv ? nu : nv;
  int64_t b = ceil_div(n > 0 ? n : 1, 256);
  const int64_t cap = kOrthMaxBlocks / orth_pairs(r) > 0 ? kOrthMaxBlocks / orth_pairs(r) : 1;
  return static_cast<int>(b < cap ? b : cap);
}

void launch_orth_gram(OrthArgs& a, cudaStream_t st) {
  const int npair = orth_pairs(a.r);
  note_launch();
  orth_gram_kernel<<<2 * a.nblk * npair, kOrthThreads, 0, st>>>(a);
  note_launch();
  orth_reduce_kernel<<<static_cast<unsigned>(ceil_div(2LL * npair * 4096, kOrthThreads)), kOrthThreads, 0, st>>>(a);
}

void launch_orth_core(const OrthArgs& a, void* ws, cudaStream_t st) {
  static bool attr = false;
  const int smax = (kOrthPackedMax * (kOrthPackedMax + 1) / 2) * 8;
  if (!attr) {
    cudaFuncSetAttribute(orth_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
    attr = true;
  }
  const int smem = a.r <= kOrthPackedMax ? (a.r * (a.r + 1) / 2) * 8 : 0;
  note_launch();
  orth_chol_kernel<<<2, kOrthCholT, smem, st>>>(a, ws);
  note_launch();
  orth_kcore_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(a.r) * a.r, kOrthThreads)), kOrthThreads, 0,
                      st>>>(a);
}

// Uo = U T_U only (the V side absent): the tiled apply, used for F = C U* by cur.cu
void launch_orth_apply_u(const OrthArgs& a, cudaStream_t st) {
  const int64_t nbu = ceil_div(a.nu, 64);
  const int ncb = static_cast<int>(ceil_div(a.lduo, 64));
  if (nbu == 0) return;
  note_launch();
  orth_apply_kernel<<<static_cast<unsigned>(nbu * ncb), kOrthThreads, 0, st>>>(a, static_cast<int>(nbu), ncb);
}

void launch_orth_finish(const OrthArgs& a, cudaStream_t st) {
  note_launch();
  orth_solve_kernel<<<2 * ((a.r + 31) / 32), 128, 0, st>>>(a);
  const int64_t nbu = ceil_div(a.nu, 64), nbv = ceil_div(a.nv, 64);
  const int64_t ldo = a.lduo > a.ldvo ? a.lduo : a.ldvo;
  const int ncb = static_cast<int>(ceil_div(ldo, 64));
  if (nbu + nbv == 0) return;
  note_launch();
  orth_apply_kernel<<<static_cast<unsigned>((nbu + nbv) * ncb), kOrthThreads, 0, st>>>(a, static_cast<int>(nbu), ncb);
}

}  // namespace cabsk
