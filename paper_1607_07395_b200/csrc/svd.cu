// svd.cu -- S4: the k x k SVD of W in FP64 ("Assuming an SVD W = U_w Sigma_w V_w^T").
//
// One-sided (Hestenes) Jacobi on the columns of W: plane rotations applied from
// the right orthogonalise the columns, W V = U Sigma.  Round-robin (circle-method)
// ordering gives k/2 disjoint column pairs per round, one warp per pair, all in
// one CTA.  Columns live in shared memory when 2 k^2 doubles fit (k <= 112),
// otherwise in the (L2-resident) workspace.  Output: sigma descending, truncation
// count r = #{sigma_i > tol sigma_1} (Z4), canonical signs (Z5).
#include <float.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cabsk {

constexpr int kSvdThreads = 1024;
constexpr int kSvdMaxSweeps = 60;
constexpr int kSvdSmemK = 112;

__device__ __forceinline__ int rr_player(int j, int r, int np) {
  return j == 0 ? 0 : 1 + ((j - 1 + r) % (np - 1));
}

__global__ void __launch_bounds__(kSvdThreads, 1)
svd_jacobi_kernel(int k, const float* __restrict__ W, int64_t ldw, double tol, double* gA, double* gV,
                  double* __restrict__ sigma_out, double* __restrict__ Uw64, double* __restrict__ Vw64,
                  float* __restrict__ uw32, float* __restrict__ vw32, int64_t ld32, int* r_out, int* r_out2,
                  bool use_smem, void* ws) {
  extern __shared__ __align__(16) double smem_d[];
  __shared__ int s_rot;
  __shared__ double s_sig[CABS_KMAX];
  __shared__ int s_perm[CABS_KMAX];  // s_perm[rank] = column
  double* A = use_smem ? smem_d : gA;
  double* V = use_smem ? smem_d + (size_t)k * k : gV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  // load: A[c*k + i] = W[i, c] (column-major), V = I
  for (int64_t e = tid; e < (int64_t)k * k; e += blockDim.x) {
    int c = static_cast<int>(e / k), i = static_cast<int>(e % k);
    float w = W[(int64_t)i * ldw + c];
    if (!isfinite(w)) set_status(ws, CABS_DEV_NONFINITE);
    A[e] = static_cast<double>(w);
    V[e] = (c == i) ? 1.0 : 0.0;
  }
  __syncthreads();

  const int np = (k + 1) & ~1;  // even number of players (dummy = k when k is odd)
  const double tol_rot = 2.0 * sqrt(static_cast<double>(k)) * DBL_EPSILON;
  const double tol_rot2 = tol_rot * tol_rot;
  int sweep = 0;
  if (k > 1) {
    for (; sweep < kSvdMaxSweeps; ++sweep) {
      if (tid == 0) s_rot = 0;
      __syncthreads();
      for (int rnd = 0; rnd < np - 1; ++rnd) {
        for (int pr = warp; pr < np / 2; pr += nwarps) {
          int p = rr_player(pr, rnd, np), q = rr_player(np - 1 - pr, rnd, np);
          if (p > q) { int t = p; p = q; q = t; }
          if (q >= k) continue;  // dummy player
          double* ap = A + (size_t)p * k;
          double* aq = A + (size_t)q * k;
          double al = 0, be = 0, ga = 0;
          for (int i = lane; i < k; i += 32) {
            double x = ap[i], y = aq[i];
            al = fma(x, x, al);
            be = fma(y, y, be);
            ga = fma(x, y, ga);
          }
          al = warp_sum_d(al);
          be = warp_sum_d(be);
          ga = warp_sum_d(ga);
          if (ga != 0.0 && ga * ga > tol_rot2 * al * be) {
            // t = sign(zeta)/(|zeta| + sqrt(1 + zeta^2)), zeta = (be - al)/(2 ga), evaluated in FP32 on
            // power-of-two-scaled operands: t's accuracy only sets the convergence rate.  c = 1/sqrt(1+t^2)
            // in FP64 and s = c t make the rotation orthogonal to FP64 rounding whatever t is.
            const double x = be - al, y = 2.0 * ga;
            int ex;
            frexp(fmax(fabs(x), fabs(y)), &ex);
            const float xf = static_cast<float>(ldexp(x, -ex)), yf = static_cast<float>(ldexp(y, -ex));
            const float tf = copysignf(1.f, xf) * yf / (fabsf(xf) + sqrtf(fmaf(xf, xf, yf * yf)));
            if (tf == 0.f) continue;
            const double t = static_cast<double>(tf);
            const double c = rsqrt(fma(t, t, 1.0)), s = c * t;
            for (int i = lane; i < k; i += 32) {
              double x = ap[i], y = aq[i];
              ap[i] = c * x - s * y;
              aq[i] = s * x + c * y;
            }
            double* vp = V + (size_t)p * k;
            double* vq = V + (size_t)q * k;
            for (int i = lane; i < k; i += 32) {
              double x = vp[i], y = vq[i];
              vp[i] = c * x - s * y;
              vq[i] = s * x + c * y;
            }
            if (lane == 0) atomicAdd(&s_rot, 1);
          }
        }
        __syncthreads();
      }
      __syncthreads();
      int rot = s_rot;
      __syncthreads();
      if (rot == 0) break;
    }
    if (sweep == kSvdMaxSweeps && tid == 0) set_status(ws, CABS_DEV_SVD_NOCONV);
    if (tid == 0) reinterpret_cast<int*>(ws)[8] = sweep;  // diagnostics: sweeps of the last SVD
  }

  // singular values = column norms
  for (int c = warp; c < k; c += nwarps) {
    const double* ac = A + (size_t)c * k;
    double ss = 0;
    for (int i = lane; i < k; i += 32) ss = fma(ac[i], ac[i], ss);
    ss = warp_sum_d(ss);
    if (lane == 0) s_sig[c] = sqrt(ss);
  }
  __syncthreads();
  // descending rank, ties -> lower column first
  for (int c = tid; c < k; c += blockDim.x) {
    double sc = s_sig[c];
    int rk = 0;
    for (int j = 0; j < k; ++j) {
      double sj = s_sig[j];
      rk += (sj > sc) || (sj == sc && j < c);
    }
    s_perm[rk] = c;
  }
  __syncthreads();
  const double smax = s_sig[s_perm[0]];
  int r = 0;
  if (smax > 0) {
    for (int j = 0; j < k; ++j) r += s_sig[j] > tol * smax;
  }
  if (tid == 0) {
    if (r_out) *r_out = r;
    if (r_out2) *r_out2 = r;
  }
  for (int j = tid; j < k; j += blockDim.x) {
    if (sigma_out) sigma_out[j] = s_sig[s_perm[j]];
  }
  // write U_w, V_w columns in rank order with canonical sign
  for (int j = warp; j < k; j += nwarps) {
    const int c = s_perm[j];
    const double sg = s_sig[c];
    const bool keep = j < r;
    const double* ac = A + (size_t)c * k;
    const double* vc = V + (size_t)c * k;
    // argmax |a_c| (lowest index on ties)
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = lane; i < k; i += 32) {
      double v = fabs(ac[i]);
      if (v > best || (v == best && i < bi)) { best = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      double ob = __shfl_xor_sync(0xffffffffu, best, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const double sign = (bi < k && ac[bi] < 0) ? -1.0 : 1.0;
    const double inv = (keep && sg > 0) ? sign / sg : 0.0;
    const double vs = keep ? sign : 0.0;
    for (int i = lane; i < k; i += 32) {
      double u = ac[i] * inv, v = vc[i] * vs;
      if (Uw64) Uw64[(size_t)i * k + j] = u;
      if (Vw64) Vw64[(size_t)i * k + j] = v;
      if (uw32) uw32[(size_t)i * ld32 + j] = static_cast<float>(u);
      if (vw32) vw32[(size_t)i * ld32 + j] = static_cast<float>(v);
    }
  }
  // zero padding columns [k, ld32)
  if (uw32) {
    for (int64_t e = tid; e < (int64_t)k * (ld32 - k); e += blockDim.x) {
      int64_t i = e / (ld32 - k), c = k + e % (ld32 - k);
      uw32[i * ld32 + c] = 0.f;
      vw32[i * ld32 + c] = 0.f;
    }
  }
}

int launch_svd(int k, const float* W, int64_t ldw, double tol, void* ws, const Ws& L, double* sigma_user,
               double* Uw64, double* Vw64, int* r_user, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(svd_jacobi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kSvdSmemK * kSvdSmemK * 8);
    attr_set = true;
  }
  const bool use_smem = k <= kSvdSmemK;
  size_t smem = use_smem ? 2 * (size_t)k * k * sizeof(double) : 0;
  double* sig = sigma_user ? sigma_user : wsp<double>(ws, L.sig64);
  int* r_ws = wsp<int>(ws, L.scal) + SCAL_R_TMP;
  note_launch();
  svd_jacobi_kernel<<<1, kSvdThreads, smem, st>>>(k, W, ldw, tol, wsp<double>(ws, L.a64), wsp<double>(ws, L.v64),
                                                  sig, Uw64, Vw64, wsp<float>(ws, L.uw32), wsp<float>(ws, L.vw32),
                                                  L.Kp, r_ws, r_user, use_smem, ws);
  if (sigma_user && sigma_user != wsp<double>(ws, L.sig64)) {
    cudaMemcpyAsync(wsp<double>(ws, L.sig64), sigma_user, sizeof(double) * k, cudaMemcpyDeviceToDevice, st);
  }
  return 0;
}

}  // namespace cabsk
