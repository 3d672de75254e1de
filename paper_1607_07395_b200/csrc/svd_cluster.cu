// svd_cluster.cu -- S4 for k > 64: the k x k SVD of W in FP64 ("Assuming an SVD
// W = U_w Sigma_w V_w^T") by block one-sided (Hestenes) Jacobi over a thread-block cluster.
//
// The k columns of A = W (and of V = I) are cut into 2P blocks of w <= 16 columns; each of
// the P CTAs of the cluster holds two blocks in shared memory (FP64, A and V side by side).
// A sweep is
//   * one round-robin pass over the pairs INSIDE each block (w - 1 rounds, all blocks at once),
//   * 2P - 1 block rounds of the circle-method tournament on the 2P blocks: in a block round a
//     CTA rotates every pair (column of its first block, column of its second block) -- w
//     inner rounds of w disjoint pairs, one warp per pair -- then the blocks move one seat
//     (DSMEM copies staged through registers, two cluster barriers),
// so every pair of columns is rotated exactly once per sweep (a cyclic Jacobi ordering), each
// inner round is CTA-local (one __syncthreads), and only the 2P - 1 seat changes cross SMs.
// Rotation formula and stopping rule are those of the single-CTA kernels (svd.cu): stop after
// a sweep without rotations or whose rotations all had |t| < CABS_SVD_TSTOP.  Output as
// svd_write: sigma descending, r = #{sigma_i > tol sigma_1}, U_w = a_c / sigma_c and V_w in rank
// order with canonical signs (Z5), dropped components zero.
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

#ifndef CABS_SVD_TSTOP
#define CABS_SVD_TSTOP 1e-6
#endif

namespace cabsk {

constexpr int kScThreads = 512;  // 16 warps: one per pair of an inner round (w <= 16)
constexpr int kScMaxSweeps = 60;
constexpr int kScKmax = 320;

// t of the Jacobi rotation of (x, y), al = x.x, be = y.y, ga = x.y (0 when orthogonal to tol),
// then c = 1 / sqrt(1 + t^2) to FP64 accuracy and s = c t (the formulas of svd.cu)
__device__ __forceinline__ double sc_rsqrt64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double sc_rcp64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double sc_angle(double al, double be, double ga, double tol2, double& c, double& s) {
  const bool need = ga != 0.0 && ga * ga > tol2 * al * be;
  const double dx = be - al, dy = 2.0 * ga;
  const double h = fma(dx, dx, dy * dy);
  const double den = fabs(dx) + h * sc_rsqrt64(h);
  const double t = need ? copysign(1.0, dx) * dy * sc_rcp64(den) : 0.0;
  const double q1 = fma(t, t, 1.0);
  double cc = sc_rsqrt64(q1);
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  c = cc;
  s = cc * t;
  return t;
}

__device__ __forceinline__ uint32_t sc_map(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(tc::smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void sc_st_f64(uint32_t a, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void sc_st_s32(uint32_t a, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ int sc_ld_s32(uint32_t a) {
  int v;
  asm volatile("ld.shared::cluster.s32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sc_cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

// Squared norm of a column (warp, fixed-order tree)
template <int EPL>
__device__ __forceinline__ double sc_norm2(const double* cp, int lane) {
  double a0 = 0, a1 = 0;
#pragma unroll
  for (int e = 0; e < EPL; e += 2) {
    a0 = fma(cp[lane + 32 * e], cp[lane + 32 * e], a0);
    if (e + 1 < EPL) a1 = fma(cp[lane + 32 * (e + 1)], cp[lane + 32 * (e + 1)], a1);
  }
  return warp_sum_d(a0 + a1);
}

// One warp rotates the column pair (p, q) of the CTA's 2w local columns, A and V: lanes hold
// rows lane + 32 e.  Column j lives at col(j) (A) and col(j) + kp (V); its squared norm is
// cached in *np / *nq (exact at every block round start, then updated by the rotation's exact
// 2 x 2 formula: x.x -= t g, y.y += t g), so only x.y is reduced across the warp.
template <int EPL>
__device__ __forceinline__ void sc_rotate(double* cp, double* cq, double* np, double* nq, int kp, double tol2,
                                          int lane, bool& rotated, double& tmax) {
  double x[EPL], y[EPL];
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    x[e] = cp[lane + 32 * e];
    y[e] = cq[lane + 32 * e];
  }
  double ga0 = 0, ga1 = 0;
#pragma unroll
  for (int e = 0; e < EPL; e += 2) {
    ga0 = fma(x[e], y[e], ga0);
    if (e + 1 < EPL) ga1 = fma(x[e + 1], y[e + 1], ga1);
  }
  const double ga = warp_sum_d(ga0 + ga1);
  const double al = *np, be = *nq;
  double c, s;
  const double t = sc_angle(al, be, ga, tol2, c, s);
  if (t != 0.0) {
    rotated = true;
    tmax = fmax(tmax, fabs(t));
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      cp[lane + 32 * e] = c * x[e] - s * y[e];
      cq[lane + 32 * e] = s * x[e] + c * y[e];
    }
    double* vp = cp + kp;
    double* vq = cq + kp;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const double a = vp[lane + 32 * e], b = vq[lane + 32 * e];
      vp[lane + 32 * e] = c * a - s * b;
      vq[lane + 32 * e] = s * a + c * b;
    }
    __syncwarp();
    if (lane == 0) {
      *np = fma(-t, ga, al);
      *nq = fma(t, ga, be);
    }
  }
}

// circle method on n (even) players: player j's seat in round r (player 0 fixed)
__device__ __forceinline__ int sc_rr(int j, int r, int n) {
  int x = j - 1 + r;
  if (x >= n - 1) x -= n - 1;
  return j == 0 ? 0 : 1 + x;
}

// ---------------------------------------------------------------- QR preconditioner, 128 < k <= 320
// The pivoted Householder QR of svd.cu's svd_qrcp_kernel (same pivot rule, same reflector
// arithmetic, same outputs Xt = R^T, Hv = reflectors + scales, piv) for matrices too large for
// one CTA's registers: a cooperative grid of ceil(k/4) CTAs, one warp per column (rows
// lane + 32 e in registers), one grid barrier per pivot step.  Every column is published to a
// double-buffered global copy each step (the next pivot column is read from there, through L2)
// and every CTA its best (key, column) of the next step.
struct QrGrid {
  double* colbuf;  // [2][k][kr]
  double* bests;   // [2][128][2]: key, column
  double* rd;      // R_jj
  unsigned* bar;   // arrival counter (zeroed before the launch)
  int kr;
};

__device__ __forceinline__ void qg_barrier(unsigned* bar, unsigned target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(bar, 1u);
    while (ld_acquire_gpu(bar) < target) __nanosleep(20);
  }
  __syncthreads();
}

template <int E>
__global__ void __launch_bounds__(128) svd_qrcp_grid_kernel(int k, const float* __restrict__ W, int64_t ldw,
                                                            double* __restrict__ Xt, double* __restrict__ Hv,
                                                            double* __restrict__ Rg, int* __restrict__ piv_out,
                                                            QrGrid g, void* ws) {
  __shared__ double s_k[4];
  __shared__ int s_i[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int q = blockIdx.x * 4 + warp;
  const int NB = gridDim.x;
  const int kr = g.kr;
  double a[E];
  bool bad = false;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane + 32 * e;
    float v = 0.f;
    if (i < k && q < k) v = W[(int64_t)i * ldw + q];
    bad |= !isfinite(v);
    a[e] = static_cast<double>(v);
  }
  if (bad) set_status(ws, CABS_DEV_NONFINITE);
  bool done = q >= k;
  unsigned nbar = 0;
  auto publish = [&](int par, double key) {  // column copy + the CTA's best (lowest column on ties)
    if (!done) {
      double* cb = g.colbuf + ((size_t)par * k + q) * kr;
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (lane + 32 * e < kr) cb[lane + 32 * e] = a[e];
    }
    if (lane == 0) { s_k[warp] = done ? -1.0 : key; s_i[warp] = q; }
    __syncthreads();
    if (tid == 0) {
      double bk = -1.0;
      int bi = 0x7fffffff;
      for (int w2 = 0; w2 < 4; ++w2)
        if (s_k[w2] > bk) { bk = s_k[w2]; bi = s_i[w2]; }
      g.bests[((size_t)par * 128 + blockIdx.x) * 2] = bk;
      g.bests[((size_t)par * 128 + blockIdx.x) * 2 + 1] = static_cast<double>(bi);
    }
  };
  {
    double n0 = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) n0 = fma(a[e], a[e], n0);
    publish(0, warp_sum_d(n0));
  }
  qg_barrier(g.bar, static_cast<unsigned>(NB) * ++nbar);
  for (int j = 0; j < k; ++j) {
    const int par = j & 1;
    // pivot: argmax of the NB CTA bests (identical in every warp)
    double bv = -1.0;
    int bq = 0x7fffffff;
    for (int c = lane; c < NB; c += 32) {
      const double kk = __ldcg(g.bests + ((size_t)par * 128 + c) * 2);
      const int ii = static_cast<int>(__ldcg(g.bests + ((size_t)par * 128 + c) * 2 + 1));
      if (kk > bv || (kk == bv && ii < bq)) { bv = kk; bq = ii; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
      if (ov > bv || (ov == bv && oq < bq)) { bv = ov; bq = oq; }
    }
    const int ph = bq;
    const double* xp = g.colbuf + ((size_t)par * k + ph) * kr;
    const double xj = __ldcg(xp + j), nn = fmax(bv, 0.0), sn = sqrt(nn);
    const double alpha = xj >= 0.0 ? -sn : sn;                           // R_jj
    const double vjj = xj - alpha;                                        // x_j + sign(x_j) ||x||
    const double beta = nn > 0.0 ? 1.0 / (sn * (sn + fabs(xj))) : 0.0;    // 2 / v^T v
    double x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = lane + 32 * e < kr ? __ldcg(xp + lane + 32 * e) : 0.0;
    if (q == ph) done = true;
    // rows above j are zero in every column (cleared as they move to R)
    const double aj = (!done && q < k) ? __ldcg(g.colbuf + ((size_t)par * k + q) * kr + j) : 0.0;
    double d0 = lane == 0 ? (vjj - xj) * aj : 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) d0 = fma(x[e], a[e], d0);
    const double f = done ? 0.0 : beta * warp_sum_d(d0);
    double n0 = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      a[e] = lane + 32 * e == j ? 0.0 : fma(-f, x[e], a[e]);
      n0 = fma(a[e], a[e], n0);
    }
    const double key = warp_sum_d(n0);  // exact ||a(j+1:)||^2
    if (!done && lane == 0) Rg[(size_t)j * k + q] = fma(-f, vjj, aj);  // R_jq
    if (blockIdx.x == 0 && warp == 0) {  // reflector j (every warp holds it)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = lane + 32 * e;
        if (i < k) Hv[(size_t)j * k + i] = i == j ? vjj : x[e];
      }
      if (lane == 0) {
        Hv[(size_t)k * k + j] = beta;
        piv_out[j] = ph;
        g.rd[j] = alpha;
      }
    }
    publish(par ^ 1, key);
    qg_barrier(g.bar, static_cast<unsigned>(NB) * ++nbar);
  }
  // X = R^T: X[i][c] = R[c][i] = Rg[c][piv[i]] above the diagonal, R_ii on it, 0 below
  for (int64_t e = (int64_t)blockIdx.x * 128 + tid; e < (int64_t)k * k; e += (int64_t)NB * 128) {
    const int i = static_cast<int>(e / k), c = static_cast<int>(e - (int64_t)i * k);
    Xt[e] = c < i ? __ldcg(Rg + (size_t)c * k + __ldcg(piv_out + i)) : (c == i ? __ldcg(g.rd + i) : 0.0);
  }
}

template <int EPL>
__global__ void __launch_bounds__(kScThreads, 1)
svd_cluster_kernel(int k, int w, const float* __restrict__ W, int64_t ldw, const double* __restrict__ Xt,
                   const double* __restrict__ Hq, const int* __restrict__ piv, double tol,
                   double* __restrict__ sigma_out, double* __restrict__ Uw64, double* __restrict__ Vw64,
                   float* __restrict__ uw32, float* __restrict__ vw32, int64_t ld32, int* r_out, int* r_out2,
                   void* ws) {
  // Xt != nullptr: QR-preconditioned (svd_qrcp_grid_kernel): A = R^T, V = Q (formed here from
  // the reflectors Hq); the V columns end as U_w = Q V_x, the A columns give V_w (rows permuted)
  const bool pre = Xt != nullptr;
  extern __shared__ __align__(16) double sm[];
  __shared__ double s_sig[kScKmax];  // CTA 0: sigma by column id
  __shared__ int s_rank[kScKmax];    // CTA 0: rank by column id
  __shared__ int s_perm[kScKmax];
  __shared__ int s_flag[2];          // CTA 0: [rotated any, all |t| small] of the sweep
  __shared__ int s_r, s_last;
  __shared__ double s_nrm[32];       // cached squared norms of the 2w local columns
  constexpr int kp = 32 * EPL;       // padded column length
  constexpr bool DB = EPL <= 5;      // double-buffered block storage (seat changes without staging)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  uint32_t cr, P;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(cr));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(P));
  const int nb = 2 * static_cast<int>(P);
  // local column j (0 <= j < 2w): slot j / w, column j % w; storage [j][A kp | V kp]
  int buf = 0;
  const size_t bufsz = (size_t)2 * w * 2 * kp;
  auto col = [&](int j) { return sm + buf * bufsz + (size_t)j * 2 * kp; };
  auto refresh_norms = [&]() {  // exact squared norms of the local columns
    for (int j = warp; j < 2 * w; j += kScThreads / 32) {
      const double n2 = sc_norm2<EPL>(col(j), lane);
      if (lane == 0) s_nrm[j] = n2;
    }
    __syncthreads();
  };
  // block ids of the two slots (the tournament moves them); global column = blk * w + local
  int blk[2] = {static_cast<int>(cr), nb - 1 - static_cast<int>(cr)};

  // ---- load A = W (columns), V = I; zero padding rows / columns
  if (pre) {
    for (int e = tid; e < 2 * w * kp; e += kScThreads) {
      const int j = e / kp, i = e - j * kp;
      const int gc = blk[j / w] * w + (j % w);
      col(j)[i] = (i < k && gc < k) ? Xt[(size_t)i * k + gc] : 0.0;
      col(j)[kp + i] = (i == gc && gc < k) ? 1.0 : 0.0;
    }
    __syncthreads();
    // V = Q = H_0 ... H_{k-1} on the local unit columns: H_j for j = k - 1 down to 0, one warp per
    // column (H_j e_c = e_c for j > c: skipped exactly)
    for (int jl = warp; jl < 2 * w; jl += kScThreads / 32) {
      const int gc = blk[jl / w] * w + (jl % w);
      if (gc >= k) continue;
      double* vc = col(jl) + kp;
      double y[EPL];
#pragma unroll
      for (int e = 0; e < EPL; ++e) y[e] = vc[lane + 32 * e];
      for (int j = gc; j >= 0; --j) {
        const double* hv = Hq + (size_t)j * k;
        double dd = 0.0, hvr[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
          const int i = lane + 32 * e;
          hvr[e] = i < k ? __ldg(hv + i) : 0.0;
          dd = fma(hvr[e], y[e], dd);
        }
        const double f = __ldg(Hq + (size_t)k * k + j) * warp_sum_d(dd);
#pragma unroll
        for (int e = 0; e < EPL; ++e) y[e] = fma(-f, hvr[e], y[e]);
      }
#pragma unroll
      for (int e = 0; e < EPL; ++e) vc[lane + 32 * e] = y[e];
    }
    __syncthreads();
  } else {
    bool bad = false;
    for (int e = tid; e < 2 * w * kp; e += kScThreads) {
      const int j = e / kp, i = e - j * kp;
      const int gc = blk[j / w] * w + (j % w);
      float v = 0.f;
      if (i < k && gc < k) v = W[(int64_t)i * ldw + gc];
      bad |= !isfinite(v);
      col(j)[i] = static_cast<double>(v);
      col(j)[kp + i] = (i == gc && gc < k) ? 1.0 : 0.0;
    }
    if (__syncthreads_or(bad) && tid == 0) set_status(ws, CABS_DEV_NONFINITE);
  }
  if (tid == 0) { s_flag[0] = 0; s_flag[1] = 1; }
  sc_cluster_sync();

  const double tol_rot = 2.0 * sqrt(static_cast<double>(k)) * DBL_EPSILON;
  const double tol2 = tol_rot * tol_rot;
  const uint32_t flag0 = sc_map(&s_flag[0], 0);
  int sweep = 0;
  bool last = k <= 1;
#ifdef CABS_PROFILE_SVDC
  long long pc[4] = {0, 0, 0, 0}, pt = clock64();
#define SC_PROF(i) do { const long long t_ = clock64(); pc[i] += t_ - pt; pt = t_; } while (0)
#else
#define SC_PROF(i) do { } while (0)
#endif
  for (; !last; ++sweep) {
    bool rotated = false;
    double tmax = 0.0;
    // (1) pairs inside each block: round-robin on w (padded to even) players, both slots at once
    refresh_norms();
    {
      const int wp = (w + 1) & ~1;
      for (int r = 0; r < wp - 1; ++r) {
        if (warp < wp) {  // warps [0, wp/2): slot 0, [wp/2, wp): slot 1
          const int half = wp / 2, sl = warp / half, pi = warp % half;
          int p = sc_rr(pi, r, wp), q = sc_rr(wp - 1 - pi, r, wp);
          if (p < w && q < w)
            sc_rotate<EPL>(col(sl * w + p), col(sl * w + q), &s_nrm[sl * w + p], &s_nrm[sl * w + q], kp, tol2, lane,
                           rotated, tmax);
        }
        __syncthreads();
      }
    }
    SC_PROF(0);
    // (2) block rounds: cross pairs, then a seat change
    for (int br = 0; br < nb - 1; ++br) {
      if (br > 0) refresh_norms();  // the blocks moved
      for (int s = 0; s < w; ++s) {
        if (warp < w) {
          const int i = warp, jq = (warp + s) % w;
          sc_rotate<EPL>(col(i), col(w + jq), &s_nrm[i], &s_nrm[w + jq], kp, tol2, lane, rotated, tmax);
        }
        __syncthreads();
      }
      SC_PROF(1);
      if (P > 1) {
        // seat change (circle method, seat 0 fixed; seat s -> s + 1, seat 2P - 1 -> 1): CTA c's
        // low block (seat c) goes to CTA c + 1's low slot (c = P - 1: its own high slot; c = 0:
        // stays); its high block (seat 2P - 1 - c) to CTA c - 1's high slot (c = 0: CTA 1's low)
        const int c = static_cast<int>(cr), Pi = static_cast<int>(P);
        int dst[2], dsl[2];
        dst[0] = c == 0 ? 0 : (c == Pi - 1 ? c : c + 1);
        dsl[0] = c == 0 ? 0 : (c == Pi - 1 ? 1 : 0);
        dst[1] = c == 0 ? 1 : c - 1;
        dsl[1] = c == 0 ? 0 : 1;
        sc_cluster_sync();  // every CTA is done with its blocks
        if (DB) {
          // straight into the destination's other buffer, 16 bytes per store
          for (int sl = 0; sl < 2; ++sl) {
            const uint32_t base = sc_map(sm + (buf ^ 1) * bufsz + (size_t)dsl[sl] * w * 2 * kp,
                                         static_cast<uint32_t>(dst[sl]));
            const double2* src = reinterpret_cast<const double2*>(col(sl * w));
            for (int e = tid; e < w * kp; e += kScThreads) {  // w columns x (A | V) = w * 2 kp doubles
              const double2 v2 = src[e];
              asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(base + 16u * e), "d"(v2.x), "d"(v2.y)
                           : "memory");
            }
          }
          sc_cluster_sync();
          buf ^= 1;
        } else {
          // stage both slots through registers in two halves (A, then V), write them to the seats
          constexpr int kPer = (16 * kScKmax + kScThreads - 1) / kScThreads;  // w * kp / threads, <= 10
          for (int part = 0; part < 2; ++part) {
            double v[2][kPer];
#pragma unroll
            for (int sl = 0; sl < 2; ++sl)
#pragma unroll
              for (int u = 0; u < kPer; ++u) {
                const int e = tid + u * kScThreads;
                const int j = e / kp, i = e - j * kp;
                v[sl][u] = (j < w) ? col(sl * w + j)[part * kp + i] : 0.0;
              }
            sc_cluster_sync();  // reads done before anyone overwrites
#pragma unroll
            for (int sl = 0; sl < 2; ++sl) {
              const uint32_t base = sc_map(col(dsl[sl] * w), static_cast<uint32_t>(dst[sl]));
#pragma unroll
              for (int u = 0; u < kPer; ++u) {
                const int e = tid + u * kScThreads;
                const int j = e / kp, i = e - j * kp;
                if (j < w) sc_st_f64(base + static_cast<uint32_t>(((size_t)j * 2 * kp + part * kp + i) * 8), v[sl][u]);
              }
            }
            sc_cluster_sync();
          }
        }
        // the tournament is deterministic: the seats' blocks from the number of seat changes
        const int rd = sweep * (nb - 1) + br + 1;  // seat changes so far
        auto seat_block = [&](int seat) {          // block at `seat` after rd changes
          if (seat == 0) return 0;
          int b0 = seat - 1 - (rd % (nb - 1));
          if (b0 < 0) b0 += nb - 1;
          return b0 + 1;
        };
        blk[0] = seat_block(c);
        blk[1] = seat_block(nb - 1 - c);
      }
      SC_PROF(2);
    }
    // convergence over the cluster: any rotation, all |t| small
    if (tid == 0) { s_flag[0] = 0; s_flag[1] = 1; }
    const int rot_cta = __syncthreads_or(rotated);
    const int small_cta = __syncthreads_and(tmax < CABS_SVD_TSTOP);
    sc_cluster_sync();  // CTA 0's flags reset before anyone reports
    if (tid == 0) {
      if (rot_cta) asm volatile("red.shared::cluster.or.b32 [%0], 1;" ::"r"(flag0) : "memory");
      if (!small_cta) asm volatile("red.shared::cluster.and.b32 [%0], 0;" ::"r"(flag0 + 4u) : "memory");
    }
    sc_cluster_sync();
    if (tid == 0) {
      const int any = sc_ld_s32(flag0), allsmall = sc_ld_s32(flag0 + 4u);
      s_last = (!any || allsmall || sweep + 1 >= kScMaxSweeps) ? 1 : 0;
    }
    __syncthreads();
    last = s_last != 0;
    sc_cluster_sync();  // everyone has read the flags before the next reset
    SC_PROF(3);
  }
#ifdef CABS_PROFILE_SVDC
  if (cr == 0 && tid == 0)
    for (int i = 0; i < 4; ++i) reinterpret_cast<long long*>(ws)[16 + i] = pc[i];
#endif
  if (cr == 0 && tid == 0) {
    if (sweep >= kScMaxSweeps && k > 1) set_status(ws, CABS_DEV_SVD_NOCONV);
    reinterpret_cast<int*>(ws)[8] = sweep;
  }

  // ---- sigma of every local column -> CTA 0; ranks there; back to everyone
  const uint32_t sig0 = sc_map(s_sig, 0), rank0 = sc_map(s_rank, 0), r0 = sc_map(&s_r, 0);
  for (int j = warp; j < 2 * w; j += kScThreads / 32) {
    const int gc = blk[j / w] * w + (j % w);
    const double* a = col(j);
    double ss = 0.0;
    for (int i = lane; i < kp; i += 32) ss = fma(a[i], a[i], ss);
    ss = warp_sum_d(ss);
    if (lane == 0 && gc < k) sc_st_f64(sig0 + 8u * gc, sqrt(ss));
  }
  sc_cluster_sync();
  if (cr == 0) {
    for (int c = tid; c < k; c += kScThreads) {
      const double sc = s_sig[c];
      int rk = 0;
      for (int j = 0; j < k; ++j) {
        const double sj = s_sig[j];
        rk += (sj > sc) || (sj == sc && j < c);
      }
      s_rank[c] = rk;
      s_perm[rk] = c;
    }
    __syncthreads();
    if (warp == 0) {
      const double smax = s_sig[s_perm[0]];
      int cnt = 0;
      for (int c = lane; c < k; c += 32) cnt += smax > 0 && s_sig[c] > tol * smax;
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (lane == 0) {
        s_r = cnt;
        if (r_out) *r_out = cnt;
        if (r_out2) *r_out2 = cnt;
      }
    }
    if (sigma_out)
      for (int j = tid; j < k; j += kScThreads) sigma_out[j] = s_sig[s_perm[j]];
    if (uw32) {  // zero padding columns [k, ld32)
      for (int64_t e = tid; e < (int64_t)k * (ld32 - k); e += kScThreads) {
        const int64_t i = e / (ld32 - k), c = k + e % (ld32 - k);
        uw32[i * ld32 + c] = 0.f;
        vw32[i * ld32 + c] = 0.f;
      }
    }
  }
  sc_cluster_sync();
  // ---- every CTA writes its columns: U_w = a / sigma and V_w, canonical signs, rank order
  {
    const int r = sc_ld_s32(r0);
    for (int j = warp; j < 2 * w; j += kScThreads / 32) {
      const int gc = blk[j / w] * w + (j % w);
      if (gc >= k) continue;
      const int jr = sc_ld_s32(rank0 + 4u * gc);
      double sg;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(sg) : "r"(sig0 + 8u * gc) : "memory");
      const double* a = col(j);
      const double* v = a + kp;
      const double* uc = pre ? v : a;  // the column holding U_w's direction fixes the sign
      double best = -1.0;
      int bi = 0x7fffffff;
      for (int i = lane; i < k; i += 32) {
        const double x = fabs(uc[i]);
        if (x > best || (x == best && i < bi)) { best = x; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      const bool keep = jr < r;
      const double sign = (bi < k && uc[bi] < 0) ? -1.0 : 1.0;
      const double inv = (keep && sg > 0) ? sign / sg : 0.0;
      const double vs = keep ? sign : 0.0;
      for (int i = lane; i < k; i += 32) {
        // plain: U_w = a / sigma, V_w = v; preconditioned: U_w = v (= Q V_x), V_w(piv) = a / sigma
        const double u = pre ? v[i] * vs : a[i] * inv, vv = pre ? a[i] * inv : v[i] * vs;
        const int iv = pre ? piv[i] : i;
        if (Uw64) Uw64[(size_t)i * k + jr] = u;
        if (Vw64) Vw64[(size_t)iv * k + jr] = vv;
        if (uw32) uw32[(size_t)i * ld32 + jr] = static_cast<float>(u);
        if (vw32) vw32[(size_t)iv * ld32 + jr] = static_cast<float>(vv);
      }
    }
  }
  sc_cluster_sync();  // no CTA exits while others still read its shared memory
}

template <int EPL>
static bool launch_sc(int k, int w, int P, const float* W, int64_t ldw, const double* Xt, const double* Hq,
                      const int* piv, double tol, double* sig, double* Uw64, double* Vw64, float* uw32, float* vw32,
                      int64_t ld32, int* r_ws, int* r_user, void* ws, cudaStream_t st) {
  const size_t smem = sizeof(double) * 2 * (size_t)w * 2 * 32 * EPL * (EPL <= 5 ? 2 : 1);
  auto kern = svd_cluster_kernel<EPL>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024) != cudaSuccess) return false;
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(P));
  cfg.blockDim = dim3(kScThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = static_cast<unsigned>(P);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, k, w, W, ldw, Xt, Hq, piv, tol, sig, Uw64, Vw64, uw32, vw32, ld32, r_ws,
                            r_user, ws) == cudaSuccess;
}

template <int E>
static bool launch_qrg(int k, const float* W, int64_t ldw, const SvdQrBufs& b, void* ws, cudaStream_t st) {
  QrGrid g{};
  g.kr = static_cast<int>(round_up(k, 32));
  g.colbuf = b.extra;
  g.bests = g.colbuf + (size_t)2 * b.K * round_up(b.K, 32);
  g.rd = g.bests + 2 * 128 * 2;
  g.bar = reinterpret_cast<unsigned*>(g.rd + b.K);
  if (cudaMemsetAsync(g.bar, 0, sizeof(unsigned), st) != cudaSuccess) return false;
  const int nb = static_cast<int>(ceil_div(k, 4));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(nb));
  cfg.blockDim = dim3(128);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeCooperative;  // one barrier per pivot step: every CTA co-resident
  at[0].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  note_launch();
  return cudaLaunchKernelEx(&cfg, svd_qrcp_grid_kernel<E>, k, W, ldw, b.Xt, b.Hv, b.Rg, b.piv, g, ws) == cudaSuccess;
}

// k in (16, 320]: 2P blocks of w <= 16 columns on a cluster of P CTAs
bool launch_svd_cluster(int k, const float* W, int64_t ldw, double tol, double* sig, double* Uw64, double* Vw64,
                        float* uw32, float* vw32, int64_t ld32, int* r_ws, int* r_user, void* ws, cudaStream_t st,
                        const SvdQrBufs* qb) {
  if (k < 2 || k > kScKmax) return false;
  const int P = static_cast<int>(ceil_div(k, 32));
  const int w = static_cast<int>(ceil_div(k, 2 * P));
  if (w > 16) return false;
  const int epl = static_cast<int>(ceil_div(k, 32));
  // QR preconditioning for k > 128 (the grid QR kernel; CABS_SVD_NOQR: plain Jacobi on W)
  const double* Xt = nullptr;
  const double* Hq = nullptr;
  const int* piv = nullptr;
  if (qb && qb->extra && k > 128 && !getenv("CABS_SVD_NOQR")) {
    bool q = false;
    if (epl <= 5) q = launch_qrg<5>(k, W, ldw, *qb, ws, st);
    else if (epl <= 8) q = launch_qrg<8>(k, W, ldw, *qb, ws, st);
    else q = launch_qrg<10>(k, W, ldw, *qb, ws, st);
    if (q) { Xt = qb->Xt; Hq = qb->Hv; piv = qb->piv; } else { cudaGetLastError(); }
  }
  bool ok;
  if (epl <= 4) ok = launch_sc<4>(k, w, P, W, ldw, Xt, Hq, piv, tol, sig, Uw64, Vw64, uw32, vw32, ld32, r_ws, r_user, ws, st);
  else if (epl <= 5) ok = launch_sc<5>(k, w, P, W, ldw, Xt, Hq, piv, tol, sig, Uw64, Vw64, uw32, vw32, ld32, r_ws, r_user, ws, st);
  else if (epl <= 7) ok = launch_sc<7>(k, w, P, W, ldw, Xt, Hq, piv, tol, sig, Uw64, Vw64, uw32, vw32, ld32, r_ws, r_user, ws, st);
  else ok = launch_sc<10>(k, w, P, W, ldw, Xt, Hq, piv, tol, sig, Uw64, Vw64, uw32, vw32, ld32, r_ws, r_user, ws, st);
  if (!ok) cudaGetLastError();
  return ok;
}

}  // namespace cabsk
