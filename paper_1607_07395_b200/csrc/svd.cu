// svd.cu -- S4: the k x k SVD of W in FP64 ("Assuming an SVD W = U_w Sigma_w V_w^T").
//
// One-sided (Hestenes) Jacobi on the columns of W: plane rotations applied from
// the right orthogonalise the columns, W V = U Sigma.  Round-robin (circle-method)
// ordering gives k/2 disjoint column pairs per round, one warp per pair, all in
// one CTA.  Columns live in shared memory when 2 k^2 doubles fit (k <= 112),
// otherwise in the (L2-resident) workspace.  Output: sigma descending, truncation
// count r = #{sigma_i > tol sigma_1} (Z4), canonical signs (Z5).
#include <float.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

#include <cooperative_groups.h>
namespace cg = cooperative_groups;

#ifndef CABS_SVD_TSTOP
// Stop after a sweep whose rotations all had |t| below this: Jacobi converges quadratically,
// so the next sweep would rotate by O(t^2) ~ 1e-12 -- U_w, V_w are then orthonormal to
// ~1e-12 (measured <= 1e-12, tools/probe.py svd), five orders below the resolution of their
// FP32 consumers; sigma errors are second order (~1e-15).  1e-8 costs one more sweep.
#define CABS_SVD_TSTOP 1e-6
#endif
namespace cabsk {

constexpr int kSvdThreads = 1024;
constexpr int kSvdMaxSweeps = 60;
constexpr int kSvdSmemK = 112;


// Circle-method tournament: player 0 fixed, the others rotate by one seat per round.
// 0 <= j - 1 + r < 2 (np - 1), so the modulo is one conditional subtraction.
__device__ __forceinline__ int rr_player(int j, int r, int np) {
  int x = j - 1 + r;
  if (x >= np - 1) x -= np - 1;
  return j == 0 ? 0 : 1 + x;
}


// Jacobi rotation for the pair (x, y) with al = x.x, be = y.y, ga = x.y:
// t = sign(zeta)/(|zeta| + sqrt(1 + zeta^2)), zeta = (be - al)/(2 ga), evaluated in FP32
// on operands scaled by an exact power of two (exponent arithmetic on the bits): t's
// accuracy only sets the convergence rate.  c = 1/sqrt(1+t^2) to FP64 accuracy (FP32
// seed + two Newton steps) and s = c t keep the rotation orthogonal to FP64 rounding.
// Returns t == 0 (c = 1, s = 0) when the pair is already orthogonal to tol_rot.
__device__ __forceinline__ float jacobi_angle(double al, double be, double ga, double tol_rot2, double& c,
                                              double& sn) {
  const bool need = ga != 0.0 && ga * ga > tol_rot2 * al * be;
  const double dx = be - al, dy = 2.0 * ga;
  const double mx = fmax(fabs(dx), fabs(dy));
  const int ex = static_cast<int>((__double_as_longlong(mx) >> 52) & 0x7ff);
  const double scl = __longlong_as_double(static_cast<long long>(2046 - ex) << 52);
  const float xf = static_cast<float>(dx * scl), yf = static_cast<float>(dy * scl);
  const float hyp = fmaf(xf, xf, yf * yf);
  const float den = fabsf(xf) + hyp * __frsqrt_rn(hyp);
  float tf = copysignf(1.f, xf) * __fdividef(yf, den);
  tf = (need && ex > 0 && ex < 2046 && den > 0.f) ? tf : 0.f;
  const double t = static_cast<double>(tf);
  const double q1 = fma(t, t, 1.0);
  double cc = static_cast<double>(__frsqrt_rn(static_cast<float>(q1)));
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  c = cc;
  sn = cc * t;
  return tf;
}

// The same rotation with FP64 approximate reciprocal / rsqrt (MUFU) for t: inputs are
// squares of FP32-born data, so dx^2 + dy^2 cannot overflow FP64.  Returns "rotated".
__device__ __forceinline__ double rsqrt_approx64(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
__device__ __forceinline__ double rcp_approx64(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}
// t of the rotation (0 when the pair is already orthogonal to tol_rot)
__device__ __forceinline__ double jacobi_t(double al, double be, double ga, double tol_rot2, bool& need) {
  need = ga != 0.0 && ga * ga > tol_rot2 * al * be;
  const double dx = be - al, dy = 2.0 * ga;
  const double h = fma(dx, dx, dy * dy);
  const double den = fabs(dx) + h * rsqrt_approx64(h);      // |dx| + sqrt(dx^2 + dy^2)
  return need ? copysign(1.0, dx) * dy * rcp_approx64(den) : 0.0;
}
// c = 1/sqrt(1 + t^2) to FP64 accuracy (approximation + two Newton steps), s = c t
__device__ __forceinline__ void rot_cs(double t, double& c, double& sn) {
  const double q1 = fma(t, t, 1.0);
  double cc = rsqrt_approx64(q1);
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  cc = cc * fma(-0.5 * q1, cc * cc, 1.5);
  c = cc;
  sn = cc * t;
}
__device__ __forceinline__ bool jacobi_angle_fast(double al, double be, double ga, double tol_rot2, double& c,
                                                  double& sn) {
  bool need;
  rot_cs(jacobi_t(al, be, ga, tol_rot2, need), c, sn);
  return need;
}

// Cyclic one-sided Jacobi sweeps until no pair needs a rotation (or the sweep cap).
// A group of LP lanes (LP | 32) runs one column pair, each lane holding E = ceil(k/LP)
// elements of both columns in registers (rows g + LP e), so a warp advances 32/LP
// pairs at once and the dot products are LP-lane butterflies.  A round is one
// dependent chain (loads -> dots -> butterfly -> angle -> update -> barrier), so the
// body is branch-free: the angle is always computed (t = 0 when no rotation is due),
// the update always stored, and the rotation count rides on the round's barrier.
template <int LP, int E>
__device__ int jacobi_sweeps(double* A, int k) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  constexpr int kGroups = 32 / LP;
  const int grp = lane / LP, gl = lane % LP;
  const int np = (k + 1) & ~1;  // even number of players (dummy = k when k is odd)
  const int npairs = np / 2;
  const double tol_rot = 2.0 * sqrt(static_cast<double>(k)) * DBL_EPSILON;
  const double tol_rot2 = tol_rot * tol_rot;
  int sweep = 0;
  for (; sweep < kSvdMaxSweeps; ++sweep) {
    int rotations = 0;
    for (int rnd = 0; rnd < np - 1; ++rnd) {
      int rotated = 0;
      // warp-uniform trip count; the pair index differs per lane group
      for (int base = warp * kGroups; base < npairs; base += nwarps * kGroups) {
        const int pr = base + grp;
        const int prc = pr < npairs ? pr : 0;
        int p = rr_player(prc, rnd, np), q = rr_player(np - 1 - prc, rnd, np);
        const int lo = p < q ? p : q, hi = p < q ? q : p;
        const bool real = pr < npairs && hi < k;  // group-uniform
        double* ap = A + (size_t)(real ? lo : 0) * k;
        double* aq = A + (size_t)(real ? hi : 0) * k;
        double x[E], y[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = gl + LP * e;
          const bool in = real && i < k;
          x[e] = in ? ap[i] : 0.0;
          y[e] = in ? aq[i] : 0.0;
        }
        // two interleaved partial sums per dot product halve the dependent FMA chains
        double al0 = 0, be0 = 0, ga0 = 0, al1 = 0, be1 = 0, ga1 = 0;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
          al0 = fma(x[e], x[e], al0);
          be0 = fma(y[e], y[e], be0);
          ga0 = fma(x[e], y[e], ga0);
          if (e + 1 < E) {
            al1 = fma(x[e + 1], x[e + 1], al1);
            be1 = fma(y[e + 1], y[e + 1], be1);
            ga1 = fma(x[e + 1], y[e + 1], ga1);
          }
        }
        double al = al0 + al1, be = be0 + be1, ga = ga0 + ga1;
#pragma unroll
        for (int o = LP / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        double c, sn;
        const float tf = jacobi_angle(al, be, ga, tol_rot2, c, sn);
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = gl + LP * e;
          if (real && i < k) {
            ap[i] = c * x[e] - sn * y[e];
            aq[i] = sn * x[e] + c * y[e];
          }
        }
        rotated |= tf != 0.f;
      }
      rotations += __syncthreads_count(rotated);
    }
    if (rotations == 0) break;
  }
  return sweep;
}


// ---------------------------------------------------------------- shared epilogue
// Singular values = column norms of the converged A; rank order descending (ties -> lower
// column); truncation count r = #{sigma_i > tol sigma_1} (Z4).  Ends with a barrier.
__device__ int svd_sigma(const double* A, int k, double tol, double* s_sig, int* s_perm, double* sigma_out,
                         int* r_out, int* r_out2) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int c = warp; c < k; c += nwarps) {
    const double* ac = A + (size_t)c * k;
    double ss = 0;
    for (int i = lane; i < k; i += 32) ss = fma(ac[i], ac[i], ss);
    ss = warp_sum_d(ss);
    if (lane == 0) s_sig[c] = sqrt(ss);
  }
  __syncthreads();
  for (int c = tid; c < k; c += blockDim.x) {
    const double sc = s_sig[c];
    int rk = 0;
    for (int j = 0; j < k; ++j) {
      const double sj = s_sig[j];
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
  return r;
}

// U_w = a_c / sigma_c and V_w in rank order, canonical sign (Z5: the largest-|.| entry of
// each U_w column positive, lowest index on ties); dropped components written as zeros.
__device__ void svd_write(const double* A, const double* V, int k, int r, const double* s_sig, const int* s_perm,
                          double* __restrict__ Uw64, double* __restrict__ Vw64, float* __restrict__ uw32,
                          float* __restrict__ vw32, int64_t ld32) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
  for (int j = warp; j < k; j += nwarps) {
    const int c = s_perm[j];
    const double sg = s_sig[c];
    const bool keep = j < r;
    const double* ac = A + (size_t)c * k;
    const double* vc = V + (size_t)c * k;
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int i = lane; i < k; i += 32) {
      const double v = fabs(ac[i]);
      if (v > best || (v == best && i < bi)) { best = v; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
    }
    const double sign = (bi < k && ac[bi] < 0) ? -1.0 : 1.0;
    const double inv = (keep && sg > 0) ? sign / sg : 0.0;
    const double vs = keep ? sign : 0.0;
    for (int i = lane; i < k; i += 32) {
      const double u = ac[i] * inv, v = vc[i] * vs;
      if (Uw64) Uw64[(size_t)i * k + j] = u;
      if (Vw64) Vw64[(size_t)i * k + j] = v;
      if (uw32) uw32[(size_t)i * ld32 + j] = static_cast<float>(u);
      if (vw32) vw32[(size_t)i * ld32 + j] = static_cast<float>(v);
    }
  }
  if (uw32) {  // zero padding columns [k, ld32)
    for (int64_t e = tid; e < (int64_t)k * (ld32 - k); e += blockDim.x) {
      const int64_t i = e / (ld32 - k), c = k + e % (ld32 - k);
      uw32[i * ld32 + c] = 0.f;
      vw32[i * ld32 + c] = 0.f;
    }
  }
}

// ---------------------------------------------------------------- k <= 64: register-resident, odd-even
// Each pair slot g (a group of LP lanes; lane l holds rows l + LP e, e < E) keeps the
// columns at positions 2g (L) and 2g+1 (R) of A AND of V in registers.  Ordering: the
// odd-even transposition network (every round swaps the columns of each active pair, so
// after n = 2P rounds every pair has met exactly once):
//   even rounds  pairs (2g, 2g+1): inside the slot, no data movement, no barrier;
//   odd rounds   pairs (2g+1, 2g+2): each slot publishes L and R through shared memory
//                (double-buffered by odd-round parity), ONE barrier, then computes both
//                pairs it takes part in (bit-identical to its neighbours' copies) and
//                keeps its own rotated halves.  Idle ends (positions 0 and n-1) use the
//                rotation (c, s) = (0, -/+1), which with the swap leaves them in place.
// Rotations are accumulated into V on the way, so V is orthogonal to FP64 rounding
// without a Gram-Schmidt pass.
template <int E>
__device__ __forceinline__ void pair_dots(const double (&x)[E], const double (&y)[E], double& al, double& be,
                                          double& ga) {
  double al0 = 0, be0 = 0, ga0 = 0, al1 = 0, be1 = 0, ga1 = 0;
#pragma unroll
  for (int e = 0; e < E; e += 2) {
    al0 = fma(x[e], x[e], al0);
    be0 = fma(y[e], y[e], be0);
    ga0 = fma(x[e], y[e], ga0);
    if (e + 1 < E) {
      al1 = fma(x[e + 1], x[e + 1], al1);
      be1 = fma(y[e + 1], y[e + 1], be1);
      ga1 = fma(x[e + 1], y[e + 1], ga1);
    }
  }
  al = al0 + al1;
  be = be0 + be1;
  ga = ga0 + ga1;
}

template <int LP>
__device__ __forceinline__ double group_sum(double v) {
#pragma unroll
  for (int o = LP / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int LP, int E>
__global__ void __launch_bounds__(128, 1)
svd_systolic_kernel(int k, const float* __restrict__ W, int64_t ldw, double tol, double* __restrict__ sigma_out,
                    double* __restrict__ Uw64, double* __restrict__ Vw64, float* __restrict__ uw32,
                    float* __restrict__ vw32, int64_t ld32, int* r_out, int* r_out2, void* ws) {
  constexpr int G = 32 / LP;        // pair slots per warp
  // doubles per published column, padded so that consecutive seats start 32 bytes apart
  // modulo 128 (the 8 slots of a warp then cover the 32 banks twice: conflict-free)
  constexpr int SEAT = E * LP + ((4 - (E * LP) % 16) + 16) % 16;
  extern __shared__ __align__(16) double smem_d[];
  __shared__ double s_sig[64];
  __shared__ int s_perm[64];
  __shared__ int s_id[2][2][34];    // [parity][L|R][seat]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int gl = lane % LP, gw = lane / LP;
  const int g = warp * G + gw;
  const int np = (k + 1) & ~1, P = np / 2;
  const int nseat = nw * G + 2;     // seat g + 1 <- slot g; seats 0 and nw G + 1 stay zero
  const bool live = g < P;
  // published columns: [parity][seat][e][LP] for A_L, A_R, V_L, V_R
  const size_t arr = (size_t)2 * nseat * SEAT;
  double* bAL = smem_d;
  double* bAR = bAL + arr;
  double* bVL = bAR + arr;
  double* bVR = bVL + arr;
  for (int e = tid; e < 4 * (int)arr; e += blockDim.x) smem_d[e] = 0.0;

  double aL[E], aR[E], vL[E], vR[E];
  int idL = 2 * g, idR = 2 * g + 1;  // column ids (>= k: dummy zero column)
  bool bad = false;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = gl + LP * e;
    float wl = 0.f, wr = 0.f;
    if (live && i < k && idL < k) wl = W[(int64_t)i * ldw + idL];
    if (live && i < k && idR < k) wr = W[(int64_t)i * ldw + idR];
    bad |= !isfinite(wl) || !isfinite(wr);
    aL[e] = wl;
    aR[e] = wr;
    vL[e] = (i == idL && idL < k) ? 1.0 : 0.0;
    vR[e] = (i == idR && idR < k) ? 1.0 : 0.0;
  }
  if (bad) set_status(ws, CABS_DEV_NONFINITE);
  __syncthreads();
  const double tol_rot = 2.0 * sqrt(static_cast<double>(k)) * DBL_EPSILON;
  const double tol_rot2 = tol_rot * tol_rot;
  const bool left_edge = g == 0, right_edge = g == P - 1;
  int sweep = 0;
  if (k > 1) {
    for (; sweep < kSvdMaxSweeps; ++sweep) {
      int rotated = 0;
      for (int rnd = 0; rnd < np; ++rnd) {
        if ((rnd & 1) == 0) {
          // ---- even round: pair (L, R) of this slot; rotate and swap
          double al, be, ga, c, sn;
          pair_dots<E>(aL, aR, al, be, ga);
          al = group_sum<LP>(al);
          be = group_sum<LP>(be);
          ga = group_sum<LP>(ga);
          rotated |= jacobi_angle_fast(al, be, ga, tol_rot2, c, sn) && live;
#pragma unroll
          for (int e = 0; e < E; ++e) {
            const double x = aL[e], y = aR[e], vx = vL[e], vy = vR[e];
            aL[e] = sn * x + c * y;  // position 2g <- y'
            aR[e] = c * x - sn * y;  // position 2g+1 <- x'
            vL[e] = sn * vx + c * vy;
            vR[e] = c * vx - sn * vy;
          }
          const int t = idL;
          idL = idR;
          idR = t;
          continue;
        }
        // ---- odd round: publish, barrier, pairs (R_{g-1}, L_g) and (R_g, L_{g+1})
        const int par = (rnd >> 1) & 1;
        const size_t pub = ((size_t)par * nseat + g + 1) * SEAT + gl;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          bAL[pub + e * LP] = aL[e];
          bAR[pub + e * LP] = aR[e];
          bVL[pub + e * LP] = vL[e];
          bVR[pub + e * LP] = vR[e];
        }
        if (gl == 0) {
          s_id[par][0][g + 1] = idL;
          s_id[par][1][g + 1] = idR;
        }
        __syncthreads();
        const size_t lft = ((size_t)par * nseat + g) * SEAT + gl;      // slot g - 1 (seat 0: zeros)
        const size_t rgt = ((size_t)par * nseat + g + 2) * SEAT + gl;  // slot g + 1
        double rm[E], lp[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
          rm[e] = bAR[lft + e * LP];
          lp[e] = bAL[rgt + e * LP];
        }
        double alA, beA, gaA, alB, beB, gaB, cA, sA, cB, sB;
        pair_dots<E>(rm, aL, alA, beA, gaA);
        pair_dots<E>(aR, lp, alB, beB, gaB);
        alA = group_sum<LP>(alA);
        beA = group_sum<LP>(beA);
        gaA = group_sum<LP>(gaA);
        alB = group_sum<LP>(alB);
        beB = group_sum<LP>(beB);
        gaB = group_sum<LP>(gaB);
        const bool rA = jacobi_angle_fast(alA, beA, gaA, tol_rot2, cA, sA);
        const bool rB = jacobi_angle_fast(alB, beB, gaB, tol_rot2, cB, sB);
        rotated |= live && ((rA && !left_edge) || (rB && !right_edge));
        if (left_edge) { cA = 0.0; sA = -1.0; }
        if (right_edge) { cB = 0.0; sB = 1.0; }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double vm = bVR[lft + e * LP], vp = bVL[rgt + e * LP];
          aL[e] = cA * rm[e] - sA * aL[e];  // x' of the left pair
          aR[e] = sB * aR[e] + cB * lp[e];  // y' of the right pair
          vL[e] = cA * vm - sA * vL[e];
          vR[e] = sB * vR[e] + cB * vp;
        }
        if (!left_edge) idL = s_id[par][1][g];
        if (!right_edge) idR = s_id[par][0][g + 2];
      }
      rotated = __syncthreads_or(rotated);
      if (!rotated) break;
    }
    if (sweep == kSvdMaxSweeps && tid == 0) set_status(ws, CABS_DEV_SVD_NOCONV);
  }
  if (tid == 0) reinterpret_cast<int*>(ws)[8] = sweep;  // diagnostics: sweeps of the last SVD
  __syncthreads();
  // ---- converged columns -> shared memory (column-major by original column id)
  double* As = smem_d;
  double* Vs = smem_d + (size_t)k * k;
  if (live) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = gl + LP * e;
      if (i < k) {
        if (idL < k) { As[(size_t)idL * k + i] = aL[e]; Vs[(size_t)idL * k + i] = vL[e]; }
        if (idR < k) { As[(size_t)idR * k + i] = aR[e]; Vs[(size_t)idR * k + i] = vR[e]; }
      }
    }
  }
  __syncthreads();
  const int r = svd_sigma(As, k, tol, s_sig, s_perm, sigma_out, r_out, r_out2);
  svd_write(As, Vs, k, r, s_sig, s_perm, Uw64, Vw64, uw32, vw32, ld32);
}

// ---------------------------------------------------------------- k <= 64: A and V on two SMs
// A cluster of two CTAs: CTA 0 runs the register-resident odd-even Jacobi on the columns of
// A only (half the data movement of carrying V) and streams every round's rotations
// (c, s) into CTA 1's shared memory through DSMEM; CTA 1 applies them to V = I with the same
// odd-even data movement, one sweep behind (a sweep buffer per parity, one mbarrier signal per
// sweep each way).  At the end CTA 1 stores V's columns (by column id) into CTA 0, which runs
// the common epilogue.  Rotation formulas, ordering and convergence test are those of
// svd_systolic_kernel; CTA 0 streams the (c, s) pairs themselves, so A and V see
// bit-identical rotations and CTA 1's round has no angle computation on it.
__device__ __forceinline__ uint32_t dsmem_map(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(tc::smem_u32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void dsmem_st_f64(uint32_t addr, double v) {
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(addr), "d"(v) : "memory");
}
// Generic-address form for stores inside the sweep loop: the peer address is mapped once
// (mapa on the generic address), and the store carries no compiler memory clobber (the
// ordering that matters -- before the cluster fence + mbarrier release at the sweep end --
// is kept because both are volatile asm).
__device__ __forceinline__ double* dsmem_map_generic(const void* p, uint32_t rank) {
  uint64_t r;
  asm volatile("mapa.u64 %0, %1, %2;" : "=l"(r) : "l"(p), "r"(rank));
  return reinterpret_cast<double*>(r);
}
__device__ __forceinline__ void dsmem_st2_f64(double* gaddr, double a, double b) {
  asm volatile("st.v2.f64 [%0], {%1, %2};" ::"l"(gaddr), "d"(a), "d"(b));
}
__device__ __forceinline__ void dsmem_st_s32(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\n"
      "bra WAIT_%=;\n"
      "DONE_%=:\n"
      "}\n" ::"r"(tc::smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}


template <int LP, int E>
__global__ void __launch_bounds__(256, 1) __cluster_dims__(2, 1, 1)
svd_split_kernel(int k, const float* __restrict__ W, int64_t ldw, double tol, double* __restrict__ sigma_out,
                 double* __restrict__ Uw64, double* __restrict__ Vw64, float* __restrict__ uw32,
                 float* __restrict__ vw32, int64_t ld32, int* r_out, int* r_out2, void* ws) {
  constexpr int G = 32 / LP;
  constexpr int SEAT = E * LP + ((LP - (E * LP) % 16) + 16) % 16;  // slot footprints tile the banks
  extern __shared__ __align__(16) double smem_d[];
  __shared__ double s_sig[64];
  __shared__ int s_perm[64];
  __shared__ int s_id[2][2][34];
  __shared__ __align__(8) uint64_t bar_full[2], bar_empty[2];  // full: in CTA 1, empty: in CTA 0
  __shared__ int s_last[2];                                    // CTA 1: last sweep flag per parity
  __shared__ double s_nrm[2][2][34];                           // CTA 0: published squared norms [parity][L|R][seat]
  const uint32_t crank = cg::this_cluster().block_rank();
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int gl = lane % LP, gw = lane / LP;
  const int g = warp * G + gw;
  const int np = (k + 1) & ~1, P = np / 2;
  const int nseat = nw * G + 2;
  const bool live = g < P;
  const bool left_edge = g == 0, right_edge = g == P - 1;
  // smem: exchange [XL|XR][parity][seat][SEAT] | (CTA 1) rotations (c, s) [parity][round][slot][4] |
  // (CTA 0) final A and V columns [k][k] each (reusing the exchange area)
  const size_t arr = (size_t)2 * nseat * SEAT;
  double* bXL = smem_d;
  double* bXR = bXL + arr;
  double* prm = bXR + arr;  // CTA 1 only
  if (tid == 0) {
    tc::mbar_init(&bar_full[0], 1); tc::mbar_init(&bar_full[1], 1);
    tc::mbar_init(&bar_empty[0], 1); tc::mbar_init(&bar_empty[1], 1);
    tc::mbar_fence_init();
  }
  for (int e = tid; e < 2 * (int)arr; e += blockDim.x) smem_d[e] = 0.0;
  for (int e = tid; e < 2 * 2 * 34; e += blockDim.x) (&s_nrm[0][0][0])[e] = 0.0;
  cluster_sync_all();

  double xL[E], xR[E];  // CTA 0: columns of A; CTA 1: columns of V
  int idL = 2 * g, idR = 2 * g + 1;
  if (crank == 0) {
    bool bad = false;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = gl + LP * e;
      float wl = 0.f, wr = 0.f;
      if (live && i < k && idL < k) wl = W[(int64_t)i * ldw + idL];
      if (live && i < k && idR < k) wr = W[(int64_t)i * ldw + idR];
      bad |= !isfinite(wl) || !isfinite(wr);
      xL[e] = wl;
      xR[e] = wr;
    }
    if (bad) set_status(ws, CABS_DEV_NONFINITE);
  } else {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = gl + LP * e;
      xL[e] = (i == idL && idL < k) ? 1.0 : 0.0;
      xR[e] = (i == idR && idR < k) ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  const double tol_rot = 2.0 * sqrt(static_cast<double>(k)) * DBL_EPSILON;
  const double tol_rot2 = tol_rot * tol_rot;
  // remote addresses (CTA 0 -> CTA 1 params and full barriers; CTA 1 -> CTA 0 empty barriers)
  const uint32_t prm_remote = dsmem_map(prm, 1);
  const uint32_t full_remote0 = dsmem_map(&bar_full[0], 1), full_remote1 = dsmem_map(&bar_full[1], 1);
  const uint32_t empty_remote0 = dsmem_map(&bar_empty[0], 0), empty_remote1 = dsmem_map(&bar_empty[1], 0);
  const uint32_t last_remote = dsmem_map(&s_last[0], 1);
#ifdef CABS_PROFILE_SVD
  long long sprof[8] = {0, 0, 0, 0, 0, 0, 0, 0}, st0 = clock64();
#define SPROF(i) do { if (crank == 0 && tid == 0) { const long long t1_ = clock64(); sprof[i] += t1_ - st0; st0 = t1_; } } while (0)
#else
#define SPROF(i) do { } while (0)
#endif
  int sweep = 0;
  bool last = k <= 1;
  for (; !last; ++sweep) {
    const int sp = sweep & 1;
    if (crank == 0 && sweep >= 2) mbar_wait_cluster(&bar_empty[sp], static_cast<uint32_t>(((sweep - 2) >> 1) & 1));
    if (crank == 1) {
      mbar_wait_cluster(&bar_full[sp], static_cast<uint32_t>((sweep >> 1) & 1));
    }
    int rotated = 0;
    double tmax = 0.0;  // largest |t| of this sweep (CTA 0)
    // squared column norms: recomputed exactly at every sweep start, then carried through
    // the rotations by the exact 2x2 formulas, so a round reduces only the cross products
    double nL = 0.0, nR = 0.0;
    if (crank == 0) {
      double t0 = 0.0, t1 = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) { t0 = fma(xL[e], xL[e], t0); t1 = fma(xR[e], xR[e], t1); }
      nL = group_sum<LP>(t0);
      nR = group_sum<LP>(t1);
    }
    for (int rnd = 0; rnd < np; ++rnd) {
      const int pidx = ((sp * np + rnd) * P + (live ? g : 0)) * 4;  // [parity][round][slot][4]
      const double* pr = prm + pidx;                                 // CTA 1 view
      const uint32_t prr = prm_remote + static_cast<uint32_t>(pidx * 8);
      if ((rnd & 1) == 0) {
        double c, sn;
        if (crank == 0) {
          SPROF(7);
          double ga0 = 0.0, ga1 = 0.0;
#pragma unroll
          for (int e = 0; e < E; e += 2) {
            ga0 = fma(xL[e], xR[e], ga0);
            if (e + 1 < E) ga1 = fma(xL[e + 1], xR[e + 1], ga1);
          }
          SPROF(0);
#ifdef SVD_NO_BFLY
          const double ga = ga0 + ga1;
#else
          const double ga = group_sum<LP>(ga0 + ga1);
#endif
          SPROF(1);
          bool need;
#ifdef SVD_FAST_ANGLE
          need = ga * ga > tol_rot2 * nL * nR;
          const double t = need ? ga * 1e-3 : 0.0;
          c = 1.0;
          sn = t;
#else
          const double t = jacobi_t(nL, nR, ga, tol_rot2, need);
          rot_cs(t, c, sn);
#endif
          rotated |= need && live;
          if (live) tmax = fmax(tmax, fabs(t));
#ifndef SVD_NO_REMOTE
          if (gl == 0 && live) { dsmem_st_f64(prr, c); dsmem_st_f64(prr + 8, sn); }
#endif
          // new L = s x + c y, new R = c x - s y (the swap of the odd-even network)
          const double cs2 = 2.0 * c * sn * ga, c2 = c * c, s2 = sn * sn;
          const double nx = fma(c2, nL, fma(s2, nR, -cs2)), ny = fma(s2, nL, fma(c2, nR, cs2));
          nL = ny;
          nR = nx;
          SPROF(2);
        } else {  // slots beyond P carry no rotations (their columns stay zero)
          c = live ? pr[0] : 1.0;
          sn = live ? pr[1] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const double x = xL[e], y = xR[e];
          xL[e] = sn * x + c * y;
          xR[e] = c * x - sn * y;
        }
        const int t = idL;
        idL = idR;
        idR = t;
        SPROF(3);
        continue;
      }
      SPROF(7);
      const int par = (rnd >> 1) & 1;
      const size_t pub = ((size_t)par * nseat + g + 1) * SEAT + gl;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        bXL[pub + e * LP] = xL[e];
        bXR[pub + e * LP] = xR[e];
      }
      if (gl == 0) {
        s_id[par][0][g + 1] = idL;
        s_id[par][1][g + 1] = idR;
        if (crank == 0) {
          s_nrm[par][0][g + 1] = nL;
          s_nrm[par][1][g + 1] = nR;
        }
      }
      SPROF(4);
      __syncthreads();
      SPROF(5);
      const size_t lft = ((size_t)par * nseat + g) * SEAT + gl;
      const size_t rgt = ((size_t)par * nseat + g + 2) * SEAT + gl;
      double rm[E], lp[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        rm[e] = bXR[lft + e * LP];
        lp[e] = bXL[rgt + e * LP];
      }
      double cA, sA, cB, sB;
      if (crank == 0) {
        SPROF(6);
        double gA0 = 0.0, gA1 = 0.0, gB0 = 0.0, gB1 = 0.0;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
          gA0 = fma(rm[e], xL[e], gA0);
          gB0 = fma(xR[e], lp[e], gB0);
          if (e + 1 < E) {
            gA1 = fma(rm[e + 1], xL[e + 1], gA1);
            gB1 = fma(xR[e + 1], lp[e + 1], gB1);
          }
        }
        const double nRm = s_nrm[par][1][g], nLp = s_nrm[par][0][g + 2];
        SPROF(0);
#ifdef SVD_NO_BFLY
        const double gaA = gA0 + gA1, gaB = gB0 + gB1;
#else
        const double gaA = group_sum<LP>(gA0 + gA1), gaB = group_sum<LP>(gB0 + gB1);
#endif
        SPROF(1);
        bool rA, rB;
#ifdef SVD_FAST_ANGLE
        rA = gaA * gaA > tol_rot2 * nRm * nL;
        rB = gaB * gaB > tol_rot2 * nR * nLp;
        const double tA = rA ? gaA * 1e-3 : 0.0, tB = rB ? gaB * 1e-3 : 0.0;
        cA = 1.0; sA = tA; cB = 1.0; sB = tB;
#else
        const double tA = jacobi_t(nRm, nL, gaA, tol_rot2, rA), tB = jacobi_t(nR, nLp, gaB, tol_rot2, rB);
        rot_cs(tA, cA, sA);
        rot_cs(tB, cB, sB);
#endif
        rotated |= live && ((rA && !left_edge) || (rB && !right_edge));
        if (live && !left_edge) tmax = fmax(tmax, fabs(tA));
        if (live && !right_edge) tmax = fmax(tmax, fabs(tB));
#ifndef SVD_NO_REMOTE
        if (gl == 0 && live) {
          dsmem_st_f64(prr, cA); dsmem_st_f64(prr + 8, sA);
          dsmem_st_f64(prr + 16, cB); dsmem_st_f64(prr + 24, sB);
        }
#endif
        if (left_edge) { cA = 0.0; sA = -1.0; }
        if (right_edge) { cB = 0.0; sB = 1.0; }
        // new L = x'_A = cA Rm - sA L, new R = y'_B = sB R + cB Lp
        const double nxA = fma(cA * cA, nRm, fma(sA * sA, nL, -2.0 * cA * sA * gaA));
        const double nyB = fma(sB * sB, nR, fma(cB * cB, nLp, 2.0 * cB * sB * gaB));
        nL = nxA;
        nR = nyB;
        SPROF(2);
      } else {
        cA = live ? pr[0] : 1.0; sA = live ? pr[1] : 0.0;
        cB = live ? pr[2] : 1.0; sB = live ? pr[3] : 0.0;
      }
      if (left_edge) { cA = 0.0; sA = -1.0; }
      if (right_edge) { cB = 0.0; sB = 1.0; }
#pragma unroll
      for (int e = 0; e < E; ++e) {
        xL[e] = cA * rm[e] - sA * xL[e];
        xR[e] = sB * xR[e] + cB * lp[e];
      }
      if (!left_edge) idL = s_id[par][1][g];
      if (!right_edge) idR = s_id[par][0][g + 2];
      SPROF(3);
    }
    if (crank == 0) {
      rotated = __syncthreads_or(rotated);
      // quadratic convergence: after a sweep whose rotations all had |t| < 1e-8 the next
      // sweep's would be below the rotation threshold (|t| ~ 1e-16), so it is not run
      const int small = __syncthreads_and(tmax < CABS_SVD_TSTOP);
      last = !rotated || small || sweep + 1 >= kSvdMaxSweeps;
      if (tid == 0) {
        dsmem_st_s32(last_remote + 4 * sp, last ? 1 : 0);
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        mbar_arrive_remote(sp ? full_remote1 : full_remote0);
      }
    } else {
      __syncthreads();
      last = s_last[sp] != 0;
      __syncthreads();
      if (tid == 0) mbar_arrive_remote(sp ? empty_remote1 : empty_remote0);
    }
  }
  if (crank == 0) {
    if (sweep >= kSvdMaxSweeps && k > 1) set_status(ws, CABS_DEV_SVD_NOCONV);
    if (tid == 0) reinterpret_cast<int*>(ws)[8] = sweep;
#ifdef CABS_PROFILE_SVD
    if (tid == 0)
      for (int i = 0; i < 8; ++i) reinterpret_cast<long long*>(ws)[8 + i] = sprof[i];
#endif
  }
  // converged columns -> CTA 0's shared memory, column-major by id: A (CTA 0) and V (CTA 1)
  cluster_sync_all();  // every exchange buffer read is done in both CTAs
  double* As = smem_d;
  double* Vs = smem_d + (size_t)k * k;
  const uint32_t vs_remote = dsmem_map(Vs, 0);
  if (live) {
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = gl + LP * e;
      if (i < k) {
        if (crank == 0) {
          if (idL < k) As[(size_t)idL * k + i] = xL[e];
          if (idR < k) As[(size_t)idR * k + i] = xR[e];
        } else {
          if (idL < k) dsmem_st_f64(vs_remote + static_cast<uint32_t>(((size_t)idL * k + i) * 8), xL[e]);
          if (idR < k) dsmem_st_f64(vs_remote + static_cast<uint32_t>(((size_t)idR * k + i) * 8), xR[e]);
        }
      }
    }
  }
  cluster_sync_all();
  if (crank != 0) return;
  const int r = svd_sigma(As, k, tol, s_sig, s_perm, sigma_out, r_out, r_out2);
  svd_write(As, Vs, k, r, s_sig, s_perm, Uw64, Vw64, uw32, vw32, ld32);
}

// Scaled rotations.  Columns are kept as actual = d * stored.  The rotation of the pair (x, y)
// at positions (p, p + 1), actual (X, Y) -> (s X + c Y, c X - s Y) (the odd-even network's swap
// included), t = s / c, is applied to the stored columns as
//   p: y + al x  (scale c dy),   p + 1: x - be y  (scale c dx),   al = t dx / dy, be = t dy / dx,
// one FMA per element, and only t (not c) is on the critical path; norms follow the exact
// 2 x 2 formulas.  One lane evaluates it for ITS position: left (p, own column x) or right
// (p + 1, own column y); (on, od, oi) its own n, d, 1 / d, (pn, pd, pi) the other position's,
// gs the stored dot.  Each lane gets its own position's new n, d, 1 / d (the column moving in
// is the partner's, scaled by c).
struct LaneRot {
  double tu, tv, t, n, d, i;
  bool need;
};
__device__ __forceinline__ void lane_rot(bool left, double on, double od, double oi, double pn, double pd, double pi,
                                         double gs, double tol_rot2, LaneRot& r) {
  // left lane: x = own, y = partner; right lane: the mirror image.  Every product below is
  // formed from the same two factors on both lanes (commutation only), dx = ny - nx exactly
  // negated on the right lane, so t is bit-identical on the pair's lanes.
  const double dl = pn - on;
  const double g = gs * (od * pd);
  r.need = g != 0.0 && g * g > tol_rot2 * (on * pn);
  const double dx = left ? dl : -dl, dy = 2.0 * g;
  const double h = fma(dx, dx, dy * dy);
  const double den = fabs(dx) + h * rsqrt_approx64(h);  // |dx| + sqrt(dx^2 + dy^2)
  const double t = r.need ? copysign(1.0, dx) * dy * rcp_approx64(den) : 0.0;
  r.t = t;
  // tu = al (left lane) / be (right lane), tv the other: al = t dx / dy, be = t dy / dx
  r.tu = t * (od * pi);
  r.tv = t * (pd * oi);
  const double q1 = fma(t, t, 1.0);
  double c = rsqrt_approx64(q1);
  c = c * fma(-0.5 * q1, c * c, 1.5);
  c = c * fma(-0.5 * q1, c * c, 1.5);
  const double kg = (left ? 2.0 : -2.0) * g;
  // |s X + c Y|^2 (left), |c X - s Y|^2 (right); the column moving in is the partner's
  r.n = (c * c) * (fma(t * t, on, pn) + t * kg);
  r.d = c * pd;
  r.i = pi * (q1 * c);
}

// ---------------------------------------------------------------- QR preconditioning (k <= 128)
// W P = Q R by Householder QR with column pivoting (largest remaining column norm first, lowest
// column on ties), FP64, one CTA.  One-sided Jacobi then runs on X = R^T instead of W: its
// columns are much closer to orthogonal (the pivoted R is graded), so the sweep count drops
// (c3's pilot W: 15 -> 8 sweeps, tools/dump_w.py + an offline replay).  With X = U_x S V_x^T:
// W = (Q V_x) S (P U_x)^T, so the Jacobi pair's CTA 1 starts its accumulator from Q instead of I
// (forming Q = H_0 ... H_{k-1} from the reflectors itself, while CTA 0 runs the first segment)
// and ends with U_w = Q V_x; CTA 0's normalised columns give V_w with rows permuted by P.
// Outputs: Xt = R^T (k x k row-major), Hv = the reflectors (row j = v_j: 0 above j, vjj at j,
// x below; then k scales beta_j = 2 / v_j^T v_j), piv[j] = the column of W at position j.
// Layout: 8 warps; a group of 8 lanes owns four columns (q = group + 32 t, rows gl + 8 e) in
// registers, stored to shared memory after every step (the next pivot column is read there).
// A step: the pivot is the argmax of the 8 per-warp bests of the previous step (every warp
// reduces the same entries in the same order); x_j and the exact ||x(j:)||^2 give the
// reflector's scalars without a reduction; row j of every column moves to R (a global scratch)
// and is cleared in the registers, so rows above j are zero everywhere and no step needs a row
// mask; every group updates its columns (v^T a: one 3-level group reduction per column; column
// slots finished in the whole warp are skipped) and forms their exact trailing
// norms ||a(j+1:)||^2 (the next pivot keys); row j of R goes to a global scratch.
constexpr int kQrThreads = 256;
constexpr int kQrK = 128;

template <int E>
__global__ void __launch_bounds__(kQrThreads, 1)
svd_qrcp_kernel(int k, const float* __restrict__ W, int64_t ldw, double* __restrict__ Xt, double* __restrict__ Hv,
                double* __restrict__ Rg, int* __restrict__ piv_out, void* ws) {
  constexpr int KP = 8 * E;                      // padded column length
  extern __shared__ __align__(16) double qa[];  // [kQrK columns][KP rows]
  __shared__ double s_wb[2][8];                 // per-warp best key (-1: nothing left), by step parity
  __shared__ int s_wi[2][8];
  __shared__ double s_rd[kQrK];
  __shared__ int s_piv[kQrK];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = tid >> 3, gl = tid & 7;  // group, lane in the group (rows gl + 8 e)
  double a[4][E];
  bool bad = false;
#pragma unroll
  for (int t = 0; t < 4; ++t)
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = gl + 8 * e, q = g + 32 * t;
      float v = 0.f;
      if (i < k && q < k) v = W[(int64_t)i * ldw + q];
      bad |= !isfinite(v);
      a[t][e] = static_cast<double>(v);
    }
  if (bad) set_status(ws, CABS_DEV_NONFINITE);
  uint32_t done = 0;  // bit t: column g + 32 t eliminated (or absent)
#pragma unroll
  for (int t = 0; t < 4; ++t)
    if (g + 32 * t >= k) done |= 1u << t;
  // (key, column) argmax over the group's four columns and the warp's four groups -> s_wb
  auto publish_best = [&](const double (&key)[4], int par) {
    double bk = -1.0;
    int bi = 0x7fffffff;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const double kk = ((done >> t) & 1) ? -1.0 : key[t];
      if (kk > bk) { bk = kk; bi = g + 32 * t; }
    }
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
      const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ok > bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
    }
    if (lane == 0) { s_wb[par][warp] = bk; s_wi[par][warp] = bi; }
  };
  {
    double key[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      double n0 = 0.0, n1 = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e & 1) n1 = fma(a[t][e], a[t][e], n1); else n0 = fma(a[t][e], a[t][e], n0);
      }
      key[t] = n0 + n1;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) key[t] = group_sum<8>(key[t]);
    publish_best(key, 0);
#pragma unroll
    for (int t = 0; t < 4; ++t)
#pragma unroll
      for (int e = 0; e < E; ++e) qa[(g + 32 * t) * KP + gl + 8 * e] = a[t][e];
  }
  __syncthreads();
  for (int j = 0; j < k; ++j) {
    const int par = j & 1;
    // pivot: argmax of the 8 warp bests (identical in every warp)
    double bv = lane < 8 ? s_wb[par][lane] : -1.0;
    int bq = lane < 8 ? s_wi[par][lane] : 0x7fffffff;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oq = __shfl_xor_sync(0xffffffffu, bq, o);
      if (ov > bv || (ov == bv && oq < bq)) { bv = ov; bq = oq; }
    }
    bv = __shfl_sync(0xffffffffu, bv, 0);
    const int ph = __shfl_sync(0xffffffffu, bq, 0);
    const double* xp = qa + ph * KP;
    const double xj = xp[j], nn = fmax(bv, 0.0), sn = sqrt(nn);
    const double alpha = xj >= 0.0 ? -sn : sn;                           // R_jj
    const double vjj = xj - alpha;                                        // x_j + sign(x_j) ||x||
    const double beta = nn > 0.0 ? 1.0 / (sn * (sn + fabs(xj))) : 0.0;    // 2 / v^T v
    // every column's rows above j are zero (cleared at their step), the pivot's too
    double x[E], mz[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      x[e] = xp[gl + 8 * e];
      mz[e] = gl + 8 * e == j ? 0.0 : 1.0;  // clears row j (it moves to R)
    }
#pragma unroll
    for (int t = 0; t < 4; ++t)
      if (g + 32 * t == ph) done |= 1u << t;
    double aj[4], d[4], key[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      aj[t] = qa[(g + 32 * t) * KP + j];
      d[t] = 0.0;
      key[t] = -1.0;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (!__any_sync(0xffffffffu, !((done >> t) & 1))) continue;  // the warp's columns t are all done
      double d0 = gl == 0 ? (vjj - xj) * aj[t] : 0.0, d1 = 0.0;  // v = x with x_j replaced by vjj
#pragma unroll
      for (int e = 0; e < E; ++e) {
        if (e & 1) d1 = fma(x[e], a[t][e], d1); else d0 = fma(x[e], a[t][e], d0);
      }
      const double gsum = group_sum<8>(d0 + d1);  // (warp-wide shuffles: outside any branch)
      d[t] = ((done >> t) & 1) ? 0.0 : beta * gsum;  // finished columns: a unchanged
      double n0 = 0.0, n1 = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        a[t][e] = fma(-d[t], x[e], a[t][e]) * mz[e];
        if (e & 1) n1 = fma(a[t][e], a[t][e], n1); else n0 = fma(a[t][e], a[t][e], n0);
      }
      key[t] = group_sum<8>(n0 + n1);  // exact ||a(j+1:)||^2: the next pivot key
    }
    publish_best(key, par ^ 1);
    if (gl == 0) {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (!((done >> t) & 1)) Rg[(size_t)j * k + g + 32 * t] = fma(-d[t], vjj, aj[t]);  // R_jq
    }
    if (g == 0) {  // reflector j
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = gl + 8 * e;
        if (i < k) Hv[(size_t)j * k + i] = i == j ? vjj : x[e];
      }
      if (gl == 0) {
        Hv[(size_t)k * k + j] = beta;
        s_piv[j] = ph;
        s_rd[j] = alpha;
      }
    }
    __syncthreads();  // every read of the pivot column is done ...
#pragma unroll
    for (int t = 0; t < 4; ++t)  // ... before the updated columns are stored (finished ones stay)
      if (!((done >> t) & 1))
#pragma unroll
        for (int e = 0; e < E; ++e) qa[(g + 32 * t) * KP + gl + 8 * e] = a[t][e];
    __syncthreads();
  }
  // X = R^T: X[i][c] = R[c][i] = Rg[c][piv[i]] above the diagonal (c < i), R_ii on it, 0 below
  for (int e = tid; e < k * k; e += kQrThreads) {
    const int i = e / k, c = e - i * k;
    Xt[e] = c < i ? Rg[(size_t)c * k + s_piv[i]] : (c == i ? s_rd[i] : 0.0);
  }
  if (tid < k) piv_out[tid] = s_piv[tid];
}

template <int E>
static void launch_qrcp_e(int k, const float* W, int64_t ldw, double* Xt, double* Hv, double* Rg, int* piv, void* ws,
                          cudaStream_t st) {
  constexpr size_t smem = sizeof(double) * kQrK * 8 * E;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svd_qrcp_kernel<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  svd_qrcp_kernel<E><<<1, kQrThreads, smem, st>>>(k, W, ldw, Xt, Hv, Rg, piv, ws);
}

static bool launch_qrcp(int k, const float* W, int64_t ldw, double* Xt, double* Hv, double* Rg, int* piv, void* ws,
                        cudaStream_t st) {
  if (k > kQrK) return false;
  note_launch();
  if (k <= 32) launch_qrcp_e<4>(k, W, ldw, Xt, Hv, Rg, piv, ws, st);
  else if (k <= 64) launch_qrcp_e<8>(k, W, ldw, Xt, Hv, Rg, piv, ws, st);
  else if (k <= 104) launch_qrcp_e<13>(k, W, ldw, Xt, Hv, Rg, piv, ws, st);
  else launch_qrcp_e<16>(k, W, ldw, Xt, Hv, Rg, piv, ws, st);
  return true;
}

// ---------------------------------------------------------------- k <= 64: four columns per slot
// As svd_split_kernel (A on CTA 0, V on CTA 1 of a cluster pair, rotations streamed through
// DSMEM), but every slot (LP lanes) holds FOUR consecutive positions of the odd-even network:
// even rounds rotate (0,1) and (2,3), odd rounds (1,2) inside the slot and (3, next slot's 0)
// across slots -- only two of the four columns move per odd round (half the shared-memory
// traffic of two-column slots), and every round has two or three independent rotation chains
// per warp.  n' = round_up(k, 4) positions (zero columns pad).
//
// KM (64 or 128) bounds k.  CTA 1 follows CTA 0 by one SEGMENT of nseg (1, 2 or 4) equal
// parts of a sweep (n4 / nseg rounds, even): the rotations of a segment are double-buffered
// [segment parity][round][slot][4] in CTA 1's shared memory, one full / empty mbarrier pair
// per parity; the scale fold and the stop decision stay at sweep boundaries.  k = 100 needs
// nseg = 2 to fit (80 KB of rotations instead of 160).
template <int LP, int E, int KM>
__global__ void __launch_bounds__(256, 1) __cluster_dims__(2, 1, 1)
svd_quad_kernel(int k, int nseg, const float* __restrict__ W, int64_t ldw, const double* __restrict__ Xt,
                const double* __restrict__ Qm, const int* __restrict__ piv, double tol, double* __restrict__ sigma_out,
                double* __restrict__ Uw64, double* __restrict__ Vw64, float* __restrict__ uw32,
                float* __restrict__ vw32, int64_t ld32, int* r_out, int* r_out2, void* ws) {
  // Xt != nullptr: QR-preconditioned (svd_qrcp_kernel): CTA 0 starts from X = R^T, CTA 1 from Q
  // (formed from the reflectors Qm = Hv);
  // at the end CTA 1 holds U_w = Q V_x and CTA 0 the columns of V_w (rows permuted by piv)
  const bool pre = Xt != nullptr;
  constexpr int G = 32 / LP;
  constexpr int SEAT = E * LP + ((LP - (E * LP) % 16) + 16) % 16;
  constexpr int NS = KM / 4 + 4;      // seats (slots + the two outer ones, rounded up)
  extern __shared__ __align__(16) double smem_d[];
  __shared__ double s_sig[KM];
  __shared__ int s_perm[KM];
  __shared__ int s_id[2][2][NS];      // [parity][col0 | col3][seat]
  __shared__ double s_st[2][NS][4][3];  // CTA 0: published n, d, 1 / d [parity][seat][position]
  __shared__ __align__(8) uint64_t bar_full[2], bar_empty[2];
  __shared__ int s_last[2];
  const uint32_t crank = cg::this_cluster().block_rank();
#ifdef CABS_PROFILE_SVD
  const long long q_k0 = clock64();
#endif
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = blockDim.x >> 5;
  const int gl = lane % LP, gw = lane / LP;
  const int g = warp * G + gw;
  const int n4 = (k + 3) & ~3, Q = n4 / 4;
  const int nseat = nw * G + 2;
  const bool live = g < Q;
  const bool first = g == 0, lastslot = g == Q - 1;
  const size_t arr = (size_t)2 * nseat * SEAT;
  double* b0 = smem_d;       // published column 0 of each slot  [parity][seat][SEAT]
  double* b3 = b0 + arr;     // published column 3
  double* prm = b3 + arr;    // CTA 1: rotations [parity][round][slot][4]
  if (tid == 0) {
    tc::mbar_init(&bar_full[0], 1); tc::mbar_init(&bar_full[1], 1);
    tc::mbar_init(&bar_empty[0], 1); tc::mbar_init(&bar_empty[1], 1);
    tc::mbar_fence_init();
  }
  for (int e = tid; e < 2 * (int)arr; e += blockDim.x) smem_d[e] = 0.0;
  for (int e = tid; e < 2 * NS * 4 * 3; e += blockDim.x) (&s_st[0][0][0][0])[e] = (e % 3 == 0) ? 0.0 : 1.0;
  for (int e = tid; e < 2 * 2 * NS; e += blockDim.x) (&s_id[0][0][0])[e] = 1 << 30;
  cluster_sync_all();

  double a[4][E];
  int id[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) id[c] = 4 * g + c;
  if (pre && crank == 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = gl + LP * e;
        a[c][e] = (live && i < k && id[c] < k) ? Xt[(size_t)i * k + id[c]] : 0.0;
      }
  } else if (pre) {
    // Q = H_0 H_1 ... H_{k-1} applied to this slot's unit columns, reflectors from the QR
    // kernel (Qm = Hv: row j = v_j, then the k scales); hidden behind CTA 0's first segment
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int e = 0; e < E; ++e) a[c][e] = (live && gl + LP * e == id[c] && id[c] < k) ? 1.0 : 0.0;
    double vn[E];
#pragma unroll
    for (int e = 0; e < E; ++e) vn[e] = gl + LP * e < k ? Qm[(size_t)(k - 1) * k + gl + LP * e] : 0.0;
    double bn = Qm[(size_t)k * k + k - 1];
    for (int j = k - 1; j >= 0; --j) {
      double v[E];
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = vn[e];
      const double bj = bn;
      if (j > 0) {  // prefetch the next reflector
#pragma unroll
        for (int e = 0; e < E; ++e) vn[e] = gl + LP * e < k ? Qm[(size_t)(j - 1) * k + gl + LP * e] : 0.0;
        bn = Qm[(size_t)k * k + j - 1];
      }
      double dq[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (e & 1) d1 = fma(v[e], a[c][e], d1); else d0 = fma(v[e], a[c][e], d0);
        }
        dq[c] = d0 + d1;
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) dq[c] = bj * group_sum<LP>(dq[c]);
#pragma unroll
      for (int c = 0; c < 4; ++c)
#pragma unroll
        for (int e = 0; e < E; ++e) a[c][e] = fma(-dq[c], v[e], a[c][e]);
    }
  } else if (crank == 0) {
    bool bad = false;
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = gl + LP * e;
        float w = 0.f;
        if (live && i < k && id[c] < k) w = W[(int64_t)i * ldw + id[c]];
        bad |= !isfinite(w);
        a[c][e] = w;
      }
    if (bad) set_status(ws, CABS_DEV_NONFINITE);
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = gl + LP * e;
        a[c][e] = (live && i == id[c] && id[c] < k) ? 1.0 : 0.0;
      }
  }
  __syncthreads();
  const double tol_rot = 2.0 * sqrt(static_cast<double>(k)) * DBL_EPSILON;
  const double tol_rot2 = tol_rot * tol_rot;
  double* const prm_remote = dsmem_map_generic(prm, 1);
  const uint32_t full_remote0 = dsmem_map(&bar_full[0], 1), full_remote1 = dsmem_map(&bar_full[1], 1);
  const uint32_t empty_remote0 = dsmem_map(&bar_empty[0], 0), empty_remote1 = dsmem_map(&bar_empty[1], 0);
  const uint32_t last_remote = dsmem_map(&s_last[0], 1);
  const int HS = n4 / nseg;                     // rounds per segment (even)
  double* dvs = prm + (size_t)2 * HS * Q * 4;   // CTA 1: column scales at sweep end [parity][position]
  const uint32_t dvs_remote = dsmem_map(dvs, 1);
  // Scaled columns: actual column = d * stored.  The scalar state of position p of the slot
  // (squared norm n, scale d, 1 / d) lives on lanes 2p, 2p + 1 of the group ("owners"), and
  // each rotation's scalar chain runs once per lane: a pair's two owner pairs of lanes compute
  // it together (bit-identical inputs), each keeping its own position's new state.  CTA 1's V
  // columns carry the same scales (they see the same rotations).
  const int own = gl >> 1;                 // position owned
  const int base = lane & ~(LP - 1);       // first lane of the group
  const bool hi = (gl & 4) != 0, mid = (gl & 2) != 0;
  double on = 0.0, od = 1.0, oi = 1.0;     // own position's n, d, 1 / d
  int sweep = 0;
  bool last = k <= 1;
#ifdef CABS_PROFILE_SVD
  long long q_wait = 0, q_t0 = clock64(), q_sweep = 0;
#endif
  for (; !last; ++sweep) {
    const int sp = sweep & 1;
#ifdef CABS_PROFILE_SVD
    const long long s0 = clock64();
#endif
    int rotated = 0;
    double tmax = 0.0;
    if (crank == 0) {  // fold the scales in; exact squared norms at every sweep start, then by formula
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const double dc = __shfl_sync(0xffffffffu, od, base + 2 * c);
        double t0 = 0.0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          a[c][e] *= dc;
          t0 = fma(a[c][e], a[c][e], t0);
        }
        t0 = group_sum<LP>(t0);
        if (c == own) on = t0;
      }
      od = 1.0;
      oi = 1.0;
    }
    int seg = 0, sro = 0;  // segment of the sweep, round offset inside it (no division in the loop)
    for (int rnd = 0; rnd < n4; rnd += 2, sro += 2) {
      if (sro == HS) { ++seg; sro = 0; }
      const int gs = sweep * nseg + seg, bp = gs & 1;  // global segment index, its buffer parity
      if (sro == 0) {  // segment start: CTA 0 needs a free buffer, CTA 1 a full one
#ifdef CABS_PROFILE_SVD
        const long long w0 = clock64();
#endif
        if (crank == 0 && gs >= 2) mbar_wait_cluster(&bar_empty[bp], static_cast<uint32_t>(((gs - 2) >> 1) & 1));
        if (crank == 1) mbar_wait_cluster(&bar_full[bp], static_cast<uint32_t>((gs >> 1) & 1));
#ifdef CABS_PROFILE_SVD
        q_wait += clock64() - w0;
#endif
      }
      // ---- even round: pairs (0,1) (lanes 0-3) and (2,3) (lanes 4-7), rotated and swapped
      const int pidx = ((bp * HS + sro) * Q + (live ? g : 0)) * 4;  // [parity][round][slot][4]
      double al01, be01, al23, be23;
      if (crank == 0) {
        double p01a = 0.0, p01b = 0.0, p23a = 0.0, p23b = 0.0;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
          p01a = fma(a[0][e], a[1][e], p01a);
          p23a = fma(a[2][e], a[3][e], p23a);
          if (e + 1 < E) {
            p01b = fma(a[0][e + 1], a[1][e + 1], p01b);
            p23b = fma(a[2][e + 1], a[3][e + 1], p23b);
          }
        }
        const double p01 = p01a + p01b, p23 = p23a + p23b;
        // reduce-scatter: lanes 0-3 end with the (0,1) dot, lanes 4-7 with the (2,3) dot
        double gsum = (hi ? p23 : p01) + __shfl_xor_sync(0xffffffffu, hi ? p01 : p23, 4);
        gsum += __shfl_xor_sync(0xffffffffu, gsum, 2);
        gsum += __shfl_xor_sync(0xffffffffu, gsum, 1);
        const double pn = __shfl_xor_sync(0xffffffffu, on, 2);
        const double pd = __shfl_xor_sync(0xffffffffu, od, 2);
        const double pi = __shfl_xor_sync(0xffffffffu, oi, 2);
        LaneRot r;
#if defined(SVQ_EXP) && (SVQ_EXP & 1)  // diagnostics: a cheap stand-in for the rotation chain
        r.t = gsum * 1e-30; r.need = false; r.tu = r.t; r.tv = r.t; r.n = on; r.d = od; r.i = oi; (void)pn; (void)pd; (void)pi;
#else
        lane_rot(!mid, on, od, oi, pn, pd, pi, gsum, tol_rot2, r);
#endif
        al01 = __shfl_sync(0xffffffffu, r.tu, base);  // lanes 0 and 4: left lanes
        be01 = __shfl_sync(0xffffffffu, r.tv, base);
        al23 = __shfl_sync(0xffffffffu, r.tu, base + 4);
        be23 = __shfl_sync(0xffffffffu, r.tv, base + 4);
        rotated |= live && r.need;
        if (live) tmax = fmax(tmax, fabs(r.t));
        if ((gl & 3) == 0 && live) dsmem_st2_f64(prm_remote + pidx + (hi ? 2 : 0), r.tu, r.tv);
        on = r.n; od = r.d; oi = r.i;
      } else {
        const double* pr = prm + pidx;
        al01 = live ? pr[0] : 0.0; be01 = live ? pr[1] : 0.0;
        al23 = live ? pr[2] : 0.0; be23 = live ? pr[3] : 0.0;
      }
      // new position 0 = y + alpha x (the old 1 moves left), new 1 = x - beta y
      double e0[E], e1[E], e2[E], e3[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        e0[e] = fma(al01, a[0][e], a[1][e]);
        e1[e] = fma(-be01, a[1][e], a[0][e]);
        e2[e] = fma(al23, a[2][e], a[3][e]);
        e3[e] = fma(-be23, a[3][e], a[2][e]);
      }
      {
        int t = id[0]; id[0] = id[1]; id[1] = t;
        t = id[2]; id[2] = id[3]; id[3] = t;
      }
      // ---- odd round: (1,2) inside (lanes 2-5), (3, right slot's 0) (lanes 6,7) and
      // (left slot's 3, 0) (lanes 0,1) across
      const int par = ((rnd + 1) >> 1) & 1;
      const size_t pub = ((size_t)par * nseat + g + 1) * SEAT + gl;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        b0[pub + e * LP] = e0[e];
        b3[pub + e * LP] = e3[e];
      }
      if (gl == 0) {
        s_id[par][0][g + 1] = id[0];
        s_id[par][1][g + 1] = id[3];
      }
      if (crank == 0 && (gl & 1) == 0) {  // every position's n, d, 1 / d: [parity][seat][position]
        s_st[par][g + 1][own][0] = on; s_st[par][g + 1][own][1] = od; s_st[par][g + 1][own][2] = oi;
      }
#if !(defined(SVQ_EXP) && (SVQ_EXP & 2))  // diagnostics: no barrier (wrong data, timing only)
      __syncthreads();
#endif
      const size_t lft = ((size_t)par * nseat + g) * SEAT + gl;      // left slot's column 3
      const size_t rgt = ((size_t)par * nseat + g + 2) * SEAT + gl;  // right slot's column 0
      double rl[E], rr[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        rl[e] = b3[lft + e * LP];
        rr[e] = b0[rgt + e * LP];
      }
      const int pido = pidx + Q * 4;  // round rnd + 1
      double al12, be12, alR, beL;
      if (crank == 0) {
        double p12a = 0.0, p12b = 0.0, pRa = 0.0, pRb = 0.0, pLa = 0.0, pLb = 0.0;
#pragma unroll
        for (int e = 0; e < E; e += 2) {
          p12a = fma(e1[e], e2[e], p12a);
          pRa = fma(e3[e], rr[e], pRa);
          pLa = fma(rl[e], e0[e], pLa);
          if (e + 1 < E) {
            p12b = fma(e1[e + 1], e2[e + 1], p12b);
            pRb = fma(e3[e + 1], rr[e + 1], pRb);
            pLb = fma(rl[e + 1], e0[e + 1], pLb);
          }
        }
        const double p12 = p12a + p12b, pR = pRa + pRb, pL = pLa + pLb;
        // reduce-scatter: lanes 0,1 end with the left crossing dot, 2-5 with (1,2), 6,7 with
        // the right crossing dot (every sum is formed in a commutation of the same tree)
        const double q12 = p12 + __shfl_xor_sync(0xffffffffu, p12, 4);
        const double qX = (hi ? pR : pL) + __shfl_xor_sync(0xffffffffu, hi ? pL : pR, 4);
        double gsum = ((hi != mid) ? q12 : qX) + __shfl_xor_sync(0xffffffffu, (hi != mid) ? qX : q12, 2);
        gsum += __shfl_xor_sync(0xffffffffu, gsum, 1);
        // partner position: 0 <- left slot's 3, 1 <-> 2, 3 <- right slot's 0
        const int pseat = own == 0 ? g : (own == 3 ? g + 2 : g + 1), ppos = own ^ 3;
        const double* ps = s_st[par][pseat][ppos];
        LaneRot r;
#if defined(SVQ_EXP) && (SVQ_EXP & 1)
        r.t = gsum * 1e-30; r.need = false; r.tu = r.t; r.tv = r.t; r.n = on; r.d = od; r.i = oi; (void)ps;
#else
        lane_rot(mid, on, od, oi, ps[0], ps[1], ps[2], gsum, tol_rot2, r);
#endif
        al12 = __shfl_sync(0xffffffffu, r.tu, base + 2);  // lanes 2 and 6: left lanes
        be12 = __shfl_sync(0xffffffffu, r.tv, base + 2);
        const double alR0 = __shfl_sync(0xffffffffu, r.tu, base + 6);
        const double beL0 = __shfl_sync(0xffffffffu, r.tu, base);  // lanes 0, 1: right lanes
        alR = lastslot ? 1.0 : alR0;
        beL = first ? -1.0 : beL0;
        const bool idle = (first && gl < 2) || (lastslot && gl >= 6);  // positions 0 and n' - 1 stay
        rotated |= live && !idle && r.need;
        if (live && !idle) tmax = fmax(tmax, fabs(r.t));
        if ((gl == 2 || gl == 6) && live) dsmem_st2_f64(prm_remote + pido + (hi ? 2 : 0), r.tu, r.tv);
        if (!idle) { on = r.n; od = r.d; oi = r.i; }
      } else {
        const double* pr = prm + pido;
        al12 = live ? pr[0] : 0.0; be12 = live ? pr[1] : 0.0;
        alR = lastslot ? 1.0 : (live ? pr[2] : 0.0);
        // the left crossing pair is the left slot's right crossing pair
        beL = first ? -1.0 : (live ? prm[pido - 4 + 3] : 0.0);
      }
      // idle end positions (0 and n' - 1) keep their column: coefficient 1 against the zero
      // column of the never-written outer seat (or of a dead slot)
#pragma unroll
      for (int e = 0; e < E; ++e) {
        a[1][e] = fma(al12, e1[e], e2[e]);
        a[2][e] = fma(-be12, e2[e], e1[e]);
        a[3][e] = fma(alR, e3[e], rr[e]);
        a[0][e] = fma(-beL, e0[e], rl[e]);
      }
      {
        const int t = id[1]; id[1] = id[2]; id[2] = t;
      }
      if (!lastslot) id[3] = s_id[par][0][g + 2];
      if (!first) id[0] = s_id[par][1][g];
      if (sro + 2 == HS && seg + 1 < nseg) {  // segment end inside the sweep: hand over
        __syncthreads();
        if (tid == 0) {
          if (crank == 0) {
            asm volatile("fence.acq_rel.cluster;" ::: "memory");
            mbar_arrive_remote(bp ? full_remote1 : full_remote0);
          } else {
            mbar_arrive_remote(bp ? empty_remote1 : empty_remote0);
          }
        }
      }
    }
    const int bpl = (sweep * nseg + nseg - 1) & 1;  // the sweep's last segment parity
#ifdef CABS_PROFILE_SVD
    q_sweep += clock64() - s0;
#endif
    if (crank == 0) {
      if ((gl & 1) == 0 && live)  // the scales the sweep ended with, for CTA 1's V columns
        dsmem_st_f64(dvs_remote + static_cast<uint32_t>((sp * n4 + 4 * g + own) * 8), od);
      rotated = __syncthreads_or(rotated);
      const int small = __syncthreads_and(tmax < CABS_SVD_TSTOP);
      last = !rotated || small || sweep + 1 >= kSvdMaxSweeps;
      if (tid == 0) {
        dsmem_st_s32(last_remote + 4 * sp, last ? 1 : 0);
        asm volatile("fence.acq_rel.cluster;" ::: "memory");
        mbar_arrive_remote(bpl ? full_remote1 : full_remote0);
      }
    } else {
      if (live) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double dc = dvs[sp * n4 + 4 * g + c];
#pragma unroll
          for (int e = 0; e < E; ++e) a[c][e] *= dc;
        }
      }
      __syncthreads();
      last = s_last[sp] != 0;
      __syncthreads();
      if (tid == 0) mbar_arrive_remote(bpl ? empty_remote1 : empty_remote0);
    }
  }
  if (crank == 0) {
    if (sweep >= kSvdMaxSweeps && k > 1) set_status(ws, CABS_DEV_SVD_NOCONV);
    if (tid == 0) reinterpret_cast<int*>(ws)[8] = sweep;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const double dc = __shfl_sync(0xffffffffu, od, base + 2 * c);
#pragma unroll
      for (int e = 0; e < E; ++e) a[c][e] *= dc;
    }
  }
#ifdef CABS_PROFILE_SVD
  if (tid == 0) {  // [CTA][wait, rounds, total]
    long long* pw = reinterpret_cast<long long*>(ws) + 8 + 3 * crank;
    pw[0] = q_wait; pw[1] = q_sweep; pw[2] = clock64() - q_t0;
  }
#endif
  // ---- epilogue from the registers: sigma_c = |a_c| and the canonical sign (the largest-|.|
  // entry of U_w's column positive, lowest row on ties) per column, rank order by one thread
  // per column, then every group writes its own columns (CTA 0: U_w, CTA 1: V_w) in rank order.
  __shared__ double s_sgn[KM];
  __shared__ int s_rank[KM];
  __shared__ int s_r;
#ifdef CABS_PROFILE_SVD
  const long long q_e0 = clock64();
#endif
  // the CTA holding U_w's columns fixes the signs (CTA 0, or CTA 1 when preconditioned)
  const bool usgn = pre ? crank == 1 : crank == 0;
  {
    const uint32_t sgn0 = dsmem_map(s_sgn, 0);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      double ss = 0.0, best = -1.0;
      int bi = 0x7fffffff;
      bool neg = false;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int i = gl + LP * e;
        ss = fma(a[c][e], a[c][e], ss);
        const double v = fabs(a[c][e]);
        if (i < k && v > best) { best = v; bi = i; neg = a[c][e] < 0.0; }
      }
      ss = group_sum<LP>(ss);
#pragma unroll
      for (int o = LP / 2; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        const bool on2 = __shfl_xor_sync(0xffffffffu, neg, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; neg = on2; }
      }
      if (gl == 0 && live && id[c] < k) {
        if (crank == 0) s_sig[id[c]] = sqrt(ss);
        if (usgn) dsmem_st_f64(sgn0 + 8u * id[c], neg ? -1.0 : 1.0);
      }
    }
  }
  cluster_sync_all();  // sigma and signs in CTA 0
  if (crank == 0) {
    const uint32_t rank_remote = dsmem_map(s_rank, 1), sgn_remote = dsmem_map(s_sgn, 1);
    for (int c = tid; c < k; c += blockDim.x) {
      const double sc = s_sig[c];
      int rk = 0;
      for (int j2 = 0; j2 < k; ++j2) {
        const double sj = s_sig[j2];
        rk += (sj > sc) || (sj == sc && j2 < c);
      }
      s_rank[c] = rk;
      s_perm[rk] = c;
      dsmem_st_s32(rank_remote + 4 * c, rk);
      dsmem_st_f64(sgn_remote + 8 * c, s_sgn[c]);
    }
    __syncthreads();
    if (warp == 0) {  // rank r: sigma_j > tol * sigma_max
      const double smax = s_sig[s_perm[0]];
      int cnt = 0;
      for (int c = lane; c < k; c += 32) cnt += smax > 0 && s_sig[c] > tol * smax;
      cnt = __reduce_add_sync(0xffffffffu, cnt);
      if (lane == 0) {
        s_r = cnt;
        dsmem_st_s32(dsmem_map(&s_r, 1), cnt);
        if (r_out) *r_out = cnt;
        if (r_out2) *r_out2 = cnt;
      }
    }
    if (sigma_out)
      for (int j2 = tid; j2 < k; j2 += blockDim.x) sigma_out[j2] = s_sig[s_perm[j2]];
  }
  cluster_sync_all();
#ifdef CABS_PROFILE_SVD
  const long long q_e1 = clock64();
#endif
  {
    const int r = s_r;
    // CTA 0: its columns / sigma (U_w; V_w when preconditioned, rows permuted by piv); CTA 1:
    // its columns (V_w; U_w = Q V_x when preconditioned)
    const bool to_u = (crank == 0) != pre;
    double* o64 = to_u ? Uw64 : Vw64;
    float* o32 = to_u ? uw32 : vw32;
    if (live) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (id[c] >= k) continue;
        const int jr = s_rank[id[c]];
        const bool keep = jr < r;
        double mul;
        if (crank == 0) {
          const double sg = s_sig[id[c]];
          mul = (keep && sg > 0) ? s_sgn[id[c]] / sg : 0.0;
        } else {
          mul = keep ? s_sgn[id[c]] : 0.0;
        }
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i0 = gl + LP * e;
          if (i0 < k) {
            const int i = (pre && crank == 0) ? piv[i0] : i0;
            const double u = a[c][e] * mul;
            if (o64) o64[(size_t)i * k + jr] = u;
            if (o32) o32[(size_t)i * ld32 + jr] = static_cast<float>(u);
          }
        }
      }
    }
    if (o32) {  // zero padding columns [k, ld32)
      for (int64_t e = tid; e < (int64_t)k * (ld32 - k); e += blockDim.x) {
        const int64_t i = e / (ld32 - k), c = k + e % (ld32 - k);
        o32[i * ld32 + c] = 0.f;
      }
    }
  }
#ifdef CABS_PROFILE_SVD
  __syncthreads();
  if (crank == 0 && tid == 0) {  // [start -> loop start, loop end -> epilogue start, sigma, write]
    long long* pw = reinterpret_cast<long long*>(ws) + 14;
    pw[0] = q_t0 - q_k0; pw[1] = q_e0 - q_t0; pw[2] = q_e1 - q_e0; pw[3] = clock64() - q_e1;
  }
#endif
}

template <int LP, int E, int KM = 64>
static bool launch_quad(int k, const float* W, int64_t ldw, double tol, double* sig, double* Uw64, double* Vw64,
                        float* uw32, float* vw32, int64_t ld32, int* r_ws, int* r_user, void* ws, cudaStream_t st,
                        const Ws* L = nullptr) {
  constexpr int G = 32 / LP;
  constexpr int SEAT = E * LP + ((LP - (E * LP) % 16) + 16) % 16;
  const int n4 = (k + 3) & ~3, Q = n4 / 4;
  const int nw = (Q + G - 1) / G;
  if (k > KM || k > E * LP || nw * G + 2 > KM / 4 + 4 || nw > 8) return false;
  const size_t xch = sizeof(double) * 2 * 2 * (size_t)(nw * G + 2) * SEAT;
  constexpr int kCap = 214 * 1024;  // (+ ~10.6 KB static: within the 227 KB opt-in)
  int nseg = 0;
  size_t smem = 0;
  for (int ns = 1; ns <= 4 && !nseg; ns *= 2) {  // fewest segments whose rotation buffers fit
    if (n4 % (2 * ns)) continue;
    smem = xch + sizeof(double) * 2 * ((size_t)(n4 / ns) * Q * 4 + n4);
    if (smem <= kCap) nseg = ns;
  }
  if (!nseg) return false;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svd_quad_kernel<LP, E, KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCap);
    attr = true;
  }
  // QR preconditioning (L given, k > 2; CABS_SVD_NOQR: plain Jacobi on W)
  const double* Xt = nullptr;
  const double* Qm = nullptr;
  const int* piv = nullptr;
  if (L && k > 2 && !getenv("CABS_SVD_NOQR")) {
    double* x = wsp<double>(ws, L->a64);
    double* hv = wsp<double>(ws, L->v64);
    double* rg = wsp<double>(ws, L->qr);
    int* pv = reinterpret_cast<int*>(rg + (size_t)L->K * L->K);
    if (launch_qrcp(k, W, ldw, x, hv, rg, pv, ws, st)) { Xt = x; Qm = hv; piv = pv; }
  }
  note_launch();
  svd_quad_kernel<LP, E, KM><<<2, 32 * nw, smem, st>>>(k, nseg, W, ldw, Xt, Qm, piv, tol, sig, Uw64, Vw64, uw32, vw32,
                                                       ld32, r_ws, r_user, ws);
  return true;
}

// ---------------------------------------------------------------- k > 64: columns in memory
template <int L, bool SMEM>
__global__ void __launch_bounds__(kSvdThreads, 1)
svd_jacobi_kernel(int k, const float* __restrict__ W, int64_t ldw, double tol, double* gA, double* gV,
                  double* __restrict__ sigma_out, double* __restrict__ Uw64, double* __restrict__ Vw64,
                  float* __restrict__ uw32, float* __restrict__ vw32, int64_t ld32, int* r_out, int* r_out2,
                  bool use_smem, void* ws) {
  extern __shared__ __align__(16) double smem_d[];
  __shared__ double s_sig[CABS_KMAX];
  __shared__ int s_perm[CABS_KMAX];  // s_perm[rank] = column
  __shared__ double s_h[CABS_KMAX];  // Gram-Schmidt coefficients
  // SMEM is a compile-time choice so the columns are addressed as shared memory (LDS/STS)
  double* A = SMEM ? smem_d : gA;
  double* V = SMEM ? smem_d + (size_t)k * k : gV;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;

  // load: A[c*k + i] = W[i, c] (column-major)
  for (int e = tid; e < k * k; e += blockDim.x) {
    const int c = e / k, i = e - c * k;
    float w = W[(int64_t)i * ldw + c];
    if (!isfinite(w)) set_status(ws, CABS_DEV_NONFINITE);
    A[e] = static_cast<double>(w);
  }
  __syncthreads();

  int sweep = 0;
  if (k > 1) {
    // L = ceil(k/32) class -> (lanes per pair, elements per lane): 8 elements per lane
    // while k <= 256, so small k packs several pairs into each warp
    sweep = jacobi_sweeps<(L <= 1 ? 4 : L == 2 ? 8 : L == 4 ? 16 : 32), (L <= 4 ? 8 : L)>(A, k);
    if (sweep == kSvdMaxSweeps && tid == 0) set_status(ws, CABS_DEV_SVD_NOCONV);
  }
  if (tid == 0) reinterpret_cast<int*>(ws)[8] = sweep;

  const int r = svd_sigma(A, k, tol, s_sig, s_perm, sigma_out, r_out, r_out2);
  __syncthreads();
  const double smax = s_sig[s_perm[0]];
  // Right singular vectors without accumulating the rotations (which would double the
  // shared-memory traffic of every round): W^T W V = V S^2 and A = W V = U S give
  // v_c = W^T a_c / sigma_c^2 for the kept components, then two passes of classical
  // Gram-Schmidt in descending sigma order restore orthonormality to FP64 rounding.
  for (int e = tid; e < k * k; e += blockDim.x) {
    const int c = e / k, i = e - c * k;
    const double sg = s_sig[c];
    double v = 0.0;
    if (sg > tol * smax && sg > 0) {
      const double* ac = A + (size_t)c * k;
      for (int rr = 0; rr < k; ++rr) v = fma(static_cast<double>(W[(int64_t)rr * ldw + i]), ac[rr], v);
      v /= sg * sg;
    }
    V[e] = v;
  }
  __syncthreads();
  for (int j = 1; j < r; ++j) {
    double* vj = V + (size_t)s_perm[j] * k;
    for (int pass = 0; pass < 2; ++pass) {
      // coefficients h_i = v_i . v_j for the j earlier (larger-sigma) columns, one warp each
      for (int i = warp; i < j; i += nwarps) {
        const double* vi = V + (size_t)s_perm[i] * k;
        double h = 0;
        for (int e = lane; e < k; e += 32) h = fma(vi[e], vj[e], h);
        h = warp_sum_d(h);
        if (lane == 0) s_h[i] = h;
      }
      __syncthreads();
      for (int e = tid; e < k; e += blockDim.x) {
        double x = vj[e];
        for (int i = 0; i < j; ++i) x = fma(-s_h[i], V[(size_t)s_perm[i] * k + e], x);
        vj[e] = x;
      }
      __syncthreads();
    }
  }
  // unit norms (column j of V now orthogonal to the earlier ones)
  for (int j = warp; j < r; j += nwarps) {
    double* vj = V + (size_t)s_perm[j] * k;
    double ss = 0;
    for (int e = lane; e < k; e += 32) ss = fma(vj[e], vj[e], ss);
    ss = warp_sum_d(ss);
    const double inv = ss > 0 ? 1.0 / sqrt(ss) : 0.0;
    for (int e = lane; e < k; e += 32) vj[e] *= inv;
  }
  __syncthreads();
  svd_write(A, V, k, r, s_sig, s_perm, Uw64, Vw64, uw32, vw32, ld32);
}

template <int LP, int E>
static void launch_systolic(int k, const float* W, int64_t ldw, double tol, double* sig, double* Uw64, double* Vw64,
                            float* uw32, float* vw32, int64_t ld32, int* r_ws, int* r_user, void* ws, cudaStream_t st) {
  constexpr int G = 32 / LP;
  const int P = ((k + 1) & ~1) / 2;
  const int nw = (P + G - 1) / G;
  constexpr int SEAT = E * LP + ((4 - (E * LP) % 16) + 16) % 16;
  const size_t seats = sizeof(double) * 4 * 2 * (size_t)(nw * G + 2) * SEAT;  // [AL|AR|VL|VR][parity][seat]
  const size_t fin = sizeof(double) * 2 * (size_t)k * k;
  const size_t smem = seats > fin ? seats : fin;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svd_systolic_kernel<LP, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr = true;
  }
  note_launch();
  svd_systolic_kernel<LP, E><<<1, 32 * nw, smem, st>>>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, ld32, r_ws,
                                                      r_user, ws);
}

template <int LP, int E>
static bool launch_split(int k, const float* W, int64_t ldw, double tol, double* sig, double* Uw64, double* Vw64,
                         float* uw32, float* vw32, int64_t ld32, int* r_ws, int* r_user, void* ws, cudaStream_t st) {
  constexpr int G = 32 / LP;
  constexpr int SEAT = E * LP + ((LP - (E * LP) % 16) + 16) % 16;
  const int np = (k + 1) & ~1, P = np / 2;
  const int nw = (P + G - 1) / G;
  const size_t xch = sizeof(double) * 2 * 2 * (size_t)(nw * G + 2) * SEAT;  // [XL|XR][parity][seat]
  const size_t prm = sizeof(double) * 2 * (size_t)np * P * 4;               // [parity][round][slot][c s c s]
  const size_t fin = sizeof(double) * 2 * (size_t)k * k;
  const size_t smem = (xch + prm > fin ? xch + prm : fin);
  constexpr int kCap = 220 * 1024;
  if (smem > kCap) return false;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(svd_split_kernel<LP, E>, cudaFuncAttributeMaxDynamicSharedMemorySize, kCap);
    attr = true;
  }
  note_launch();
  svd_split_kernel<LP, E><<<2, 32 * nw, smem, st>>>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, ld32, r_ws, r_user,
                                                    ws);
  return true;
}

int launch_svd(int k, const float* W, int64_t ldw, double tol, void* ws, const Ws& L, double* sigma_user,
               double* Uw64, double* Vw64, int* r_user, cudaStream_t st) {
  double* sig = sigma_user ? sigma_user : wsp<double>(ws, L.sig64);
  int* r_ws = wsp<int>(ws, L.scal) + SCAL_R_TMP;
  float* uw32 = wsp<float>(ws, L.uw32);
  float* vw32 = wsp<float>(ws, L.vw32);
  // (every launcher notes its own kernel launches: the QR preconditioner adds one)
  SvdQrBufs qbufs{};
  {
    qbufs.K = L.K;
    qbufs.Xt = wsp<double>(ws, L.a64);
    qbufs.Hv = wsp<double>(ws, L.v64);
    qbufs.Rg = wsp<double>(ws, L.qr);
    qbufs.piv = reinterpret_cast<int*>(qbufs.Rg + (size_t)L.K * L.K);
    const size_t off = ((sizeof(double) * (size_t)L.K * L.K + sizeof(int) * (size_t)L.K) + 15) & ~size_t(15);
    qbufs.extra = L.K > 128 ? reinterpret_cast<double*>(reinterpret_cast<char*>(qbufs.Rg) + off) : nullptr;
  }
  if (k <= 64 && !getenv("CABS_SVD_SMEM") && !getenv("CABS_SVD_ONE_SM")) {
    // A on one SM, V on its cluster partner; four columns per 8-lane slot (the two-column
    // svd_split_kernel stays selectable for comparison)
    if (!getenv("CABS_SVD_SPLIT")) {
      if (k <= 16) launch_quad<8, 2>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st, &L);
      else if (k <= 32) launch_quad<8, 4>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st, &L);
      else if (k <= 56) launch_quad<8, 7>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st, &L);
      else launch_quad<8, 8>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st, &L);
    } else if (k <= 16) {
      launch_split<8, 2>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st);
    } else if (k <= 32) {
      launch_split<8, 4>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st);
    } else if (k <= 56) {
      launch_split<8, 7>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st);
    } else {
      launch_split<8, 8>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st);
    }
  } else if (k > 64 && k <= 128 && !getenv("CABS_SVD_CLUSTER") && !getenv("CABS_SVD_ONE_CTA") &&
             (k <= 104 ? launch_quad<8, 13, 128>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st,
                                                 &L)
                       : launch_quad<8, 16, 128>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws,
                                                 st, &L))) {
    // 64 < k <= 128: the four-column slots of k <= 64 with 7-8 warps and segment handover
  } else if (k <= 64 && !getenv("CABS_SVD_SMEM")) {
    // register-resident systolic Jacobi, 4 lanes per column pair
    if (k <= 16) launch_systolic<4, 4>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st);
    else if (k <= 32) launch_systolic<4, 8>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st);
    else if (k <= 52) launch_systolic<4, 13>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st);
    else launch_systolic<4, 16>(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st);
  } else if (k <= 320 && !getenv("CABS_SVD_ONE_CTA") &&
             launch_svd_cluster(k, W, ldw, tol, sig, Uw64, Vw64, uw32, vw32, L.Kp, r_ws, r_user, ws, st, &qbufs)) {
    // k > 64: block Jacobi over a thread-block cluster (svd_cluster.cu)
  } else {
    static bool attr_set = false;
    if (!attr_set) {
      const int smax = 2 * kSvdSmemK * kSvdSmemK * 8;
      cudaFuncSetAttribute(svd_jacobi_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
      cudaFuncSetAttribute(svd_jacobi_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
      cudaFuncSetAttribute(svd_jacobi_kernel<4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smax);
      attr_set = true;
    }
    const bool use_smem = k <= kSvdSmemK;
    const size_t smem = use_smem ? 2 * (size_t)k * k * sizeof(double) : 0;
    auto kern = k <= 32 ? svd_jacobi_kernel<1, true> : k <= 64 ? svd_jacobi_kernel<2, true>
              : k <= kSvdSmemK ? svd_jacobi_kernel<4, true> : k <= 128 ? svd_jacobi_kernel<4, false>
              : k <= 256 ? svd_jacobi_kernel<8, false> : k <= 320 ? svd_jacobi_kernel<10, false>
                         : svd_jacobi_kernel<32, false>;
    note_launch();
    kern<<<1, kSvdThreads, smem, st>>>(k, W, ldw, tol, wsp<double>(ws, L.a64), wsp<double>(ws, L.v64), sig, Uw64, Vw64,
                                       uw32, vw32, L.Kp, r_ws, r_user, use_smem, ws);
  }
  if (sigma_user && sigma_user != wsp<double>(ws, L.sig64)) {
    cudaMemcpyAsync(wsp<double>(ws, L.sig64), sigma_user, sizeof(double) * k, cudaMemcpyDeviceToDevice, st);
  }
  return 0;
}

}  // namespace cabsk
