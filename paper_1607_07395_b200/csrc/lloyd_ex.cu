// lloyd_ex.cu -- the whole Lloyd loop of one or two k-means problems (rows and columns of
// CABS, Alg. 2 steps 6-7; Eq. 6) in ONE persistent kernel that prunes the
// distance computations EXACTLY by the triangle inequality, for large point sets (c3: 1.5e5
// points, k2 = d = 100).
//
// Assignment, iteration t >= 1 (per point x with previous label a):
//   pass 1 (thread = point): Hamerly's test -- U >= ||x - c_a|| and L <= ||x - c_j|| (j != a)
//   carried over from the previous iteration, less / plus the centre drifts of this update; if
//   L' > (1 + eps) U' no other centre is nearer or within the near-tie band and the label stays
//   without reading x; else U is tightened to the exact ||x - c_a|| (the FFMA kernels' chain:
//   FP32 direct differences, dimensions ascending, one fmaf chain) and the test repeated.
//   pass 2 (warp = 32 queued points in label order): the candidates are the centres whose lower
//   bound -- the per-centre bound stored at the point's last search less the cumulative drift
//   since (Elkan), or ||c_a - c_j|| - ||x - c_a|| (triangle inequality) -- is <= (1 + eps) u;
//   the warp evaluates the union of its lanes' candidates by the same chain, and every exact
//   distance becomes the point's stored bound.  Every centre that could be nearer than c_a, or
//   within the near-tie band of the nearest, is a candidate (eps = 2e-4 covers the FP32 rounding
//   of the three chains, 30x over; bounds are rounded down, drifts up), so the label (lowest j on
//   ties), the nearest distance, the near-tie count and the near-tie log are bit-identical to a
//   search over all k2 centres.  ||c_i - c_j|| is computed once per iteration, split over the
//   thread-block cluster (rows i = rank mod csize) and exchanged through DSMEM.  Iteration 0 (no
//   previous label) searches all centres.
// Update (exact int64 fixed point, km_fixed.cuh): per cluster the sums of w x, of w and of
// w ||x||^2.  A FULL iteration adds every point into a dense per-CTA partial (shared memory),
// reduced over the cluster through DSMEM into the iteration's global slot (the totals); a DELTA
// iteration adds + to the new and - to the old cluster of every point whose label changed,
// straight into the global slot (red.add), and every CTA keeps the running totals in shared
// memory.  Integer sums do not depend on the order of the additions, so both modes give the
// totals of a full recomputation bit for bit.  The mode of iteration t is full iff more than
// N/8 points changed label at iteration t - 1 (iteration 0 is full), read from a global
// counter after the grid barrier: uniform per problem.
// Objective (Eq. 6): J_t = sum_j (Q_j - 2 c_j . S_j + W_j ||c_j||^2) from the exact totals of
// iteration t and its FP32 centres, in FP64 (relative rounding ~1e-16 x sum w ||x||^2 / J: 1e-12
// on c3), not the FP64 sum of FP32 distances the FFMA kernels form (they agree to FP32 rounding).
#include <cooperative_groups.h>
#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"
#include "km_fixed.cuh"
#include "km_tile.cuh"
#include "tc_ptx.cuh"

namespace cg = cooperative_groups;

namespace cabsk {

constexpr int kLxT = 384;  // 12 warps, one thread per point
constexpr float kCandSlack = 2e-4f;

#ifdef CABS_PROFILE_LEX
// global-timer stamps of CTA 0 per iteration (<= 64): [0] start, [1] centres, [2] D, [6] bound
// pass, [3] search pass, [4] reduce, [5] barrier; [7] candidates visited (all CTAs, all points)
__device__ long long g_lex_tl[64][16];
#define LEX_STAMP(i) do { if (blockIdx.x == 0 && tid == 0 && it < 64) { long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_lex_tl[it][i] = t_; } } while (0)
#define LEX_CAND(n_) do { if (it < 64) atomicAdd(reinterpret_cast<unsigned long long*>(&g_lex_tl[it][7]), \
    static_cast<unsigned long long>(n_)); } while (0)
__device__ unsigned long long g_lex_q[64];
#define LEX_QUEUE(n_) do { if (it < 64 && tid == 0) atomicAdd(&g_lex_q[it], static_cast<unsigned long long>(n_)); } while (0)
#else
#define LEX_CAND(n_) do { } while (0)
#define LEX_QUEUE(n_) do { } while (0)
#define LEX_STAMP(i) do { } while (0)
#endif

void lex_debug_timeline(long long* out, int n) {
#ifdef CABS_PROFILE_LEX
  const int m = n < 64 * 16 ? n : 64 * 16;
  cudaMemcpyFromSymbol(out, g_lex_tl, sizeof(long long) * m);
  if (n >= 64 * 16 + 64) cudaMemcpyFromSymbol(out + 64 * 16, g_lex_q, sizeof(long long) * 64);
#else
  for (int i = 0; i < n; ++i) out[i] = 0;
#endif
}

struct LexProb {
  const float* X;
  int64_t ldx, N;
  int d, k2;
  const float* w;
  const unsigned* bounds;
  float* centres;
  int64_t ldc;
  int* labels;
  double* objective;
  int* near_ties;
  double* cluster_w;
  long long* fsum;  // [3][Eqp] global slots
  double* pobj;     // [iters][Gq]
  int* ptie;        // [iters][Gq]
  int* chg;         // [iters] points whose label changed (all CTAs of the problem)
  int* tie_log;
  int tie_cap;
  int64_t row_off;
  float* eb;  // [N][k2p] per-centre lower bounds on ||x - c_j||, offset by the cumulative drift
  long long* qv;  // [N] w ||x||^2 in fixed point (scale_q), formed once at the start
};

struct LexArgs {
  LexProb pr[2];
  int nprob, iters, g0;
  unsigned* gbar[2];
  int capn;  // max points per CTA
  int cp;    // centre pitch (floats): >= DP, 16-byte rows
  int k2p;   // D row pitch: round_up(k2max, 4)
  float cand_factor;  // pass-2 candidates: lower bound <= cand_factor u (>= 1 + eps)
  int dperiod;        // ||c_i - c_j|| recomputed exactly every dperiod-th iteration (decayed between)
  int fulldiv;        // an iteration accumulates every point iff > N / fulldiv labels changed before
  uint32_t off_s, off_c, off_d, off_lab, off_ord, off_bd, off_lb, off_qs, off_wd, off_dl, off_cd, total;
};

__host__ __device__ inline uint32_t lex_align(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

inline void lex_plan(LexArgs& a, int dp, int k2max, int64_t capn) {
  a.capn = static_cast<int>(capn);
  a.cp = dp + 4;
  a.k2p = static_cast<int>(round_up(k2max, 4));
  const size_t E = ((size_t)k2max * dp + 2 * k2max + 1) & ~size_t(1);  // dp >= d: covers every problem
  uint32_t o = 0;
  a.off_s = o;
  o = lex_align(o + static_cast<uint32_t>(E * 8), 16);
  a.off_c = o;
  o = lex_align(o + sizeof(float) * k2max * a.cp, 16);
  a.off_d = o;
  o = lex_align(o + sizeof(float) * k2max * a.k2p, 16);
  a.off_lab = o;
  o = lex_align(o + sizeof(int) * static_cast<uint32_t>(capn), 16);
  a.off_ord = o;
  o = lex_align(o + sizeof(int) * static_cast<uint32_t>(capn), 16);
  a.off_bd = o;
  o = lex_align(o + sizeof(float) * static_cast<uint32_t>(capn), 16);
  a.off_lb = o;
  o = lex_align(o + sizeof(float) * static_cast<uint32_t>(capn), 16);
  a.off_qs = o;
  o = lex_align(o + sizeof(int) * static_cast<uint32_t>(capn), 16);
  a.off_wd = o;
  o = lex_align(o + sizeof(double) * k2max, 16);
  a.off_dl = o;
  o = lex_align(o + sizeof(float) * a.k2p, 16);
  a.off_cd = o;
  o = lex_align(o + sizeof(float) * a.k2p, 16);
  a.total = o;
}

// sum_i (x_i - c_i)^2, i ascending, one fmaf chain per centre; n centres interleaved (ILP)
template <int DP, int NC>
__device__ __forceinline__ void lex_chain(const float (&x)[DP], const float* const (&c)[NC], float (&acc)[NC]) {
#pragma unroll
  for (int q = 0; q < NC; ++q) acc[q] = 0.f;
#pragma unroll
  for (int i4 = 0; i4 < DP / 4; ++i4) {
    float4 cv[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) cv[q] = *reinterpret_cast<const float4*>(c[q] + 4 * i4);
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      float f = x[4 * i4] - cv[q].x;
      acc[q] = fmaf(f, f, acc[q]);
      f = x[4 * i4 + 1] - cv[q].y;
      acc[q] = fmaf(f, f, acc[q]);
      f = x[4 * i4 + 2] - cv[q].z;
      acc[q] = fmaf(f, f, acc[q]);
      f = x[4 * i4 + 3] - cv[q].w;
      acc[q] = fmaf(f, f, acc[q]);
    }
  }
}

// the first PD dimensions of the same chain (a prefix of the FP32 sum of non-negative terms, so
// <= the full chain's value bit for bit: an exact lower bound)
template <int DP, int PD, int NC>
__device__ __forceinline__ void lex_chain_part(const float (&x)[DP], const float* const (&c)[NC], float (&acc)[NC]) {
#pragma unroll
  for (int q = 0; q < NC; ++q) acc[q] = 0.f;
#pragma unroll
  for (int i4 = 0; i4 < PD / 4; ++i4) {
    float4 cv[NC];
#pragma unroll
    for (int q = 0; q < NC; ++q) cv[q] = *reinterpret_cast<const float4*>(c[q] + 4 * i4);
#pragma unroll
    for (int q = 0; q < NC; ++q) {
      float f = x[4 * i4] - cv[q].x;
      acc[q] = fmaf(f, f, acc[q]);
      f = x[4 * i4 + 1] - cv[q].y;
      acc[q] = fmaf(f, f, acc[q]);
      f = x[4 * i4 + 2] - cv[q].z;
      acc[q] = fmaf(f, f, acc[q]);
      f = x[4 * i4 + 3] - cv[q].w;
      acc[q] = fmaf(f, f, acc[q]);
    }
  }
}

template <int DP>
__device__ __forceinline__ void lex_load_x(const float* row, int d, float (&x)[DP]) {
#pragma unroll
  for (int i4 = 0; i4 < DP / 4; ++i4) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (4 * i4 + 3 < d) {
      v = __ldg(reinterpret_cast<const float4*>(row + 4 * i4));
    } else if (4 * i4 < d) {
      v.x = __ldg(row + 4 * i4);
      if (4 * i4 + 1 < d) v.y = __ldg(row + 4 * i4 + 1);
      if (4 * i4 + 2 < d) v.z = __ldg(row + 4 * i4 + 2);
    }
    x[4 * i4] = v.x; x[4 * i4 + 1] = v.y; x[4 * i4 + 2] = v.z; x[4 * i4 + 3] = v.w;
  }
}

// Stable counting sort of keys[0..n) (values in [0, k2), k2 <= 128) by ONE warp: out[] = the
// positions in key order, ties in index order.  cnt: shared int[128] scratch.
__device__ __forceinline__ void lex_warp_sort(const int* keys, const int* idx, int n, int k2, int* cnt, int* out) {
  const int lane = threadIdx.x & 31;
  for (int l = lane; l < 128; l += 32) cnt[l] = 0;
  __syncwarp();
  for (int q = lane; q < n; q += 32) atomicAdd(&cnt[keys[idx ? idx[q] : q]], 1);
  __syncwarp();
  int v[4], t = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    v[q] = cnt[4 * lane + q];
    t += v[q];
  }
  int incl = t;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  int run = incl - t;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    cnt[4 * lane + q] = run;
    run += v[q];
  }
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  for (int c0 = 0; c0 < n; c0 += 32) {
    const int q = c0 + lane;
    const int e = q < n ? (idx ? idx[q] : q) : -1;
    const int l = e >= 0 ? keys[e] : -1;
    const unsigned m = __match_any_sync(0xffffffffu, l);
    if (l >= 0) out[cnt[l] + __popc(m & lt)] = e;
    __syncwarp();
    if (l >= 0 && (m & lt) == 0) cnt[l] += __popc(m);
    __syncwarp();
  }
  (void)k2;
}

template <int DP>
__global__ void __launch_bounds__(kLxT, 1) lloyd_prune_kernel(LexArgs a) {
  extern __shared__ __align__(16) uint8_t lx_smem[];
  long long* Sl = reinterpret_cast<long long*>(lx_smem + a.off_s);  // running totals / dense partial
  float* c32 = reinterpret_cast<float*>(lx_smem + a.off_c);          // centres (FP32, pitch cp)
  float* Dn = reinterpret_cast<float*>(lx_smem + a.off_d);           // ||c_i - c_j|| (pitch k2p)
  int* lab = reinterpret_cast<int*>(lx_smem + a.off_lab);            // labels (point order)
  int* queue = reinterpret_cast<int*>(lx_smem + a.off_ord);          // points needing a search
  float* ubv = reinterpret_cast<float*>(lx_smem + a.off_bd);         // upper bound on ||x - c_label||
  float* lbv = reinterpret_cast<float*>(lx_smem + a.off_lb);         // lower bound, other centres
  int* qsort = reinterpret_cast<int*>(lx_smem + a.off_qs);           // queue in label order
  float* dlt = reinterpret_cast<float*>(lx_smem + a.off_dl);         // centre drift of this update
  float* cdr = reinterpret_cast<float*>(lx_smem + a.off_cd);         // cumulative drift (rounded up)
  __shared__ int s_tie[kLxT / 32];
  __shared__ double s_obj[kLxT / 32];
  __shared__ int s_full, s_nq, s_next;
  __shared__ float s_dmax;
  __shared__ int s_cnt[128];

  cg::cluster_group cluster = cg::this_cluster();
  const int crank = static_cast<int>(cluster.block_rank()), csize = static_cast<int>(cluster.num_blocks());
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  const int myq = (a.nprob > 1 && static_cast<int>(blockIdx.x) >= a.g0) ? 1 : 0;
  const int b = myq ? static_cast<int>(blockIdx.x) - a.g0 : static_cast<int>(blockIdx.x);
  const int Gb = a.nprob > 1 ? (myq ? G - a.g0 : a.g0) : G;
  const LexProb& pr = a.pr[myq];
  const int d = pr.d, k2 = pr.k2, cp = a.cp, k2p = a.k2p;
  const int64_t pbeg = (pr.N * b) / Gb, pend = (pr.N * (b + 1)) / Gb;
  const int npts = static_cast<int>(pend - pbeg);
  // exact int64 totals per cluster: [k2 d sums of w x | k2 weights | k2 sums of w ||x||^2]
  const int nsum = k2 * d, oq = nsum + k2;
  const int64_t Eq = (int64_t)nsum + 2 * k2, Eqp = (Eq + 1) & ~int64_t(1);
  const int64_t ebeg = Eq * crank / csize, eend = Eq * (crank + 1) / csize;
  double scale, scale_w, scale_q;
  fx_scales(pr.bounds, pr.N, scale, scale_w);
  {
    const double xm = static_cast<double>(__uint_as_float(__ldcg(pr.bounds)));
    const double wm = static_cast<double>(__uint_as_float(__ldcg(pr.bounds + 1)));
    scale_q = ldexp(1.0, fx_scale_exp(static_cast<double>(pr.N) * wm * d * xm * xm));
  }
  const double inv_scale = 1.0 / scale;
  constexpr float kEps = kCandSlack;

  // centres of iteration 0 (global) -> FP32 copy, zero-padded to the pitch; Dn padding = +inf
  for (int e = tid; e < k2 * cp; e += kLxT) {
    const int j = e / cp, i = e - j * cp;
    c32[e] = i < d ? __ldcg(pr.centres + (int64_t)j * pr.ldc + i) : 0.f;
  }
  for (int e = tid; e < k2 * k2p; e += kLxT) Dn[e] = (e % k2p) < k2 ? 0.f : FLT_MAX;
  for (int j = tid; j < k2p; j += kLxT) { dlt[j] = 0.f; cdr[j] = 0.f; }
  // w ||x||^2 of the CTA's points in fixed point (one warp per point, coalesced, FP64 in a fixed
  // order): the per-point term of the per-cluster sums Q_j
  for (int pl = warp; pl < npts; pl += kLxT / 32) {
    const int64_t p = pbeg + pl;
    double x2 = 0.0;
    for (int i = lane; i < d; i += 32) {
      const double v = static_cast<double>(__ldg(pr.X + p * pr.ldx + i));
      x2 = fma(v, v, x2);
    }
    x2 = warp_sum_d(x2);
    if (lane == 0) pr.qv[p] = llrint(static_cast<double>(__ldg(pr.w + p)) * x2 * scale_q);
  }
  __syncthreads();

  // J_t = sum_j (Q_j - 2 c_j . S_j + W_j ||c_j||^2) (Eq. 6 expanded over the exact per-cluster sums;
  // the FP32 centres c_j of iteration t) -> objective[t]; CTA 0 of the problem, FP64, fixed order
  auto objective_of = [&](int t) {
    double acc = 0.0;
    for (int j = tid; j < k2; j += kLxT) {  // thread = centre, dimensions in order
      double cs = 0.0, cc = 0.0;
      for (int i = 0; i < d; ++i) {
        const double c = static_cast<double>(c32[j * cp + i]);
        cs = fma(c, static_cast<double>(Sl[j * d + i]), cs);
        cc = fma(c, c, cc);
      }
      acc += static_cast<double>(Sl[oq + j]) / scale_q - 2.0 * cs / scale + static_cast<double>(Sl[nsum + j]) / scale_w * cc;
    }
    acc = warp_sum_d(acc);
    if (lane == 0) s_obj[warp] = acc;
    __syncthreads();
    if (tid == 0) {
      double o = 0.0;
      for (int w = 0; w < kLxT / 32; ++w) o += s_obj[w];
      pr.objective[t] = o;
    }
  };

  bool prev_full = true;
  for (int it = 0; it < a.iters; ++it) {
    LEX_STAMP(0);
    // ------------------------------------------------------------ centres of this iteration
    if (it > 0) {
      // the totals of iteration it - 1 (or their change): every CTA reads the whole slot, starting
      // at a CTA-dependent offset so that the 148 readers spread over the L2 slices
      const long long* slot = pr.fsum + (size_t)((it - 1) % 3) * Eqp;
      {
        const int64_t rot = ((int64_t)blockIdx.x * 997) % Eq;
        constexpr int kU = 8;  // loads in flight per thread
        for (int64_t e0 = tid; e0 < Eq; e0 += kU * kLxT) {
          long long v[kU];
          int64_t ee[kU];
#pragma unroll
          for (int u = 0; u < kU; ++u) {
            const int64_t e1 = e0 + u * kLxT;
            ee[u] = e1 + rot < Eq ? e1 + rot : e1 + rot - Eq;
            v[u] = e1 < Eq ? __ldcg(slot + ee[u]) : 0;
          }
#pragma unroll
          for (int u = 0; u < kU; ++u)
            if (e0 + u * kLxT < Eq) Sl[ee[u]] = prev_full ? v[u] : Sl[ee[u]] + v[u];
        }
      }
      // zero this CTA's share of the slot iteration it + 1 accumulates into
      long long* fs_next = pr.fsum + (size_t)((it + 1) % 3) * Eqp;
      for (int64_t e = (int64_t)b * kLxT + tid; e < Eq; e += (int64_t)Gb * kLxT) fs_next[e] = 0;
      if (tid == 0) {
        s_full = __ldcg(pr.chg + it - 1) * static_cast<long long>(a.fulldiv) > pr.N;
        s_dmax = 0.f;
      }
      __syncthreads();
      LEX_STAMP(8);
      if (b == 0) objective_of(it - 1);
      LEX_STAMP(9);
      // new centres (an empty cluster keeps its centre) and their drift ||c_new - c_old||: one
      // thread per centre, dimensions in order
      for (int j = tid; j < k2; j += kLxT) {
        const long long wj = Sl[nsum + j];
        const double rw = wj > 0 ? 1.0 / (static_cast<double>(wj) * (1.0 / scale_w)) : 0.0;
        float s2 = 0.f;
        if (rw > 0) {
          for (int i = 0; i < d; ++i) {
            const float v = static_cast<float>((static_cast<double>(Sl[j * d + i]) * inv_scale) * rw);
            const float f = v - c32[j * cp + i];
            s2 = fmaf(f, f, s2);
            c32[j * cp + i] = v;
          }
        }
        const float dj = sqrtf(s2) * (1.f + 2e-5f);  // rounded up (FP32 chain): a valid drift bound
        dlt[j] = dj;
        cdr[j] = __fadd_ru(cdr[j], dj);
        atomicMax(reinterpret_cast<int*>(&s_dmax), __float_as_int(dj));  // non-negative floats order as ints
      }
      __syncthreads();
      LEX_STAMP(1);
      if (it % a.dperiod == 1 % a.dperiod) {
      // Dn_ij = ||c_i - c_j||: one warp per row i of this CTA's share (rows i = crank mod csize),
      // lane l takes j = l + 32 q (consecutive lanes on consecutive rows of c32: odd pitch in
      // 16-byte units, conflict-free; c_i is a broadcast); then every CTA copies the other rows
      // from their owners in the cluster (DSMEM).  (c_i - c_j)^2 = (c_j - c_i)^2 bit for bit, so
      // Dn is exactly symmetric.
      for (int i = crank + csize * warp; i < k2; i += csize * (kLxT / 32)) {
        const float* ci = c32 + i * cp;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
        const float* cj[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) cj[q] = c32 + (lane + 32 * q < k2 ? lane + 32 * q : i) * cp;
        for (int i4 = 0; i4 < cp / 4; ++i4) {
          const float4 u = *reinterpret_cast<const float4*>(ci + 4 * i4);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const float4 v = *reinterpret_cast<const float4*>(cj[q] + 4 * i4);
            float f = u.x - v.x;
            acc[q] = fmaf(f, f, acc[q]);
            f = u.y - v.y;
            acc[q] = fmaf(f, f, acc[q]);
            f = u.z - v.z;
            acc[q] = fmaf(f, f, acc[q]);
            f = u.w - v.w;
            acc[q] = fmaf(f, f, acc[q]);
          }
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int jj = lane + 32 * q;
          if (jj < k2) Dn[i * k2p + jj] = jj == i ? 0.f : sqrtf(acc[q]) * (1.f - 2e-5f);  // rounded down
        }
      }
      cluster.sync();
      if (csize > 1) {
        const int n4 = k2p / 4;
        for (int e = tid; e < k2 * n4; e += kLxT) {
          const int i = e / n4, r = i % csize;
          if (r == crank) continue;
          const float4* src = reinterpret_cast<const float4*>(cluster.map_shared_rank(Dn, r) + i * k2p) + (e - i * n4);
          reinterpret_cast<float4*>(Dn + i * k2p)[e - i * n4] = *src;
        }
      }
      } else {
        // in between, a lower bound: ||c_i' - c_j'|| >= ||c_i - c_j|| - dlt_i - dlt_j (rounded down)
        for (int e = tid; e < k2 * k2; e += kLxT) {
          const int i = e / k2, jj = e - i * k2;
          if (jj != i) Dn[i * k2p + jj] = fmaxf(__fsub_rd(__fsub_rd(Dn[i * k2p + jj], dlt[i]), dlt[jj]), 0.f);
        }
      }
      LEX_STAMP(2);
    } else {
      if (tid == 0) s_full = 1;
    }
    if (tid == 0) { s_nq = 0; s_next = 0; }
    __syncthreads();
    const bool full = s_full != 0;
    long long* slot = pr.fsum + (size_t)(it % 3) * Eqp;
    if (full) {  // the dense partial overlays the running totals (not needed until the next iteration)
      for (int64_t e = tid; e < Eqp; e += kLxT) Sl[e] = 0;
      __syncthreads();
    }
    const float dmax = s_dmax;

    int ties = 0, nchg = 0;
    unsigned* pw = reinterpret_cast<unsigned*>(Sl);
    auto add64 = [&](int e, long long v) {  // exact int64 add into the shared partial by two 32-bit atomics
      const unsigned lo = static_cast<unsigned>(v);
      const unsigned old = atomicAdd(pw + 2 * e, lo);
      atomicAdd(reinterpret_cast<int*>(pw + 2 * e + 1), static_cast<int>(v >> 32) + ((old + lo) < old ? 1 : 0));
    };
    // the update of point pl (label bj, previous label a0, x in registers)
    auto update = [&](int pl, int64_t p, const float (&x)[DP], int bj, int a0) {
      if (full || bj != a0) {
        const float wv = __ldg(pr.w + p);
        const double ws = static_cast<double>(wv) * scale;
        const long long iw = llrint(static_cast<double>(wv) * scale_w);
        const long long iq = __ldcg(pr.qv + p);
        if (full) {
#pragma unroll
          for (int i = 0; i < DP; ++i)
            if (i < d) add64(bj * d + i, fx_prod_magic(ws, x[i]));
          add64(nsum + bj, iw);
          add64(oq + bj, iq);
        } else {
#pragma unroll
          for (int i = 0; i < DP; ++i) {
            if (i < d) {
              const long long v = fx_prod_magic(ws, x[i]);
              if (v != 0) {
                red_add_u64(slot + bj * d + i, v);
                red_add_u64(slot + a0 * d + i, -v);
              }
            }
          }
          if (iw != 0) {
            red_add_u64(slot + nsum + bj, iw);
            red_add_u64(slot + nsum + a0, -iw);
          }
          if (iq != 0) {
            red_add_u64(slot + oq + bj, iq);
            red_add_u64(slot + oq + a0, -iq);
          }
        }
      }
      lab[pl] = bj;
      if (it == a.iters - 1) pr.labels[p] = bj;
    };

    // ------------------------------------------------------------ assignment, pass 1: bound test
    // (thread = point, index order).  U >= ||x - c_a|| and L <= ||x - c_j|| for every j != a from
    // the previous iteration; the centres moved by dlt_j <= dmax, so U + dlt_a and L - dmax bound the
    // new distances.  If L - dmax > (1 + eps) U', no other centre is nearer or within the near-tie
    // band: the label stays (x is not even read unless this iteration accumulates every point).
    // Otherwise U is tightened to the exact distance, the test repeated, and failing points queued.
    if (it > 0) {
      for (int pl = tid; pl < npts; pl += kLxT) {
        const int64_t p = pbeg + pl;
        const int a0 = lab[pl];
        const float Lm = lbv[pl] - dmax;
        const float U1 = __fadd_ru(ubv[pl], dlt[a0]);
        if (!full && Lm > (1.f + kEps) * U1) {
          ubv[pl] = U1;
          lbv[pl] = Lm;
          if (it == a.iters - 1) pr.labels[p] = a0;
          continue;
        }
        if (!(Lm > 0.f)) {  // cannot pass whatever u is
          queue[atomicAdd(&s_nq, 1)] = pl;
          continue;
        }
        float x[DP];
        lex_load_x<DP>(pr.X + p * pr.ldx, d, x);
        float acc[1];
        const float* c[1] = {c32 + a0 * cp};
        lex_chain<DP, 1>(x, c, acc);
        const float u = sqrtf(acc[0]) * (1.f + 2e-5f);
        if (Lm > (1.f + kEps) * u) {
          ubv[pl] = u;
          lbv[pl] = Lm;
          update(pl, p, x, a0, a0);
        } else {
          queue[atomicAdd(&s_nq, 1)] = pl;
        }
      }
      __syncthreads();
      // the queue in the order of the labels (stable): a warp's points then share their label, so
      // the union of their candidate sets is small and the lanes read the same centre rows
      if (warp == 0) lex_warp_sort(lab, queue, s_nq, k2, s_cnt, qsort);
      __syncthreads();
    } else {
      if (tid == 0) s_nq = npts;
      __syncthreads();
    }
    LEX_STAMP(6);
    // ------------------------------------------------------------ pass 2: candidate search
    // (warp = 32 queued points, chunks taken dynamically).  Candidates of a point with label a:
    // every j whose lower bound -- the per-centre bound stored at its last search less the drift
    // since (eb), or ||c_a - c_j|| - u -- is <= (1 + eps) u (triangle inequality; see the header);
    // iteration 0: every centre.  The warp visits the union of its lanes' candidates, and every
    // exact distance it computes becomes the point's stored bound for that centre.
    const int nq = s_nq;
    LEX_QUEUE(nq);
    for (;;) {
      int q0 = 0;
      if (lane == 0) q0 = atomicAdd(&s_next, 32);
      q0 = __shfl_sync(0xffffffffu, q0, 0);
      if (q0 >= nq) break;
      const bool act = q0 + lane < nq;
      const int qq = act ? q0 + lane : q0;
      const int pl = it > 0 ? qsort[qq] : qq;
      const int64_t p = pbeg + pl;
      float x[DP];
      lex_load_x<DP>(pr.X + p * pr.ldx, d, x);
      float bd = FLT_MAX, sd = FLT_MAX;
      int bj = 0x7fffffff, sj = -1;
      auto take = [&](float val, int j) {
        if (val < bd || (val == bd && j < bj)) { sd = bd; sj = bj; bd = val; bj = j; }
        else if (val < sd) { sd = val; sj = j; }
      };
      const int a0 = it > 0 ? lab[pl] : -1;
      uint32_t rem[4] = {0u, 0u, 0u, 0u};
      float lbo = FLT_MAX;  // min lower bound over the centres NOT evaluated
      float* ebr = pr.eb + p * k2p;
      auto store_lb = [&](int j, float d2) {  // exact distance -> the stored bound (rounded down)
        if (act) ebr[j] = __fadd_rd(sqrtf(d2) * (1.f - 2e-5f), cdr[j]);
      };
      if (a0 < 0) {
#pragma unroll
        for (int w = 0; w < 4; ++w) rem[w] = 32 * w + 32 <= k2 ? 0xffffffffu : (32 * w < k2 ? (1u << (k2 - 32 * w)) - 1u : 0u);
      } else {
        {
          const float* c[1] = {c32 + a0 * cp};
          float acc[1];
          lex_chain<DP, 1>(x, c, acc);
          take(acc[0], a0);
        }
        const float u = sqrtf(bd) * (1.f + 2e-5f);
        const float tu = a.cand_factor * u;  // >= (1 + eps) u: every centre that could be nearer or near-tied
        const float* drow = Dn + a0 * k2p;
        for (int j4 = 0; j4 < k2p / 4; ++j4) {
          const float4 v = *reinterpret_cast<const float4*>(drow + 4 * j4);
          const float4 e = __ldcg(reinterpret_cast<const float4*>(ebr + 4 * j4));
          const float4 g = *reinterpret_cast<const float4*>(cdr + 4 * j4);
          const float vv[4] = {v.x, v.y, v.z, v.w}, ee[4] = {e.x, e.y, e.z, e.w}, gg[4] = {g.x, g.y, g.z, g.w};
          uint32_t m = 0u;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = 4 * j4 + q;
            if (j < k2 && j != a0) {
              // lower bound on ||x - c_j||: the stored bound less the drift since, or the triangle
              // inequality through c_a
              const float lbj = fmaxf(__fsub_rd(ee[q], gg[q]), __fsub_rd(vv[q], u));
              if (lbj <= tu) m |= 1u << q;
              else lbo = fminf(lbo, lbj);
            }
          }
          rem[j4 >> 3] |= m << ((4 * j4) & 31);
        }
        if (!act) rem[0] = rem[1] = rem[2] = rem[3] = 0u;
        store_lb(a0, bd);
      }
#pragma unroll
      for (int w = 0; w < 4; ++w) rem[w] = __reduce_or_sync(0xffffffffu, rem[w]);
      LEX_CAND(act ? __popc(rem[0]) + __popc(rem[1]) + __popc(rem[2]) + __popc(rem[3]) : 0);
      // partial distance search: the first PD dimensions of every union candidate's chain (warp-
      // uniform, shared-memory broadcasts) are an exact lower bound of its distance; a candidate
      // whose prefix exceeds (1 + eps) times the best distance known so far cannot be nearer or in
      // the near-tie band, and its prefix becomes its stored bound.  The lane's survivors then
      // complete their chains (from dimension 0: the same FP32 sums).  Iteration 0 first guesses
      // the label as the centre of smallest prefix and evaluates it fully.
#ifndef CABS_LEX_PD
#define CABS_LEX_PD 24  // measured on c3: 8 / 16 / 24 / 32 -> 4.23 / 4.16 / 4.10 / 4.20 ms
#endif
      constexpr int PD = DP >= 48 ? CABS_LEX_PD : 0;
      int guess = -1;
      auto each4 = [&](const uint32_t (&msk)[4], auto&& fn) {  // warp-uniform visit, 4 centres per step
        uint32_t r[4] = {msk[0], msk[1], msk[2], msk[3]};
        for (;;) {
          int jj[4], cnt = 0;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            int j = -1;
#pragma unroll
            for (int w = 0; w < 4; ++w)
              if (j < 0 && r[w]) { j = 32 * w + __ffs(r[w]) - 1; r[w] &= r[w] - 1; }
            jj[q] = j;
            cnt += j >= 0;
          }
          if (cnt == 0) break;
          fn(jj);
        }
      };
      uint32_t sv[4] = {rem[0], rem[1], rem[2], rem[3]};
      if (PD > 0) {
        if (a0 < 0) {
          float pmin = FLT_MAX;
          int pj = 0;
          each4(rem, [&](const int (&jj)[4]) {
            const float* c[4] = {c32 + (jj[0] < 0 ? 0 : jj[0]) * cp, c32 + (jj[1] < 0 ? 0 : jj[1]) * cp,
                                 c32 + (jj[2] < 0 ? 0 : jj[2]) * cp, c32 + (jj[3] < 0 ? 0 : jj[3]) * cp};
            float acc[4];
            lex_chain_part<DP, PD, 4>(x, c, acc);
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (jj[q] >= 0 && (acc[q] < pmin || (acc[q] == pmin && jj[q] < pj))) { pmin = acc[q]; pj = jj[q]; }
          });
          const float* c[1] = {c32 + pj * cp};
          float acc[1];
          lex_chain<DP, 1>(x, c, acc);
          take(acc[0], pj);
          store_lb(pj, acc[0]);
          guess = pj;
        }
        const float thrp = bd * (1.f + kEps);
        sv[0] = sv[1] = sv[2] = sv[3] = 0u;
        each4(rem, [&](const int (&jj)[4]) {
          const float* c[4] = {c32 + (jj[0] < 0 ? 0 : jj[0]) * cp, c32 + (jj[1] < 0 ? 0 : jj[1]) * cp,
                               c32 + (jj[2] < 0 ? 0 : jj[2]) * cp, c32 + (jj[3] < 0 ? 0 : jj[3]) * cp};
          float acc[4];
          lex_chain_part<DP, PD, 4>(x, c, acc);
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int j = jj[q];
            if (j < 0 || j == a0 || j == guess) continue;
            if (acc[q] <= thrp) {
              sv[j >> 5] |= 1u << (j & 31);
            } else {
              lbo = fminf(lbo, sqrtf(acc[q]) * (1.f - 2e-5f));
              store_lb(j, acc[q]);
            }
          }
        });
      } else if (a0 >= 0) {
        sv[a0 >> 5] &= ~(1u << (a0 & 31));
      }
      // the lane's survivors: full chains, two at a time
      auto nxt = [&]() {
        int j = -1;
#pragma unroll
        for (int w = 0; w < 4; ++w)
          if (j < 0 && sv[w]) { j = 32 * w + __ffs(sv[w]) - 1; sv[w] &= sv[w] - 1; }
        return j;
      };
      if (!act) sv[0] = sv[1] = sv[2] = sv[3] = 0u;
      for (;;) {
        const int j0 = nxt();
        if (j0 < 0) break;
        const int j1 = nxt();
        const float* c[2] = {c32 + j0 * cp, c32 + (j1 < 0 ? j0 : j1) * cp};
        float acc[2];
        lex_chain<DP, 2>(x, c, acc);
        take(acc[0], j0);
        store_lb(j0, acc[0]);
        if (j1 >= 0) { take(acc[1], j1); store_lb(j1, acc[1]); }
      }
      if (act) {
        ubv[pl] = sqrtf(bd) * (1.f + 2e-5f);
        // every centre other than bj: evaluated ones are >= sqrt(sd), the others >= lbo
        lbv[pl] = fminf(sd < FLT_MAX ? sqrtf(sd) * (1.f - 2e-5f) : FLT_MAX, lbo);
        const bool tie = (sd - bd) < kNearTie * sd;
        ties += tie;
        if (tie && pr.tie_log) km_log_tie(pr.tie_log, pr.tie_cap, it, pr.row_off + p, bj, sj, bd, sd);
        nchg += bj != a0;
        update(pl, p, x, bj, a0);
      }
    }
    LEX_STAMP(3);
    // near ties / label changes of this CTA
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      ties += __shfl_xor_sync(0xffffffffu, ties, o);
      nchg += __shfl_xor_sync(0xffffffffu, nchg, o);
    }
    if (lane == 0) {
      s_tie[warp] = ties;
      if (nchg) atomicAdd(pr.chg + it, nchg);
    }
    if (full) {
      // cluster reduction of the dense partials (DSMEM), one global integer add per entry
      cluster.sync();
      for (int64_t e = ebeg + tid; e < eend; e += kLxT) {
        long long s = 0;
        for (int rr = 0; rr < csize; ++rr) s += cluster.map_shared_rank(Sl, rr)[e];
        if (s != 0) red_add_u64(slot + e, s);
      }
      cluster.sync();  // the cluster's partials are read: the buffer may be overwritten
    } else {
      __syncthreads();
    }
    if (tid == 0) {
      int qq = 0;
      for (int w = 0; w < kLxT / 32; ++w) qq += s_tie[w];
      pr.ptie[(size_t)it * Gb + b] = qq;
    }
    LEX_STAMP(4);
    // grid barrier of the problem (monotonic arrival counter)
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      unsigned* bar = a.gbar[myq];
      atomicAdd(bar, 1u);
      const unsigned target = static_cast<unsigned>(Gb) * static_cast<unsigned>(it + 1);
      while (ld_acquire_gpu(bar) < target) __nanosleep(20);
    }
    __syncthreads();
    prev_full = full;
    LEX_STAMP(5);
  }
  // ---------------- epilogue (CTA 0 of each problem): final centres, cluster weights, objective
  if (b == 0) {
    const long long* slot = pr.fsum + (size_t)((a.iters - 1) % 3) * Eqp;
    if (prev_full) {
      for (int64_t e = tid; e < Eq; e += kLxT) Sl[e] = __ldcg(slot + e);
    } else {
      for (int64_t e = tid; e < Eq; e += kLxT) Sl[e] += __ldcg(slot + e);
    }
    __syncthreads();
    objective_of(a.iters - 1);
    const double inv_scale_w = 1.0 / scale_w;
    for (int e = tid; e < nsum; e += kLxT) {
      const int j = e / d, i = e - j * d;
      const long long wj = Sl[nsum + j];
      pr.centres[(int64_t)j * pr.ldc + i] =
          wj > 0 ? static_cast<float>((static_cast<double>(Sl[e]) * inv_scale) *
                                      (1.0 / (static_cast<double>(wj) * inv_scale_w)))
                 : c32[j * cp + i];
    }
    for (int j = tid; j < k2; j += kLxT) pr.cluster_w[j] = static_cast<double>(Sl[nsum + j]) / scale_w;
    for (int t = tid; t < a.iters; t += kLxT) {
      long long qq = 0;
      for (int g = 0; g < Gb; ++g) qq += __ldcg(pr.ptie + (size_t)t * Gb + g);
      if (pr.near_ties) pr.near_ties[t] = static_cast<int>(qq);
    }
  }
}

// ---------------------------------------------------------------- host side
constexpr size_t kLexSmemCap = 225 * 1024;

static int lex_dp(int d) { return static_cast<int>(round_up(d, 16)); }

// Selected for k2 d >= 4096 (c3: k2 = d = 100); below that the FFMA kernel's full search is as
// cheap (c2: k2 = d = 50 on noise-dominated embeddings, where every centre stays a candidate).
// CABS_KMEANS_PRUNE=1 forces it wherever it applies; CABS_KMEANS_FFMA / CABS_KMEANS_TC select those.
bool kmeans_prune_selected(int k2, int d) {
  if (getenv("CABS_KMEANS_FFMA") || getenv("CABS_KMEANS_TC")) return false;
  if (k2 < 1 || k2 > 128 || d < 1 || d > 128) return false;
  if (!getenv("CABS_KMEANS_PRUNE") && k2 * d < 4096) return false;
  LexArgs a{};
  lex_plan(a, lex_dp(d), k2, 2048);
  return a.total <= kLexSmemCap;
}

template <int DP>
static bool lex_launch(LexArgs& a, int njobs, const LloydJob* jobs, int iters, int dmax, int k2max, int nsm,
                       cudaStream_t st) {
  auto kern = lloyd_prune_kernel<DP>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kLexSmemCap)) !=
        cudaSuccess)
      return false;
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kLxT);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  const double Ntot = static_cast<double>(jobs[0].N) + (njobs > 1 ? static_cast<double>(jobs[1].N) : 0.0);
  int csize = 0;
  int64_t Gq[2] = {0, 0}, Gt = 0;
  LexArgs plan{};
  for (int c = 8; c >= 1 && csize == 0; c >>= 1) {
    const int64_t tot = (int64_t)nsm / c * c;
    if (tot < c * njobs) continue;
    int64_t g[2] = {tot, 0};
    if (njobs > 1) {
      // CTAs in proportion to the points (CABS_KM_SPLIT = the first problem's share, diagnostics)
      double share = static_cast<double>(jobs[0].N) / Ntot;
      if (const char* e = getenv("CABS_KM_SPLIT")) share = atof(e);
      g[0] = (int64_t)llround(static_cast<double>(tot) * share / c) * c;
      g[0] = g[0] < c ? c : (g[0] > tot - c ? tot - c : g[0]);
      g[1] = tot - g[0];
    }
    bool ok = true;
    int64_t capn = 0;
    for (int q = 0; q < njobs; ++q) {
      if (g[q] > jobs[q].N) ok = false;
      const int64_t per = ceil_div(jobs[q].N, g[q] > 0 ? g[q] : 1);
      capn = per > capn ? per : capn;
    }
    if (!ok) continue;
    LexArgs t{};
    lex_plan(t, DP, k2max, round_up(capn, 4));
    if (t.total > kLexSmemCap) continue;
    at[0].val.clusterDim.x = static_cast<unsigned>(c);
    cfg.gridDim = dim3(static_cast<unsigned>(tot));
    cfg.dynamicSmemBytes = t.total;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) == cudaSuccess && (int64_t)ncl * c >= tot) {
      csize = c;
      Gt = tot;
      Gq[0] = g[0];
      Gq[1] = g[1];
      plan = t;
    }
  }
  cudaGetLastError();
  if (csize == 0) return false;
  (void)dmax;
  a = plan;
  {
    const char* cf = getenv("CABS_KMEANS_CAND");
    // measured on c3 (tools/kcand.py): 1.0003 / 1.01 / 1.05 / 1.2 -> 4.02 / 4.05 / 4.12 / 4.29 ms
    a.cand_factor = cf ? static_cast<float>(atof(cf)) : 1.0003f;
    if (!(a.cand_factor >= 1.f + kCandSlack)) a.cand_factor = 1.f + kCandSlack;
    // measured on c3 (tools/ktune.py, period:divisor): 4:16 4.02, 8:16 3.97, 4:8 3.95, 8:8 3.90,
    // 16:8 3.91, 1:16 4.25, 4:64 4.38 ms
    const char* dp = getenv("CABS_KM_DPERIOD");  // (diagnostics)
    a.dperiod = dp ? atoi(dp) : 8;
    if (a.dperiod < 1) a.dperiod = 1;
    const char* fd = getenv("CABS_KM_FULLDIV");
    a.fulldiv = fd ? atoi(fd) : 8;
    if (a.fulldiv < 1) a.fulldiv = 1;
  }
  a.nprob = njobs;
  a.iters = iters;
  a.g0 = static_cast<int>(Gq[0]);
  for (int q = 0; q < njobs; ++q) {
    const LloydJob& j = jobs[q];
    const size_t E = ((size_t)j.k2 * j.d + 2 * j.k2 + 1) & ~size_t(1);
    const size_t need = sizeof(long long) * 3 * E + 16 + (sizeof(double) + sizeof(int)) * iters * Gt + sizeof(int) * iters;
    if (need > j.scratch_bytes) return false;
    char* base = static_cast<char*>(j.scratch);
    LexProb& p = a.pr[q];
    p.X = j.X; p.ldx = j.ldx; p.N = j.N; p.d = j.d; p.k2 = j.k2; p.w = j.w; p.bounds = j.bounds;
    p.centres = j.centres; p.ldc = j.ldc; p.labels = j.labels; p.objective = j.objective;
    p.near_ties = j.near_ties; p.cluster_w = j.cluster_w;
    p.fsum = reinterpret_cast<long long*>(base);
    unsigned* gb = reinterpret_cast<unsigned*>(p.fsum + 3 * E);
    a.gbar[q] = gb;
    p.pobj = reinterpret_cast<double*>(gb + 4);
    p.ptie = reinterpret_cast<int*>(p.pobj + (size_t)iters * Gt);
    p.chg = p.ptie + (size_t)iters * Gt;
    p.tie_log = j.tie_log;
    p.tie_cap = j.tie_cap;
    p.row_off = j.row_off;
    if (!j.ebuf || sizeof(float) * (size_t)j.N * (size_t)a.k2p > j.ebuf_bytes) return false;
    p.eb = j.ebuf;
    if (!j.qbuf) return false;
    p.qv = j.qbuf;
    if (cudaMemsetAsync(base, 0, sizeof(long long) * 3 * E + 16, st) != cudaSuccess) return false;
    if (cudaMemsetAsync(p.chg, 0, sizeof(int) * iters, st) != cudaSuccess) return false;
  }
  (void)k2max;
  cfg.gridDim = dim3(static_cast<unsigned>(Gt));
  cfg.dynamicSmemBytes = a.total;
  at[0].val.clusterDim.x = static_cast<unsigned>(csize);
  note_launch();
  return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess;
}

bool launch_lloyd_prune(const LloydJob* jobs, int njobs, int iters, cudaStream_t st) {
  if (njobs < 1 || njobs > 2) return false;
  int dmax = 0, k2max = 0;
  for (int q = 0; q < njobs; ++q) {
    if (!kmeans_prune_selected(jobs[q].k2, jobs[q].d) || jobs[q].N <= 0) return false;
    if ((jobs[q].ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(jobs[q].X) & 15) != 0) return false;
    dmax = jobs[q].d > dmax ? jobs[q].d : dmax;
    k2max = jobs[q].k2 > k2max ? jobs[q].k2 : k2max;
  }
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  LexArgs a{};
  switch (lex_dp(dmax)) {
    case 16: return lex_launch<16>(a, njobs, jobs, iters, dmax, k2max, nsm, st);
    case 32: return lex_launch<32>(a, njobs, jobs, iters, dmax, k2max, nsm, st);
    case 48: return lex_launch<48>(a, njobs, jobs, iters, dmax, k2max, nsm, st);
    case 64: return lex_launch<64>(a, njobs, jobs, iters, dmax, k2max, nsm, st);
    case 80: return lex_launch<80>(a, njobs, jobs, iters, dmax, k2max, nsm, st);
    case 96: return lex_launch<96>(a, njobs, jobs, iters, dmax, k2max, nsm, st);
    case 112: return lex_launch<112>(a, njobs, jobs, iters, dmax, k2max, nsm, st);
    case 128: return lex_launch<128>(a, njobs, jobs, iters, dmax, k2max, nsm, st);
    default: return false;
  }
}

}  // namespace cabsk
