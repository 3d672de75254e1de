// lloyd.cu -- the whole Lloyd loop of one or two k-means problems (the row side and the
// column side of CABS, Alg. 2 steps 6-7) in ONE persistent kernel (single GPU):
// c iterations x {centres | assign | accumulate | cluster reduce | grid barrier}, no host
// round trips, no per-iteration launches, ONE grid-wide barrier per iteration for both
// problems.  Every CTA (one per SM) holds a balanced contiguous slice of the points of EACH
// problem, so the two problems share the synchronisation latency instead of paying it twice.
//
// Arithmetic (Eq. 6; c iterations P:204):
//  * distances by direct differences in FP32, dimensions ascending (= km_tile.cuh), lowest
//    centre index on ties; two centres per packed FP32x2 instruction (FADD2/FFMA2: the same
//    IEEE rounding as the scalar ops, half the instructions);
//  * sums w_l X_l and w_l accumulated EXACTLY as int64 fixed point (km_fixed.cuh): a dense
//    int64 partial per CTA in shared memory (warp w owns the clusters j = w mod 8, so the
//    read-modify-writes need no atomics), the CTAs of a thread-block cluster add their
//    partials through distributed shared memory (each CTA one slice), and one
//    red.global.add.u64 per (cluster, entry) lands in the global sums -- order-free, so
//    deterministic and identical to the per-iteration kernels of kmeans.cu;
//  * centres = (sum / 2^S) * (1 / (weight / 2^Sw)) in FP64, formed by every CTA for all
//    entries straight from the global sums; an empty cluster keeps its centre (Z12).
// Global sums rotate over three slots: slot it%3 accumulates, slot (it-1)%3 is read by
// every CTA to form this iteration's centres, slot (it+1)%3 is zeroed for the next one.
// Synchronisation per iteration: one cluster barrier (partials complete) and one grid
// barrier (a monotonic arrival counter; the partials and the rotating slots make every
// other hazard one iteration apart).
#include <cooperative_groups.h>
#include <float.h>
#include <limits.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"
#include "km_fixed.cuh"
#include "km_tile.cuh"
#include "tc_ptx.cuh"

namespace cg = cooperative_groups;

namespace cabsk {

constexpr int kLT = 256;       // threads per CTA (one CTA per SM)
constexpr int kLA = 7;         // max point rows per thread
constexpr int kLP = 16 * kLA;  // max points per chunk: thread (pt = tid & 15, ct = tid >> 4) owns points pt + 16u
constexpr int kLC = 64;        // centres per block: ... and centres j0 + ct + 16v, v < 4
constexpr int kMaxProb = 2;
#ifdef CABS_PROFILE_LLOYD
// per-CTA global-timer stamps of iteration kTlIter (phase boundaries), for cabs_debug_counters
constexpr int kTlIter = 10;
__device__ long long g_ll_tl[320][16];
__device__ __forceinline__ long long globaltimer_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

struct LloydProb {
  const float* X;
  int64_t ldx, N;
  int d, k2;
  const float* w;
  float* centres;  // in: initial centres; out: final centres
  int64_t ldc;
  int* labels;
  double* objective;
  int* near_ties;
  double* cluster_w;
  long long* fsum;         // [3][k2*d + k2] fixed-point sums | weights
  const unsigned* bounds;  // [2] max|x|, max w (km_weights)
  double* pobj;            // [iters][G]
  int* ptie;               // [iters][G]
  int* tie_log;            // near-tie log ([0] count, then 5 ints per entry) or null
  int tie_cap;
  int64_t row_off;         // global index of local point 0 (for the log)
  int cap;                 // points per chunk (multiple of 16, <= kLP): all of the CTA's when resident
  int pitch;               // cap + 1: odd, so a warp reading one point's dimensions is conflict-free
};

struct LloydArgs {
  LloydProb pr[kMaxProb];
  int nprob, iters, resident;
  int g0;           // CTAs of problem 0 (the rest, gridDim.x - g0, run problem 1)
  unsigned* gbar[kMaxProb];  // per-problem grid barriers: monotonic arrival counters (zeroed at launch)
  long long* prof;  // diagnostics (CABS_PROFILE_LLOYD builds): per-phase cycles of the last CTA
};

// dynamic smem per problem: centre pairs [k2p/64][d][2][16][2] | points x [d][pitch] |
// w 2^S (FP64) | llrint(w 2^Sw) | w | dense partial [k2*d + k2] | 1 / cluster weight.
// (X is never re-read from global memory: cluster.sync invalidates L1.)
struct LloydSmem {
  size_t cs, xs, wsc, iw, wts, part, wd, total;
};
__host__ __device__ inline LloydSmem lloyd_smem(int d, int k2, int pitch, size_t base) {
  LloydSmem L;
  size_t o = base;
  auto take = [&](size_t b) { size_t r = o; o += (b + 15) & ~size_t(15); return r; };
  const int d2 = (d + 1) >> 1;  // dimension pairs (an odd d gets a zero dimension)
  L.cs = take(sizeof(float) * round_up(k2, kLC) * 2 * d2);
  L.xs = take(sizeof(float) * (size_t)2 * d2 * pitch);
  L.wsc = take(sizeof(double) * (size_t)pitch);
  L.iw = take(sizeof(long long) * (size_t)pitch);
  L.wts = take(sizeof(float) * (size_t)pitch);
  L.part = take(sizeof(long long) * (((size_t)k2 * d + k2 + 1) & ~size_t(1)));
  L.wd = take(sizeof(double) * (size_t)k2);
  L.total = o;
  return L;
}

// centre j, dimension i -> float index of the pair layout [j/64][i][q][ct][half] with
// jj = j % 64 = 32 q + 16 half + ct: thread ct of the distance loop reads (c_{ct+32q},
// c_{ct+32q+16}), q < 2, as two 8-byte words per dimension.
__device__ __forceinline__ int cpair_idx(int j, int i, int d2) {
  const int jj = j & 63;
  return (((((j >> 6) * d2 + (i >> 1)) * 2 + (jj >> 5)) * 16 + (jj & 15)) * 2 + (i & 1)) * 2 + ((jj >> 4) & 1);
}

__device__ __forceinline__ unsigned long long f2_dup(float x) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ unsigned long long f2_sub(unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__device__ __forceinline__ float f2_lo(unsigned long long v) { return __uint_as_float(static_cast<unsigned>(v)); }
__device__ __forceinline__ float f2_hi(unsigned long long v) { return __uint_as_float(static_cast<unsigned>(v >> 32)); }

// per-problem views of the CTA's shared memory
struct ProbSmem {
  float *cs, *xs, *wts;
  double *wsc, *wd;
  long long *iw, *part;
};
__device__ __forceinline__ ProbSmem prob_smem(unsigned char* dyn, const LloydSmem& L) {
  ProbSmem s;
  s.cs = reinterpret_cast<float*>(dyn + L.cs);
  s.xs = reinterpret_cast<float*>(dyn + L.xs);
  s.wsc = reinterpret_cast<double*>(dyn + L.wsc);
  s.iw = reinterpret_cast<long long*>(dyn + L.iw);
  s.wts = reinterpret_cast<float*>(dyn + L.wts);
  s.part = reinterpret_cast<long long*>(dyn + L.part);
  s.wd = reinterpret_cast<double*>(dyn + L.wd);
  return s;
}

// chunk of np <= cap points -> x [i][pitch], w 2^S, llrint(w 2^Sw), w (zeros beyond)
__device__ __forceinline__ void stage_chunk(const LloydProb& pr, int64_t p0, int np, const ProbSmem& S, double scale,
                                            double scale_w) {
  const int d = pr.d, P = pr.pitch, cap = pr.cap, dd = 2 * ((d + 1) >> 1);
  for (int e = threadIdx.x; e < cap * dd; e += blockDim.x) {
    const int pp = e / dd, i = e - pp * dd;
    S.xs[((i >> 1) * P + pp) * 2 + (i & 1)] = (pp < np && i < d) ? __ldg(pr.X + (p0 + pp) * pr.ldx + i) : 0.f;
  }
  for (int pp = threadIdx.x; pp < cap; pp += blockDim.x) {
    const float w = pp < np ? pr.w[p0 + pp] : 0.f;
    S.wsc[pp] = static_cast<double>(w) * scale;  // exact (power-of-two scale)
    S.iw[pp] = llrint(static_cast<double>(w) * scale_w);
    S.wts[pp] = w;
  }
}

// Exact sums of the chunk (km_fixed.cuh) into the CTA's dense partial: warp w owns the
// clusters j = w mod 8; for each it collects the chunk's points with label j (ballots over
// the labels, held in registers), lanes over dimensions, and keeps the sums in registers --
// one store (ADD when the CTA streams several chunks) per entry, no atomics, no sort.
template <bool ADD>
__device__ __forceinline__ void accumulate_owned(const int* lab, int np, const ProbSmem& S, int P, int d, int k2) {
  constexpr int NB = (kLP + 31) / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nsum = k2 * d;
  long long* __restrict__ part = S.part;
  int labr[NB];
#pragma unroll
  for (int t = 0; t < NB; ++t) labr[t] = lane + 32 * t < np ? lab[lane + 32 * t] : -1;
  for (int j = warp; j < k2; j += kLT / 32) {
    for (int i0 = 0; i0 < d; i0 += 64) {
      const int ia = i0 + lane, ib = i0 + 32 + lane;
      long long sa = 0, sb = 0, sw = 0;
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        unsigned m = __ballot_sync(0xffffffffu, labr[t] == j);
        while (m) {
          const int p = 32 * t + __ffs(m) - 1;
          m &= m - 1;
          const double ws = S.wsc[p];
          if (ia < d) sa += fx_prod_magic(ws, S.xs[((ia >> 1) * P + p) * 2 + (ia & 1)]);
          if (ib < d) sb += fx_prod_magic(ws, S.xs[((ib >> 1) * P + p) * 2 + (ib & 1)]);
          sw += S.iw[p];
        }
      }
      if (ia < d) part[j * d + ia] = ADD ? part[j * d + ia] + sa : sa;
      if (ib < d) part[j * d + ib] = ADD ? part[j * d + ib] + sb : sb;
      if (i0 == 0 && lane == 0) part[nsum + j] = ADD ? part[nsum + j] + sw : sw;
    }
  }
}

// One block of centres jc + 16 v, v < NV (jc = j0 + ct), against the points pt + 16 u: pairs
// (v, v + 1) in one FFMA2 lane pair, an odd last centre in scalar FP32 (the same IEEE ops).
template <int NA, int NV>
__device__ __forceinline__ void dist_block(const float2* __restrict__ xq, int P, const ulonglong2* cq, int d2,
                                           int jc, int k2, float* bd, float* sd, int* bj, int* sj) {
  unsigned long long acc0[NA], acc1[NA];
  float accs[NA];
#pragma unroll
  for (int u = 0; u < NA; ++u) { acc0[u] = 0ull; acc1[u] = 0ull; accs[u] = 0.f; }
  for (int i2 = 0; i2 < d2; ++i2) {  // dimensions 2 i2, 2 i2 + 1: one 8-byte x load, one 16-byte centre load
    const ulonglong2 c0 = cq[i2 * 32];
    const ulonglong2 c1 = NV >= 3 ? cq[i2 * 32 + 16] : make_ulonglong2(0ull, 0ull);
    float2 x2[NA];
#pragma unroll
    for (int u = 0; u < NA; ++u) x2[u] = xq[i2 * P + 16 * u];
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // the sums stay in dimension order
      const unsigned long long cc0 = h ? c0.y : c0.x, cc1 = h ? c1.y : c1.x;
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        const float xv = h ? x2[u].y : x2[u].x;
        if (NV >= 2) {
          const unsigned long long xx = f2_dup(xv);
          const unsigned long long df0 = f2_sub(xx, cc0);
          acc0[u] = f2_fma(df0, df0, acc0[u]);
          if (NV == 4) {
            const unsigned long long df1 = f2_sub(xx, cc1);
            acc1[u] = f2_fma(df1, df1, acc1[u]);
          } else if (NV == 3) {
            const float df = xv - f2_lo(cc1);
            accs[u] = fmaf(df, df, accs[u]);
          }
        } else {
          const float df = xv - f2_lo(cc0);
          accs[u] = fmaf(df, df, accs[u]);
        }
      }
    }
  }
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    const int j = jc + 16 * v;
    if (j >= k2) continue;
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      float val;
      if (NV == 1) val = accs[u];
      else if (v == 0) val = f2_lo(acc0[u]);
      else if (v == 1) val = f2_hi(acc0[u]);
      else if (v == 2) val = NV == 3 ? accs[u] : f2_lo(acc1[u]);
      else val = f2_hi(acc1[u]);
      if (val < bd[u] || (val == bd[u] && j < bj[u])) { sd[u] = bd[u]; sj[u] = bj[u]; bd[u] = val; bj[u] = j; }
      else if (val < sd[u]) { sd[u] = val; sj[u] = j; }
    }
  }
}

// merge (b2, j2, s2, sj2) into the running (best, index, runner-up, index); lowest index on ties
__device__ __forceinline__ void merge_best2(float& bd, int& bj, float& sd, int& sj, float b2, int j2, float s2,
                                            int sj2) {
  if (b2 < bd || (b2 == bd && j2 < bj)) {
    if (bd < s2) { sd = bd; sj = bj; } else { sd = s2; sj = sj2; }
    bd = b2; bj = j2;
  } else {
    if (b2 < sd) { sd = b2; sj = j2; }
    if (s2 < sd) { sd = s2; sj = sj2; }
  }
}

// Distances of the chunk's points pt + 16u (u < NA) to all centres (two per FFMA2; direct
// differences, dimensions ascending), running (best, index, runner-up) per point, merged over
// the two centre lanes of the warp and written to the per-warp slots sb_*[warp][point].
template <int NA>
__device__ __forceinline__ void dist_rows(const float* __restrict__ xs, int P, const float* cs, int d, int k2, int pt,
                                          int ct, int lane, int warp, float (*sb_d)[kLP], int (*sb_j)[kLP],
                                          float (*ss_d)[kLP], int (*ss_j)[kLP]) {
  float bd[NA], sd[NA];
  int bj[NA], sj[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) { bd[q] = FLT_MAX; sd[q] = FLT_MAX; bj[q] = 0x7fffffff; sj[q] = -1; }
  const float2* xq = reinterpret_cast<const float2*>(xs) + pt;
  const int d2 = (d + 1) >> 1;
  for (int j0 = 0; j0 < k2; j0 += kLC) {
    // centres ct + 16 v (v < nv) of the block hold real centres for this warp (its two ct are
    // 2 warp and 2 warp + 1): the padding of the last block costs no arithmetic
    const int rem = k2 - j0 - 2 * warp;
    const int nv = rem <= 0 ? 0 : (rem >= 64 ? 4 : (rem + 15) >> 4);
    const ulonglong2* cq = reinterpret_cast<const ulonglong2*>(cs) + (size_t)(j0 >> 6) * d2 * 32 + ct;
    if (nv == 4) dist_block<NA, 4>(xq, P, cq, d2, j0 + ct, k2, bd, sd, bj, sj);
    else if (nv == 3) dist_block<NA, 3>(xq, P, cq, d2, j0 + ct, k2, bd, sd, bj, sj);
    else if (nv == 2) dist_block<NA, 2>(xq, P, cq, d2, j0 + ct, k2, bd, sd, bj, sj);
    else if (nv == 1) dist_block<NA, 1>(xq, P, cq, d2, j0 + ct, k2, bd, sd, bj, sj);
  }
  // merge the two centre lanes of this warp (lanes l and l ^ 16 hold the same points)
#pragma unroll
  for (int u = 0; u < NA; ++u) {
    const float b2 = __shfl_xor_sync(0xffffffffu, bd[u], 16), s2 = __shfl_xor_sync(0xffffffffu, sd[u], 16);
    const int j2 = __shfl_xor_sync(0xffffffffu, bj[u], 16), sj2 = __shfl_xor_sync(0xffffffffu, sj[u], 16);
    merge_best2(bd[u], bj[u], sd[u], sj[u], b2, j2, s2, sj2);
  }
  if (lane < 16) {
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      sb_d[warp][pt + 16 * u] = bd[u];
      sb_j[warp][pt + 16 * u] = bj[u];
      ss_d[warp][pt + 16 * u] = sd[u];
      ss_j[warp][pt + 16 * u] = sj[u];
    }
  }
}

void lloyd_debug_timeline(long long* out, int n) {
#ifdef CABS_PROFILE_LLOYD
  const int m = n < 320 * 16 ? n : 320 * 16;
  cudaMemcpyFromSymbol(out, g_ll_tl, sizeof(long long) * m);
#else
  for (int i = 0; i < n; ++i) out[i] = 0;
#endif
}

static_assert(kLT == 256, "8 warps: cluster ownership j % 8 and the 16 x 16 distance lanes");
static_assert(kLA == 7, "dist_rows instantiations cover up to 7 rows");
__global__ void __launch_bounds__(kLT, 2) lloyd_persistent_kernel(LloydArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ float sb_d[8][kLP];  // per point: best / runner-up of each warp's two centre lanes
  __shared__ int sb_j[8][kLP];
  __shared__ float ss_d[8][kLP];
  __shared__ int ss_j[8][kLP];
  __shared__ int lab_s[kLP];
  __shared__ double s_red[kMaxProb][kLT / 32];
  __shared__ int s_tie[kMaxProb][kLT / 32];
  __shared__ __align__(8) uint64_t s_mbar;  // the multicast sums of one iteration landed
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = static_cast<int>(cluster.block_rank()), csize = static_cast<int>(cluster.num_blocks());
  const int tid = threadIdx.x, pt = tid & 15, ct = tid >> 4, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, np_ = a.nprob;
  // each CTA runs ONE problem (two CTAs per SM: the problems' latency-bound phases overlap);
  // b / Gb: the CTA's index / count among its problem's CTAs (clusters never mix problems)
  const int myq = (np_ > 1 && static_cast<int>(blockIdx.x) >= a.g0) ? 1 : 0;
  const int b = myq ? static_cast<int>(blockIdx.x) - a.g0 : static_cast<int>(blockIdx.x);
  const int Gb = np_ > 1 ? (myq ? G - a.g0 : a.g0) : G;

  // per problem: smem views, point range, scales, reduction slice
  LloydSmem Ls[kMaxProb];
  int64_t pbeg[kMaxProb], pend[kMaxProb], Eq[kMaxProb], Eqp[kMaxProb], ebeg[kMaxProb], eend[kMaxProb];
  double scale[kMaxProb], scale_w[kMaxProb];
  {
#pragma unroll
    for (int q = 0; q < kMaxProb; ++q) {
      if (q >= np_) break;
      if (q != myq) continue;
      const LloydProb& pr = a.pr[q];
      Ls[q] = lloyd_smem(pr.d, pr.k2, pr.pitch, 0);
      pbeg[q] = (pr.N * b) / Gb;
      pend[q] = (pr.N * (b + 1)) / Gb;
      Eq[q] = (int64_t)pr.k2 * pr.d + pr.k2;
      Eqp[q] = (Eq[q] + 1) & ~int64_t(1);  // slot stride: 16-byte aligned slots for the bulk copies
      ebeg[q] = Eq[q] * crank / csize;
      eend[q] = Eq[q] * (crank + 1) / csize;
      fx_scales(pr.bounds, pr.N, scale[q], scale_w[q]);
    }
  }

  // ---------------- prologue: resident chunks, initial centres (padding centres = 0)
  if (tid == 0) {
    tc::mbar_init(&s_mbar, 1);
    tc::mbar_fence_init();  // visible to the cluster by the first cluster barrier
  }
#pragma unroll
  for (int q = 0; q < kMaxProb; ++q) {
    if (q >= np_) break;
    if (q != myq) continue;
    const LloydProb& pr = a.pr[q];
    const ProbSmem S = prob_smem(dyn, Ls[q]);
    if (a.resident) stage_chunk(pr, pbeg[q], static_cast<int>(pend[q] - pbeg[q]), S, scale[q], scale_w[q]);
    const int k2p = static_cast<int>(round_up(pr.k2, kLC));
    const int dd = 2 * ((pr.d + 1) >> 1);
    for (int e = tid; e < k2p * dd; e += blockDim.x) {  // padding centres and the padding dimension = 0
      const int j = e / dd, i = e - j * dd;
      S.cs[cpair_idx(j, i, dd >> 1)] = (j < pr.k2 && i < pr.d) ? __ldcg(pr.centres + (int64_t)j * pr.ldc + i) : 0.f;
    }
  }

#ifdef CABS_PROFILE_LLOYD
  long long prof[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, t0 = clock64();
  int tl_n = 0;
#define LPROF(i) do { if (blockIdx.x == G - 1 && tid == 0) { long long t1 = clock64(); prof[i] += t1 - t0; t0 = t1; } \
                      if (it == kTlIter && tid == 0 && tl_n < 16) g_ll_tl[blockIdx.x][tl_n++] = globaltimer_ns(); } while (0)
#else
#define LPROF(i) do { } while (0)
#endif
  for (int it = 0; it < a.iters; ++it) {
    LPROF(9);
    if (it > 0) {
      // centres of this iteration from the previous iteration's exact sums, all entries, in
      // every CTA (an empty cluster keeps its centre).  The sums reach every CTA of the
      // cluster by bulk copies multicast from the CTAs' slices (one L2 read per cluster) into
      // the partial buffers (free: read by the cluster before the last grid barrier).
      if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        uint32_t total = 0;
#pragma unroll
        for (int q = 0; q < kMaxProb; ++q)
          if (q == myq) total += static_cast<uint32_t>(Eqp[q] * 8);
        tc::mbar_expect_tx(&s_mbar, total);
#pragma unroll
        for (int q = 0; q < kMaxProb; ++q) {
          if (q >= np_) break;
          if (q != myq) continue;
          const ProbSmem S = prob_smem(dyn, Ls[q]);
          const int64_t n16 = Eqp[q] / 2;  // 16-byte units
          const int64_t c0 = n16 * crank / csize, c1 = n16 * (crank + 1) / csize;
          if (c1 > c0) {
            const long long* src = a.pr[q].fsum + (size_t)((it + 2) % 3) * Eqp[q] + 2 * c0;
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
                "[%0], [%1], %2, [%3], %4;" ::"r"(tc::smem_u32(S.part + 2 * c0)),
                "l"(src), "r"(static_cast<uint32_t>((c1 - c0) * 16)), "r"(tc::smem_u32(&s_mbar)),
                "h"(static_cast<uint16_t>((1u << csize) - 1u))
                : "memory");
          }
        }
      }
      tc::mbar_wait(&s_mbar, static_cast<uint32_t>((it - 1) & 1));
      LPROF(8);
#pragma unroll
      for (int q = 0; q < kMaxProb; ++q) {
        if (q >= np_) break;
        if (q != myq) continue;
        const LloydProb& pr = a.pr[q];
        const ProbSmem S = prob_smem(dyn, Ls[q]);
        const int nsum = pr.k2 * pr.d;
        for (int j = tid; j < pr.k2; j += blockDim.x) {
          const long long wj = S.part[nsum + j];
          S.wd[j] = wj > 0 ? 1.0 / (static_cast<double>(wj) * (1.0 / scale_w[q])) : 0.0;
        }
      }
      __syncthreads();  // wd ready
#pragma unroll
      for (int q = 0; q < kMaxProb; ++q) {
        if (q >= np_) break;
        if (q != myq) continue;
        const LloydProb& pr = a.pr[q];
        const ProbSmem S = prob_smem(dyn, Ls[q]);
        const int d = pr.d;
        const double inv_scale = 1.0 / scale[q];
        // thread (j mod 64, i group): lanes over centres, so the stores into the pair layout
        // are conflict-free; no division per entry
        for (int j = tid & 63; j < pr.k2; j += 64) {
          const double rw = S.wd[j];
          if (rw > 0) {
#pragma unroll 4
            for (int i = tid >> 6; i < d; i += kLT / 64)
              S.cs[cpair_idx(j, i, (d + 1) >> 1)] =
                  static_cast<float>((static_cast<double>(S.part[j * d + i]) * inv_scale) * rw);
          }
        }
        // zero this CTA's share of the slot the next iteration accumulates into (last read
        // before the previous grid barrier)
        long long* fs_next = pr.fsum + (size_t)((it + 1) % 3) * Eqp[q];
        for (int64_t e = (int64_t)b * blockDim.x + tid; e < Eq[q]; e += (int64_t)Gb * blockDim.x) fs_next[e] = 0;
      }
      __syncthreads();  // staged sums consumed: the partial buffers are free
    }
    if (!a.resident) {
#pragma unroll
      for (int q = 0; q < kMaxProb; ++q) {  // the partials the streamed chunks add into
        if (q >= np_) break;
        if (q != myq) continue;
        const ProbSmem S = prob_smem(dyn, Ls[q]);
        for (int64_t e = tid; e < Eq[q]; e += blockDim.x) S.part[e] = 0;
      }
    }
    __syncthreads();
    LPROF(0);
#pragma unroll
    for (int q = 0; q < kMaxProb; ++q) {
      if (q >= np_) break;
      if (q != myq) continue;
      const LloydProb& pr = a.pr[q];
      const ProbSmem S = prob_smem(dyn, Ls[q]);
      const int d = pr.d, k2 = pr.k2;
      double obj = 0.0;
      int ties = 0;
      for (int64_t p0 = pbeg[q]; p0 < pend[q]; p0 += pr.cap) {
        const int np = static_cast<int>(pend[q] - p0 < pr.cap ? pend[q] - p0 : pr.cap);
        if (!a.resident) {
          __syncthreads();  // previous chunk fully consumed
          stage_chunk(pr, p0, np, S, scale[q], scale_w[q]);
          __syncthreads();
        }
        // distances: rows u < ceil(np / 16)
        {
          const int na = (np + 15) >> 4;
          if (na <= 3) dist_rows<3>(S.xs, pr.pitch, S.cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d, ss_j);
          else if (na <= 5) dist_rows<5>(S.xs, pr.pitch, S.cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d, ss_j);
          else dist_rows<7>(S.xs, pr.pitch, S.cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d, ss_j);
        }
        __syncthreads();
        for (int p = tid; p < np; p += kLT) {  // merge the 8 warps (lowest index on ties)
          float B = sb_d[0][p], Sd = ss_d[0][p];
          int Bj = sb_j[0][p], Sj = ss_j[0][p];
          for (int t = 1; t < kLT / 32; ++t) merge_best2(B, Bj, Sd, Sj, sb_d[t][p], sb_j[t][p], ss_d[t][p], ss_j[t][p]);
          lab_s[p] = Bj;
          pr.labels[p0 + p] = Bj;
          obj += static_cast<double>(S.wts[p]) * static_cast<double>(B);
          const bool tie = (Sd - B) < kNearTie * Sd;
          ties += tie;
          if (tie && pr.tie_log) km_log_tie(pr.tie_log, pr.tie_cap, it, pr.row_off + p0 + p, Bj, Sj, B, Sd);
        }
        __syncthreads();
        LPROF(1);
        if (a.resident) {
          accumulate_owned<false>(lab_s, np, S, pr.pitch, d, k2);
        } else {
          accumulate_owned<true>(lab_s, np, S, pr.pitch, d, k2);
          __syncthreads();  // lab_s and the chunk are reused
        }
        LPROF(2);
      }
      obj = warp_sum_d(obj);
      int tt = ties;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, o);
      if (lane == 0) { s_red[q][warp] = obj; s_tie[q][warp] = tt; }
    }
    // cluster reduction of the dense partials (DSMEM), one global integer add per entry
    cluster.sync();
    LPROF(5);
#pragma unroll
    for (int q = 0; q < kMaxProb; ++q) {
      if (q >= np_) break;
      if (q != myq) continue;
      const ProbSmem S = prob_smem(dyn, Ls[q]);
      long long* fs_cur = a.pr[q].fsum + (size_t)(it % 3) * Eqp[q];
      const long long* rp[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) rp[r] = r < csize ? cluster.map_shared_rank(S.part, r) : S.part;
      for (int64_t e = ebeg[q] + tid; e < eend[q]; e += blockDim.x) {
        long long v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = r < csize ? rp[r][e] : 0;
        long long s = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) s += v[r];
        if (s != 0) red_add_u64(fs_cur + e, s);
      }
    }
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < kMaxProb; ++q) {
        if (q >= np_) break;
        if (q != myq) continue;
        double sacc = 0;
        int qq = 0;
        for (int w = 0; w < kLT / 32; ++w) { sacc += s_red[q][w]; qq += s_tie[q][w]; }
        a.pr[q].pobj[(size_t)it * Gb + b] = sacc;
        a.pr[q].ptie[(size_t)it * Gb + b] = qq;
      }
    }
    // the partial buffers are overwritten next by the async proxy (the multicast sums)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    LPROF(6);
    // grid barrier: monotonic arrival counter.  The partials are re-zeroed only after it (no
    // CTA still reads them), and the slots rotate, so nothing else needs a barrier.
    __syncthreads();
    LPROF(7);
    if (tid == 0) {
      __threadfence();
      // one counter per problem: the two problems never wait for each other, so the two CTAs
      // of an SM drift out of phase and overlap their latency-bound phases
      unsigned* bar = a.gbar[myq];
      atomicAdd(bar, 1u);
      const unsigned target = static_cast<unsigned>(Gb) * static_cast<unsigned>(it + 1);
      while (ld_acquire_gpu(bar) < target) __nanosleep(20);
    }
    __syncthreads();
    LPROF(3);
  }
#ifdef CABS_PROFILE_LLOYD
  if (blockIdx.x == G - 1 && tid == 0)
    for (int i = 0; i < 10; ++i) a.prof[i] = prof[i];
#endif
  // ---------------- epilogue (CTA 0): final centres, cluster weights, objective history
  if (b == 0) {
#pragma unroll
    for (int q = 0; q < kMaxProb; ++q) {
      if (q >= np_) break;
      if (q != myq) continue;
      const LloydProb& pr = a.pr[q];
      const ProbSmem S = prob_smem(dyn, Ls[q]);
      const int d = pr.d, k2 = pr.k2, nsum = k2 * d;
      const double inv_scale = 1.0 / scale[q], inv_scale_w = 1.0 / scale_w[q];
      const long long* fs_last = pr.fsum + (size_t)((a.iters - 1) % 3) * Eqp[q];
      for (int e = tid; e < nsum; e += blockDim.x) {
        const int j = e / d, i = e - j * d;
        const long long wj = __ldcg(fs_last + nsum + j);
        pr.centres[(int64_t)j * pr.ldc + i] =
            wj > 0 ? static_cast<float>((static_cast<double>(__ldcg(fs_last + e)) * inv_scale) *
                                        (1.0 / (static_cast<double>(wj) * inv_scale_w)))
                   : S.cs[cpair_idx(j, i, (d + 1) >> 1)];
      }
      for (int j = tid; j < k2; j += blockDim.x)
        pr.cluster_w[j] = static_cast<double>(__ldcg(fs_last + nsum + j)) / scale_w[q];
      for (int it = tid; it < a.iters; it += blockDim.x) {
        double s = 0;
        long long qq = 0;
        for (int g = 0; g < Gb; ++g) {
          s += __ldcg(pr.pobj + (size_t)it * Gb + g);
          qq += __ldcg(pr.ptie + (size_t)it * Gb + g);
        }
        pr.objective[it] = s;
        if (pr.near_ties) pr.near_ties[it] = static_cast<int>(qq);
      }
    }
  }
}

// Returns false when the fast path does not apply (caller uses the per-iteration kernels).
bool launch_lloyd_persistent(const LloydJob* jobs, int njobs, int iters, long long* prof, cudaStream_t st) {
  if (njobs < 1 || njobs > kMaxProb) return false;
  for (int q = 0; q < njobs; ++q)
    if (jobs[q].k2 > CABS_KMAX) return false;
  for (int q = 0; q < njobs; ++q)
    if (jobs[q].N <= 0) return false;
  constexpr size_t kSmemCap = 200 * 1024;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(lloyd_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kSmemCap)) != cudaSuccess)
      return false;
    attr = true;
  }
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  // grid: two CTAs per SM when they fit (else one), each running ONE problem -- the problems
  // get CTAs in proportion to their points (whole clusters each) -- and the largest cluster
  // size (8, 4, 2, 1) whose clusters can all be resident
  LloydArgs a{};
  a.nprob = njobs;
  a.iters = iters;
  a.prof = prof;
  int cap[kMaxProb] = {kLP, kLP};
  int resident = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kLT);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  int csize = 0;
  int64_t G = 0, Gq[kMaxProb] = {0, 0};
  size_t smem = 0;
  const double Ntot = static_cast<double>(jobs[0].N) + (njobs > 1 ? static_cast<double>(jobs[1].N) : 0.0);
  const int per_sm0 = getenv("CABS_LLOYD_ONE_PER_SM") ? 1 : 2;
  for (int per_sm = per_sm0; per_sm >= 1 && csize == 0; --per_sm) {
    const int cmax = getenv("CABS_LLOYD_MAX_CLUSTER") ? atoi(getenv("CABS_LLOYD_MAX_CLUSTER")) : 8;
    for (int c = 8; c >= 1 && csize == 0; c >>= 1) {
      if (c > cmax) continue;
      const int64_t tot = (int64_t)nsm * per_sm / c * c;
      if (tot < c * njobs) continue;
      int64_t g[kMaxProb] = {tot, 0};
      if (njobs > 1) {
        g[0] = (int64_t)llround(static_cast<double>(tot) * static_cast<double>(jobs[0].N) / Ntot / c) * c;
        g[0] = g[0] < c ? c : (g[0] > tot - c ? tot - c : g[0]);
        g[1] = tot - g[0];
      }
      bool ok = true;
      int r = 1, cp[kMaxProb] = {kLP, kLP};
      size_t sm = 0;
      for (int q = 0; q < njobs; ++q) {
        if (g[q] > jobs[q].N) ok = false;
        const int64_t per = ceil_div(jobs[q].N, g[q] > 0 ? g[q] : 1);
        cp[q] = per <= kLP ? static_cast<int>(round_up(per, 16)) : kLP;
        if (per > kLP) r = 0;
        const size_t t = lloyd_smem(jobs[q].d, jobs[q].k2, cp[q] + 1, 0).total;
        sm = t > sm ? t : sm;
      }
      if (!ok || sm > kSmemCap) continue;
      at[0].val.clusterDim.x = static_cast<unsigned>(c);
      cfg.gridDim = dim3(static_cast<unsigned>(tot));
      cfg.dynamicSmemBytes = sm;
      int ncl = 0;
      if (cudaOccupancyMaxActiveClusters(&ncl, lloyd_persistent_kernel, &cfg) == cudaSuccess &&
          (int64_t)ncl * c >= tot) {
        csize = c;
        G = tot;
        Gq[0] = g[0];
        Gq[1] = g[1];
        smem = sm;
        resident = r;
        cap[0] = cp[0];
        cap[1] = cp[1];
      }
    }
  }
  cudaGetLastError();
  if (csize == 0) return false;
  cfg.gridDim = dim3(static_cast<unsigned>(G));
  cfg.dynamicSmemBytes = smem;
  at[0].val.clusterDim.x = static_cast<unsigned>(csize);
  a.resident = resident;
  a.g0 = static_cast<int>(Gq[0]);
  // scratch of each job: fsum [3][k2*d + k2] | pobj [iters][G] | ptie [iters][G]; barrier in job 0's
  for (int q = 0; q < njobs; ++q) {
    const LloydJob& j = jobs[q];
    const size_t E = ((size_t)j.k2 * j.d + j.k2 + 1) & ~size_t(1);  // slot stride (16-byte aligned)
    const size_t need = sizeof(long long) * 3 * E + 16 + (sizeof(double) + sizeof(int)) * iters * G;
    if (need > j.scratch_bytes) return false;
    char* base = static_cast<char*>(j.scratch);
    LloydProb& p = a.pr[q];
    p.X = j.X; p.ldx = j.ldx; p.N = j.N; p.d = j.d; p.k2 = j.k2; p.w = j.w;
    p.centres = j.centres; p.ldc = j.ldc; p.labels = j.labels; p.objective = j.objective;
    p.near_ties = j.near_ties; p.cluster_w = j.cluster_w; p.bounds = j.bounds; p.cap = cap[q];
    p.tie_log = j.tie_log; p.tie_cap = j.tie_cap; p.row_off = j.row_off;
    p.pitch = cap[q] + 1;
    p.fsum = reinterpret_cast<long long*>(base);
    unsigned* gb = reinterpret_cast<unsigned*>(p.fsum + 3 * E);
    a.gbar[q] = gb;
    p.pobj = reinterpret_cast<double*>(gb + 4);
    p.ptie = reinterpret_cast<int*>(p.pobj + (size_t)iters * G);
    if (cudaMemsetAsync(base, 0, sizeof(long long) * 3 * E + 16, st) != cudaSuccess) return false;
  }
  note_launch();
  return cudaLaunchKernelEx(&cfg, lloyd_persistent_kernel, a) == cudaSuccess;
}

}  // namespace cabsk
