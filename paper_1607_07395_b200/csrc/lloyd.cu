// lloyd.cu -- the whole Lloyd loop of one or two k-means problems (the row side and the
// column side of CABS, Alg. 2 steps 6-7) in ONE persistent kernel (single GPU):
// c iterations x {centres | assign | accumulate | cluster reduce | grid sync}, no host round
// trips, no per-iteration launches, ONE grid-wide barrier per iteration for both problems.
// Every CTA (one per SM) holds a balanced contiguous slice of the points of EACH problem, so
// the two problems share the synchronisation latency instead of paying it twice.
//
// Arithmetic (Eq. 6; c iterations P:204):
//  * distances by direct differences in FP32, dimensions ascending (= km_tile.cuh), lowest
//    centre index on ties; two centres per packed FP32x2 instruction (FADD2/FFMA2: the same
//    IEEE rounding as the scalar ops, half the instructions);
//  * sums w_l X_l and w_l accumulated EXACTLY as int64 fixed point (km_fixed.cuh): a dense
//    int64 partial per CTA in shared memory, the CTAs of a thread-block cluster add their
//    partials through distributed shared memory (each CTA one slice), and one
//    red.global.add.u64 per (cluster, entry) lands in the global sums -- order-free, so
//    deterministic and identical to the per-iteration kernels of kmeans.cu;
//  * centres = (sum / 2^S) * (1 / (weight / 2^Sw)) in FP64; an empty cluster keeps its
//    centre (Z12).
// Global sums rotate over three slots: slot it%3 accumulates, slot (it-1)%3 is read by
// every CTA to form this iteration's centres, slot (it+1)%3 is zeroed for the next one.
#include <cooperative_groups.h>
#include <float.h>
#include <limits.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"
#include "km_fixed.cuh"
#include "km_tile.cuh"

namespace cg = cooperative_groups;

namespace cabsk {

constexpr int kLT = 256;       // threads per CTA (one CTA per SM)
constexpr int kLA = 9;         // max point rows per thread
constexpr int kLP = 16 * kLA;  // max points per chunk: thread (pt = tid & 15, ct = tid >> 4) owns points pt + 16u
constexpr int kLC = 64;        // centres per block: ... and centres j0 + ct + 16v, v < 4
constexpr int kMaxProb = 2;

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
  int pitch;               // resident chunk pitch (points, multiple of 16), or kLP when streaming
};

struct LloydArgs {
  LloydProb pr[kMaxProb];
  int nprob, iters, resident;
  unsigned* gbar;   // [2] grid barrier {arrivals, generation}
  long long* prof;  // diagnostics (CABS_PROFILE_LLOYD builds): per-phase cycles of the last CTA
};

// dynamic smem per problem: centre pairs [k2p/64][d][2][16][2] | points x [d][pitch] |
// rows [pitch][d] | w 2^S (FP64) | llrint(w 2^Sw) | w | dense partial [k2*d + k2] |
// 1 / cluster weight.  (X is never re-read from global memory: cluster.sync invalidates L1.)
struct LloydSmem {
  size_t cs, xs, xr, wsc, iw, wts, part, wd, total;
};
__host__ __device__ inline LloydSmem lloyd_smem(int d, int k2, int pitch, size_t base) {
  LloydSmem L;
  size_t o = base;
  auto take = [&](size_t b) { size_t r = o; o += (b + 15) & ~size_t(15); return r; };
  L.cs = take(sizeof(float) * round_up(k2, kLC) * d);
  L.xs = take(sizeof(float) * (size_t)d * pitch);
  L.xr = take(sizeof(float) * (size_t)d * pitch);
  L.wsc = take(sizeof(double) * (size_t)pitch);
  L.iw = take(sizeof(long long) * (size_t)pitch);
  L.wts = take(sizeof(float) * (size_t)pitch);
  L.part = take(sizeof(long long) * ((size_t)k2 * d + k2));
  L.wd = take(sizeof(double) * (size_t)k2);
  L.total = o;
  return L;
}

// centre j, dimension i -> float index of the pair layout [j/64][i][q][ct][half] with
// jj = j % 64 = 32 q + 16 half + ct: thread ct of the distance loop reads (c_{ct+32q},
// c_{ct+32q+16}), q < 2, as two 8-byte words per dimension.
__device__ __forceinline__ int cpair_idx(int j, int i, int d) {
  const int jj = j & 63;
  return ((((j >> 6) * d + i) * 2 + (jj >> 5)) * 16 + (jj & 15)) * 2 + ((jj >> 4) & 1);
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
  float *cs, *xs, *xr, *wts;
  double *wsc, *wd;
  long long *iw, *part;
};
__device__ __forceinline__ ProbSmem prob_smem(unsigned char* dyn, const LloydSmem& L) {
  ProbSmem s;
  s.cs = reinterpret_cast<float*>(dyn + L.cs);
  s.xs = reinterpret_cast<float*>(dyn + L.xs);
  s.xr = reinterpret_cast<float*>(dyn + L.xr);
  s.wsc = reinterpret_cast<double*>(dyn + L.wsc);
  s.iw = reinterpret_cast<long long*>(dyn + L.iw);
  s.wts = reinterpret_cast<float*>(dyn + L.wts);
  s.part = reinterpret_cast<long long*>(dyn + L.part);
  s.wd = reinterpret_cast<double*>(dyn + L.wd);
  return s;
}

// chunk of np <= pitch points -> x [i][pitch], rows [p][d], w 2^S, llrint(w 2^Sw), w (zeros beyond)
__device__ __forceinline__ void stage_chunk(const LloydProb& pr, int64_t p0, int np, const ProbSmem& S, double scale,
                                            double scale_w) {
  const int d = pr.d, P = pr.pitch;
  for (int e = threadIdx.x; e < P * d; e += blockDim.x) {
    const int pp = e / d, i = e - pp * d;
    const float x = pp < np ? __ldg(pr.X + (p0 + pp) * pr.ldx + i) : 0.f;
    S.xs[i * P + pp] = x;
    S.xr[e] = x;
  }
  for (int pp = threadIdx.x; pp < P; pp += blockDim.x) {
    const float w = pp < np ? pr.w[p0 + pp] : 0.f;
    S.wsc[pp] = static_cast<double>(w) * scale;  // exact (power-of-two scale)
    S.iw[pp] = llrint(static_cast<double>(w) * scale_w);
    S.wts[pp] = w;
  }
}

// Distances of the chunk's points pt + 16u (u < NA) to all centres (two per FFMA2; direct
// differences, dimensions ascending), running (best, index, runner-up) per point, merged over
// the two centre lanes of the warp and written to the per-warp slots sb_*[warp][point].
template <int NA>
__device__ __forceinline__ void dist_rows(const float* __restrict__ xs, int P, const float* cs, int d, int k2, int pt,
                                          int ct, int lane, int warp, float (*sb_d)[kLP], int (*sb_j)[kLP],
                                          float (*ss_d)[kLP]) {
  float bd[NA], sd[NA];
  int bj[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) { bd[q] = FLT_MAX; sd[q] = FLT_MAX; bj[q] = 0x7fffffff; }
  const float* xq = xs + pt;
  for (int j0 = 0; j0 < k2; j0 += kLC) {
    unsigned long long acc[2][NA] = {};
    const unsigned long long* cq = reinterpret_cast<const unsigned long long*>(cs) + (size_t)(j0 >> 6) * d * 32 + ct;
    for (int i = 0; i < d; ++i) {
      const unsigned long long c0 = cq[i * 32], c1 = cq[i * 32 + 16];
      float x[NA];
#pragma unroll
      for (int u = 0; u < NA; ++u) x[u] = xq[i * P + 16 * u];
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        const unsigned long long xx = f2_dup(x[u]);
        const unsigned long long df0 = f2_sub(xx, c0), df1 = f2_sub(xx, c1);
        acc[0][u] = f2_fma(df0, df0, acc[0][u]);
        acc[1][u] = f2_fma(df1, df1, acc[1][u]);
      }
    }
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = j0 + ct + 16 * v;
      if (j >= k2) continue;
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        const float val = (v & 1) ? f2_hi(acc[v >> 1][u]) : f2_lo(acc[v >> 1][u]);
        if (val < bd[u] || (val == bd[u] && j < bj[u])) { sd[u] = bd[u]; bd[u] = val; bj[u] = j; }
        else sd[u] = fminf(sd[u], val);
      }
    }
  }
  // merge the two centre lanes of this warp (lanes l and l ^ 16 hold the same points)
#pragma unroll
  for (int u = 0; u < NA; ++u) {
    const float b2 = __shfl_xor_sync(0xffffffffu, bd[u], 16), s2 = __shfl_xor_sync(0xffffffffu, sd[u], 16);
    const int j2 = __shfl_xor_sync(0xffffffffu, bj[u], 16);
    if (b2 < bd[u] || (b2 == bd[u] && j2 < bj[u])) { sd[u] = fminf(fminf(sd[u], s2), bd[u]); bd[u] = b2; bj[u] = j2; }
    else sd[u] = fminf(fminf(sd[u], s2), b2);
  }
  if (lane < 16) {
#pragma unroll
    for (int u = 0; u < NA; ++u) {
      sb_d[warp][pt + 16 * u] = bd[u];
      sb_j[warp][pt + 16 * u] = bj[u];
      ss_d[warp][pt + 16 * u] = sd[u];
    }
  }
}

static_assert(kLT == 256, "8 warps: cluster ownership j % 8 and the 16 x 16 distance lanes");
__global__ void __launch_bounds__(kLT, 1) lloyd_persistent_kernel(LloydArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ float sb_d[8][kLP];  // per point: best / runner-up of each warp's two centre lanes
  __shared__ int sb_j[8][kLP];
  __shared__ float ss_d[8][kLP];
  __shared__ int lab_s[kLP], order_s[kLP], slab_s[kLP];
  __shared__ int hist_s[CABS_KMAX];
  __shared__ int wstart_s[kLT / 32 + 1];
  __shared__ double s_red[kMaxProb][kLT / 32];
  __shared__ int s_tie[kMaxProb][kLT / 32];
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = static_cast<int>(cluster.block_rank()), csize = static_cast<int>(cluster.num_blocks());
  unsigned gen = 0;  // grid-barrier generation
  const int tid = threadIdx.x, pt = tid & 15, ct = tid >> 4, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, b = blockIdx.x, np_ = a.nprob;

  // per problem: smem views, point range, scales, reduction slice
  LloydSmem Ls[kMaxProb];
  int64_t pbeg[kMaxProb], pend[kMaxProb], Eq[kMaxProb], ebeg[kMaxProb], eend[kMaxProb];
  double scale[kMaxProb], scale_w[kMaxProb];
  {
    size_t off = 0;
#pragma unroll
    for (int q = 0; q < kMaxProb; ++q) {
      if (q >= np_) break;
      const LloydProb& pr = a.pr[q];
      Ls[q] = lloyd_smem(pr.d, pr.k2, pr.pitch, off);
      off = Ls[q].total;
      pbeg[q] = (pr.N * b) / G;
      pend[q] = (pr.N * (b + 1)) / G;
      Eq[q] = (int64_t)pr.k2 * pr.d + pr.k2;
      ebeg[q] = Eq[q] * crank / csize;
      eend[q] = Eq[q] * (crank + 1) / csize;
      fx_scales(pr.bounds, pr.N, scale[q], scale_w[q]);
    }
  }

  // ---------------- prologue: resident chunks, initial centres (padding centres = 0)
#pragma unroll
  for (int q = 0; q < kMaxProb; ++q) {
    if (q >= np_) break;
    const LloydProb& pr = a.pr[q];
    const ProbSmem S = prob_smem(dyn, Ls[q]);
    if (a.resident) stage_chunk(pr, pbeg[q], static_cast<int>(pend[q] - pbeg[q]), S, scale[q], scale_w[q]);
    const int k2p = static_cast<int>(round_up(pr.k2, kLC));
    for (int e = tid; e < k2p * pr.d; e += blockDim.x) {
      const int j = e / pr.d, i = e - j * pr.d;
      S.cs[cpair_idx(j, i, pr.d)] = j < pr.k2 ? __ldcg(pr.centres + (int64_t)j * pr.ldc + i) : 0.f;
    }
  }

#ifdef CABS_PROFILE_LLOYD
  long long prof[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, t0 = clock64();
#define LPROF(i) do { if (b == G - 1 && tid == 0) { long long t1 = clock64(); prof[i] += t1 - t0; t0 = t1; } } while (0)
#else
#define LPROF(i) do { } while (0)
#endif
  for (int it = 0; it < a.iters; ++it) {
    if (it > 0) {
      // centres of this iteration from the previous iteration's exact sums (empty cluster: keep).
      // Each CTA forms the centres of ITS slice of the entries (the slice it reduced) and stores
      // them into the centre arrays of all CTAs of its cluster (DSMEM); one cluster barrier.
#pragma unroll
      for (int q = 0; q < kMaxProb; ++q) {
        if (q >= np_) break;
        const LloydProb& pr = a.pr[q];
        const ProbSmem S = prob_smem(dyn, Ls[q]);
        const int64_t nsum = (int64_t)pr.k2 * pr.d;
        const long long* fs_prev = pr.fsum + (size_t)((it + 2) % 3) * Eq[q];
        for (int j = tid; j < pr.k2; j += blockDim.x) {
          const long long wj = __ldcg(fs_prev + nsum + j);
          S.wd[j] = wj > 0 ? 1.0 / (static_cast<double>(wj) * (1.0 / scale_w[q])) : 0.0;
        }
      }
      constexpr int U = 4;  // slice entries per thread per problem (c2: ~2.5)
      long long sv[kMaxProb][U];
#pragma unroll
      for (int q = 0; q < kMaxProb; ++q) {
        if (q >= np_) break;
        const LloydProb& pr = a.pr[q];
        const int64_t nsum = (int64_t)pr.k2 * pr.d;
        const long long* fs_prev = pr.fsum + (size_t)((it + 2) % 3) * Eq[q];
        const int64_t se = eend[q] < nsum ? eend[q] : nsum;
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int64_t e = ebeg[q] + tid + (int64_t)u * kLT;
          sv[q][u] = e < se ? __ldcg(fs_prev + e) : 0;
        }
      }
      __syncthreads();  // wd ready
#pragma unroll
      for (int q = 0; q < kMaxProb; ++q) {
        if (q >= np_) break;
        const LloydProb& pr = a.pr[q];
        const ProbSmem S = prob_smem(dyn, Ls[q]);
        const int d = pr.d;
        const int64_t nsum = (int64_t)pr.k2 * d;
        const double inv_scale = 1.0 / scale[q];
        const long long* fs_prev = pr.fsum + (size_t)((it + 2) % 3) * Eq[q];
        const int64_t se = eend[q] < nsum ? eend[q] : nsum;
        float* rcs[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) rcs[r] = r < csize ? cluster.map_shared_rank(S.cs, r) : S.cs;
        for (int64_t e0 = ebeg[q] + tid, u0 = 0; e0 < se; e0 += (int64_t)U * kLT, u0 += U) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int64_t e = e0 + (int64_t)u * kLT;
            if (e >= se) break;
            const long long v = u0 == 0 ? sv[q][u] : __ldcg(fs_prev + e);
            const int j = static_cast<int>(e / d), i = static_cast<int>(e - (int64_t)j * d);
            const double rw = S.wd[j];
            if (rw > 0) {
              const float c = static_cast<float>((static_cast<double>(v) * inv_scale) * rw);
              const int ci = cpair_idx(j, i, d);
#pragma unroll
              for (int r = 0; r < 8; ++r)
                if (r < csize) rcs[r][ci] = c;
            }
          }
        }
        // zero the slot the next iteration accumulates into (last read before the previous barrier)
        long long* fs_next = pr.fsum + (size_t)((it + 1) % 3) * Eq[q];
        for (int64_t e = (int64_t)b * blockDim.x + tid; e < Eq[q]; e += (int64_t)G * blockDim.x) fs_next[e] = 0;
      }
    }
#pragma unroll
    for (int q = 0; q < kMaxProb; ++q) {
      if (q >= np_) break;
      const ProbSmem S = prob_smem(dyn, Ls[q]);
      for (int64_t e = tid; e < Eq[q]; e += blockDim.x) S.part[e] = 0;
    }
    if (it > 0) cluster.sync();  // every CTA of the cluster has stored its slice of the centres
    else __syncthreads();
    LPROF(0);
#pragma unroll
    for (int q = 0; q < kMaxProb; ++q) {
      if (q >= np_) break;
      const LloydProb& pr = a.pr[q];
      const ProbSmem S = prob_smem(dyn, Ls[q]);
      const int d = pr.d, k2 = pr.k2;
      const int64_t nsum = (int64_t)k2 * d;
      double obj = 0.0;
      int ties = 0;
      for (int64_t p0 = pbeg[q]; p0 < pend[q]; p0 += pr.pitch) {
        const int np = static_cast<int>(pend[q] - p0 < pr.pitch ? pend[q] - p0 : pr.pitch);
        if (!a.resident) {
          __syncthreads();  // previous chunk fully consumed
          stage_chunk(pr, p0, np, S, scale[q], scale_w[q]);
          __syncthreads();
        }
        // distances: rows u < ceil(np / 16)
        {
          const int na = (np + 15) >> 4;
          if (na <= 3) dist_rows<3>(S.xs, pr.pitch, S.cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d);
          else if (na <= 5) dist_rows<5>(S.xs, pr.pitch, S.cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d);
          else if (na <= 7) dist_rows<7>(S.xs, pr.pitch, S.cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d);
          else dist_rows<9>(S.xs, pr.pitch, S.cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d);
        }
        __syncthreads();
        for (int p = tid; p < np; p += kLT) {  // merge the 8 warps (lowest index on ties)
          float B = sb_d[0][p], Sd = ss_d[0][p];
          int Bj = sb_j[0][p];
          for (int t = 1; t < kLT / 32; ++t) {
            const float b2 = sb_d[t][p], s2 = ss_d[t][p];
            const int j2 = sb_j[t][p];
            if (b2 < B || (b2 == B && j2 < Bj)) { Sd = fminf(fminf(Sd, s2), B); B = b2; Bj = j2; }
            else Sd = fminf(fminf(Sd, s2), b2);
          }
          lab_s[p] = Bj;
          pr.labels[p0 + p] = Bj;
          obj += static_cast<double>(S.wts[p]) * static_cast<double>(B);
          ties += (Sd - B) < kNearTie * Sd;
        }
        __syncthreads();
        LPROF(1);
        // exact sums (km_fixed.cuh).  Counting sort of the chunk's points by label (the order
        // inside a label is irrelevant: integer sums), then warp w takes a contiguous range of
        // the sorted points aligned to label-run starts (every cluster belongs to ONE warp) and
        // keeps the running sums of the current run in registers, lanes over dimensions:
        // no read-modify-write chains, one flush per run.
        {
          for (int j = tid; j < k2; j += kLT) hist_s[j] = 0;
          __syncthreads();
          for (int p = tid; p < np; p += kLT) atomicAdd(&hist_s[lab_s[p]], 1);
          __syncthreads();
          if (warp == 0) {  // exclusive scan of the k2 counts: lane owns a contiguous block
            const int per = (k2 + 31) >> 5;
            const int b0 = lane * per, b1 = b0 + per < k2 ? b0 + per : k2;
            int sl = 0;
            for (int j = b0; j < b1; ++j) sl += hist_s[j];
            int inc = sl;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int t = __shfl_up_sync(0xffffffffu, inc, o);
              if (lane >= o) inc += t;
            }
            int run = inc - sl;
            for (int j = b0; j < b1; ++j) {
              const int c = hist_s[j];
              hist_s[j] = run;
              run += c;
            }
          }
          __syncthreads();
          for (int p = tid; p < np; p += kLT) {
            const int l = lab_s[p];
            const int pos = atomicAdd(&hist_s[l], 1);
            order_s[pos] = p;
            slab_s[pos] = l;
          }
          __syncthreads();
          if (tid <= kLT / 32) {
            int q = (tid * np) / (kLT / 32);
            if (tid < kLT / 32) {
              while (q > 0 && q < np && slab_s[q] == slab_s[q - 1]) ++q;
            } else {
              q = np;
            }
            wstart_s[tid] = q;
          }
          __syncthreads();
          const int qb = wstart_s[warp], qe = wstart_s[warp + 1];
          long long* __restrict__ pp = S.part;
          const float* __restrict__ xr = S.xr;
          if (qb < qe) {
            for (int i0 = 0; i0 < d; i0 += 64) {
              const int ia = i0 + lane, ib = i0 + 32 + lane;
              const bool wl = i0 == 0 && lane == 0;
              long long sa = 0, sbv = 0, sw = 0;
              int jc = slab_s[qb];
#pragma unroll 4
              for (int q = qb; q < qe; ++q) {
                const int j = slab_s[q];
                if (j != jc) {  // run of cluster jc ends: flush (this warp owns jc)
                  if (ia < d) pp[(int64_t)jc * d + ia] += sa;
                  if (ib < d) pp[(int64_t)jc * d + ib] += sbv;
                  if (wl) pp[nsum + jc] += sw;
                  sa = 0; sbv = 0; sw = 0;
                  jc = j;
                }
                const int p = order_s[q];
                const double ws = S.wsc[p];
                const float* xrow = xr + p * d;
                if (ia < d) sa += fx_prod_magic(ws, xrow[ia]);
                if (ib < d) sbv += fx_prod_magic(ws, xrow[ib]);
                if (wl) sw += S.iw[p];
              }
              if (ia < d) pp[(int64_t)jc * d + ia] += sa;
              if (ib < d) pp[(int64_t)jc * d + ib] += sbv;
              if (wl) pp[nsum + jc] += sw;
            }
          }
        }
        __syncthreads();
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
      const ProbSmem S = prob_smem(dyn, Ls[q]);
      long long* fs_cur = a.pr[q].fsum + (size_t)(it % 3) * Eq[q];
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
    LPROF(6);
    if (tid == 0) {
#pragma unroll
      for (int q = 0; q < kMaxProb; ++q) {
        if (q >= np_) break;
        double sacc = 0;
        int qq = 0;
        for (int w = 0; w < kLT / 32; ++w) { sacc += s_red[q][w]; qq += s_tie[q][w]; }
        a.pr[q].pobj[(size_t)it * G + b] = sacc;
        a.pr[q].ptie[(size_t)it * G + b] = qq;
      }
    }
    __threadfence();
    LPROF(7);
    cluster.sync();  // partials free again; this cluster's global adds issued and fenced
    LPROF(8);
    // grid barrier between cluster leaders only, then the cluster barrier releases the members
    if (crank == 0 && tid == 0) {
      unsigned* bar = a.gbar;
      const unsigned nb = static_cast<unsigned>(G / csize);
      if (atomicAdd(bar, 1u) == nb - 1) {
        atomicExch(bar, 0u);
        __threadfence();
        atomicExch(bar + 1, gen + 1);
      } else {
        while (ld_acquire_gpu(bar + 1) == gen) __nanosleep(20);
      }
    }
    ++gen;
    LPROF(3);
    cluster.sync();
    LPROF(4);
  }
#ifdef CABS_PROFILE_LLOYD
  if (b == G - 1 && tid == 0)
    for (int i = 0; i < 10; ++i) a.prof[i] = prof[i];
#endif
  // ---------------- epilogue (CTA 0): final centres, cluster weights, objective history
  if (b == 0) {
#pragma unroll
    for (int q = 0; q < kMaxProb; ++q) {
      if (q >= np_) break;
      const LloydProb& pr = a.pr[q];
      const ProbSmem S = prob_smem(dyn, Ls[q]);
      const int d = pr.d, k2 = pr.k2, nsum = k2 * d;
      const double inv_scale = 1.0 / scale[q], inv_scale_w = 1.0 / scale_w[q];
      const long long* fs_last = pr.fsum + (size_t)((a.iters - 1) % 3) * Eq[q];
      for (int e = tid; e < nsum; e += blockDim.x) {
        const int j = e / d, i = e - j * d;
        const long long wj = __ldcg(fs_last + nsum + j);
        pr.centres[(int64_t)j * pr.ldc + i] =
            wj > 0 ? static_cast<float>((static_cast<double>(__ldcg(fs_last + e)) * inv_scale) *
                                        (1.0 / (static_cast<double>(wj) * inv_scale_w)))
                   : S.cs[cpair_idx(j, i, d)];
      }
      for (int j = tid; j < k2; j += blockDim.x)
        pr.cluster_w[j] = static_cast<double>(__ldcg(fs_last + nsum + j)) / scale_w[q];
      for (int it = tid; it < a.iters; it += blockDim.x) {
        double s = 0;
        long long qq = 0;
        for (int g = 0; g < G; ++g) {
          s += __ldcg(pr.pobj + (size_t)it * G + g);
          qq += __ldcg(pr.ptie + (size_t)it * G + g);
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
  int64_t Nmin = jobs[0].N;
  for (int q = 1; q < njobs; ++q) Nmin = jobs[q].N < Nmin ? jobs[q].N : Nmin;
  // grid: one CTA per SM (every CTA holds ~N / #SM points of each problem); the largest
  // cluster size (8, 4, 2, 1) whose clusters can all be resident
  int64_t G = nsm;
  if (G > Nmin) G = Nmin;
  auto smem_for = [&](int64_t g, int& resident, int* pitch) {
    resident = 1;
    size_t total = 0;
    for (int q = 0; q < njobs; ++q) {
      const int64_t per = ceil_div(jobs[q].N, g);
      pitch[q] = per <= kLP ? static_cast<int>(round_up(per, 16)) : kLP;
      if (per > kLP) resident = 0;
      total = lloyd_smem(jobs[q].d, jobs[q].k2, pitch[q], total).total;
    }
    return total;
  };
  LloydArgs a{};
  a.nprob = njobs;
  a.iters = iters;
  a.prof = prof;
  int pitch[kMaxProb] = {kLP, kLP};
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
  size_t smem = 0;
  for (int c = 8; c >= 1 && csize == 0; c >>= 1) {
    const int64_t g = G / c * c;  // round down: every CTA still gets <= ceil(N / g) points
    if (g < 1) continue;
    smem = smem_for(g, resident, pitch);
    if (smem > kSmemCap) continue;
    at[0].val.clusterDim.x = static_cast<unsigned>(c);
    cfg.gridDim = dim3(static_cast<unsigned>(g));
    cfg.dynamicSmemBytes = smem;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, lloyd_persistent_kernel, &cfg) == cudaSuccess && (int64_t)ncl * c >= g) {
      csize = c;
      G = g;
    }
  }
  cudaGetLastError();
  if (csize == 0) return false;
  a.resident = resident;
  // scratch of each job: fsum [3][k2*d + k2] | pobj [iters][G] | ptie [iters][G]; barrier in job 0's
  for (int q = 0; q < njobs; ++q) {
    const LloydJob& j = jobs[q];
    const size_t E = (size_t)j.k2 * j.d + j.k2;
    const size_t need = sizeof(long long) * 3 * E + 16 + (sizeof(double) + sizeof(int)) * iters * G;
    if (need > j.scratch_bytes) return false;
    char* base = static_cast<char*>(j.scratch);
    LloydProb& p = a.pr[q];
    p.X = j.X; p.ldx = j.ldx; p.N = j.N; p.d = j.d; p.k2 = j.k2; p.w = j.w;
    p.centres = j.centres; p.ldc = j.ldc; p.labels = j.labels; p.objective = j.objective;
    p.near_ties = j.near_ties; p.cluster_w = j.cluster_w; p.bounds = j.bounds; p.pitch = pitch[q];
    p.fsum = reinterpret_cast<long long*>(base);
    unsigned* gb = reinterpret_cast<unsigned*>(p.fsum + 3 * E);
    if (q == 0) a.gbar = gb;
    p.pobj = reinterpret_cast<double*>(gb + 4);
    p.ptie = reinterpret_cast<int*>(p.pobj + (size_t)iters * G);
    if (cudaMemsetAsync(base, 0, sizeof(long long) * 3 * E + 16, st) != cudaSuccess) return false;
  }
  note_launch();
  return cudaLaunchKernelEx(&cfg, lloyd_persistent_kernel, a) == cudaSuccess;
}

}  // namespace cabsk
