// lloyd.cu -- the whole Lloyd loop of one k-means call in ONE persistent kernel (single
// GPU): c iterations x {centres | assign | accumulate | cluster reduce | grid sync}, no
// host round trips, no per-iteration launches, ONE grid-wide barrier per iteration.
//
// Arithmetic (Eq. 6; c iterations P:204):
//  * distances by direct differences in FP32, dimensions ascending (= km_tile.cuh), lowest
//    centre index on ties; two centres per packed FP32x2 instruction (FADD2/FFMA2: the same
//    IEEE rounding as the scalar ops, half the instructions), 8 points x 8 centres per
//    thread so that shared-memory operands are reused 8 times;
//  * sums w_l X_l and w_l accumulated EXACTLY as int64 fixed point (km_fixed.cuh): every
//    CTA buckets its 128 points by label into a dense int64 partial in shared memory, the
//    CTAs of a thread-block cluster (8) add their partials through distributed shared
//    memory (each CTA one slice), and one red.global.add.u64 per (cluster, entry) lands in
//    the global sums -- order-free, so deterministic and identical to the per-iteration
//    kernels of kmeans.cu;
//  * centres = (sum / 2^S) / (weight / 2^Sw) in FP64; an empty cluster keeps its centre (Z12).
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
constexpr int kLA = 9;         // point rows per thread
constexpr int kLP = 16 * kLA;  // points per chunk: thread (pt = tid & 15, ct = tid >> 4) owns points pt + 16u, u < 9
constexpr int kLC = 64;        // centres per block: ... and centres j0 + ct + 16v, v < 4

struct LloydArgs {
  const float* X;
  int64_t ldx, N;
  int d, k2, iters;
  const float* w;
  float* centres;  // in: initial centres; out: final centres
  int64_t ldc;
  int* labels;
  double* objective;
  int* near_ties;
  double* cluster_w;
  long long* fsum;         // [3][k2*d + k2] fixed-point sums | weights
  const unsigned* bounds;  // [2] max|x|, max w (km_weights)
  unsigned* gbar;          // [2] grid barrier {arrivals, generation}
  double* pobj;            // [iters][G]
  int* ptie;               // [iters][G]
  int resident, cpc;       // X chunks resident in smem; max chunks per CTA
  long long* prof;         // diagnostics (CABS_PROFILE_LLOYD builds): per-phase cycles of the last CTA
};

// dynamic smem: centre pairs | per resident chunk: point pairs [d][kLP], point rows [kLP][d],
// w * 2^S (FP64), llrint(w * 2^Sw), weights | dense partial | 1 / cluster weight (FP64).
// (X is not re-read from global memory: every cluster.sync invalidates L1.)
struct LloydSmem {
  size_t cs, xp, xr, wsc, iw, wts, part, wd, total;
};
__host__ __device__ inline LloydSmem lloyd_smem(int d, int k2, int nchunk_buf) {
  LloydSmem L;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 15) & ~size_t(15); return r; };
  L.cs = take(sizeof(float) * round_up(k2, kLC) * d);
  L.xp = take(sizeof(float) * 2 * (size_t)nchunk_buf * d * kLP);
  L.xr = take(sizeof(float) * (size_t)nchunk_buf * d * kLP);
  L.wsc = take(sizeof(double) * (size_t)nchunk_buf * kLP);
  L.iw = take(sizeof(long long) * (size_t)nchunk_buf * kLP);
  L.wts = take(sizeof(float) * (size_t)nchunk_buf * kLP);
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

struct ChunkBufs {
  float *xp, *xr;
  double* wsc;
  long long* iw;
  float* wts;
};
__device__ __forceinline__ ChunkBufs chunk_bufs(unsigned char* dyn, const LloydSmem& L, int d, int c) {
  ChunkBufs cb;
  cb.xp = reinterpret_cast<float*>(dyn + L.xp) + (size_t)c * d * kLP * 2;
  cb.xr = reinterpret_cast<float*>(dyn + L.xr) + (size_t)c * d * kLP;
  cb.wsc = reinterpret_cast<double*>(dyn + L.wsc) + (size_t)c * kLP;
  cb.iw = reinterpret_cast<long long*>(dyn + L.iw) + (size_t)c * kLP;
  cb.wts = reinterpret_cast<float*>(dyn + L.wts) + (size_t)c * kLP;
  return cb;
}
// chunk of up to kLP points -> (x, x) pairs [i][kLP], w 2^S, llrint(w 2^Sw), w (zeros beyond)
__device__ __forceinline__ void stage_chunk(const LloydArgs& a, int64_t p0, int np, const ChunkBufs& cb, double scale,
                                            double scale_w) {
  const int d = a.d;
  for (int e = threadIdx.x; e < kLP * d; e += blockDim.x) {
    const int pp = e / d, i = e - pp * d;
    const float x = pp < np ? __ldg(a.X + (p0 + pp) * a.ldx + i) : 0.f;
    reinterpret_cast<float2*>(cb.xp)[i * kLP + pp] = make_float2(x, x);
    cb.xr[e] = x;
  }
  for (int pp = threadIdx.x; pp < kLP; pp += blockDim.x) {
    const float w = pp < np ? a.w[p0 + pp] : 0.f;
    cb.wsc[pp] = static_cast<double>(w) * scale;  // exact (power-of-two scale)
    cb.iw[pp] = llrint(static_cast<double>(w) * scale_w);
    cb.wts[pp] = w;
  }
}

// Distances of the chunk's points pt + 16u (u < NA) to all centres (two per FFMA2; direct
// differences, dimensions ascending), running (best, index, runner-up) per point, merged over
// the two centre lanes of the warp and written to the per-warp slots sb_*[warp][point].
template <int NA>
__device__ __forceinline__ void dist_rows(const unsigned long long* __restrict__ xq, const float* cs, int d, int k2,
                                          int pt, int ct, int lane, int warp, float (*sb_d)[kLP], int (*sb_j)[kLP],
                                          float (*ss_d)[kLP]) {
  float bd[NA], sd[NA];
  int bj[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) { bd[q] = FLT_MAX; sd[q] = FLT_MAX; bj[q] = 0x7fffffff; }
  for (int j0 = 0; j0 < k2; j0 += kLC) {
    unsigned long long acc[2][NA] = {};
    const unsigned long long* cq = reinterpret_cast<const unsigned long long*>(cs) + (size_t)(j0 >> 6) * d * 32 + ct;
    for (int i = 0; i < d; ++i) {
      const unsigned long long c0 = cq[i * 32], c1 = cq[i * 32 + 16];
      unsigned long long x[NA];
#pragma unroll
      for (int u = 0; u < NA; ++u) x[u] = xq[i * kLP + 16 * u];
#pragma unroll
      for (int u = 0; u < NA; ++u) {
        const unsigned long long df0 = f2_sub(x[u], c0), df1 = f2_sub(x[u], c1);
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

static_assert(kLT == 256, "the accumulation maps 8 warps x 8 clusters onto 64-cluster blocks");
__global__ void __launch_bounds__(kLT, 1) lloyd_persistent_kernel(LloydArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ float sb_d[8][kLP];  // per point: best / runner-up of each warp's two centre lanes
  __shared__ int sb_j[8][kLP];
  __shared__ float ss_d[8][kLP];
  __shared__ int lab_s[kLP];
  __shared__ double s_red[kLT / 32];
  __shared__ int s_tie[kLT / 32];
  cg::cluster_group cluster = cg::this_cluster();
  const int crank = static_cast<int>(cluster.block_rank()), csize = static_cast<int>(cluster.num_blocks());
  unsigned gen = 0;  // grid-barrier generation
  const int tid = threadIdx.x, pt = tid & 15, ct = tid >> 4, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, b = blockIdx.x;
  const int k2 = a.k2, d = a.d;
  const int64_t nsum = (int64_t)k2 * d, E = nsum + k2;
  const LloydSmem L = lloyd_smem(d, k2, a.resident ? a.cpc : 1);
  float* cs = reinterpret_cast<float*>(dyn + L.cs);
  long long* part = reinterpret_cast<long long*>(dyn + L.part);  // [E]
  double* wd = reinterpret_cast<double*>(dyn + L.wd);           // 1 / weight_j (0: empty cluster)
  const int k2p = static_cast<int>(round_up(k2, kLC));
  // balanced contiguous point range of this CTA, in chunks of kLP
  const int64_t p_beg = (a.N * b) / G, p_end = (a.N * (b + 1)) / G;
  double scale, scale_w;
  fx_scales(a.bounds, a.N, scale, scale_w);
  const double inv_scale = 1.0 / scale, inv_scale_w = 1.0 / scale_w;  // exact: powers of two
  // this CTA's slice of the cluster reduction
  const int64_t e_beg = E * crank / csize, e_end = E * (crank + 1) / csize;

  // ---------------- prologue: resident chunks, initial centres (padding centres = 0)
  if (a.resident)
    for (int64_t p0 = p_beg, c = 0; p0 < p_end; p0 += kLP, ++c) {
      const int np = static_cast<int>(p_end - p0 < kLP ? p_end - p0 : kLP);
      stage_chunk(a, p0, np, chunk_bufs(dyn, L, d, static_cast<int>(c)), scale, scale_w);
    }
  for (int e = tid; e < k2p * d; e += blockDim.x) {
    const int j = e / d, i = e - j * d;
    cs[cpair_idx(j, i, d)] = j < k2 ? __ldcg(a.centres + (int64_t)j * a.ldc + i) : 0.f;
  }

#ifdef CABS_PROFILE_LLOYD
  long long prof[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, t0 = clock64();
#define LPROF(i) do { if (b == G - 1 && tid == 0) { long long t1 = clock64(); prof[i] += t1 - t0; t0 = t1; } } while (0)
#else
#define LPROF(i) do { } while (0)
#endif
  for (int it = 0; it < a.iters; ++it) {
    long long* fs_cur = a.fsum + (size_t)(it % 3) * E;
    if (it > 0) {
      // centres of this iteration from the previous iteration's exact sums (empty cluster: keep)
      const long long* fs_prev = a.fsum + (size_t)((it + 2) % 3) * E;
      for (int j = tid; j < k2; j += blockDim.x) {
        const long long wj = __ldcg(fs_prev + nsum + j);
        wd[j] = wj > 0 ? 1.0 / (static_cast<double>(wj) * inv_scale_w) : 0.0;
      }
      constexpr int U = 8;  // independent L2 loads in flight per thread
      long long sv[U];
      const int ns = static_cast<int>(nsum);
#pragma unroll
      for (int u = 0; u < U; ++u) sv[u] = tid + u * kLT < ns ? __ldcg(fs_prev + tid + u * kLT) : 0;
      __syncthreads();  // wd ready
      for (int e0 = tid; e0 < ns; e0 += U * kLT) {
        if (e0 != tid) {
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int e = e0 + u * kLT;
            sv[u] = e < ns ? __ldcg(fs_prev + e) : 0;
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int e = e0 + u * kLT;
          if (e < ns) {
            const int j = e / d, i = e - j * d;
            const double rw = wd[j];
            if (rw > 0) cs[cpair_idx(j, i, d)] = static_cast<float>((static_cast<double>(sv[u]) * inv_scale) * rw);
          }
        }
      }
      // zero the slot the next iteration accumulates into (last read before the previous barrier)
      long long* fs_next = a.fsum + (size_t)((it + 1) % 3) * E;
      for (int64_t e = (int64_t)b * blockDim.x + tid; e < E; e += (int64_t)G * blockDim.x) fs_next[e] = 0;
    }
    for (int64_t e = tid; e < E; e += blockDim.x) part[e] = 0;
    double obj = 0.0;
    int ties = 0;
    __syncthreads();
    LPROF(0);
    for (int64_t p0 = p_beg, c = 0; p0 < p_end; p0 += kLP, ++c) {
      const int np = static_cast<int>(p_end - p0 < kLP ? p_end - p0 : kLP);
      const ChunkBufs cb = chunk_bufs(dyn, L, d, a.resident ? static_cast<int>(c) : 0);
      if (!a.resident) {
        __syncthreads();  // previous chunk fully consumed
        stage_chunk(a, p0, np, cb, scale, scale_w);
        __syncthreads();
      }
      // distances: points pt + 16u x centres j0 + ct + 16v (v < 4), rows u < NA = ceil(np / 16)
      {
        const unsigned long long* xq = reinterpret_cast<const unsigned long long*>(cb.xp) + pt;
        const int na = (np + 15) >> 4;
        if (na <= 3) dist_rows<3>(xq, cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d);
        else if (na <= 5) dist_rows<5>(xq, cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d);
        else if (na <= 7) dist_rows<7>(xq, cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d);
        else dist_rows<9>(xq, cs, d, k2, pt, ct, lane, warp, sb_d, sb_j, ss_d);
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
        if (p < np) {
          a.labels[p0 + p] = Bj;
          obj += static_cast<double>(cb.wts[p]) * static_cast<double>(B);
          ties += (Sd - B) < kNearTie * Sd;
        }
      }
      __syncthreads();
      LPROF(1);
      // exact sums (km_fixed.cuh): warp w owns the clusters j = jb + w + 8t (t < 8) and keeps
      // their sums over the chunk in registers, lanes over dimensions; a ballot over 32 labels
      // at a time finds its points, whose llrint(w 2^S x_pi) it adds (integer adds: any order).
      for (int jb = 0; jb < k2; jb += 64) {
        for (int i0 = 0; i0 < d; i0 += 64) {
          const int ia = i0 + lane, ib = i0 + 32 + lane;
          long long sa[8], sbv[8], sw[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) { sa[t] = 0; sbv[t] = 0; sw[t] = 0; }
          for (int q0 = 0; q0 < np; q0 += 32) {
            const int q = q0 + lane;
            const int jr = q < np ? lab_s[q] - jb - warp : -1;
            unsigned m = __ballot_sync(0xffffffffu, jr >= 0 && jr < 64 && (jr & 7) == 0);
            while (m) {  // two points per step: independent load -> convert chains
              const int p1 = q0 + __ffs(m) - 1;
              m &= m - 1;
              const bool two = m != 0;
              const int p2 = two ? q0 + __ffs(m) - 1 : p1;
              if (two) m &= m - 1;
              const int t1 = (lab_s[p1] - jb - warp) >> 3, t2 = (lab_s[p2] - jb - warp) >> 3;
              const double ws1 = cb.wsc[p1], ws2 = two ? cb.wsc[p2] : 0.0;
              const float* x1 = cb.xr + p1 * d;
              const float* x2 = cb.xr + p2 * d;
              const long long va1 = ia < d ? fx_prod_magic(ws1, x1[ia]) : 0;
              const long long vb1 = ib < d ? fx_prod_magic(ws1, x1[ib]) : 0;
              const long long va2 = ia < d ? fx_prod_magic(ws2, x2[ia]) : 0;
              const long long vb2 = ib < d ? fx_prod_magic(ws2, x2[ib]) : 0;
              const long long vw1 = cb.iw[p1], vw2 = two ? cb.iw[p2] : 0;
#pragma unroll
              for (int tt = 0; tt < 8; ++tt) {
                if (tt == t1) { sa[tt] += va1; sbv[tt] += vb1; sw[tt] += vw1; }
                if (tt == t2) { sa[tt] += va2; sbv[tt] += vb2; sw[tt] += vw2; }
              }
            }
          }
#pragma unroll
          for (int t = 0; t < 8; ++t) {
            const int j = jb + warp + 8 * t;
            if (j < k2) {
              if (ia < d) part[j * d + ia] += sa[t];
              if (ib < d) part[j * d + ib] += sbv[t];
              if (i0 == 0 && lane == 0) part[nsum + j] += sw[t];
            }
          }
        }
      }
      __syncthreads();
    }
    LPROF(2);
    // cluster reduction of the dense partials (DSMEM), one global integer add per entry
    cluster.sync();
    LPROF(5);
    {
      const long long* rp[8];
#pragma unroll
      for (int r = 0; r < 8; ++r) rp[r] = r < csize ? cluster.map_shared_rank(part, r) : part;
      for (int64_t e = e_beg + tid; e < e_end; e += blockDim.x) {
        long long v[8];
#pragma unroll
        for (int r = 0; r < 8; ++r) v[r] = r < csize ? rp[r][e] : 0;
        long long s = 0;
#pragma unroll
        for (int r = 0; r < 8; ++r) s += v[r];
        if (s != 0) red_add_u64(fs_cur + e, s);
      }
    }
    obj = warp_sum_d(obj);
    int tt = ties;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, o);
    if (lane == 0) { s_red[warp] = obj; s_tie[warp] = tt; }
    LPROF(6);
    __threadfence();
    LPROF(7);
    cluster.sync();  // partials free again; this cluster's global adds issued and fenced
    LPROF(8);
    if (tid == 0) {
      double s = 0;
      int q = 0;
      for (int w = 0; w < kLT / 32; ++w) { s += s_red[w]; q += s_tie[w]; }
      a.pobj[(size_t)it * G + b] = s;
      a.ptie[(size_t)it * G + b] = q;
    }
    LPROF(3);
    grid_barrier(a.gbar, gen);
    LPROF(4);
  }
#ifdef CABS_PROFILE_LLOYD
  if (b == G - 1 && tid == 0)
    for (int i = 0; i < 10; ++i) a.prof[i] = prof[i];
#endif
  // ---------------- epilogue (CTA 0): final centres, cluster weights, objective history
  if (b == 0) {
    const long long* fs_last = a.fsum + (size_t)((a.iters - 1) % 3) * E;
    for (int e = tid; e < nsum; e += blockDim.x) {
      const int j = e / d, i = e - j * d;
      const long long wj = __ldcg(fs_last + nsum + j);
      a.centres[(int64_t)j * a.ldc + i] =
          wj > 0 ? static_cast<float>((static_cast<double>(__ldcg(fs_last + e)) * inv_scale) *
                                      (1.0 / (static_cast<double>(wj) * inv_scale_w)))
                 : cs[cpair_idx(j, i, d)];
    }
    for (int j = tid; j < k2; j += blockDim.x) a.cluster_w[j] = static_cast<double>(__ldcg(fs_last + nsum + j)) / scale_w;
    for (int it = tid; it < a.iters; it += blockDim.x) {
      double s = 0;
      long long q = 0;
      for (int g = 0; g < G; ++g) { s += __ldcg(a.pobj + (size_t)it * G + g); q += __ldcg(a.ptie + (size_t)it * G + g); }
      a.objective[it] = s;
      if (a.near_ties) a.near_ties[it] = static_cast<int>(q);
    }
  }
}

// Returns false when the fast path does not apply (caller uses the per-iteration kernels).
bool launch_lloyd_persistent(const float* X, int64_t ldx, int64_t N, int d, int k2, int iters, const float* w,
                             const unsigned* bounds, float* centres, int64_t ldc, int* labels, double* objective,
                             int* near_ties, double* cluster_w, void* scratch, size_t scratch_bytes, long long* prof,
                             cudaStream_t st) {
  if (N <= 0) return false;
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
  // grid: one CTA per SM, every CTA a balanced contiguous range of ~N / #SM points (chunks of
  // kLP); the largest cluster size (8, 4, 2, 1) whose clusters can all be resident
  int64_t G = nsm;  // all SMs: the per-CTA point count sets the iteration time
  if (G > N) G = N;
  const int cpc = static_cast<int>(ceil_div(ceil_div(N, G), kLP));
  int resident = 1;
  size_t smem = lloyd_smem(d, k2, cpc).total;
  if (smem > kSmemCap) {
    resident = 0;
    smem = lloyd_smem(d, k2, 1).total;
  }
  if (smem > kSmemCap) return false;
  // co-residency of all CTAs (the grid barrier) is checked, not assumed
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kLT);
  cfg.dynamicSmemBytes = smem;
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
  for (int c = 8; c >= 1 && csize == 0; c >>= 1) {
    const int64_t g = G / c * c;  // round down: every CTA still gets <= ceil(N / g) points
    if (g < 1) continue;
    at[0].val.clusterDim.x = static_cast<unsigned>(c);
    cfg.gridDim = dim3(static_cast<unsigned>(g));
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, lloyd_persistent_kernel, &cfg) == cudaSuccess && (int64_t)ncl * c >= g) {
      csize = c;
      G = g;
    }
  }
  cudaGetLastError();
  if (csize == 0) return false;
  const int cpc_final = static_cast<int>(ceil_div(ceil_div(N, G), kLP));  // <= cpc: smem suffices
  // scratch: fsum [3][k2*d + k2] | gbar [2] (+pad) | pobj [iters][G] | ptie [iters][G]
  const size_t E = (size_t)k2 * d + k2;
  const size_t need = sizeof(long long) * 3 * E + 16 + (sizeof(double) + sizeof(int)) * iters * G;
  if (need > scratch_bytes) return false;
  char* base = static_cast<char*>(scratch);
  long long* fsum = reinterpret_cast<long long*>(base);
  unsigned* gbar = reinterpret_cast<unsigned*>(fsum + 3 * E);
  double* pobj = reinterpret_cast<double*>(gbar + 4);
  int* ptie = reinterpret_cast<int*>(pobj + (size_t)iters * G);
  if (cudaMemsetAsync(base, 0, sizeof(long long) * 3 * E + 16, st) != cudaSuccess) return false;
  LloydArgs a{X, ldx, N, d, k2, iters, w, centres, ldc, labels, objective, near_ties, cluster_w,
              fsum, bounds, gbar, pobj, ptie, resident, cpc_final, prof};
  note_launch();
  return cudaLaunchKernelEx(&cfg, lloyd_persistent_kernel, a) == cudaSuccess;
}

}  // namespace cabsk
