// lloyd.cu -- the whole Lloyd loop of one k-means call in ONE persistent cooperative
// kernel (single GPU): c iterations x {assign + accumulate | grid sync | reduce +
// update | grid sync}, no host round trips and no per-iteration launches.
//
// Same arithmetic as the multi-kernel path (kmeans.cu): direct-difference FP32
// distances (km_tile.cuh), per-CTA FP32 partial sums over a fixed contiguous point
// range in index order, fixed-order FP64 cross-CTA reduction, empty clusters keep
// their centre (Z12).  Eq. 6, c iterations.
#include <cooperative_groups.h>
#include <float.h>

#include "common.cuh"
#include "kernels.cuh"
#include "km_tile.cuh"

namespace cg = cooperative_groups;

namespace cabsk {

struct LloydArgs {
  const float* X;
  int64_t ldx, N;
  int d, k2, iters;
  const float* w;
  float* centres;
  int64_t ldc;
  int* labels;
  double* objective;
  int* near_ties;
  double* cluster_w;
  float* psum;  // [G][k2][d]
  double* pw;   // [G][k2]
  double* pobj; // [G]
  int* ptie;    // [G]
  int groups;   // accumulation thread groups (256 / dgroup)
  int dgroup;   // threads per group (>= d, multiple of 32)
};

constexpr int kLloydThreads = 256;
constexpr int kXt = kTileP + 1;  // row pitch of the transposed point tile (conflict-free both ways)

// Dynamic shared memory layout (floats unless noted):
//   cs   [round_up(k2,64)][d+1]   centres of this iteration
//   xt   [d][65]                  the current 64-point tile, transposed
//   acc  [groups][k2][d]          per-group partial sums
//   wacc [groups][k2] (double)    per-group partial weights
//   ws_  [64]                     weights of the tile's points
struct LloydSmem {
  size_t cs, xt, acc, wacc, wts, total;
};
__host__ __device__ inline LloydSmem lloyd_smem(int d, int k2, int groups) {
  LloydSmem L;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 15) & ~size_t(15); return r; };
  L.cs = take(sizeof(float) * round_up(k2, 64) * (d + 1));
  L.xt = take(sizeof(float) * (size_t)d * kXt);
  L.acc = take(sizeof(float) * (size_t)groups * k2 * d);
  L.wacc = take(sizeof(double) * (size_t)groups * k2);
  L.wts = take(sizeof(float) * kTileP);
  L.total = o;
  return L;
}

__global__ void __launch_bounds__(kLloydThreads) lloyd_persistent_kernel(LloydArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ float sb_d[16][kTileP + 1];
  __shared__ int sb_j[16][kTileP + 1];
  __shared__ float ss_d[16][kTileP + 1];
  __shared__ int lab_s[kTileP];
  __shared__ double s_red[8];
  __shared__ int s_tie[8];
  cg::grid_group grid = cg::this_grid();
  const int tid = threadIdx.x, tp = tid & 15, tc = tid >> 4;
  const int G = gridDim.x, b = blockIdx.x;
  const int k2 = a.k2, d = a.d, cst = d + 1;
  const LloydSmem L = lloyd_smem(d, k2, a.groups);
  float* cs = reinterpret_cast<float*>(dyn + L.cs);
  float* xt = reinterpret_cast<float*>(dyn + L.xt);
  float* acc = reinterpret_cast<float*>(dyn + L.acc);
  double* wacc = reinterpret_cast<double*>(dyn + L.wacc);
  float* wts = reinterpret_cast<float*>(dyn + L.wts);
  const int grp = tid / a.dgroup, gi = tid % a.dgroup;  // accumulation group / dimension
  const int k2p = static_cast<int>(round_up(k2, 64));
  const int64_t ntiles = ceil_div(a.N, kTileP);
  const int64_t t_beg = (ntiles * b) / G, t_end = (ntiles * (b + 1)) / G;  // contiguous tiles

  for (int it = 0; it < a.iters; ++it) {
    // ---------------- phase A: assign + per-CTA partial sums
    for (int e = tid; e < k2p * d; e += blockDim.x) {
      const int j = e / d, i = e - j * d;
      cs[j * cst + i] = j < k2 ? __ldcg(a.centres + (int64_t)j * a.ldc + i) : 0.f;
    }
    for (int e = tid; e < a.groups * k2 * d; e += blockDim.x) acc[e] = 0.f;
    for (int e = tid; e < a.groups * k2; e += blockDim.x) wacc[e] = 0.0;
    double obj = 0.0;
    int ties = 0;
    __syncthreads();
    for (int64_t tile = t_beg; tile < t_end; ++tile) {
      const int64_t p0 = tile * kTileP;
      // stage the tile transposed: xt[i][pp] (coalesced global reads along i)
      for (int e = tid; e < kTileP * d; e += blockDim.x) {
        const int pp = e / d, i = e - pp * d;
        const int64_t p = p0 + pp;
        xt[i * kXt + pp] = p < a.N ? __ldg(a.X + p * a.ldx + i) : 0.f;
      }
      if (tid < kTileP) wts[tid] = (p0 + tid < a.N) ? a.w[p0 + tid] : 0.f;
      __syncthreads();
      // distances (direct differences, ascending i -- identical arithmetic to km_tile.cuh)
      float bd[4], sd[4];
      int bj[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) { bd[q] = FLT_MAX; sd[q] = FLT_MAX; bj[q] = 0x7fffffff; }
      for (int j0 = 0; j0 < k2; j0 += kTileC) {
        float accd[4][4] = {};
        const float* c0 = cs + (j0 + tc) * cst;
        for (int i = 0; i < d; ++i) {
          float x[4], c[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) x[q] = xt[i * kXt + tp + 16 * q];
#pragma unroll
          for (int q = 0; q < 4; ++q) c[q] = c0[16 * q * cst + i];
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
              const float df = x[u] - c[v];
              accd[u][v] = fmaf(df, df, accd[u][v]);
            }
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) {
          const int j = j0 + tc + 16 * v;
          if (j >= k2) continue;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const float val = accd[u][v];
            if (val < bd[u] || (val == bd[u] && j < bj[u])) { sd[u] = bd[u]; bd[u] = val; bj[u] = j; }
            else sd[u] = fminf(sd[u], val);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        sb_d[tc][tp + 16 * u] = bd[u];
        sb_j[tc][tp + 16 * u] = bj[u];
        ss_d[tc][tp + 16 * u] = sd[u];
      }
      __syncthreads();
      if (tid < kTileP) {
        float B = sb_d[0][tid], Sd = ss_d[0][tid];
        int Bj = sb_j[0][tid];
        for (int t = 1; t < 16; ++t) {
          const float b2 = sb_d[t][tid], s2 = ss_d[t][tid];
          const int j2 = sb_j[t][tid];
          if (b2 < B || (b2 == B && j2 < Bj)) { Sd = fminf(fminf(Sd, s2), B); B = b2; Bj = j2; }
          else Sd = fminf(fminf(Sd, s2), b2);
        }
        lab_s[tid] = Bj;
        const int64_t p = p0 + tid;
        if (p < a.N) {
          a.labels[p] = Bj;
          obj += static_cast<double>(wts[tid]) * static_cast<double>(B);
          ties += (Sd - B) < kNearTie * Sd;
        }
      }
      __syncthreads();
      // group grp accumulates points [grp*per, (grp+1)*per) of the tile in index order;
      // thread gi owns dimension gi (and gi + dgroup, ... when d > dgroup)
      const int per = kTileP / a.groups;
      float* ag = acc + (size_t)grp * k2 * d;
      double* wg = wacc + (size_t)grp * k2;
      for (int pp = grp * per; pp < (grp + 1) * per; ++pp) {
        if (p0 + pp >= a.N) break;
        const int j = lab_s[pp];
        const float wl = wts[pp];
        for (int i = gi; i < d; i += a.dgroup) ag[j * d + i] = fmaf(wl, xt[i * kXt + pp], ag[j * d + i]);
        if (gi == 0) wg[j] += static_cast<double>(wl);
      }
      __syncthreads();
    }
    // combine the groups in fixed order and publish this CTA's partials
    for (int e = tid; e < k2 * d; e += blockDim.x) {
      float s = acc[e];
      for (int g = 1; g < a.groups; ++g) s += acc[(size_t)g * k2 * d + e];
      a.psum[(size_t)b * k2 * d + e] = s;
    }
    for (int j = tid; j < k2; j += blockDim.x) {
      double s = wacc[j];
      for (int g = 1; g < a.groups; ++g) s += wacc[(size_t)g * k2 + j];
      a.pw[(size_t)b * k2 + j] = s;
    }
    obj = warp_sum_d(obj);
    int tt = ties;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, o);
    if ((tid & 31) == 0) { s_red[tid >> 5] = obj; s_tie[tid >> 5] = tt; }
    __syncthreads();
    if (tid == 0) {
      double s = 0;
      int q = 0;
      for (int w = 0; w < kLloydThreads / 32; ++w) { s += s_red[w]; q += s_tie[w]; }
      a.pobj[b] = s;
      a.ptie[b] = q;
    }
    grid.sync();
    // ---------------- phase B: fixed-order FP64 reduction over CTAs + centre update.
    // 8 lanes per output element, lane l sums CTAs l, l+8, ...; xor-butterfly combine.
    const int64_t nsum = (int64_t)k2 * d;
    const int64_t nel = nsum + k2 + 2;
    const int64_t gt = (int64_t)b * blockDim.x + tid;
    const int sub = static_cast<int>(gt & 7);
    const unsigned gmask = 0xffu << (tid & 24);  // the 8-lane group sharing one element
    const int64_t gstride = ((int64_t)G * blockDim.x) >> 3;
    for (int64_t e = gt >> 3; e < nel; e += gstride) {
      double s = 0.0, wsum = 0.0;
      if (e < nsum) {
        const int j = static_cast<int>(e / d);
        for (int q = sub; q < G; q += 8) {
          s += static_cast<double>(__ldcg(a.psum + (size_t)q * nsum + e));
          wsum += __ldcg(a.pw + (size_t)q * k2 + j);
        }
      } else if (e < nsum + k2) {
        const int j = static_cast<int>(e - nsum);
        for (int q = sub; q < G; q += 8) s += __ldcg(a.pw + (size_t)q * k2 + j);
      } else if (e == nsum + k2) {
        for (int q = sub; q < G; q += 8) s += __ldcg(a.pobj + q);
      } else {
        for (int q = sub; q < G; q += 8) s += static_cast<double>(__ldcg(a.ptie + q));
      }
#pragma unroll
      for (int o = 4; o > 0; o >>= 1) {
        s += __shfl_xor_sync(gmask, s, o);
        wsum += __shfl_xor_sync(gmask, wsum, o);
      }
      if (sub == 0) {
        if (e < nsum) {
          const int j = static_cast<int>(e / d), i = static_cast<int>(e % d);
          if (wsum > 0) a.centres[(int64_t)j * a.ldc + i] = static_cast<float>(s / wsum);
        } else if (e < nsum + k2) {
          a.cluster_w[e - nsum] = s;
        } else if (e == nsum + k2) {
          a.objective[it] = s;
        } else if (a.near_ties) {
          a.near_ties[it] = static_cast<int>(s);
        }
      }
    }
    grid.sync();
  }
}

// Returns false when the fast path does not apply (caller uses the multi-kernel loop).
bool launch_lloyd_persistent(const float* X, int64_t ldx, int64_t N, int d, int k2, int iters, const float* w,
                             float* centres, int64_t ldc, int* labels, double* objective, int* near_ties,
                             double* cluster_w, float* psum, double* pw, double* pobj, int* ptie, int max_grid,
                             cudaStream_t st) {
  if (N <= 0) return false;
  const int dgroup = static_cast<int>(round_up(d < 256 ? d : 256, 32));
  const int groups = kLloydThreads / dgroup;
  const size_t smem = lloyd_smem(d, k2, groups).total;
  if (smem > 160 * 1024) return false;
  static int attr_smem = -1;
  if (attr_smem < 0) {
    cudaFuncSetAttribute(lloyd_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    attr_smem = 1;
  }
  int dev = 0, nsm = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lloyd_persistent_kernel, kLloydThreads, smem);
  if (occ < 1) return false;
  int64_t G = (int64_t)nsm * (occ > 2 ? 2 : occ);
  const int64_t ntiles = ceil_div(N, kTileP);
  if (G > ntiles) G = ntiles;
  if (G > max_grid) G = max_grid;
  LloydArgs a{X, ldx, N, d, k2, iters, w, centres, ldc, labels, objective, near_ties, cluster_w,
              psum, pw, pobj, ptie, groups, dgroup};
  void* params[] = {&a};
  note_launch();
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lloyd_persistent_kernel), dim3(static_cast<unsigned>(G)),
                                              dim3(kLloydThreads), params, smem, st);
  return e == cudaSuccess;
}

}  // namespace cabsk
