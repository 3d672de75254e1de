// lloyd.cu -- the whole Lloyd loop of one k-means call in ONE persistent cooperative
// kernel (single GPU): c iterations x {assign + accumulate | grid sync}, no host round
// trips, no per-iteration launches, ONE grid-wide barrier per iteration.
//
// Arithmetic (Eq. 6; c iterations P:204):
//  * distances by direct differences in FP32, dimensions ascending (= km_tile.cuh), lowest
//    centre index on ties;
//  * each CTA accumulates w_l X_l of its own contiguous points in FP32 (dimension-owned,
//    index order), then adds its partial to the global sums as int64 fixed point
//    (scale 2^S from the global bound N * max w * max|x|).  Integer addition is
//    associative, so the sums -- and the centres -- do not depend on CTA scheduling:
//    deterministic run to run, with ~2^-40 relative resolution;
//  * centres = sums / weights in FP64; an empty cluster keeps its centre (Z12).
// Sum buffers rotate over three slots: slot it%3 accumulates, slot (it-1)%3 is read by
// every CTA to form this iteration's centres, slot (it+1)%3 is zeroed for the next one.
#include <cooperative_groups.h>
#include <float.h>
#include <math.h>

#include "common.cuh"
#include "kernels.cuh"
#include "km_tile.cuh"

namespace cg = cooperative_groups;

namespace cabsk {

constexpr int kLloydThreads = 256;
constexpr int kXt = kTileP + 1;  // row pitch of a transposed point tile (conflict-free both ways)

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
  long long* fsum;  // [3][k2*d] fixed-point sums
  long long* fw;    // [3][k2]   fixed-point weights
  unsigned* gmax;   // [4] bit patterns of max|x|, max w; grid barrier {arrivals, generation}
  double* pobj;     // [iters][G]
  int* ptie;        // [iters][G]
  int groups, dgroup, resident, tpc;
  long long* prof;  // diagnostics (CABS_PROFILE_LLOYD builds): per-phase cycles of CTA 0
};

struct LloydSmem {
  size_t cs, xt, acc, wacc, wts, winv, total;
};
__host__ __device__ inline LloydSmem lloyd_smem(int d, int k2, int groups, int ntile_buf) {
  LloydSmem L;
  size_t o = 0;
  auto take = [&](size_t b) { size_t r = o; o += (b + 15) & ~size_t(15); return r; };
  L.cs = take(sizeof(float) * round_up(k2, 64) * (d + 1));
  L.xt = take(sizeof(float) * (size_t)ntile_buf * d * kXt);
  L.acc = take(sizeof(float) * (size_t)groups * k2 * d);
  L.wacc = take(sizeof(double) * (size_t)groups * k2);
  L.wts = take(sizeof(float) * (size_t)ntile_buf * kTileP);
  L.winv = take(sizeof(double) * (size_t)k2);
  L.total = o;
  return L;
}

__device__ __forceinline__ void stage_tile(const LloydArgs& a, int64_t p0, float* xt, float* wts) {
  const int d = a.d;
  for (int e = threadIdx.x; e < kTileP * d; e += blockDim.x) {
    const int pp = e / d, i = e - pp * d;
    const int64_t p = p0 + pp;
    xt[i * kXt + pp] = p < a.N ? __ldg(a.X + p * a.ldx + i) : 0.f;
  }
  for (int pp = threadIdx.x; pp < kTileP; pp += blockDim.x) wts[pp] = (p0 + pp < a.N) ? a.w[p0 + pp] : 0.f;
}

__device__ __forceinline__ int scale_exp(double bound) {
  // largest S with bound * 2^S < 2^61 (headroom for the int64 sum), clamped to [0, 60]
  if (!(bound > 0)) return 60;
  int e = static_cast<int>(ceil(log2(bound)));
  int S = 61 - e;
  return S < 0 ? 0 : (S > 60 ? 60 : S);
}

__global__ void __launch_bounds__(kLloydThreads) lloyd_persistent_kernel(LloydArgs a) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ float sb_d[16][kTileP + 1];
  __shared__ int sb_j[16][kTileP + 1];
  __shared__ float ss_d[16][kTileP + 1];
  __shared__ int lab_s[kTileP];
  __shared__ double s_red[8];
  __shared__ int s_tie[8];
  __shared__ float s_max[2][8];
  unsigned gen = 0;  // grid-barrier generation (a.gmax + 2 = {arrivals, generation})
  const int tid = threadIdx.x, tp = tid & 15, tc = tid >> 4, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x, b = blockIdx.x;
  const int k2 = a.k2, d = a.d, cst = d + 1;
  const int64_t nsum = (int64_t)k2 * d;
  const LloydSmem L = lloyd_smem(d, k2, a.groups, a.resident ? a.tpc : 1);
  float* cs = reinterpret_cast<float*>(dyn + L.cs);
  float* xt_all = reinterpret_cast<float*>(dyn + L.xt);
  float* acc = reinterpret_cast<float*>(dyn + L.acc);
  double* wacc = reinterpret_cast<double*>(dyn + L.wacc);
  float* wts_all = reinterpret_cast<float*>(dyn + L.wts);
  double* winv = reinterpret_cast<double*>(dyn + L.winv);
  const int grp = tid / a.dgroup, gi = tid % a.dgroup;
  const int k2p = static_cast<int>(round_up(k2, 64));
  const int64_t ntiles = ceil_div(a.N, kTileP);
  const int64_t t_beg = (ntiles * b) / G, t_end = (ntiles * (b + 1)) / G;

  // ---------------- prologue: global bounds for the fixed-point scale; resident tiles
  {
    float mx = 0.f, mw = 0.f;
    const int64_t pb = t_beg * kTileP, pe = t_end * kTileP < a.N ? t_end * kTileP : a.N;
    for (int64_t e = tid; e < (pe - pb) * d; e += blockDim.x) {
      const int64_t p = pb + e / d;
      mx = fmaxf(mx, fabsf(__ldg(a.X + p * a.ldx + e % d)));
    }
    for (int64_t p = pb + tid; p < pe; p += blockDim.x) mw = fmaxf(mw, a.w[p]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mw = fmaxf(mw, __shfl_xor_sync(0xffffffffu, mw, o));
    }
    if (lane == 0) { s_max[0][warp] = mx; s_max[1][warp] = mw; }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < 8; ++q) { mx = fmaxf(mx, s_max[0][q]); mw = fmaxf(mw, s_max[1][q]); }
      atomicMax(a.gmax, __float_as_uint(mx));
      atomicMax(a.gmax + 1, __float_as_uint(mw));
    }
    if (a.resident)
      for (int64_t t = t_beg; t < t_end; ++t)
        stage_tile(a, t * kTileP, xt_all + (t - t_beg) * d * kXt, wts_all + (t - t_beg) * kTileP);
    for (int e = tid; e < k2p * d; e += blockDim.x) {
      const int j = e / d, i = e - j * d;
      cs[j * cst + i] = j < k2 ? __ldcg(a.centres + (int64_t)j * a.ldc + i) : 0.f;
    }
  }
  grid_barrier(a.gmax + 2, gen);
  const double xmax = static_cast<double>(__uint_as_float(__ldcg(a.gmax)));
  const double wmax = static_cast<double>(__uint_as_float(__ldcg(a.gmax + 1)));
  const int S = scale_exp(static_cast<double>(a.N) * wmax * xmax);
  const int Sw = scale_exp(static_cast<double>(a.N) * wmax);
  const double scale = ldexp(1.0, S), scale_w = ldexp(1.0, Sw);

#ifdef CABS_PROFILE_LLOYD
  long long prof[6] = {0, 0, 0, 0, 0, 0}, t0 = clock64();
#define LPROF(i) do { if (b == 0 && tid == 0) { long long t1 = clock64(); prof[i] += t1 - t0; t0 = t1; } } while (0)
#else
#define LPROF(i) do { } while (0)
#endif
  for (int it = 0; it < a.iters; ++it) {
    long long* fs_cur = a.fsum + (size_t)(it % 3) * nsum;
    long long* fw_cur = a.fw + (size_t)(it % 3) * k2;
    // centres of this iteration from the previous iteration's sums (empty cluster: keep)
    if (it > 0) {
      const long long* fs_prev = a.fsum + (size_t)((it + 2) % 3) * nsum;
      const long long* fw_prev = a.fw + (size_t)((it + 2) % 3) * k2;
      // 1 / (weight_j * scale) once per cluster (0 marks an empty cluster), then one multiply per entry
      for (int j = tid; j < k2; j += blockDim.x) {
        const long long wj = __ldcg(fw_prev + j);
        winv[j] = wj > 0 ? scale_w / (static_cast<double>(wj) * scale) : 0.0;
      }
      __syncthreads();
      for (int e = tid; e < nsum; e += blockDim.x) {
        const int j = e / d, i = e - j * d;
        const double wi = winv[j];
        if (wi > 0) cs[j * cst + i] = static_cast<float>(static_cast<double>(__ldcg(fs_prev + e)) * wi);
      }
      // zero the slot the next iteration accumulates into (last read before the previous barrier)
      long long* fs_next = a.fsum + (size_t)((it + 1) % 3) * nsum;
      long long* fw_next = a.fw + (size_t)((it + 1) % 3) * k2;
      for (int64_t e = (int64_t)b * blockDim.x + tid; e < nsum + k2; e += (int64_t)G * blockDim.x) {
        if (e < nsum) fs_next[e] = 0;
        else fw_next[e - nsum] = 0;
      }
    }
    for (int e = tid; e < a.groups * k2 * d; e += blockDim.x) acc[e] = 0.f;
    for (int e = tid; e < a.groups * k2; e += blockDim.x) wacc[e] = 0.0;
    double obj = 0.0;
    int ties = 0;
    __syncthreads();
    LPROF(0);
    for (int64_t tile = t_beg; tile < t_end; ++tile) {
      const int64_t p0 = tile * kTileP;
      float* xt = xt_all;
      float* wts = wts_all;
      if (a.resident) {
        xt += (tile - t_beg) * d * kXt;
        wts += (tile - t_beg) * kTileP;
      } else {
        stage_tile(a, p0, xt, wts);
        __syncthreads();
      }
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
      LPROF(1);
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
    LPROF(2);
    // publish: groups combined in fixed order, added to the global sums in fixed point
    for (int e = tid; e < nsum; e += blockDim.x) {
      float s = acc[e];
      for (int g = 1; g < a.groups; ++g) s += acc[(size_t)g * nsum + e];
      if (s != 0.f) atomicAdd(reinterpret_cast<unsigned long long*>(fs_cur + e),
                              static_cast<unsigned long long>(llrint(static_cast<double>(s) * scale)));
    }
    for (int j = tid; j < k2; j += blockDim.x) {
      double s = wacc[j];
      for (int g = 1; g < a.groups; ++g) s += wacc[(size_t)g * k2 + j];
      if (s != 0.0) atomicAdd(reinterpret_cast<unsigned long long*>(fw_cur + j),
                              static_cast<unsigned long long>(llrint(s * scale_w)));
    }
    obj = warp_sum_d(obj);
    int tt = ties;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, o);
    if (lane == 0) { s_red[warp] = obj; s_tie[warp] = tt; }
    __syncthreads();
    if (tid == 0) {
      double s = 0;
      int q = 0;
      for (int w = 0; w < kLloydThreads / 32; ++w) { s += s_red[w]; q += s_tie[w]; }
      a.pobj[(size_t)it * G + b] = s;
      a.ptie[(size_t)it * G + b] = q;
    }
    LPROF(3);
    grid_barrier(a.gmax + 2, gen);
    LPROF(4);
  }
#ifdef CABS_PROFILE_LLOYD
  if (b == 0 && tid == 0)
    for (int i = 0; i < 5; ++i) a.prof[i] = prof[i];
#endif
  // ---------------- epilogue (CTA 0): final centres, cluster weights, objective history
  if (b == 0) {
    const long long* fs_last = a.fsum + (size_t)((a.iters - 1) % 3) * nsum;
    const long long* fw_last = a.fw + (size_t)((a.iters - 1) % 3) * k2;
    for (int e = tid; e < nsum; e += blockDim.x) {
      const int j = e / d, i = e - j * d;
      const long long wj = __ldcg(fw_last + j);
      a.centres[(int64_t)j * a.ldc + i] =
          wj > 0 ? static_cast<float>((static_cast<double>(__ldcg(fs_last + e)) / scale) /
                                      (static_cast<double>(wj) / scale_w))
                 : cs[j * cst + i];
    }
    for (int j = tid; j < k2; j += blockDim.x)
      a.cluster_w[j] = static_cast<double>(__ldcg(fw_last + j)) / scale_w;
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
                             float* centres, int64_t ldc, int* labels, double* objective, int* near_ties,
                             double* cluster_w, void* scratch, size_t scratch_bytes, long long* prof,
                             cudaStream_t st) {
  if (N <= 0) return false;
  const int dgroup = static_cast<int>(round_up(d < 256 ? d : 256, 32));
  const int groups = kLloydThreads / dgroup;
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
  const int64_t ntiles = ceil_div(N, kTileP);
  // grid: up to 2 CTAs per SM; X resident in smem when every CTA's tiles fit
  int64_t G = 0;
  int resident = 0, tpc = 1;
  size_t smem = 0;
  for (int per_sm = 2; per_sm >= 1 && G == 0; --per_sm) {
    int64_t g = (int64_t)nsm * per_sm;
    if (g > ntiles) g = ntiles;
    g = ceil_div(ntiles, ceil_div(ntiles, g));  // balanced: every CTA gets the same tile count (+-1)
    const int t = static_cast<int>(ceil_div(ntiles, g));
    size_t s_res = lloyd_smem(d, k2, groups, t).total;
    size_t s_str = lloyd_smem(d, k2, groups, 1).total;
    const size_t cap = per_sm == 2 ? kSmemCap / 2 - 8 * 1024 : kSmemCap;
    if (s_res <= cap) { G = g; resident = 1; tpc = t; smem = s_res; }
    else if (s_str <= cap) { G = g; resident = 0; tpc = t; smem = s_str; }
  }
  if (G == 0) return false;
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lloyd_persistent_kernel, kLloydThreads, smem);
  if (occ < 1) return false;
  if (G > (int64_t)occ * nsm) {
    G = (int64_t)occ * nsm;
    if (resident && ceil_div(ntiles, G) > tpc) {  // fewer CTAs than planned: stream the tiles instead
      resident = 0;
      smem = lloyd_smem(d, k2, groups, 1).total;
    }
    tpc = static_cast<int>(ceil_div(ntiles, G));
  }
  // scratch: fsum [3][k2*d] | fw [3][k2] | gmax [2] (+pad) | pobj [iters][G] | ptie [iters][G]
  const size_t nsum = (size_t)k2 * d;
  const size_t need = sizeof(long long) * (3 * nsum + 3 * k2) + 16 + (sizeof(double) + sizeof(int)) * iters * G;
  if (need > scratch_bytes) return false;
  char* base = static_cast<char*>(scratch);
  long long* fsum = reinterpret_cast<long long*>(base);
  long long* fw = fsum + 3 * nsum;
  unsigned* gmax = reinterpret_cast<unsigned*>(fw + 3 * k2);
  double* pobj = reinterpret_cast<double*>(gmax + 4);
  int* ptie = reinterpret_cast<int*>(pobj + (size_t)iters * G);
  if (cudaMemsetAsync(base, 0, sizeof(long long) * (3 * nsum + 3 * k2) + 16, st) != cudaSuccess) return false;
  LloydArgs a{X, ldx, N, d, k2, iters, w, centres, ldc, labels, objective, near_ties, cluster_w,
              fsum, fw, gmax, pobj, ptie, groups, dgroup, resident, tpc, prof};
  void* params[] = {&a};
  note_launch();
  cudaError_t e = cudaLaunchCooperativeKernel(reinterpret_cast<void*>(lloyd_persistent_kernel),
                                              dim3(static_cast<unsigned>(G)), dim3(kLloydThreads), params, smem, st);
  return e == cudaSuccess;
}

}  // namespace cabsk
