// km_tile.cuh -- the 64-point x all-centres distance tile shared by the k-means kernels.
// Squared distances by DIRECT differences in FP32, dimensions in ascending order
// (the same arithmetic in every kernel, so labels never depend on the launch shape).
#pragma once
#include <float.h>

#include "common.cuh"

namespace cabsk {

constexpr int kTileP = 64, kTileC = 64, kTileD = 16;
constexpr float kNearTie = 1e-5f;  // north_star near-tie rule: relative gap (d2 - d1)/d2 < 1e-5

// one entry of a near-tie log (int32 [0] = count of near ties seen, then per entry: iteration,
// global point index, nearest centre, runner-up centre, relative gap (FP32 bits)); entries past
// cap are counted, not stored
__device__ __forceinline__ void km_log_tie(int* log, int cap, int it, int64_t p, int j1, int j2, float d1, float d2) {
  const int slot = atomicAdd(log, 1);
  if (slot < cap) {
    int* e = log + 1 + 5 * slot;
    e[0] = it;
    e[1] = static_cast<int>(p);
    e[2] = j1;
    e[3] = j2;
    e[4] = __float_as_int(d2 > 0.f ? (d2 - d1) / d2 : 0.f);
  }
}

struct KmTileSmem {
  __align__(16) float Xs[kTileD][kTileP + 4];  // rows of 68 floats: 16-byte aligned float4 reads
  __align__(16) float Cs[kTileD][kTileC + 4];
  float sb_d[16][kTileP + 1];
  int sb_j[16][kTileP + 1];
  float ss_d[16][kTileP + 1];
  int ss_j[16][kTileP + 1];
};

// centres may be rewritten by other CTAs inside a persistent kernel: COHERENT loads
// them through L2 only (ld.global.cg) instead of the read-only path.
template <bool COHERENT>
__device__ __forceinline__ float ld_centre(const float* p) {
  if (COHERENT) return __ldcg(p);
  return __ldg(p);
}

__device__ __forceinline__ unsigned long long kt_dup(float x) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ unsigned long long kt_pack(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}

// acc[a][b] = ||X_{p0 + 4 tp + a} - c_{j0 + 4 tc + b}||^2 for one 64 x 64 block: per dimension
// one 16-byte shared-memory read of the thread's four point values and one of its four centre
// values, and the 16 (point, centre) terms as packed FP32 pairs (sub.rn.f32x2 / fma.rn.f32x2:
// per lane the IEEE results of FADD / FFMA, so every distance is the same ascending-dimension
// fmaf chain as a scalar loop).
template <bool COHERENT>
__device__ __forceinline__ void km_tile_block(const float* __restrict__ X, int64_t ldx, int64_t N, int d,
                                              const float* __restrict__ centres, int64_t ldc, int k2, int64_t p0,
                                              int j0, KmTileSmem& sm, float (&acc)[4][4]) {
  const int tid = threadIdx.x, tp = tid & 15, tc = tid >> 4;
  unsigned long long acc2[4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a) acc2[a][0] = acc2[a][1] = 0ull;
  // stage i0 + kTileD is loaded into registers while stage i0 is computed from shared memory
  const int pp = tid >> 2, ii = (tid & 3) * 4;
  const int64_t p = p0 + pp;
  const int jr = j0 + pp;
  float xr[4], cr[4];
  auto load_stage = [&](int i0) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int i = i0 + ii + q;
      xr[q] = (p < N && i < d) ? __ldg(X + p * ldx + i) : 0.f;
      cr[q] = (jr < k2 && i < d) ? ld_centre<COHERENT>(centres + (int64_t)jr * ldc + i) : 0.f;
    }
  };
  load_stage(0);
  for (int i0 = 0; i0 < d; i0 += kTileD) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      sm.Xs[ii + q][pp] = xr[q];
      sm.Cs[ii + q][pp] = cr[q];
    }
    __syncthreads();
    if (i0 + kTileD < d) load_stage(i0 + kTileD);
#pragma unroll
    for (int ii2 = 0; ii2 < kTileD; ++ii2) {
      const float4 xv = *reinterpret_cast<const float4*>(&sm.Xs[ii2][4 * tp]);
      const float4 cv = *reinterpret_cast<const float4*>(&sm.Cs[ii2][4 * tc]);
      const unsigned long long c01 = kt_pack(cv.x, cv.y), c23 = kt_pack(cv.z, cv.w);
      const float xa[4] = {xv.x, xv.y, xv.z, xv.w};
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const unsigned long long x2 = kt_dup(xa[a]);
        unsigned long long df;
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(df) : "l"(x2), "l"(c01));
        asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc2[a][0]) : "l"(df));
        asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(df) : "l"(x2), "l"(c23));
        asm("fma.rn.f32x2 %0, %1, %1, %0;" : "+l"(acc2[a][1]) : "l"(df));
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    acc[a][0] = __uint_as_float(static_cast<unsigned>(acc2[a][0]));
    acc[a][1] = __uint_as_float(static_cast<unsigned>(acc2[a][0] >> 32));
    acc[a][2] = __uint_as_float(static_cast<unsigned>(acc2[a][1]));
    acc[a][3] = __uint_as_float(static_cast<unsigned>(acc2[a][1] >> 32));
  }
}

// Nearest centre (lowest index on ties), its distance and the runner-up distance for the
// 64 points starting at p0 -> lab_s, d1_s, d2_s (shared).  Block-wide; ends synchronised.
template <bool COHERENT>
__device__ __forceinline__ void km_tile_argmin(const float* __restrict__ X, int64_t ldx, int64_t N, int d,
                                               const float* __restrict__ centres, int64_t ldc, int k2, int64_t p0,
                                               KmTileSmem& sm, int* lab_s, float* d1_s, float* d2_s, int* j2_s) {
  const int tid = threadIdx.x, tp = tid & 15, tc = tid >> 4;
  float bd[4], sd[4];
  int bj[4], sj[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) { bd[a] = FLT_MAX; sd[a] = FLT_MAX; bj[a] = 0x7fffffff; sj[a] = -1; }
  for (int j0 = 0; j0 < k2; j0 += kTileC) {
    float acc[4][4];
    km_tile_block<COHERENT>(X, ldx, N, d, centres, ldc, k2, p0, j0, sm, acc);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = j0 + 4 * tc + b;
      if (j >= k2) continue;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const float v = acc[a][b];
        if (v < bd[a] || (v == bd[a] && j < bj[a])) {
          sd[a] = bd[a];
          sj[a] = bj[a];
          bd[a] = v;
          bj[a] = j;
        } else if (v < sd[a]) {
          sd[a] = v;
          sj[a] = j;
        }
      }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    sm.sb_d[tc][4 * tp + a] = bd[a];
    sm.sb_j[tc][4 * tp + a] = bj[a];
    sm.ss_d[tc][4 * tp + a] = sd[a];
    sm.ss_j[tc][4 * tp + a] = sj[a];
  }
  __syncthreads();
  if (tid < kTileP) {
    float B = sm.sb_d[0][tid], S = sm.ss_d[0][tid];
    int Bj = sm.sb_j[0][tid], Sj = sm.ss_j[0][tid];
    for (int t = 1; t < 16; ++t) {
      const float b2 = sm.sb_d[t][tid], s2 = sm.ss_d[t][tid];
      const int j2 = sm.sb_j[t][tid], sj2 = sm.ss_j[t][tid];
      if (b2 < B || (b2 == B && j2 < Bj)) {
        if (B < s2) { S = B; Sj = Bj; } else { S = s2; Sj = sj2; }
        B = b2;
        Bj = j2;
      } else {
        if (b2 < S) { S = b2; Sj = j2; }
        if (s2 < S) { S = s2; Sj = sj2; }
      }
    }
    lab_s[tid] = Bj;
    d1_s[tid] = B;
    d2_s[tid] = S;
    if (j2_s) j2_s[tid] = Sj;
  }
  __syncthreads();
}

// D[j, p] for the 64 points starting at p0 and every centre.
__device__ __forceinline__ void km_tile_distmat(const float* __restrict__ X, int64_t ldx, int64_t N, int d,
                                                const float* __restrict__ centres, int64_t ldc, int k2, int64_t p0,
                                                KmTileSmem& sm, float* __restrict__ D, int64_t ldd) {
  const int tid = threadIdx.x, tp = tid & 15, tc = tid >> 4;
  for (int j0 = 0; j0 < k2; j0 += kTileC) {
    float acc[4][4];
    km_tile_block<false>(X, ldx, N, d, centres, ldc, k2, p0, j0, sm, acc);
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int j = j0 + 4 * tc + b;
      if (j >= k2) continue;
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int64_t p = p0 + 4 * tp + a;
        if (p < N) D[(int64_t)j * ldd + p] = acc[a][b];
      }
    }
  }
}

}  // namespace cabsk
