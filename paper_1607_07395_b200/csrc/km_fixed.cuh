// km_fixed.cuh -- exact, order-free accumulation of the weighted Lloyd sums (Eq. 6,
// P:166-169): sum_{l in cluster j} w_l X_l and sum_{l in cluster j} w_l.
//
// Every product w_l x_li is formed exactly in FP64 (24 x 24 bits), scaled by 2^S and
// rounded once to int64; the sums are then integer additions, so they do not depend on
// the order or the grouping of the points (CTA count, tile size, atomics order, number
// of ranks): deterministic run to run and identical between the persistent kernel and
// the per-iteration kernels.  S is the largest exponent with N * max w * max|x| * 2^S
// < 2^61, so no partial or total sum can overflow; the resolution 2^-S is ~2^-61 of that
// global bound (far below FP32 centre precision).
#pragma once
#include "common.cuh"

namespace cabsk {

__device__ __forceinline__ int fx_scale_exp(double bound) {
  if (!(bound > 0)) return 60;
  const int e = static_cast<int>(ceil(log2(bound)));
  const int S = 61 - e;
  return S < 0 ? 0 : (S > 60 ? 60 : S);
}

// bounds[0] = max|x| bits, bounds[1] = max w bits (non-negative floats order as uints).
// S also keeps every single product below 2^50, so that it can be rounded to an integer by
// the FP64 magic-number addition (fx_prod_magic) as well as by llrint.
__device__ __forceinline__ void fx_scales(const unsigned* bounds, int64_t N, double& scale, double& scale_w) {
  const double xmax = static_cast<double>(__uint_as_float(__ldcg(bounds)));
  const double wmax = static_cast<double>(__uint_as_float(__ldcg(bounds + 1)));
  int S = fx_scale_exp(static_cast<double>(N) * wmax * xmax);
  const int S1 = fx_scale_exp(wmax * xmax) - 11;  // per product < 2^50
  if (S1 < S) S = S1 < 0 ? 0 : S1;
  scale = ldexp(1.0, S);
  scale_w = ldexp(1.0, fx_scale_exp(static_cast<double>(N) * wmax));
}

// llrint(ws * x) for |ws * x| < 2^51 (round half to even): one FP64 FMA against 1.5 * 2^52
// and an integer subtraction of the bit patterns.  ws = w * 2^S (exact), so ws * x is the
// exact product and the result equals fx_prod(w, x, 2^S).
__device__ __forceinline__ long long fx_prod_magic(double ws, float x) {
  constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  return __double_as_longlong(fma(ws, static_cast<double>(x), kMagic)) - __double_as_longlong(kMagic);
}

__device__ __forceinline__ long long fx_prod(float w, float x, double scale) {
  return llrint(static_cast<double>(w) * static_cast<double>(x) * scale);
}

__device__ __forceinline__ void red_add_u64(long long* p, long long v) {
  asm volatile("red.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Stable bucket of the np <= 256 points of a tile by label: order[pos] = point, slab[pos] =
// its label, then the compact list of the non-empty clusters: ucl[u] = label, points
// order[ustart[u] .. ustart[u+1]).  lab must be padded with INT_MAX to a multiple of 4
// entries (read as int4).  Scratch smask[8]; returns nu (block-uniform).  Block-wide
// (blockDim a multiple of 32), ends synchronised.
__device__ __forceinline__ int fx_bucket(int np, const int* lab, int* order, int* slab, int* ustart, int* ucl,
                                         unsigned* smask, int* s_nu) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int4* lab4 = reinterpret_cast<const int4*>(lab);
  for (int p = tid; p < np; p += nt) {  // stable rank of point p by (label, index)
    const int l = lab[p];
    int pos = 0;
    for (int q4 = 0; q4 < (np + 3) >> 2; ++q4) {
      const int4 v = lab4[q4];
      const int q = 4 * q4;
      pos += (v.x < l) || (v.x == l && q < p);
      pos += (v.y < l) || (v.y == l && q + 1 < p);
      pos += (v.z < l) || (v.z == l && q + 2 < p);
      pos += (v.w < l) || (v.w == l && q + 3 < p);
    }
    order[pos] = p;
    slab[pos] = l;
  }
  __syncthreads();
  const int ng = (np + 31) >> 5;
  for (int q = tid; q < 32 * ng; q += nt) {
    const bool start = q < np && (q == 0 || slab[q] != slab[q - 1]);
    const unsigned m = __ballot_sync(0xffffffffu, start);
    if ((q & 31) == 0) smask[q >> 5] = m;
  }
  __syncthreads();
  for (int q = tid; q < np; q += nt) {
    if (q == 0 || slab[q] != slab[q - 1]) {
      int rank = __popc(smask[q >> 5] & ((1u << (q & 31)) - 1u));
      for (int g = 0; g < (q >> 5); ++g) rank += __popc(smask[g]);
      ucl[rank] = slab[q];
      ustart[rank] = q;
    }
  }
  if (tid == 0) {
    int nu = 0;
    for (int g = 0; g < ng; ++g) nu += __popc(smask[g]);
    ustart[nu] = np;
    *s_nu = nu;
  }
  __syncthreads();
  return *s_nu;
}

// Per-tile bucket (fx_bucket), then ONE integer per (non-empty cluster, dimension) of the
// tile handed to sink_sum(j * d + i, v) and one per non-empty cluster to sink_w(j, v).
// wts: the tile's weights (0 for padding points); xat(i, p): coordinate i of point p.
// Four (cluster, dimension) sums per thread are advanced together so that their dependent
// load -> convert -> add chains overlap.  Ends synchronised.
template <class XAT, class SINK, class SINKW>
__device__ __forceinline__ void fx_tile_accumulate(int np, const int* lab, const float* wts, XAT xat, int d,
                                                   double scale, double scale_w, SINK sink_sum, SINKW sink_w,
                                                   int* order, int* slab, int* ustart, int* ucl, unsigned* smask,
                                                   int* s_nu) {
  const int tid = threadIdx.x, nt = blockDim.x;
  fx_bucket(np, lab, order, slab, ustart, ucl, smask, s_nu);
  const int nu = *s_nu, ne = nu * d;
  constexpr int R = 4;
  for (int e0 = tid; e0 < ne; e0 += R * nt) {  // consecutive threads: consecutive clusters
    int q[R], qe[R], ii[R];
    long long s[R];
    int len = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = e0 + r * nt;
      const int i = e / nu, u = e - i * nu;
      const bool ok = e < ne;
      q[r] = ok ? ustart[u] : 0;
      qe[r] = ok ? ustart[u + 1] : 0;
      ii[r] = i;
      s[r] = 0;
      len = max(len, qe[r] - q[r]);
    }
    for (int t = 0; t < len; ++t) {
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (q[r] + t < qe[r]) {
          const int p = order[q[r] + t];
          s[r] += fx_prod(wts[p], xat(ii[r], p), scale);
        }
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int e = e0 + r * nt;
      if (e < ne) {
        const int i = e / nu, u = e - i * nu;
        sink_sum(ucl[u] * d + i, s[r]);
      }
    }
  }
  for (int u = tid; u < nu; u += nt) {
    long long s = 0;
    for (int q = ustart[u]; q < ustart[u + 1]; ++q) s += llrint(static_cast<double>(wts[order[q]]) * scale_w);
    sink_w(ucl[u], s);
  }
  __syncthreads();
}

}  // namespace cabsk
