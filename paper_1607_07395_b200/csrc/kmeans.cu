// kmeans.cu -- S6/S7: weighted Lloyd k-means (Eq. 6; c iterations P:204).
//
// assign : s(l) = argmin_j ||X_l - c_j||^2 by DIRECT differences in FP32 (SURVEY F3:
//          the expanded form flips labels on clustered data), lowest j on ties;
//          objective partial sum_l w_l d_min in FP64 per CTA; near-tie count.
// accum  : exact int64 fixed-point sums of w_l X_l and w_l by label (km_fixed.cuh):
//          order-free, so identical to the persistent kernel (lloyd.cu).
// reduce : sums / 2^S -> one FP64 payload [k2*d sums | k2 weights | objective | near
//          ties] (the allreduce buffer); the integer sums are re-zeroed for the next pass.
// finalize: c_j = sums_j / weight_j, empty clusters keep their centre (Z12).
#include <float.h>
#include <limits.h>

#include "common.cuh"
#include "kernels.cuh"
#include "km_fixed.cuh"
#include "km_tile.cuh"

namespace cabsk {


// ---------------------------------------------------------------- weights
// Also the fixed-point bounds max|x| and max w (bounds[0], bounds[1]; km_fixed.cuh).
// blockIdx.y selects one of two jobs (the two sides of cabs_kmeans_pair in one launch).
__global__ void __launch_bounds__(256) km_weights_kernel(KmWeightJob j0, KmWeightJob j1, int kind, float p) {
  const KmWeightJob j = blockIdx.y == 0 ? j0 : j1;
  const float* __restrict__ X = j.X;
  const int64_t ldx = j.ldx, N = j.N;
  const int d = j.d;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int pos = 0;
  float mx = 0.f, mw = 0.f;
  for (int64_t l = warp; l < N; l += nw) {
    float ss = 0.f;
    for (int i = lane; i < d; i += 32) {
      float x = X[l * ldx + i];
      ss = fmaf(x, x, ss);
      mx = fmaxf(mx, fabsf(x));
    }
    ss = warp_sum_f(ss);
    float wl;
    if (kind == CABS_WEIGHT_CONST) wl = 1.f;
    else if (p == 2.f) wl = ss;
    else wl = powf(sqrtf(ss), p);
    if (lane == 0) {
      j.w[l] = wl;
      pos += wl > 0.f;
      mw = fmaxf(mw, wl);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  // block-level combine: one set of atomics per CTA (the bounds are maxima: order-free)
  __shared__ float s_mx[8], s_mw[8];
  __shared__ int s_pos[8];
  const int wib = threadIdx.x >> 5;
  if (lane == 0) { s_mx[wib] = mx; s_mw[wib] = mw; s_pos[wib] = pos; }
  __syncthreads();
  if (threadIdx.x == 0) {
    int tp = 0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { mx = fmaxf(mx, s_mx[q]); mw = fmaxf(mw, s_mw[q]); tp += s_pos[q]; }
    if (tp) atomicAdd(j.cnt, tp);
    atomicMax(j.bounds, __float_as_uint(mx));
    atomicMax(j.bounds + 1, __float_as_uint(mw));
  }
}

// Constant weights (CABS_WEIGHT_CONST): w = 1, cnt += N, bounds = {max|x|, 1} -- no per-point
// reduction; thread per 4 consecutive entries (16-byte loads when the rows allow), entries
// beyond d masked out.  blockIdx.y: job.
__global__ void __launch_bounds__(256) km_weights_const_kernel(KmWeightJob j0, KmWeightJob j1) {
  const KmWeightJob j = blockIdx.y == 0 ? j0 : j1;
  const int64_t N = j.N;
  const int d = j.d;
  const int q4 = (d + 3) >> 2;
  const bool vec = (j.ldx & 3) == 0 && (reinterpret_cast<uintptr_t>(j.X) & 15) == 0;
  float mx = 0.f;
  const int64_t total = N * q4;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = e / q4;
    const int i = static_cast<int>(e - l * q4) * 4;
    const float* row = j.X + l * j.ldx;
    float4 v;
    if (vec && i + 3 < d) {
      v = __ldg(reinterpret_cast<const float4*>(row + i));
    } else {
      v.x = row[i];
      v.y = i + 1 < d ? row[i + 1] : 0.f;
      v.z = i + 2 < d ? row[i + 2] : 0.f;
      v.w = i + 3 < d ? row[i + 3] : 0.f;
    }
    mx = fmaxf(mx, fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w))));
  }
  for (int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; l < N; l += (int64_t)gridDim.x * blockDim.x)
    j.w[l] = 1.f;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ float s_mx[8];
  if ((threadIdx.x & 31) == 0) s_mx[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) mx = fmaxf(mx, s_mx[q]);
    atomicMax(j.bounds, __float_as_uint(mx));
    if (blockIdx.x == 0) {
      if (N > 0) atomicAdd(j.cnt, static_cast<int>(N));
      atomicMax(j.bounds + 1, __float_as_uint(N > 0 ? 1.f : 0.f));
    }
  }
}

void launch_km_weights2(const KmWeightJob& j0, const KmWeightJob* j1, int kind, float p, cudaStream_t st) {
  const int64_t N1 = j1 ? j1->N : 0;
  const int64_t N = j0.N > N1 ? j0.N : N1;
  if (N <= 0) return;
  if (kind == CABS_WEIGHT_CONST) {
    int64_t blocks = ceil_div(N * 16, 256);
    if (blocks > 2 * kNumSM) blocks = 2 * kNumSM;
    note_launch();
    km_weights_const_kernel<<<dim3(static_cast<unsigned>(blocks), j1 ? 2 : 1), 256, 0, st>>>(j0, j1 ? *j1 : j0);
    return;
  }
  int64_t blocks = ceil_div(N, 8);
  if (blocks > 2 * kNumSM) blocks = 2 * kNumSM;
  note_launch();
  km_weights_kernel<<<dim3(static_cast<unsigned>(blocks), j1 ? 2 : 1), 256, 0, st>>>(j0, j1 ? *j1 : j0, kind, p);
}

void launch_km_weights(const float* X, int64_t ldx, int64_t N, int d, int kind, float p, float* w, int* cnt,
                       unsigned* bounds, cudaStream_t st) {
  const KmWeightJob j{X, ldx, N, d, w, cnt, bounds};
  launch_km_weights2(j, nullptr, kind, p, st);
}

// ---------------------------------------------------------------- init
// centres[j] = X[idx[j]] if this rank owns that row (zeros otherwise: the
// caller's sum-allreduce completes it), or a copy of init_c.  blockIdx.y: job.
__global__ void km_init_kernel(KmInitJob j0, KmInitJob j1) {
  const KmInitJob jb = blockIdx.y == 0 ? j0 : j1;
  const int j = blockIdx.x;
  if (j >= jb.k2) return;
  const float* src = nullptr;
  if (jb.init_c) src = jb.init_c + (int64_t)j * jb.ldic;
  else {
    int64_t g = jb.idx[j] - jb.row_off;
    if (g >= 0 && g < jb.n_loc) src = jb.X + g * jb.ldx;
  }
  // a centre another rank owns starts as -0.0 (bit-exact sum-allreduce, see fill_neg_zero_kernel)
  for (int i = threadIdx.x; i < jb.ldc; i += blockDim.x)
    jb.centres[(int64_t)j * jb.ldc + i] = (src && i < jb.d) ? src[i] : (i < jb.d ? -0.f : 0.f);
}

void launch_km_init2(const KmInitJob& j0, const KmInitJob* j1, cudaStream_t st) {
  const int k1 = j1 ? j1->k2 : 0;
  const int kx = j0.k2 > k1 ? j0.k2 : k1;
  note_launch();
  km_init_kernel<<<dim3(kx, j1 ? 2 : 1), 128, 0, st>>>(j0, j1 ? *j1 : j0);
}

void launch_km_init(const float* X, int64_t ldx, int64_t n_loc, int64_t row_off, int d, int k2, const int64_t* idx,
                    const float* init_c, int64_t ldic, float* centres, int64_t ldc, cudaStream_t st) {
  const KmInitJob j{X, ldx, n_loc, row_off, d, k2, idx, init_c, ldic, centres, ldc};
  launch_km_init2(j, nullptr, st);
}

// ---------------------------------------------------------------- assign / distance matrix
// Tile: 64 points x 64 centres; thread (tp = tid & 15, tc = tid >> 4) owns points
// tp + 16a and centres tc + 16b (a, b = 0..3).  Dimensions are staged 16 at a time;
// every distance is accumulated over i = 0..d-1 in ascending order (km_tile.cuh).
template <bool DISTMAT>
__global__ void __launch_bounds__(256) km_assign_kernel(const float* __restrict__ X, int64_t ldx, int64_t N, int d,
                                                        const float* __restrict__ centres, int64_t ldc, int k2,
                                                        const float* __restrict__ w, int* __restrict__ labels,
                                                        double* __restrict__ pobj, int* __restrict__ ptie,
                                                        float* __restrict__ D, int64_t ldd, int* tie_log, int tie_cap,
                                                        int it, int64_t row_off) {
  __shared__ KmTileSmem sm;
  __shared__ int lab_s[kTileP], j2_s[kTileP];
  __shared__ float d1_s[kTileP], d2_s[kTileP];
  __shared__ double s_red[8];
  __shared__ int s_tie[8];
  const int tid = threadIdx.x;
  const int64_t ntiles = ceil_div(N, kTileP);
  double obj = 0.0;
  int ties = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t p0 = tile * kTileP;
    if (DISTMAT) {
      km_tile_distmat(X, ldx, N, d, centres, ldc, k2, p0, sm, D, ldd);
    } else {
      km_tile_argmin<false>(X, ldx, N, d, centres, ldc, k2, p0, sm, lab_s, d1_s, d2_s, j2_s);
      if (tid < kTileP) {
        const int64_t p = p0 + tid;
        if (p < N) {
          const float B = d1_s[tid], S = d2_s[tid];
          labels[p] = lab_s[tid];
          obj += static_cast<double>(w[p]) * static_cast<double>(B);
          const bool tie = (S - B) < kNearTie * S;
          ties += tie;
          if (tie && tie_log) km_log_tie(tie_log, tie_cap, it, row_off + p, lab_s[tid], j2_s[tid], B, S);
        }
      }
      __syncthreads();
    }
  }
  if (!DISTMAT) {
    obj = warp_sum_d(obj);
    int t = ties;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if ((tid & 31) == 0) {
      s_red[tid >> 5] = obj;
      s_tie[tid >> 5] = t;
    }
    __syncthreads();
    if (tid == 0) {
      double s = 0;
      int tt = 0;
      for (int q = 0; q < 8; ++q) { s += s_red[q]; tt += s_tie[q]; }
      pobj[blockIdx.x] = s;
      ptie[blockIdx.x] = tt;
    }
  }
}

static int assign_grid(int64_t N) {
  int64_t t = ceil_div(N, kTileP);
  if (t > kAssignGrid) t = kAssignGrid;
  return static_cast<int>(t < 1 ? 1 : t);
}

void launch_km_assign(const float* X, int64_t ldx, int64_t N, int d, const float* centres, int64_t ldc, int k2,
                      const float* w, int* labels, double* pobj, int* ptie, int* grid_out, cudaStream_t st,
                      int* tie_log, int tie_cap, int it, int64_t row_off) {
  const int g = assign_grid(N);
  *grid_out = g;
  note_launch();
  km_assign_kernel<false><<<g, 256, 0, st>>>(X, ldx, N, d, centres, ldc, k2, w, labels, pobj, ptie, nullptr, 0, tie_log,
                                             tie_cap, it, row_off);
}

void launch_km_distmat(const float* X, int64_t ldx, int64_t N, int d, const float* centres, int64_t ldc, int k2,
                       float* D, int64_t ldd, cudaStream_t st) {
  if (N <= 0) return;
  const int g = assign_grid(N);
  note_launch();
  km_assign_kernel<true><<<g, 256, 0, st>>>(X, ldx, N, d, centres, ldc, k2, nullptr, nullptr, nullptr, nullptr, D, ldd,
                                            nullptr, 0, 0, 0);
}

// ---------------------------------------------------------------- accumulate
// CTA b takes tiles b, b + G, ... of 64 points; each tile is bucketed by label and added
// to the global int64 sums (km_fixed.cuh).
__global__ void __launch_bounds__(256) km_accum_kernel(const float* __restrict__ X, int64_t ldx, int64_t N, int d,
                                                       const int* __restrict__ labels, const float* __restrict__ w,
                                                       const unsigned* bounds, long long* fsum, long long* fw) {
  extern __shared__ float xs[];  // [d][64]
  __shared__ __align__(16) int lab_s[kTileP];
  __shared__ int order_s[kTileP], slab_s[kTileP], ustart_s[kTileP + 1], ucl_s[kTileP];
  __shared__ float wts[kTileP];
  __shared__ unsigned smask_s[8];
  __shared__ int nu_s;
  double scale, scale_w;
  fx_scales(bounds, N, scale, scale_w);
  const int64_t ntiles = ceil_div(N, kTileP);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t p0 = t * kTileP;
    const int np = static_cast<int>(N - p0 < kTileP ? N - p0 : kTileP);
    for (int e = threadIdx.x; e < np * d; e += blockDim.x) {
      const int pp = e / d, i = e - pp * d;
      xs[i * kTileP + pp] = __ldg(X + (p0 + pp) * ldx + i);
    }
    for (int pp = threadIdx.x; pp < kTileP; pp += blockDim.x) {
      lab_s[pp] = pp < np ? labels[p0 + pp] : INT_MAX;
      wts[pp] = pp < np ? w[p0 + pp] : 0.f;
    }
    __syncthreads();
    fx_tile_accumulate(
        np, lab_s, wts, [&](int i, int p) { return xs[i * kTileP + p]; }, d, scale, scale_w,
        [&](int e, long long v) { if (v != 0) red_add_u64(fsum + e, v); },
        [&](int j, long long v) { if (v != 0) red_add_u64(fw + j, v); }, order_s, slab_s, ustart_s, ucl_s, smask_s,
        &nu_s);
  }
}

void launch_km_accum(const float* X, int64_t ldx, int64_t N, int d, const int* labels, const float* w,
                     const unsigned* bounds, long long* fsum, long long* fw, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(km_accum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr = true;
  }
  int64_t G = ceil_div(N, kTileP);
  if (G > 4 * kNumSM) G = 4 * kNumSM;
  if (G < 1) G = 1;
  note_launch();
  km_accum_kernel<<<static_cast<unsigned>(G), 256, sizeof(float) * (size_t)d * kTileP, st>>>(X, ldx, N, d, labels, w,
                                                                                             bounds, fsum, fw);
}

// ---------------------------------------------------------------- reduce
// red = [k2*d sums | k2 weights | objective | near ties]: integer sums / 2^S (then zeroed
// for the next pass); objective / near ties as fixed-order FP64 sums over the assign CTAs
// (8 lanes per element, lane l sums CTAs l, l+8, ..., xor-butterfly combine).
__global__ void km_reduce_kernel(long long* fsum, long long* fw, const unsigned* bounds, int64_t N, int k2, int d,
                                 const double* __restrict__ pobj, const int* __restrict__ ptie, int Gobj,
                                 double* __restrict__ red) {
  const int64_t nsum = (int64_t)k2 * d;
  double scale, scale_w;
  fx_scales(bounds, N, scale, scale_w);
  const int64_t gt = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (gt < nsum) {
    red[gt] = static_cast<double>(fsum[gt]) / scale;
    fsum[gt] = 0;
  } else if (gt < nsum + k2) {
    red[gt] = static_cast<double>(fw[gt - nsum]) / scale_w;
    fw[gt - nsum] = 0;
  }
  if (blockIdx.x == 0 && threadIdx.x < 16) {  // two 8-lane groups: objective, near ties
    const int sub = threadIdx.x & 7;
    double s = 0.0;
    if (threadIdx.x < 8) {
      for (int b = sub; b < Gobj; b += 8) s += pobj[b];
    } else {
      for (int b = sub; b < Gobj; b += 8) s += static_cast<double>(ptie[b]);
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffu, s, o);
    if (sub == 0) red[nsum + k2 + (threadIdx.x >> 3)] = s;
  }
}

void launch_km_reduce(long long* fsum, long long* fw, const unsigned* bounds, int64_t N, int k2, int d,
                      const double* pobj, const int* ptie, int Gobj, double* red, cudaStream_t st) {
  const int64_t total = (int64_t)k2 * d + k2;
  note_launch();
  km_reduce_kernel<<<static_cast<unsigned>(ceil_div(total, 256)), 256, 0, st>>>(fsum, fw, bounds, N, k2, d, pobj, ptie,
                                                                                 Gobj, red);
}

__global__ void km_finalize_kernel(const double* __restrict__ red, int k2, int d, float* __restrict__ centres,
                                   int64_t ldc, double* __restrict__ objective, int* __restrict__ near_ties,
                                   double* __restrict__ cluster_w, int t) {
  const int64_t nsum = (int64_t)k2 * d;
  const double* wts = red + nsum;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nsum; e += (int64_t)gridDim.x * blockDim.x) {
    const int j = static_cast<int>(e / d), i = static_cast<int>(e % d);
    const double wj = wts[j];
    if (wj > 0) centres[(int64_t)j * ldc + i] = static_cast<float>(red[e] * (1.0 / wj));  // = lloyd.cu
  }
  if (blockIdx.x == 0) {
    for (int j = threadIdx.x; j < k2; j += blockDim.x)
      if (cluster_w) cluster_w[j] = wts[j];
    if (threadIdx.x == 0) {
      if (objective) objective[t] = red[nsum + k2];
      if (near_ties) near_ties[t] = static_cast<int>(red[nsum + k2 + 1]);
    }
  }
}

void launch_km_finalize(const double* red, int k2, int d, float* centres, int64_t ldc, double* objective,
                        int* near_ties, double* cluster_w, int t, cudaStream_t st) {
  int64_t blocks = ceil_div((int64_t)k2 * d, 256);
  if (blocks > 4 * kNumSM) blocks = 4 * kNumSM;
  if (blocks < 1) blocks = 1;
  note_launch();
  km_finalize_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(red, k2, d, centres, ldc, objective, near_ties,
                                                                     cluster_w, t);
}

}  // namespace cabsk
