// Micro-timings of the persistent Lloyd kernel's per-iteration phases on one CTA (256 threads):
// centre formation from the int64 sums (conversion variants) and the owned-cluster
// accumulation, c2 shapes (d = 50, k2 = 50, 135 points).  Build:
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_lloyd tools/ubench_lloyd.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int D = 50, K2 = 50, NP = 135, P = 145;
__device__ __forceinline__ int cpair_idx(int j, int i, int d) {
  const int jj = j & 63;
  return ((((j >> 6) * d + i) * 2 + (jj >> 5)) * 16 + (jj & 15)) * 2 + ((jj >> 4) & 1);
}
__device__ __forceinline__ long long fx_prod_magic(double ws, float x) {
  constexpr double kMagic = 6755399441055744.0;
  return __double_as_longlong(fma(ws, static_cast<double>(x), kMagic)) - __double_as_longlong(kMagic);
}
template <int V>
__global__ void centres(const long long* gpart, float* out, long long* cyc) {
  __shared__ long long part[K2 * D + K2];
  __shared__ double wd[K2];
  __shared__ float cs[64 * D];
  const int tid = threadIdx.x;
  for (int e = tid; e < K2 * D + K2; e += 256) part[e] = gpart[e];
  for (int j = tid; j < K2; j += 256) wd[j] = 1.0 / (double)(part[K2 * D + j] + 1);
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    const int rows = 256 / D;
    if (tid < rows * D) {
      const int jr = tid / D, i = tid - jr * D;
#pragma unroll 4
      for (int j = jr; j < K2; j += rows) {
        const double rw = wd[j];
        const long long v = part[j * D + i];
        double dv;
        if (V == 0) dv = static_cast<double>(v);
        else dv = fma(static_cast<double>(static_cast<int>(v >> 32)), 4294967296.0, static_cast<double>(static_cast<unsigned>(v)));
        if (rw > 0) cs[cpair_idx(j, i, D)] = static_cast<float>((dv * 0x1p-40) * rw);
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[0] = (t1 - t0) / 4;
  for (int e = tid; e < 64 * D; e += 256) out[e] = cs[e];
}
__global__ void accum(const int* glab, const float* gx, long long* gout, long long* cyc) {
  extern __shared__ float xs[];
  __shared__ double wsc[P];
  __shared__ long long iw[P];
  __shared__ int lab[NP];
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < D * P; e += 256) xs[e] = gx[e];
  for (int p = tid; p < P; p += 256) { wsc[p] = 0x1p30; iw[p] = 1 << 20; }
  for (int p = tid; p < NP; p += 256) lab[p] = glab[p];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    constexpr int NB = 5;
    int labr[NB];
#pragma unroll
    for (int t = 0; t < NB; ++t) labr[t] = lane + 32 * t < NP ? lab[lane + 32 * t] : -1;
    for (int j = warp; j < K2; j += 8) {
      const int ia = lane, ib = 32 + lane;
      long long sa = 0, sb = 0, sw = 0;
#pragma unroll
      for (int t = 0; t < NB; ++t) {
        unsigned m = __ballot_sync(0xffffffffu, labr[t] == j);
        while (m) {
          const int p = 32 * t + __ffs(m) - 1;
          m &= m - 1;
          const double ws = wsc[p];
          if (ia < D) sa += fx_prod_magic(ws, xs[ia * P + p]);
          if (ib < D) sb += fx_prod_magic(ws, xs[ib * P + p]);
          sw += iw[p];
        }
      }
      if (ia < D) part[j * D + ia] = sa;
      if (ib < D) part[j * D + ib] = sb;
      if (lane == 0) part[K2 * D + j] = sw;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[1] = (t1 - t0) / 4;
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}
// counting sort of the chunk by label, then warp w sums clusters j = w mod 8, lanes over
// dimensions, four points of the cluster's contiguous list per step (independent loads)
__global__ void accum2(const int* glab, const float* gx, long long* gout, long long* cyc) {
  extern __shared__ float xs[];
  __shared__ double wsc[P];
  __shared__ long long iw[P];
  __shared__ int lab[NP], order[NP], cnt[K2 + 1], pos[K2];
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < D * P; e += 256) xs[e] = gx[e];
  for (int p = tid; p < P; p += 256) { wsc[p] = 0x1p30; iw[p] = 1 << 20; }
  for (int p = tid; p < NP; p += 256) lab[p] = glab[p];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    for (int j = tid; j < K2; j += 256) cnt[j] = 0;
    __syncthreads();
    int myl = tid < NP ? lab[tid] : -1;
    if (myl >= 0) atomicAdd(&cnt[myl], 1);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the counts -> list starts (pos) and ends (cnt)
      int run = 0;
      for (int j0 = 0; j0 < K2; j0 += 32) {
        const int j = j0 + lane;
        const int c = j < K2 ? cnt[j] : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int t = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += t; }
        if (j < K2) { pos[j] = run + inc - c; cnt[j] = run + inc; }
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    if (myl >= 0) order[atomicAdd(&pos[myl], 1)] = tid;  // pos[j] ends at the list end
    __syncthreads();
    if (tid == 0 && rep == 3) cyc[4] = clock64() - t0;
    const long long tw0 = clock64();
    for (int j = warp; j < K2; j += 8) {
      const int q1 = cnt[j], q0 = j > 0 ? cnt[j - 1] : 0;
      const int ia = lane, ib = 32 + lane;
      long long sa = 0, sb = 0, sw = 0;
      for (int q = q0; q < q1; q += 4) {
        int pp[4]; double wv[4]; float xa[4], xb[4]; long long iv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pp[u] = q + u < q1 ? order[q + u] : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = q + u < q1;
          wv[u] = ok ? wsc[pp[u]] : 0.0;
          iv[u] = ok ? iw[pp[u]] : 0;
          xa[u] = ia < D ? xs[ia * P + pp[u]] : 0.f;
          xb[u] = ib < D ? xs[ib * P + pp[u]] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) { sa += fx_prod_magic(wv[u], xa[u]); sb += fx_prod_magic(wv[u], xb[u]); sw += iv[u]; }
      }
      if (ia < D) part[j * D + ia] = sa;
      if (ib < D) part[j * D + ib] = sb;
      if (lane == 0) part[K2 * D + j] = sw;
    }
    if (rep == 3 && lane == 0) cyc[8 + warp] = clock64() - tw0;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[2] = (t1 - t0) / 4;
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}
template <int MODE>
__global__ void accum4(const int* glab, const float* gx, long long* gout, long long* cyc) {
  extern __shared__ float xs[];
  __shared__ double wsc[P];
  __shared__ long long iw[P];
  __shared__ int lab[NP], order[NP], cnt[K2 + 1], pos[K2];
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < D * P; e += 256) xs[e] = gx[e];
  for (int p = tid; p < P; p += 256) { wsc[p] = 0x1p30; iw[p] = 1 << 20; }
  for (int p = tid; p < NP; p += 256) lab[p] = glab[p];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    for (int j = tid; j < K2; j += 256) cnt[j] = 0;
    __syncthreads();
    int myl = tid < NP ? lab[tid] : -1;
    if (myl >= 0) atomicAdd(&cnt[myl], 1);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the counts -> list starts (pos) and ends (cnt)
      int run = 0;
      for (int j0 = 0; j0 < K2; j0 += 32) {
        const int j = j0 + lane;
        const int c = j < K2 ? cnt[j] : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int t = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += t; }
        if (j < K2) { pos[j] = run + inc - c; cnt[j] = run + inc; }
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    if (myl >= 0) order[atomicAdd(&pos[myl], 1)] = tid;  // pos[j] ends at the list end
    __syncthreads();
    if (tid == 0 && rep == 3) cyc[33] = clock64() - t0;
    const long long tw0 = clock64();
    for (int j = warp; j < K2; j += 8) {
      const int q1 = cnt[j], q0 = j > 0 ? cnt[j - 1] : 0;
      const int ia = lane, ib = 32 + lane;
      long long sa = 0, sb = 0, sw = 0;
      const uint32_t s_order = (uint32_t)__cvta_generic_to_shared(order), s_wsc = (uint32_t)__cvta_generic_to_shared(wsc);
      const uint32_t s_iw = (uint32_t)__cvta_generic_to_shared(iw);
      const uint32_t s_xa = (uint32_t)__cvta_generic_to_shared(xs) + 4u * (uint32_t)(ia * P);
      const uint32_t s_xb = s_xa + 4u * 32u * P;
      for (int q = q0; q < q1; q += 4) {
        int pp[4]; double wv[4]; float xa[4], xb[4]; long long iv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          int v = 0;
          if (q + u < q1) asm volatile("ld.shared.s32 %0, [%1];" : "=r"(v) : "r"(s_order + 4u * (q + u)));
          pp[u] = v;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = q + u < q1;
          double w = 0.0; long long iwl = 0; float fa = 0.f, fb = 0.f;
          asm volatile("ld.shared.f64 %0, [%1];" : "=d"(w) : "r"(s_wsc + 8u * pp[u]));
          asm volatile("ld.shared.s64 %0, [%1];" : "=l"(iwl) : "r"(s_iw + 8u * pp[u]));
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(fa) : "r"(s_xa + 4u * pp[u]));
          if (ib < D) asm volatile("ld.shared.f32 %0, [%1];" : "=f"(fb) : "r"(s_xb + 4u * pp[u]));
          wv[u] = ok ? w : 0.0; iv[u] = ok ? iwl : 0; xa[u] = ia < D ? fa : 0.f; xb[u] = fb;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (MODE == 0) { sa += fx_prod_magic(wv[u], xa[u]); sb += fx_prod_magic(wv[u], xb[u]); sw += iv[u]; }
          else if (MODE == 1) { sa += pp[u]; }
          else { sa += __float_as_int(xa[u]) + __double_as_longlong(wv[u]); sb += __float_as_int(xb[u]); sw += iv[u]; }
        }
      }
      if (ia < D) part[j * D + ia] = sa;
      if (ib < D) part[j * D + ib] = sb;
      if (lane == 0) part[K2 * D + j] = sw;
    }
    if (rep == 3 && lane == 0) cyc[24 + warp] = clock64() - tw0;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[32] = (t1 - t0) / 4;
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}
__global__ void accum3(const int* glab, const float* gx, long long* gout, long long* cyc) {
  extern __shared__ double xsd[];
  __shared__ double wsc[P];
  __shared__ long long iw[P];
  __shared__ int lab[NP], order[NP], cnt[K2 + 1], pos[K2];
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < D * P; e += 256) xsd[e] = gx[e];
  for (int p = tid; p < P; p += 256) { wsc[p] = 0x1p30; iw[p] = 1 << 20; }
  for (int p = tid; p < NP; p += 256) lab[p] = glab[p];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    for (int j = tid; j < K2; j += 256) cnt[j] = 0;
    __syncthreads();
    int myl = tid < NP ? lab[tid] : -1;
    if (myl >= 0) atomicAdd(&cnt[myl], 1);
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the counts -> list starts (pos) and ends (cnt)
      int run = 0;
      for (int j0 = 0; j0 < K2; j0 += 32) {
        const int j = j0 + lane;
        const int c = j < K2 ? cnt[j] : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int t = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += t; }
        if (j < K2) { pos[j] = run + inc - c; cnt[j] = run + inc; }
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    if (myl >= 0) order[atomicAdd(&pos[myl], 1)] = tid;  // pos[j] ends at the list end
    __syncthreads();
    if (tid == 0 && rep == 3) cyc[6] = clock64() - t0;
    const long long tw0 = clock64();
    for (int j = warp; j < K2; j += 8) {
      const int q1 = cnt[j], q0 = j > 0 ? cnt[j - 1] : 0;
      const int ia = lane, ib = 32 + lane;
      long long sa = 0, sb = 0, sw = 0;
      for (int q = q0; q < q1; q += 4) {
        int pp[4]; double wv[4]; double xa[4], xb[4]; long long iv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) pp[u] = q + u < q1 ? order[q + u] : 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const bool ok = q + u < q1;
          wv[u] = ok ? wsc[pp[u]] : 0.0;
          iv[u] = ok ? iw[pp[u]] : 0;
          xa[u] = ia < D ? xsd[ia * P + pp[u]] : 0.0;
          xb[u] = ib < D ? xsd[ib * P + pp[u]] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) { sa += __double_as_longlong(fma(wv[u], xa[u], 6755399441055744.0)) - 0x4338000000000000LL; sb += __double_as_longlong(fma(wv[u], xb[u], 6755399441055744.0)) - 0x4338000000000000LL; sw += iv[u]; }
      }
      if (ia < D) part[j * D + ia] = sa;
      if (ib < D) part[j * D + ib] = sb;
      if (lane == 0) part[K2 * D + j] = sw;
    }
    if (rep == 3 && lane == 0) cyc[16 + warp] = clock64() - tw0;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[5] = (t1 - t0) / 4;
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}
__global__ void centres2(const long long* gpart, float* out, long long* cyc) {
  __shared__ long long part[K2 * D + K2];
  __shared__ double wd[K2];
  __shared__ float cs[64 * D];
  const int tid = threadIdx.x;
  for (int e = tid; e < K2 * D + K2; e += 256) part[e] = gpart[e];
  for (int j = tid; j < K2; j += 256) wd[j] = 1.0 / (double)(part[K2 * D + j] + 1);
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    const int j = tid & 63, ig = tid >> 6;  // lanes over centres: conflict-free stores
    if (j < K2) {
      const double rw = wd[j];
#pragma unroll 4
      for (int i = ig; i < D; i += 4) {
        const long long v = part[j * D + i];
        if (rw > 0) cs[cpair_idx(j, i, D)] = static_cast<float>((static_cast<double>(v) * 0x1p-40) * rw);
      }
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[3] = (t1 - t0) / 4;
  for (int e = tid; e < 64 * D; e += 256) out[e] = cs[e];
}

// accumulate_sorted of lloyd.cu (sort, scatter rows, per-(group, dimension) segment sums)
template <int VAR>
__global__ void accum5(const int* glab, const float* gx, long long* gout, long long* cyc) {
  extern __shared__ float dyn5[];
  float* xs = dyn5;                 // [D][P]
  float* txs = dyn5 + D * P;        // [D][P]
  __shared__ double wsc[P], tws[P];
  __shared__ long long iw[P], tiw[P];
  __shared__ int lab[NP], tlab[P], cnt[K2], start[K2];
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < D * P; e += 256) xs[e] = gx[e];
  for (int p = tid; p < P; p += 256) { wsc[p] = 0x1p30; iw[p] = 1 << 20; }
  for (int p = tid; p < NP; p += 256) lab[p] = glab[p];
  for (int e = tid; e < K2 * D + K2; e += 256) part[e] = 0;
  __syncthreads();
  long long t0 = clock64(), ts[4];
  const int np = NP, d = D, k2 = K2, P2 = P;
  for (int rep = 0; rep < 4; ++rep) {
    for (int j = tid; j < k2; j += 256) cnt[j] = 0;
    __syncthreads();
    ts[0] = clock64();
    for (int p = tid; p < np; p += 256) atomicAdd(&cnt[lab[p]], 1);
    __syncthreads();
    if (warp == 0) {
      int run = 0;
      for (int j0 = 0; j0 < k2; j0 += 32) {
        const int j = j0 + lane;
        const int c = j < k2 ? cnt[j] : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int t = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += t; }
        if (j < k2) { start[j] = run + inc - c; cnt[j] = run + inc; }
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    ts[1] = clock64();
    for (int p = tid; p < np; p += 256) {
      const int l = lab[p];
      const int pos = atomicAdd(&start[l], 1);
      tlab[pos] = l; tws[pos] = wsc[p]; tiw[pos] = iw[p];
      for (int i = 0; i < d; ++i) txs[i * P2 + pos] = xs[i * P + p];
    }
    __syncthreads();
    ts[2] = clock64();
    const int nsum = k2 * d;
    const int G = 256 / d;
    for (int t = tid; t < G * d; t += 256) {
      const int g = t / d, i = t - g * d;
      const int j0 = g * k2 / G, j1 = (g + 1) * k2 / G;
      const int r0 = j0 > 0 ? cnt[j0 - 1] : 0, r1 = j1 > 0 ? cnt[j1 - 1] : 0;
      if (r0 >= r1) continue;
      long long s = 0, sw = 0;
      int jc = tlab[r0];
      if (VAR == 0) {
#pragma unroll 4
        for (int r = r0; r < r1; ++r) {
          const int l = tlab[r];
          const long long v = fx_prod_magic(tws[r], txs[i * P2 + r]);
          const long long vw = tiw[r];
          if (l != jc) { part[jc * d + i] += s; if (i == 0) part[nsum + jc] += sw; s = 0; sw = 0; jc = l; }
          s += v; sw += vw;
        }
      } else if (VAR == 2) {  // no flush branch (sum everything)
#pragma unroll 4
        for (int r = r0; r < r1; ++r) { s += fx_prod_magic(tws[r], txs[i * P2 + r]); sw += tiw[r]; }
      } else if (VAR == 3) {  // no F2F / DFMA: integer only
#pragma unroll 4
        for (int r = r0; r < r1; ++r) { s += __float_as_int(txs[i * P2 + r]) + (long long)tws[r]; sw += tiw[r]; }
      } else if (VAR == 4) {  // loads only, 32-bit sum
        int si = 0;
#pragma unroll 4
        for (int r = r0; r < r1; ++r) si += __float_as_int(txs[i * P2 + r]);
        s = si;
      } else {
        // explicit batches of 4 rows: all loads first
        for (int r = r0; r < r1; r += 4) {
          int l4[4]; double w4[4]; float x4[4]; long long i4[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int rr = r + u < r1 ? r + u : r1 - 1;
            l4[u] = tlab[rr]; w4[u] = tws[rr]; x4[u] = txs[i * P2 + rr]; i4[u] = tiw[rr];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            if (r + u < r1) {
              const long long v = fx_prod_magic(w4[u], x4[u]);
              if (l4[u] != jc) { part[jc * d + i] += s; if (i == 0) part[nsum + jc] += sw; s = 0; sw = 0; jc = l4[u]; }
              s += v; sw += i4[u];
            }
          }
        }
      }
      part[jc * d + i] += s;
      if (i == 0) part[nsum + jc] += sw;
    }
    ts[3] = clock64();
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) { cyc[40] = (t1 - t0) / 4; cyc[41] = ts[1] - ts[0]; cyc[42] = ts[2] - ts[1]; cyc[43] = ts[3] - ts[2]; }
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}

// warp w owns clusters j = w mod 8; register accumulators per owned cluster, points of the warp
// taken four at a time from the per-block ballot of owned labels
template <int NC>
__global__ void accum6(const int* glab, const float* gx, long long* gout, long long* cyc) {
  extern __shared__ float xs[];
  __shared__ double wsc[P];
  __shared__ long long iw[P];
  __shared__ int lab[NP];
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < D * P; e += 256) xs[e] = gx[e];
  for (int p = tid; p < P; p += 256) { wsc[p] = 0x1p30; iw[p] = 1 << 20; }
  for (int p = tid; p < NP; p += 256) lab[p] = glab[p];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    const int ia = lane, ib = 32 + lane;
    long long sa[NC], sb[NC], sw[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) { sa[c] = 0; sb[c] = 0; sw[c] = 0; }
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const int l = lane + 32 * t < NP ? lab[lane + 32 * t] : -1;
      unsigned m = __ballot_sync(0xffffffffu, l >= 0 && (l & 7) == warp);
      while (m) {
        int pp[4], cc[4];
        bool ok[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          ok[u] = m != 0;
          const int src = ok[u] ? __ffs(m) - 1 : 0;
          pp[u] = 32 * t + src;
          cc[u] = __shfl_sync(0xffffffffu, l, src) >> 3;
          m &= m - 1;
        }
        long long va[4], vb[4], vw[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const double w = ok[u] ? wsc[pp[u]] : 0.0;
          va[u] = fx_prod_magic(w, ia < D ? xs[ia * P + pp[u]] : 0.f);
          vb[u] = fx_prod_magic(w, ib < D ? xs[ib * P + pp[u]] : 0.f);
          vw[u] = ok[u] ? iw[pp[u]] : 0;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int c = 0; c < NC; ++c)
            if (cc[u] == c) { sa[c] += va[u]; sb[c] += vb[u]; sw[c] += vw[u]; }
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const int j = warp + 8 * c;
      if (j < K2) {
        if (ia < D) part[j * D + ia] = sa[c];
        if (ib < D) part[j * D + ib] = sb[c];
        if (lane == 0) part[K2 * D + j] = sw[c];
      }
    }
    if (rep == 3 && lane == 0) cyc[48 + warp] = clock64() - t0;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[56] = (t1 - t0) / 4;
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}

// precomputed products v[p][i] (int64, constant across Lloyd iterations)
__global__ void accum7(const int* glab, const float* gx, long long* gout, long long* cyc) {
  extern __shared__ long long vp[];  // [NP][D]
  __shared__ long long iw[P];
  __shared__ int lab[NP];
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < NP * D; e += 256) vp[e] = fx_prod_magic(0x1p30, gx[e % (D * P)]);
  for (int p = tid; p < P; p += 256) iw[p] = 1 << 20;
  for (int p = tid; p < NP; p += 256) lab[p] = glab[p];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    int labr[5];
#pragma unroll
    for (int t = 0; t < 5; ++t) labr[t] = lane + 32 * t < NP ? lab[lane + 32 * t] : -1;
    for (int j = warp; j < K2; j += 8) {
      const int ia = lane, ib = 32 + lane;
      long long sa = 0, sb = 0, sw = 0;
#pragma unroll
      for (int t = 0; t < 5; ++t) {
        unsigned m = __ballot_sync(0xffffffffu, labr[t] == j);
        while (m) {
          const int p = 32 * t + __ffs(m) - 1;
          m &= m - 1;
          sa += vp[p * D + ia];
          if (ib < D) sb += vp[p * D + ib];
          sw += iw[p];
        }
      }
      part[j * D + ia] = sa;
      if (ib < D) part[j * D + ib] = sb;
      if (lane == 0) part[K2 * D + j] = sw;
    }
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[57] = (t1 - t0) / 4;
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}
// counting sort, warp-contiguous ranges of the sorted rows aligned to cluster starts, running
// sums in registers (lanes over dimensions), rows four at a time
__global__ void accum8(const int* glab, const float* gx, long long* gout, long long* cyc) {
  extern __shared__ long long vp[];  // [NP][D]
  __shared__ long long iw[P];
  __shared__ int lab[NP], order[NP], slab[NP], cnt[K2], start[K2], wst[9];
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < NP * D; e += 256) vp[e] = fx_prod_magic(0x1p30, gx[e % (D * P)]);
  for (int p = tid; p < P; p += 256) iw[p] = 1 << 20;
  for (int p = tid; p < NP; p += 256) lab[p] = glab[p];
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    for (int j = tid; j < K2; j += 256) cnt[j] = 0;
    for (int e = tid; e < K2 * D + K2; e += 256) part[e] = 0;
    __syncthreads();
    const int myl = tid < NP ? lab[tid] : -1;
    if (rep == 3 && tid == 0) cyc[60 + 0] = clock64();
    if (myl >= 0) atomicAdd(&cnt[myl], 1);
    __syncthreads();
    if (rep == 3 && tid == 0) cyc[60 + 1] = clock64();
    if (warp == 0) {
      int run = 0;
      for (int j0 = 0; j0 < K2; j0 += 32) {
        const int j = j0 + lane;
        const int c = j < K2 ? cnt[j] : 0;
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) { const int t = __shfl_up_sync(0xffffffffu, inc, o); if (lane >= o) inc += t; }
        if (j < K2) start[j] = run + inc - c;
        run += __shfl_sync(0xffffffffu, inc, 31);
      }
    }
    __syncthreads();
    if (rep == 3 && tid == 0) cyc[60 + 2] = clock64();
    if (myl >= 0) { const int pos = atomicAdd(&start[myl], 1); order[pos] = tid; slab[pos] = myl; }
    __syncthreads();
    if (rep == 3 && tid == 0) cyc[60 + 3] = clock64();
    if (tid <= 8) {  // warp ranges aligned to label runs
      int q = tid * NP / 8;
      if (tid < 8) { while (q > 0 && q < NP && slab[q] == slab[q - 1]) ++q; } else q = NP;
      wst[tid] = q;
    }
    __syncthreads();
    if (rep == 3 && tid == 0) cyc[60 + 4] = clock64();
    const int qb = wst[warp], qe = wst[warp + 1];
    const int ia = lane, ib = 32 + lane;
    long long sa = 0, sb = 0, sw = 0;
    int jc = qb < qe ? slab[qb] : 0;
    for (int q = qb; q < qe; q += 4) {
      int l4[4], p4[4];
      long long a4[4], b4[4], w4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { const int qq = q + u < qe ? q + u : qe - 1; l4[u] = slab[qq]; p4[u] = order[qq]; }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        a4[u] = vp[p4[u] * D + ia];
        b4[u] = ib < D ? vp[p4[u] * D + ib] : 0;
        w4[u] = iw[p4[u]];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (q + u < qe) {
          if (l4[u] != jc) {
            part[jc * D + ia] = sa; if (ib < D) part[jc * D + ib] = sb; if (lane == 0) part[K2 * D + jc] = sw;
            sa = 0; sb = 0; sw = 0; jc = l4[u];
          }
          sa += a4[u]; sb += b4[u]; sw += w4[u];
        }
      }
    }
    if (qb < qe) { part[jc * D + ia] = sa; if (ib < D) part[jc * D + ib] = sb; if (lane == 0) part[K2 * D + jc] = sw; }
    if (rep == 3 && lane == 0) cyc[66 + warp] = clock64();
    __syncthreads();
    if (rep == 3 && tid == 0) cyc[65] = clock64();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[58] = (t1 - t0) / 4;
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}

// warp w owns clusters j = w mod 8: its matches (from 5 ballots) are ranked by (label, point) inside
// the warp, written in that order to a per-warp list, then summed eight rows at a time with all
// loads hoisted and the running sums of the current cluster in registers (one store per cluster)
__global__ void accum10(const int* glab, const float* gx, long long* gout, long long* cyc) {
  extern __shared__ float xs[];
  __shared__ double wsc[P];
  __shared__ long long iw[P];
  __shared__ int lab[NP];
  __shared__ int wlist[8][64];
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int e = tid; e < D * P; e += 256) xs[e] = gx[e];
  for (int p = tid; p < P; p += 256) { wsc[p] = 0x1p30; iw[p] = 1 << 20; }
  for (int p = tid; p < NP; p += 256) lab[p] = glab[p];
  for (int e = tid; e < K2 * D + K2; e += 256) part[e] = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    // 1. owned matches -> (key = label * 256 + point) per lane slot, M of them (M <= 64 here)
    int key0 = 0x7fffffff, key1 = 0x7fffffff, M = 0;
#pragma unroll
    for (int t = 0; t < 5; ++t) {
      const int p = lane + 32 * t;
      const int l = p < NP ? lab[p] : -1;
      const bool own = l >= 0 && (l & 7) == warp;
      const unsigned m = __ballot_sync(0xffffffffu, own);
      const int slot = M + __popc(m & ((1u << lane) - 1u));
      if (own) wlist[warp][slot] = (l << 8) | p;
      M += __popc(m);
    }
    __syncwarp();
    if (lane < M) key0 = wlist[warp][lane];
    if (lane + 32 < M) key1 = wlist[warp][lane + 32];
    // 2. rank by key (all distinct) and write back sorted
    int r0 = 0, r1 = 0;
    for (int u = 0; u < M; ++u) {
      const int ku = wlist[warp][u];
      r0 += ku < key0;
      r1 += ku < key1;
    }
    __syncwarp();
    if (lane < M) wlist[warp][r0] = key0;
    if (lane + 32 < M) wlist[warp][r1] = key1;
    __syncwarp();
    // 3. run sums, eight rows per step, loads hoisted
    const int ia = lane, ib = 32 + lane;
    long long sa = 0, sb = 0, sw = 0;
    int jc = M > 0 ? (wlist[warp][0] >> 8) : 0;
    for (int q0 = 0; q0 < M; q0 += 8) {
      int kk[8];
      double w8[8];
      float xa[8], xb[8];
      long long i8[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) kk[u] = q0 + u < M ? wlist[warp][q0 + u] : -1;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int p = kk[u] >= 0 ? (kk[u] & 255) : 0;
        w8[u] = kk[u] >= 0 ? wsc[p] : 0.0;
        i8[u] = kk[u] >= 0 ? iw[p] : 0;
        xa[u] = xs[ia * P + p];
        xb[u] = ib < D ? xs[ib * P + p] : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const long long va = fx_prod_magic(w8[u], xa[u]), vb = fx_prod_magic(w8[u], xb[u]);
        const int l = kk[u] >> 8;
        if (kk[u] >= 0 && l != jc) {
          part[jc * D + ia] = sa; if (ib < D) part[jc * D + ib] = sb; if (lane == 0) part[K2 * D + jc] = sw;
          sa = 0; sb = 0; sw = 0; jc = l;
        }
        sa += va; sb += vb; sw += i8[u];
      }
    }
    if (M > 0) { part[jc * D + ia] = sa; if (ib < D) part[jc * D + ib] = sb; if (lane == 0) part[K2 * D + jc] = sw; }
    if (rep == 3 && lane == 0) cyc[80 + warp] = clock64() - t0;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[79] = (t1 - t0) / 4;
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}

__global__ void empty_rep(long long* gout, long long* cyc) {
  __shared__ long long part[K2 * D + K2];
  const int tid = threadIdx.x;
  for (int e = tid; e < K2 * D + K2; e += 256) part[e] = 0;
  __syncthreads();
  long long t0 = clock64();
  for (int rep = 0; rep < 4; ++rep) {
    for (int e = tid; e < K2 * D + K2; e += 256) part[e] += e;
    __syncthreads();
  }
  long long t1 = clock64();
  if (tid == 0) cyc[90] = (t1 - t0) / 4;
  for (int e = tid; e < K2 * D + K2; e += 256) gout[e] = part[e];
}
int main() {
  long long *gp, *cyc, *go; float *out, *gx; int* gl;
  cudaMalloc(&gp, 8 * 4096); cudaMalloc(&out, 4 * 64 * D); cudaMallocManaged(&cyc, 1024); cudaMalloc(&go, 8 * 4096);
  cudaMalloc(&gx, 4 * D * P); cudaMalloc(&gl, 4 * NP);
  long long hp[K2 * D + K2]; for (int i = 0; i < K2 * D + K2; ++i) hp[i] = (long long)i * 123456789012345LL;
  cudaMemcpy(gp, hp, sizeof(hp), cudaMemcpyHostToDevice);
  int hl[NP]; unsigned s = 12345; for (int i = 0; i < NP; ++i) { s = s * 1103515245u + 12345u; hl[i] = (s >> 16) % K2; }
  cudaMemcpy(gl, hl, sizeof(hl), cudaMemcpyHostToDevice);
  float hx[D * P]; for (int i = 0; i < D * P; ++i) hx[i] = 0.001f * (i % 997);
  cudaMemcpy(gx, hx, sizeof(hx), cudaMemcpyHostToDevice);
  for (int r = 0; r < 2; ++r) { centres<0><<<1, 256>>>(gp, out, cyc); cudaDeviceSynchronize(); }
  printf("centres I2F.S64   : %lld cycles (one problem)\n", cyc[0]);
  for (int r = 0; r < 2; ++r) { centres<1><<<1, 256>>>(gp, out, cyc); cudaDeviceSynchronize(); }
  printf("centres hi/lo I2F : %lld cycles\n", cyc[0]);
  cudaFuncSetAttribute(accum, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int r = 0; r < 2; ++r) { accum<<<1, 256, 4 * D * P>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  cudaFuncSetAttribute(accum2, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int r = 0; r < 2; ++r) { accum2<<<1, 256, 4 * D * P>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); }
  printf("accum sort+lists  : %lld cycles (%s)\n", cyc[2], cudaGetErrorString(cudaGetLastError()));
  for (int r = 0; r < 2; ++r) { centres2<<<1, 256>>>(gp, out, cyc); cudaDeviceSynchronize(); }
  printf("centres lanes/j   : %lld cycles\n", cyc[3]);
  printf("accum2 per-warp sums:"); for (int w = 0; w < 8; ++w) printf(" %lld", cyc[8 + w]); printf("\n");
  cudaFuncSetAttribute(accum3, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int r = 0; r < 2; ++r) { accum3<<<1, 256, 8 * D * P>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); }
  printf("accum3 (x as double): %lld cycles (%s); per-warp:", cyc[5], cudaGetErrorString(cudaGetLastError()));
  for (int w = 0; w < 8; ++w) printf(" %lld", cyc[16 + w]); printf("\n");
#define RUN4(M) \
  cudaFuncSetAttribute(accum4<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024); \
  for (int r = 0; r < 2; ++r) { accum4<M><<<1, 256, 4 * D * P>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); } \
  printf("accum4 mode %d: %lld cycles (%s); per-warp:", M, cyc[32], cudaGetErrorString(cudaGetLastError())); \
  for (int w = 0; w < 8; ++w) printf(" %lld", cyc[24 + w]); printf("\n");
  RUN4(0) RUN4(1) RUN4(2)
#define RUN5(V) \
  cudaFuncSetAttribute(accum5<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024); \
  for (int r = 0; r < 2; ++r) { accum5<V><<<1, 256, 8 * D * P>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); } \
  printf("accum5 var %d: %lld cycles (%s); thread 0: hist+scan %lld scatter %lld sums %lld\n", V, cyc[40], \
         cudaGetErrorString(cudaGetLastError()), cyc[41], cyc[42], cyc[43]);
  RUN5(0) RUN5(1) RUN5(2) RUN5(3) RUN5(4)
  cudaFuncSetAttribute(accum6<7>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int r = 0; r < 2; ++r) { accum6<7><<<1, 256, 4 * D * P>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); }
  printf("accum6 regs: %lld cycles (%s)\n", cyc[56], cudaGetErrorString(cudaGetLastError()));
  cudaFuncSetAttribute(accum7, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int r = 0; r < 2; ++r) { accum7<<<1, 256, 8 * NP * D>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); }
  printf("accum7 ballot, precomputed v: %lld cycles (%s)\n", cyc[57], cudaGetErrorString(cudaGetLastError()));
  cudaFuncSetAttribute(accum8, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  for (int r = 0; r < 2; ++r) { accum8<<<1, 256, 8 * NP * D>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); }
  printf("accum8 sort+runs, precomputed v: %lld cycles (%s)\n", cyc[58], cudaGetErrorString(cudaGetLastError()));
  printf("  phases: zero %lld hist %lld scan %lld scatter %lld ranges %lld sums(warp max) ", 0LL, cyc[61] - cyc[60], cyc[62] - cyc[61], cyc[63] - cyc[62], cyc[64] - cyc[63]);
  { long long mx = 0; for (int w = 0; w < 8; ++w) mx = cyc[66 + w] - cyc[64] > mx ? cyc[66 + w] - cyc[64] : mx; printf("%lld, end %lld\n", mx, cyc[65] - cyc[64]); }
  cudaFuncSetAttribute(accum10, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  for (int r = 0; r < 2; ++r) { accum10<<<1, 256, 4 * D * P>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); }
  printf("accum10 warp-ranked runs: %lld cycles (%s); per warp (rep 3, from t0):", cyc[79], cudaGetErrorString(cudaGetLastError()));
  for (int w = 0; w < 8; ++w) printf(" %lld", cyc[80 + w]); printf("\n");
  {
    long long ref[K2 * D + K2], got[K2 * D + K2];
    accum<<<1, 256, 4 * D * P>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); cudaMemcpy(ref, go, sizeof(ref), cudaMemcpyDeviceToHost);
    accum10<<<1, 256, 4 * D * P>>>(gl, gx, go, cyc); cudaDeviceSynchronize(); cudaMemcpy(got, go, sizeof(got), cudaMemcpyDeviceToHost);
    int bad = 0; for (int e = 0; e < K2 * D + K2; ++e) bad += ref[e] != got[e];
    printf("accum10 vs accum: %d mismatches\n", bad);
  }
  for (int r = 0; r < 2; ++r) { empty_rep<<<1, 256>>>(go, cyc); cudaDeviceSynchronize(); }
  printf("empty rep (part += e, sync): %lld cycles\n", cyc[90]);
  printf("accum2 sort part at rep 3: %lld cycles after 3 full reps (=> sort %lld)\n", cyc[4], cyc[4] - 3 * cyc[2]);
  printf("accum owned-ballot: %lld cycles (one problem, 135 points)\n", cyc[1]);
  return 0;
}
