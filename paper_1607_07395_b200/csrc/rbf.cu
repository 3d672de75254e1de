// rbf.cu -- the implicit RBF source (BASELINE.json configs[4], reading Z23) and the sampled
// residual (P:313 on a seeded uniform subset of entries, readings Z17 / Z23).
//
// Entries are generated on access ("never knowing the remaining entries"):
//   A_ij = exp(-|x_i - y_j|^2 g),  g = 1 / (2 sigma^2),
// in FP32: direct differences summed over the d coordinates in order, then exp through
// ex2.approx (MUFU.EX2).  x (m x d) and y (n x d) are replicated on every rank; no gather
// crosses ranks.  The three gathers of a sketch (C = A(:, J) for the rank's rows, R = A(I, :),
// W = A(I, J)) are FFMA + MUFU bound with coalesced stores; the point rows they need are staged
// in shared memory or held in registers.
//
// Sampled residual: pair t of T has position (i_t, j_t) from the Philox block
// (t lo, t hi, 5, attempt) with Lemire bounded integers; the rank owning
// row i_t adds (A_{i_t j_t} - F_{i_t} diag(s) G_{j_t}^T)^2 and A_{i_t j_t}^2.  One warp per 32
// pairs: each lane draws one pair (and generates / loads its entry), then the warp computes the
// 32 dot products with coalesced float4 reads of the two factor rows, reduces them with a
// 31-shuffle transpose reduction, and each lane squares its own pair's error.  Per-warp FP64
// sums -> fixed-order block and grid reductions: deterministic for a given launch shape.
#include <float.h>

#include "common.cuh"
#include "kernels.cuh"
#include "philox.cuh"

namespace cabsk {

constexpr int kRbfMaxD = 64;

__device__ __forceinline__ float rbf_entry(float d2, float g) { return __expf(-d2 * g); }

// ---------------------------------------------------------------- R = A(I, :)   (k x n, ldr)
// block (256 columns) x (up to 32 rows of I): each thread keeps y_c in registers and walks the
// block's rows of x from shared memory; stores are coalesced along c.
template <int D>
__global__ void __launch_bounds__(256) rbf_rows_kernel(RbfSrc s, const int64_t* __restrict__ I, int k, int64_t n,
                                                       float* __restrict__ R, int64_t ldr) {
  __shared__ float xs[32][kRbfMaxD];
  const int d = D > 0 ? D : s.d;
  const int a0 = blockIdx.y * 32;
  const int na = k - a0 < 32 ? k - a0 : 32;
  for (int e = threadIdx.x; e < na * d; e += blockDim.x) {
    const int a = e / d, l = e - a * d;
    xs[a][l] = s.x[I[a0 + a] * s.ldx + l];
  }
  __syncthreads();
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c >= n) return;
  float yc[D > 0 ? D : kRbfMaxD];
#pragma unroll
  for (int l = 0; l < (D > 0 ? D : kRbfMaxD); ++l)
    if (l < d) yc[l] = s.y[c * s.ldy + l];
  for (int a = 0; a < na; ++a) {
    float d2 = 0.f;
#pragma unroll
    for (int l = 0; l < (D > 0 ? D : kRbfMaxD); ++l) {
      if (l < d) {
        const float df = xs[a][l] - yc[l];
        d2 = fmaf(df, df, d2);
      }
    }
    R[(int64_t)(a0 + a) * ldr + c] = rbf_entry(d2, s.g);
  }
}

// ---------------------------------------------------------------- C = A(rows, J)  (m_loc x k)
// block = 32 local rows (x in shared memory); warp w handles column chunks w, w + 8, ... of 32:
// lane b holds y_{J[b]} in registers, loops over the 32 rows; each store is one 128-byte row
// segment of C.
template <int D>
__global__ void __launch_bounds__(256) rbf_cols_kernel(RbfSrc s, int64_t row_begin, int64_t m_loc,
                                                       const int64_t* __restrict__ J, int k,
                                                       float* __restrict__ C, int64_t ldc) {
  __shared__ float xs[32][kRbfMaxD];
  const int d = D > 0 ? D : s.d;
  const int64_t i0 = blockIdx.x * 32ll;
  const int ni = m_loc - i0 < 32 ? static_cast<int>(m_loc - i0) : 32;
  for (int e = threadIdx.x; e < ni * d; e += blockDim.x) {
    const int a = e / d, l = e - a * d;
    xs[a][l] = s.x[(row_begin + i0 + a) * s.ldx + l];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int b0 = warp * 32; b0 < k; b0 += 256) {
    const int b = b0 + lane;
    float yb[D > 0 ? D : kRbfMaxD];
    const int64_t jb = b < k ? J[b] : 0;
#pragma unroll
    for (int l = 0; l < (D > 0 ? D : kRbfMaxD); ++l)
      if (l < d) yb[l] = s.y[jb * s.ldy + l];
    for (int a = 0; a < ni; ++a) {
      float d2 = 0.f;
#pragma unroll
      for (int l = 0; l < (D > 0 ? D : kRbfMaxD); ++l) {
        if (l < d) {
          const float df = xs[a][l] - yb[l];
          d2 = fmaf(df, df, d2);
        }
      }
      if (b < k) C[(i0 + a) * ldc + b] = rbf_entry(d2, s.g);
    }
  }
}

// ---------------------------------------------------------------- W = A(I, J)  (k x k)
__global__ void __launch_bounds__(128) rbf_w_kernel(RbfSrc s, const int64_t* __restrict__ I,
                                                    const int64_t* __restrict__ J, int k, float* __restrict__ W,
                                                    int64_t ldw) {
  const int a = blockIdx.x;
  const float* xa = s.x + I[a] * s.ldx;
  for (int b = threadIdx.x; b < k; b += blockDim.x) {
    const float* yb = s.y + J[b] * s.ldy;
    float d2 = 0.f;
    for (int l = 0; l < s.d; ++l) {
      const float df = xa[l] - yb[l];
      d2 = fmaf(df, df, d2);
    }
    W[(int64_t)a * ldw + b] = rbf_entry(d2, s.g);
  }
}

void launch_rbf_rows(const RbfSrc& s, const int64_t* I, int k, int64_t n, float* R, int64_t ldr, cudaStream_t st) {
  dim3 grid(static_cast<unsigned>(ceil_div(n, 256)), static_cast<unsigned>(ceil_div(k, 32)));
  note_launch();
  if (s.d == 16) rbf_rows_kernel<16><<<grid, 256, 0, st>>>(s, I, k, n, R, ldr);
  else rbf_rows_kernel<0><<<grid, 256, 0, st>>>(s, I, k, n, R, ldr);
}

void launch_rbf_cols(const RbfSrc& s, int64_t row_begin, int64_t m_loc, const int64_t* J, int k, float* C,
                     int64_t ldc, cudaStream_t st) {
  if (m_loc <= 0) return;
  note_launch();
  const unsigned grid = static_cast<unsigned>(ceil_div(m_loc, 32));
  if (s.d == 16) rbf_cols_kernel<16><<<grid, 256, 0, st>>>(s, row_begin, m_loc, J, k, C, ldc);
  else rbf_cols_kernel<0><<<grid, 256, 0, st>>>(s, row_begin, m_loc, J, k, C, ldc);
}

void launch_rbf_w(const RbfSrc& s, const int64_t* I, const int64_t* J, int k, float* W, int64_t ldw,
                  cudaStream_t st) {
  note_launch();
  rbf_w_kernel<<<k, 128, 0, st>>>(s, I, J, k, W, ldw);
}

// ---------------------------------------------------------------- residual pairs
// Lemire step on one word: accept unless lo32 < (2^32 - s) mod s (thr, precomputed).
__device__ __forceinline__ bool lemire_step(uint32_t w, uint64_t s, uint64_t thr, uint64_t& v) {
  const uint64_t p = static_cast<uint64_t>(w) * s;
  v = p >> 32;
  return (p & 0xFFFFFFFFull) >= thr;
}

// (i_t, j_t) of pair t: block (t lo, t hi, 5, attempt); i from words 0, 1,
// j from words 2, 3, next attempt while both words of a coordinate are rejected.
__device__ __forceinline__ void residual_pair(uint64_t t, uint2 key, uint64_t m, uint64_t thr_m, uint64_t n,
                                              uint64_t thr_n, int64_t& i, int64_t& j) {
  uint4 w = philox4x32_10(make_uint4(static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32), 5u, 0u), key);
  uint64_t vi, vj;
  bool ok_i = lemire_step(w.x, m, thr_m, vi) || lemire_step(w.y, m, thr_m, vi);
  bool ok_j = lemire_step(w.z, n, thr_n, vj) || lemire_step(w.w, n, thr_n, vj);
  for (uint32_t att = 1; !(ok_i && ok_j); ++att) {  // rare: P(reject) <= s / 2^32 per word
    w = philox4x32_10(make_uint4(static_cast<uint32_t>(t), static_cast<uint32_t>(t >> 32), 5u, att), key);
    if (!ok_i) ok_i = lemire_step(w.x, m, thr_m, vi) || lemire_step(w.y, m, thr_m, vi);
    if (!ok_j) ok_j = lemire_step(w.z, n, thr_n, vj) || lemire_step(w.w, n, thr_n, vj);
  }
  i = static_cast<int64_t>(vi);
  j = static_cast<int64_t>(vj);
}

__global__ void residual_pairs_kernel(uint64_t seed, uint64_t t0, int64_t T, uint64_t m, uint64_t thr_m, uint64_t n,
                                      uint64_t thr_n, int64_t* __restrict__ oi, int64_t* __restrict__ oj) {
  const uint2 key = seed_key(seed);
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i, j;
    residual_pair(t0 + t, key, m, thr_m, n, thr_n, i, j);
    oi[t] = i;
    oj[t] = j;
  }
}

static uint64_t lemire_thr(uint64_t s) { return ((1ull << 32) - s) % s; }

void launch_residual_pairs(uint64_t seed, uint64_t t0, int64_t T, int64_t m, int64_t n, int64_t* oi, int64_t* oj,
                           cudaStream_t st) {
  if (T <= 0) return;
  int64_t b = ceil_div(T, 256);
  if (b > 8 * kNumSM) b = 8 * kNumSM;
  note_launch();
  residual_pairs_kernel<<<static_cast<unsigned>(b), 256, 0, st>>>(seed, t0, T, m, lemire_thr(m), n, lemire_thr(n),
                                                                  oi, oj);
}

// ---------------------------------------------------------------- sampled residual
constexpr int kSampBlocks = 4 * kNumSM;  // persistent grid: 4 CTAs of 8 warps per SM
constexpr int kSampQ = 8;                // float4 slots per lane: ncomp <= 32 * 4 * 8 = 1024

template <bool RBF>
__global__ void __launch_bounds__(256) residual_sampled_kernel(SampArgs a, double* __restrict__ part) {
  __shared__ double red[2][8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gw = blockIdx.x * 8ll + warp, nw = gridDim.x * 8ll;
  const uint2 key = seed_key(a.seed);
  const int nq = (a.ncomp + 127) / 128;  // float4 slots of a factor row per lane
  const bool vec = (a.ldf % 4 == 0) && (a.ldg % 4 == 0) && (a.ncomp % 4 == 0) &&
                   ((reinterpret_cast<uintptr_t>(a.F) | reinterpret_cast<uintptr_t>(a.G)) & 15) == 0;
  float4 sv[kSampQ];  // this lane's entries of s (columns (q * 32 + lane) * 4 + 0..3)
#pragma unroll
  for (int q = 0; q < kSampQ; ++q) {
    const int c = (q * 32 + lane) * 4;
    sv[q] = make_float4(1.f, 1.f, 1.f, 1.f);
    if (a.s && vec && c < a.ncomp) sv[q] = make_float4(a.s[c], a.s[c + 1], a.s[c + 2], a.s[c + 3]);
  }
  double acc_e = 0.0, acc_a = 0.0;
  const int64_t nb = ceil_div(a.T, 32);
  for (int64_t bt = gw; bt < nb; bt += nw) {
    const int64_t t = bt * 32 + lane;
    int64_t i = 0, j = 0;
    bool mine = false;
    float aij = 0.f;
    if (t < a.T) {
      residual_pair(static_cast<uint64_t>(t), key, a.m, a.thr_m, a.n, a.thr_n, i, j);
      mine = i >= a.row_begin && i < a.row_end;  // owner filter
      if (mine) {
        if (RBF) {
          const float* xi = a.rbf.x + i * a.rbf.ldx;
          const float* yj = a.rbf.y + j * a.rbf.ldy;
          float d2 = 0.f;
          for (int l = 0; l < a.rbf.d; ++l) {
            const float df = __ldg(xi + l) - __ldg(yj + l);
            d2 = fmaf(df, df, d2);
          }
          aij = rbf_entry(d2, a.rbf.g);
        } else {
          aij = __ldg(a.transposed ? a.A + j * a.lda + (i - a.row_begin) : a.A + (i - a.row_begin) * a.lda + j);
        }
      }
    }
    unsigned todo = __ballot_sync(0xffffffffu, mine);
    // the warp's dot products F_{i_p} diag(s) G_{j_p}^T, four pairs at a time
    float dotv = 0.f;  // lane p ends with pair p's dot product
    while (todo) {
      int pp[4];
      int np = 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        pp[u] = todo ? __ffs(todo) - 1 : -1;
        if (todo) { todo &= todo - 1; ++np; }
      }
      float part4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (pp[u] < 0) continue;
        const int64_t iu = __shfl_sync(0xffffffffu, i, pp[u]);
        const int64_t ju = __shfl_sync(0xffffffffu, j, pp[u]);
        const float* fr = a.F + (iu - a.row_begin) * a.ldf;
        const float* gr = a.G + ju * a.ldg;
        float sacc = 0.f;
        if (vec) {
#pragma unroll
          for (int q = 0; q < kSampQ; ++q) {
            const int c = (q * 32 + lane) * 4;
            if (q < nq && c < a.ncomp) {
              const float4 f = __ldg(reinterpret_cast<const float4*>(fr + c));
              const float4 g = __ldg(reinterpret_cast<const float4*>(gr + c));
              sacc = fmaf(f.x * sv[q].x, g.x, sacc);
              sacc = fmaf(f.y * sv[q].y, g.y, sacc);
              sacc = fmaf(f.z * sv[q].z, g.z, sacc);
              sacc = fmaf(f.w * sv[q].w, g.w, sacc);
            }
          }
        } else {
          for (int c = lane; c < a.ncomp; c += 32)
            sacc = fmaf(__ldg(fr + c) * (a.s ? __ldg(a.s + c) : 1.f), __ldg(gr + c), sacc);
        }
        part4[u] = sacc;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (u >= np) break;
        float v = part4[u];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == pp[u]) dotv = v;
      }
    }
    if (mine) {
      const double e = static_cast<double>(aij) - static_cast<double>(dotv);
      acc_e += e * e;
      acc_a += static_cast<double>(aij) * static_cast<double>(aij);
    }
  }
  // fixed-order reductions: warp butterfly, then the 8 warps in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    acc_e += __shfl_xor_sync(0xffffffffu, acc_e, o);
    acc_a += __shfl_xor_sync(0xffffffffu, acc_a, o);
  }
  if (lane == 0) { red[0][warp] = acc_e; red[1][warp] = acc_a; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double se = 0.0, sa = 0.0;
    for (int w = 0; w < 8; ++w) { se += red[0][w]; sa += red[1][w]; }
    part[2 * blockIdx.x] = se;
    part[2 * blockIdx.x + 1] = sa;
  }
}

__global__ void residual_sampled_final_kernel(const double* __restrict__ part, int nblocks, double scale,
                                              double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double se = 0.0, sa = 0.0;
  for (int b = 0; b < nblocks; ++b) { se += part[2 * b]; sa += part[2 * b + 1]; }
  out[0] = scale * se;
  out[1] = scale * sa;
}

void launch_residual_sampled(const SampArgs& a0, double* part, double* out, cudaStream_t st) {
  SampArgs a = a0;
  a.thr_m = lemire_thr(a.m);
  a.thr_n = lemire_thr(a.n);
  int blocks = static_cast<int>(ceil_div(ceil_div(a.T, 32), 8));
  if (blocks > kSampBlocks) blocks = kSampBlocks;
  if (blocks < 1) blocks = 1;
  note_launch();
  if (a.rbf.x) residual_sampled_kernel<true><<<blocks, 256, 0, st>>>(a, part);
  else residual_sampled_kernel<false><<<blocks, 256, 0, st>>>(a, part);
  note_launch();
  residual_sampled_final_kernel<<<1, 32, 0, st>>>(part, blocks, static_cast<double>(a.m) * static_cast<double>(a.n) /
                                                                    static_cast<double>(a.T), out);
}

int residual_sampled_part_doubles() { return 2 * kSampBlocks; }

}  // namespace cabsk
