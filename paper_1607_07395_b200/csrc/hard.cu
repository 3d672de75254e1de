// Hard-threshold follow-up (PAPER.md P:312 variant (f), "top-k samples with largest weighting
// coefficients (Equation eq:wkmeans)"; Z26).
//
// The weighting coefficient of point l is Upsilon(||X_l||) (Eq. 6) with a monotone Upsilon, so
// the selection is the top-k of the key ||X_l||^2: the FP64 sum of the exact squares of the
// FP32 entries, in column order.  Ties go to the lowest index; the output is ascending.
//
//   hard_local_kernel  CTAs of 2048 rows: 32 x 32 tiles staged through shared memory with
//                      coalesced loads, each lane sums ITS row in column order; then the CTA's
//                      own top-k (below) -> (key, index) candidates, ascending, per CTA slot
//   hard_topk_kernel   one CTA per side over the candidates: MSB radix select on the 64-bit
//                      key (8-bit digits, early exit once the boundary bucket is taken whole),
//                      then one ordered compaction pass (block scans) that writes the winners
//                      in ascending index order -- boundary ties are the first `need` in order
// A top-k winner is a winner inside its own CTA's rows, so the candidates contain the answer,
// and the slot order (CTA by CTA) is ascending index order, so ties resolve identically.
// Multi-rank: each rank's local winners (key, global index) go to its slot of a zeroed
// [nranks][k] pair buffer, one sum-allreduce completes it, and the same top-k kernel runs over
// the nranks*k candidates (rank slots are in ascending global-index order; empty entries carry
// key -1 and never win).
#include "common.cuh"
#include "kernels.cuh"
#include "philox.cuh"

namespace cabsk {

constexpr int kHtThreads = 1024;
constexpr int kHlRows = kHardLocalRows;  // rows per CTA of the key + local top-k kernel (2 tiles per warp)
constexpr int kHtCache = 25600;  // top-k kernel: keys cached in shared memory up to this many

// Order-preserving map: valid keys (>= 0, finite or +inf) -> bits + 1; empty slots (key < 0)
// and NaN -> 0 (never preferred over a valid key).
__device__ __forceinline__ uint64_t hard_ukey(double v) {
  return v >= 0.0 ? static_cast<uint64_t>(__double_as_longlong(v)) + 1ull : 0ull;
}

// Exclusive block scan of one int per thread (kHtThreads threads); returns the block total.
__device__ __forceinline__ int hard_block_scan(int v, int* s_w, int& excl) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[w] = x;
  __syncthreads();
  if (w == 0) {
    int t = s_w[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    s_w[32 + lane] = t;  // inclusive warp totals
  }
  __syncthreads();
  excl = x - v + (w > 0 ? s_w[32 + w - 1] : 0);
  const int total = s_w[32 + 31];
  __syncthreads();  // s_w reused by the next call
  return total;
}

struct HardSel {
  uint64_t prefix, maskhi;
  int need;
};
struct HardScratch {
  uint64_t mn[32], mx[32];
  int hist[256];
  int w[64];
  int digit, above, cnt;
};

// MSB radix select (8-bit digits) of the kk-th largest mapped key among N: afterwards the
// winners are the keys with (u & maskhi) > prefix plus the first `need` (in index order) with
// (u & maskhi) == prefix.  CACHED: u = s_u[l]; else u = hard_ukey(key[l * ks]) from global
// memory, eight loads in flight per thread.  Early exit once the boundary bucket is taken whole.
template <bool CACHED>
__device__ HardSel hard_radix_select(const uint64_t* s_u, const double* __restrict__ key, int64_t ks, int64_t N,
                                     int kk, HardScratch& sc) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  HardSel r{0ull, 0ull, kk};
  if (kk <= 0) return r;
  // bits above the highest one in which the valid keys differ are common: skip them
  uint64_t umin = ~0ull, umax = 0ull;
  if (CACHED) {
    for (int64_t l = tid; l < N; l += kHtThreads) {
      const uint64_t u = s_u[l];
      if (u) umin = umin < u ? umin : u;
      umax = umax > u ? umax : u;
    }
  } else {
    for (int64_t l = tid; l < N; l += kHtThreads) {
      const uint64_t u = hard_ukey(key[l * ks]);
      if (u) umin = umin < u ? umin : u;
      umax = umax > u ? umax : u;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t a = __shfl_xor_sync(0xffffffffu, umin, o), b = __shfl_xor_sync(0xffffffffu, umax, o);
    umin = umin < a ? umin : a;
    umax = umax > b ? umax : b;
  }
  if (lane == 0) {
    sc.mn[warp] = umin;
    sc.mx[warp] = umax;
  }
  __syncthreads();
  umin = ~0ull;
  umax = 0ull;
  for (int w = 0; w < kHtThreads / 32; ++w) {
    umin = umin < sc.mn[w] ? umin : sc.mn[w];
    umax = umax > sc.mx[w] ? umax : sc.mx[w];
  }
  if (umin >= umax) {  // one distinct valid key: the first kk valid ones in order
    r.prefix = umax;
    r.maskhi = ~0ull;
    return r;
  }
  const int p = 63 - __clzll(static_cast<long long>(umin ^ umax));  // highest differing bit
  r.maskhi = p == 63 ? 0ull : ~((2ull << p) - 1ull);
  r.prefix = umax & r.maskhi;
  for (int shift = p - 7; shift > -8; shift -= 8) {
    // digit = bits [shift, shift + 8) (for shift < 0: bits [0, shift + 8), shifted up)
    const uint64_t wmask = shift >= 0 ? 0xffull << shift : 0xffull >> (-shift);
    auto digit = [shift](uint64_t u) -> int {
      return static_cast<int>((shift >= 0 ? u >> shift : u << (-shift)) & 255);
    };
    for (int b = tid; b < 256; b += kHtThreads) sc.hist[b] = 0;
    __syncthreads();
    if (CACHED) {
      for (int64_t l = tid; l < N; l += kHtThreads) {
        const uint64_t u = s_u[l];
        if ((u & r.maskhi) == r.prefix) atomicAdd(&sc.hist[digit(u)], 1);
      }
    } else {
      for (int64_t b0 = tid; b0 < N; b0 += 8 * kHtThreads) {
        uint64_t u[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int64_t l = b0 + (int64_t)j * kHtThreads;
          u[j] = l < N ? hard_ukey(key[l * ks]) : 0ull;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          if (b0 + (int64_t)j * kHtThreads < N && (u[j] & r.maskhi) == r.prefix)
            atomicAdd(&sc.hist[digit(u[j])], 1);
      }
    }
    __syncthreads();
    if (warp == 0) {  // bins in descending order: lane L holds 255 - 8L .. 248 - 8L
      int sum = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) sum += sc.hist[255 - 8 * lane - b];
      int inc = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
      }
      const unsigned hit = __ballot_sync(0xffffffffu, inc >= r.need);
      if (lane == __ffs(hit) - 1) {
        int cum = inc - sum;
        for (int b = 0; b < 8; ++b) {
          const int dg = 255 - 8 * lane - b, h = sc.hist[dg];
          if (cum + h >= r.need) {
            sc.digit = dg;
            sc.above = cum;
            sc.cnt = h;
            break;
          }
          cum += h;
        }
      }
    }
    __syncthreads();
    const uint64_t dg = static_cast<uint64_t>(sc.digit);
    r.prefix |= shift >= 0 ? dg << shift : dg >> (-shift);
    r.maskhi |= wmask;
    r.need -= sc.above;
    const bool whole = sc.cnt == r.need;  // the boundary bucket is taken whole: done
    __syncthreads();
    if (whole) break;
  }
  return r;
}

// Ordered compaction of the winners of `sel`: emit(j, l) for the j-th winner (ascending l).
template <bool CACHED, typename Emit>
__device__ void hard_compact(const uint64_t* s_u, const double* __restrict__ key, int64_t ks, int64_t N, int kk,
                             const HardSel& sel, HardScratch& sc, Emit emit) {
  int taken = 0, eq_seen = 0;
  for (int64_t base = 0; base < N && taken < kk; base += kHtThreads) {
    const int64_t l = base + threadIdx.x;
    int gt = 0, eq = 0;
    if (l < N) {
      const uint64_t u = (CACHED ? s_u[l] : hard_ukey(key[l * ks])) & sel.maskhi;
      gt = u > sel.prefix;
      eq = u == sel.prefix;
    }
    int eq_ex;
    const int eq_tot = hard_block_scan(eq, sc.w, eq_ex);
    const int take = gt || (eq && eq_seen + eq_ex < sel.need);
    int pos;
    const int tk_tot = hard_block_scan(take, sc.w, pos);
    if (take) emit(taken + pos, l);
    taken += tk_tot;
    eq_seen += eq_tot;
  }
}

// Keys + local top-k: CTA b of a side owns rows [b * kHlRows, (b + 1) * kHlRows).  Each warp
// stages 32 x 32 tiles of its rows through shared memory (coalesced loads), each lane sums ITS
// row's exact squares in column order (FP64 FMA of an exact square == the oracle's add); the
// CTA then selects its min(k, rows) winners and writes them as (key, index) pairs, ascending,
// to its slot cand[side][b][k] ((-1, -1) padding).
__global__ void __launch_bounds__(kHtThreads, 1) hard_local_kernel(HardArgs a, double* cand, int64_t side_stride,
                                                                   void* ws) {
  extern __shared__ __align__(16) unsigned char hl_smem[];
  uint64_t* s_u = reinterpret_cast<uint64_t*>(hl_smem);                      // [kHlRows]
  float (*tile)[32][33] = reinterpret_cast<float (*)[32][33]>(s_u + kHlRows);  // [32 warps]
  __shared__ HardScratch sc;
  const int side = static_cast<int>(blockIdx.x) >= a.nb0;
  const HardSide& h = a.s[side];
  const float* __restrict__ X = h.X;
  const int64_t ldx = h.ldx, N = h.N;
  const int d = h.d, k = h.k;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t blk = side ? blockIdx.x - a.nb0 : blockIdx.x;
  const int64_t r0 = blk * kHlRows;
  const int nblk_rows = N - r0 < kHlRows ? static_cast<int>(N - r0) : kHlRows;
  for (int t = 0; t < kHlRows / 32 / 32; ++t) {
    const int rb = (t * 32 + w) * 32;  // first row of this warp's tile, within the CTA
    const int nrow = nblk_rows - rb < 32 ? nblk_rows - rb : 32;
    double acc = 0.0;
    if (nrow > 0) {  // warp-uniform
      for (int c0 = 0; c0 < d; c0 += 32) {
        const int nc = d - c0 < 32 ? d - c0 : 32;
#pragma unroll 8
        for (int r = 0; r < nrow; ++r)
          if (lane < nc) tile[w][r][lane] = X[(r0 + rb + r) * ldx + c0 + lane];
        __syncwarp();
        for (int c = 0; c < nc; ++c) {
          const double v = tile[w][lane][c];
          acc = fma(v, v, acc);
        }
        __syncwarp();
      }
    }
    const bool valid = lane < nrow;
    if (valid) {
      if (!isfinite(acc)) set_status(ws, CABS_DEV_NONFINITE);
      if (h.mode == 1) {  // Efraimidis-Spirakis key (l / r) / (-log u) of the leverage score (Z27)
        const uint64_t gi = static_cast<uint64_t>(h.off + r0 + rb + lane);
        const uint4 w4 = philox4x32_10(make_uint4(static_cast<uint32_t>(gi), static_cast<uint32_t>(gi >> 32), h.tag, 1u),
                                       seed_key(h.seed));
        const double u = (static_cast<double>(w4.x >> 5) * 67108864.0 + static_cast<double>(w4.y >> 6) + 0.5) *
                         1.1102230246251565e-16;  // 2^-53
        acc = (acc / static_cast<double>(d)) / -log(u);
      }
      if (h.key) h.key[r0 + rb + lane] = acc;
    }
    s_u[rb + lane] = valid ? hard_ukey(acc) : 0ull;
  }
  __syncthreads();
  const int kk = nblk_rows < k ? nblk_rows : k;
  const HardSel sel = hard_radix_select<true>(s_u, nullptr, 1, nblk_rows, kk, sc);
  double* slot = cand + side * side_stride + blk * 2LL * k;
  hard_compact<true>(s_u, nullptr, 1, nblk_rows, kk, sel, sc, [&](int j, int64_t l) {
    const uint64_t u = s_u[l];
    slot[2 * j] = __longlong_as_double(static_cast<long long>(u - 1));
    slot[2 * j + 1] = static_cast<double>(h.off + r0 + l);
  });
  for (int j = kk + threadIdx.x; j < k; j += kHtThreads) {
    slot[2 * j] = -1.0;
    slot[2 * j + 1] = -1.0;
  }
}

// Top-k over a candidate list: key[l * ks] for l < N, index (int64) cidx[l * ks] (or off + l
// when cidx is NULL).  Writes the min(k, N) winners ascending to out (if set) and as (key,
// index) pairs to slot (if set; (-1, -1) padding up to k).  One CTA per side.
template <bool CACHED>
__global__ void __launch_bounds__(kHtThreads, 1) hard_topk_kernel(HardArgs a) {
  extern __shared__ uint64_t s_c[];
  __shared__ HardScratch sc;
  const HardSide& h = a.s[blockIdx.x];
  const double* __restrict__ key = h.key;
  const double* __restrict__ cidx = h.cidx;
  const int64_t ks = h.ks, N = h.N, off = h.off;
  const int k = h.k;
  const int kk = N < k ? static_cast<int>(N) : k;
  if (CACHED)
    for (int64_t l = threadIdx.x; l < N; l += kHtThreads) s_c[l] = hard_ukey(key[l * ks]);
  __syncthreads();
  const HardSel sel = hard_radix_select<CACHED>(s_c, key, ks, N, kk, sc);
  hard_compact<CACHED>(s_c, key, ks, N, kk, sel, sc, [&](int j, int64_t l) {
    const int64_t idx = cidx ? static_cast<int64_t>(cidx[l * ks]) : off + l;
    if (h.out) h.out[j] = idx;
    if (h.slot) {
      h.slot[2 * j] = key[l * ks];
      h.slot[2 * j + 1] = static_cast<double>(idx);
    }
  });
  if (h.slot)
    for (int j = kk + threadIdx.x; j < k; j += kHtThreads) {
      h.slot[2 * j] = -1.0;
      h.slot[2 * j + 1] = -1.0;
    }
}

int64_t hard_local_blocks(int64_t N) { return ceil_div(N, kHlRows); }

void launch_hard_local(const HardArgs& a0, int nside, double* cand, int64_t side_stride, void* ws, cudaStream_t st) {
  HardArgs a = a0;
  const int64_t nb0 = hard_local_blocks(a.s[0].N);
  const int64_t nb1 = nside > 1 ? hard_local_blocks(a.s[1].N) : 0;
  a.nb0 = static_cast<int>(nb0);
  if (nb0 + nb1 == 0) return;
  note_launch();
  constexpr size_t smem = sizeof(uint64_t) * kHlRows + sizeof(float) * 32 * 32 * 33;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(hard_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  hard_local_kernel<<<static_cast<unsigned>(nb0 + nb1), kHtThreads, smem, st>>>(a, cand, side_stride, ws);
}

void launch_hard_topk(const HardArgs& a, int nside, cudaStream_t st) {
  note_launch();
  const int64_t nmax = nside > 1 && a.s[1].N > a.s[0].N ? a.s[1].N : a.s[0].N;
  if (nmax <= kHtCache) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(hard_topk_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(sizeof(uint64_t) * kHtCache));
      attr = true;
    }
    hard_topk_kernel<true><<<nside, kHtThreads, sizeof(uint64_t) * (nmax > 0 ? nmax : 1), st>>>(a);
  } else {
    hard_topk_kernel<false><<<nside, kHtThreads, 0, st>>>(a);
  }
}

}  // namespace cabsk
