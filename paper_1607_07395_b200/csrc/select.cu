// select.cu -- S8: the snap ("any k-means clustering center will be replaced
// with its closest in-sample point").  Readings Z13/Z14: nearest over ALL points,
// duplicates resolved greedily in order (-omega_j, j), each centre taking its
// nearest untaken point, ties -> lowest point index.
//
// distmat (kmeans.cu) writes D[j, p] = ||X_p - c_j||^2 (FP32 direct differences);
// topT keeps each centre's T nearest (d, index) pairs; dedupe runs the greedy
// pass in one CTA, rescanning D for a centre whose list is exhausted.
#include <float.h>

#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cabsk {

// ---------------------------------------------------------------- per-centre top-T
// grid (k2, S): block (j, s) keeps the T nearest (d, index) of centre j among points of
// segment s and writes them as list (slot0 + s) of the packed candidate array
// all[list][k2][T][{d, idx}] (doubles; idx < 2^53 exact).  Empty entries: idx = -1.
// (d, local index) packed as one 64-bit key: d >= 0, so its FP32 bit pattern orders like d,
// and the low word breaks ties by index -- the lexicographic (d, idx) order is the integer
// order of the key, and a sorted-list insertion is a chain of 64-bit min / max.
__device__ __forceinline__ uint64_t snap_key(float d, int64_t p) {
  return (static_cast<uint64_t>(__float_as_uint(d)) << 32) | static_cast<uint32_t>(p);
}

template <int T>
__global__ void __launch_bounds__(256) snap_topT_kernel(const float* __restrict__ D, int64_t ldd, int64_t N,
                                                        int64_t row_off, int k2, int slot0,
                                                        double* __restrict__ all) {
  __shared__ uint64_t hk[256];
  const int j = blockIdx.x, tid = threadIdx.x;
  const int64_t seg = ceil_div(N, gridDim.y);
  const int64_t pbeg = blockIdx.y * seg, pend = pbeg + seg < N ? pbeg + seg : N;
  uint64_t lk[T];
#pragma unroll
  for (int q = 0; q < T; ++q) lk[q] = ~0ull;
  const float* row = D + (int64_t)j * ldd;
  constexpr int kU = 8;  // distances loaded per batch (independent loads in flight)
  for (int64_t p0 = pbeg + tid; p0 < pend; p0 += kU * (int64_t)blockDim.x) {
    float vb[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t p = p0 + (int64_t)u * blockDim.x;
      vb[u] = p < pend ? __ldg(row + p) : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t p = p0 + (int64_t)u * blockDim.x;
      uint64_t c = p < pend ? snap_key(vb[u], p) : ~0ull;
      if (c < lk[T - 1]) {  // insertion into the sorted list
#pragma unroll
        for (int q = 0; q < T; ++q) {
          const uint64_t lo = c < lk[q] ? c : lk[q];
          c = c < lk[q] ? lk[q] : c;
          lk[q] = lo;
        }
      }
    }
  }
  // merge, two levels: T rounds of warp argmin over the lanes' list heads (shuffles only) give
  // each warp its sorted top T (lane r keeps the r-th); then one warp takes the top T of the
  // 8 warps' lists the same way, each lane holding 8T / 32 of those entries
  const int lane = tid & 31, wid = tid >> 5;
  int head = 0;
  uint64_t mine = ~0ull;
  for (int round = 0; round < T; ++round) {
    uint64_t b = ~0ull;
#pragma unroll
    for (int q = 0; q < T; ++q)
      if (q == head) b = lk[q];
    const uint64_t own = b;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t ob = __shfl_xor_sync(0xffffffffu, b, o);
      b = ob < b ? ob : b;
    }
    if (own == b && b != ~0ull) ++head;  // keys are unique: exactly one lane owns the winner
    if (lane == round) mine = b;
  }
  if (lane < T) hk[wid * T + lane] = mine;
  __syncthreads();
  if (wid == 0) {
    constexpr int kE = 8 * T / 32;  // entries per lane
    uint64_t e[kE];
#pragma unroll
    for (int q = 0; q < kE; ++q) e[q] = hk[q * 32 + lane];
    for (int round = 0; round < T; ++round) {
      uint64_t b = ~0ull;
#pragma unroll
      for (int q = 0; q < kE; ++q) b = e[q] < b ? e[q] : b;
      const uint64_t own = b;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint64_t ob = __shfl_xor_sync(0xffffffffu, b, o);
        b = ob < b ? ob : b;
      }
      if (own == b && b != ~0ull) {
#pragma unroll
        for (int q = 0; q < kE; ++q)
          if (e[q] == b) e[q] = ~0ull;
      }
      if (lane == round) mine = b;
    }
    if (lane < T) {
      const int64_t o = ((((int64_t)slot0 + blockIdx.y) * k2 + j) * T + lane) * 2;
      const bool empty = mine == ~0ull;
      all[o] = empty ? static_cast<double>(FLT_MAX) : static_cast<double>(__uint_as_float(static_cast<uint32_t>(mine >> 32)));
      all[o + 1] = empty ? -1.0 : static_cast<double>(row_off + static_cast<int64_t>(static_cast<uint32_t>(mine)));
    }
  }
}

void launch_snap_topT(const float* D, int64_t ldd, int64_t N, int k2, int64_t row_off, int T, int nseg, int slot0,
                      double* all, cudaStream_t st) {
  dim3 grid(k2, nseg);
  note_launch();
  if (T == kSnapT) {
    snap_topT_kernel<kSnapT><<<grid, 256, 0, st>>>(D, ldd, N, row_off, k2, slot0, all);
  } else {
    snap_topT_kernel<kSnapTMulti><<<grid, 256, 0, st>>>(D, ldd, N, row_off, k2, slot0, all);
  }
}

// ---------------------------------------------------------------- multi-rank candidate exchange
// Merge of the packed per-segment (and per-rank) lists: the global T nearest per centre,
// ordered by (d, idx).  Lists of other ranks are zero-filled slots completed by a sum-allreduce.
// One warp per centre: T rounds of a warp-wide search for the lexicographic successor of
// the previous winner over all nlists * T entries (indices are distinct across lists:
// segments and ranks partition the points).
__global__ void __launch_bounds__(128) snap_merge_kernel(const double* __restrict__ all, int k2, int T, int nlists,
                                                         float* __restrict__ cand_d, int64_t* __restrict__ cand_i) {
  const int j = blockIdx.x * 4 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (j >= k2) return;
  const int ne = nlists * T;
  if (ne <= 64) {  // every entry loaded once into registers (two per lane), then T warp argmins
    float ed[2];
    int64_t ei[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = lane + 32 * h;
      ed[h] = FLT_MAX;
      ei[h] = INT64_MAX;
      if (e < ne) {
        const int r = e / T, q = e - r * T;
        const int64_t off = (((int64_t)r * k2 + j) * T + q) * 2;
        const int64_t i = static_cast<int64_t>(all[off + 1]);
        if (i >= 0) { ed[h] = static_cast<float>(all[off]); ei[h] = i; }
      }
    }
    for (int t = 0; t < T; ++t) {
      const bool first = lex_less(ed[0], ei[0], ed[1], ei[1]);
      float bd = first ? ed[0] : ed[1];
      int64_t bi = first ? ei[0] : ei[1];
      const int64_t own = bi;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float od = __shfl_xor_sync(0xffffffffu, bd, o);
        const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (lex_less(od, oi, bd, bi)) { bd = od; bi = oi; }
      }
      if (bi != INT64_MAX && own == bi) {  // (d, idx) pairs are unique: the owner drops it
        if (first) { ed[0] = FLT_MAX; ei[0] = INT64_MAX; }
        else { ed[1] = FLT_MAX; ei[1] = INT64_MAX; }
      }
      if (lane == 0) {
        cand_d[(int64_t)j * T + t] = bi == INT64_MAX ? FLT_MAX : bd;
        cand_i[(int64_t)j * T + t] = bi == INT64_MAX ? -1 : bi;
      }
    }
    return;
  }
  float pd = -FLT_MAX;
  int64_t pi = -1;  // previous winner
  for (int t = 0; t < T; ++t) {
    float bd = FLT_MAX;
    int64_t bi = INT64_MAX;
    for (int e = lane; e < ne; e += 32) {
      const int r = e / T, q = e - r * T;
      const int64_t off = (((int64_t)r * k2 + j) * T + q) * 2;
      const int64_t i = static_cast<int64_t>(all[off + 1]);
      if (i < 0) continue;
      const float d = static_cast<float>(all[off]);
      if (lex_less(pd, pi, d, i) && lex_less(d, i, bd, bi)) { bd = d; bi = i; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float od = __shfl_xor_sync(0xffffffffu, bd, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (lex_less(od, oi, bd, bi)) { bd = od; bi = oi; }
    }
    if (lane == 0) {
      cand_d[(int64_t)j * T + t] = bd;
      cand_i[(int64_t)j * T + t] = bi == INT64_MAX ? -1 : bi;
    }
    if (bi == INT64_MAX) {  // lists exhausted: the remaining slots stay empty
      for (int t2 = t + 1 + lane; t2 < T; t2 += 32) {
        cand_d[(int64_t)j * T + t2] = FLT_MAX;
        cand_i[(int64_t)j * T + t2] = -1;
      }
      break;
    }
    pd = bd;
    pi = bi;
  }
}

void launch_snap_merge(const double* all, int k2, int T, int nlists, float* cand_d, int64_t* cand_i, cudaStream_t st) {
  note_launch();
  snap_merge_kernel<<<static_cast<unsigned>(ceil_div(k2, 4)), 128, 0, st>>>(all, k2, T, nlists, cand_d, cand_i);
}

// ---------------------------------------------------------------- greedy dedupe (one CTA)
constexpr int kTakenBits = 11;  // capacity 2048 >= 2 * CABS_KMAX
constexpr int kTakenCap = 1 << kTakenBits;

__device__ __forceinline__ uint32_t taken_hash(int64_t x) {
  return static_cast<uint32_t>((static_cast<uint64_t>(x) * 0x9E3779B97F4A7C15ull) >> (64 - kTakenBits));
}
__device__ __forceinline__ bool taken_has(const int64_t* tab, int64_t x) {
  uint32_t h = taken_hash(x);
  while (tab[h] != -1) {
    if (tab[h] == x) return true;
    h = (h + 1) & (kTakenCap - 1);
  }
  return false;
}
__device__ __forceinline__ void taken_put(int64_t* tab, int64_t x) {
  uint32_t h = taken_hash(x);
  while (tab[h] != -1) h = (h + 1) & (kTakenCap - 1);
  tab[h] = x;
}

#ifdef CABS_PROFILE_SNAP
__device__ unsigned long long g_snap_prof[4];  // rescans, greedy-pass cycles
#endif
// The taken set of the greedy pass: a bitmap over the local point indices when the rank owns
// all points (single GPU) and the bitmap fits shared memory (one BIT per point: 1.3e6 points in
// 160 KB; a put is one plain read-modify-write by the single writing lane), else the
// open-addressing hash table of global indices.
constexpr int64_t kBitmapMax = int64_t(1) << 22;
struct TakenSet {
  unsigned* bits;  // one bit per local point; null: hash table
  int64_t* tab;
  int64_t off;
  __device__ __forceinline__ bool has(int64_t x) const {
    if (bits) {
      const int64_t l = x - off;
      return (bits[l >> 5] >> (l & 31)) & 1u;
    }
    return taken_has(tab, x);
  }
  __device__ __forceinline__ void put(int64_t x) {
    if (bits) {
      const int64_t l = x - off;
      bits[l >> 5] |= 1u << (l & 31);
    } else {
      taken_put(tab, x);
    }
  }
};

constexpr int kDedupeThreads = 1024;  // the greedy pass is one warp; the rescans use every thread

__global__ void __launch_bounds__(kDedupeThreads) snap_dedupe_kernel(const float* cand_d, const int64_t* cand_i, int k2, int T,
                                                          const double* __restrict__ cluster_w,
                                                          const float* __restrict__ D, int64_t ldd, int64_t N,
                                                          int64_t row_off, bool can_rescan,
                                                          int64_t* __restrict__ rep_of_centre, float* __restrict__ gap,
                                                          int64_t* __restrict__ reps_sorted, void* ws,
                                                          bool staged, bool use_bitmap, int* unresolved) {
  __shared__ int64_t tab[kTakenCap];
  __shared__ int order[CABS_KMAX];
  __shared__ int64_t reps[CABS_KMAX];
  __shared__ float r_d1[CABS_KMAX], r_d2[CABS_KMAX];  // per centre: its distance, the runner-up's
  __shared__ double s_w[CABS_KMAX];
  __shared__ int s_next;      // next position in `order` to process
  __shared__ int s_rescan;    // centre needing a rescan, or -1
  __shared__ float rd[kDedupeThreads / 32], rs[kDedupeThreads / 32];
  __shared__ int64_t ri[kDedupeThreads / 32], ri2[kDedupeThreads / 32];
  __shared__ unsigned char s_t1[CABS_KMAX], s_t2[CABS_KMAX];  // fast path: chosen candidate slots
  // dynamic: candidates in visiting order [k2][T] (int64 | float), then the bitmap
  extern __shared__ __align__(16) unsigned char cand_smem[];
  const int tid = threadIdx.x;
  // candidates by visiting position: staged in shared memory in that order, or (too large)
  // read from global memory through order[]
  int64_t* csi = reinterpret_cast<int64_t*>(cand_smem);
  float* csd = reinterpret_cast<float*>(csi + (size_t)(staged ? k2 * T : 0));
  auto cand_at = [&](int o, int t) -> int64_t { return staged ? csi[(int64_t)o * T + t] : cand_i[(int64_t)order[o] * T + t]; };
  auto dist_at = [&](int o, int t) -> float { return staged ? csd[(int64_t)o * T + t] : cand_d[(int64_t)order[o] * T + t]; };
  TakenSet taken;
  taken.tab = tab;
  taken.off = row_off;
  taken.bits = nullptr;
  if (use_bitmap) {
    taken.bits = reinterpret_cast<unsigned*>(
        cand_smem + (staged ? (((size_t)k2 * T * (sizeof(int64_t) + sizeof(float)) + 15) & ~size_t(15)) : 0));
    for (int64_t e = tid; e < (N + 31) / 32; e += blockDim.x) taken.bits[e] = 0u;
  } else {
    for (int e = tid; e < kTakenCap; e += blockDim.x) tab[e] = -1;
  }
  // visiting order (-omega_j, j)
  for (int j = tid; j < k2; j += blockDim.x) s_w[j] = cluster_w[j];
  __syncthreads();
  for (int j = tid; j < k2; j += blockDim.x) {
    const double wj = s_w[j];
    int rk = 0;
    for (int q = 0; q < k2; ++q) {
      const double wq = s_w[q];
      rk += (wq > wj) || (wq == wj && q < j);
    }
    order[rk] = j;
  }
  __syncthreads();
  // candidates staged in visiting order: the greedy pass reads position o without first
  // looking up order[o]
  if (staged) {
    for (int e = tid; e < k2 * T; e += blockDim.x) {
      const int o = e / T, t = e - o * T;
      const int j = order[o];
      csi[e] = cand_i[(int64_t)j * T + t];
      csd[e] = cand_d[(int64_t)j * T + t];
    }
  }
  if (tid == 0) s_next = 0;
  __syncthreads();
#ifdef CABS_PROFILE_SNAP
  long long tp0 = clock64();
#endif
  for (;;) {
    if (tid < 32) {  // warp 0: the greedy pass, lane t checks candidate t of the current centre
      const int lane = tid;
      if (lane == 0) s_rescan = -1;
      const int o0 = s_next;
      int o = o0;
      int64_t ci = (o < k2 && lane < T) ? cand_at(o, lane) : -1;
      if (staged && taken.bits) {
        // fast path: the only loop-carried dependency is the taken set, so the chain per centre
        // is probe -> ballot -> the winning lane's one-byte store -> __syncwarp; the choices
        // (t1, t2 per visiting position) are turned into outputs after the pass
        for (; o < k2; ++o) {
          const bool ok = ci >= 0 && !taken.has(ci);
          const int64_t cn = (o + 1 < k2 && lane < T) ? cand_at(o + 1, lane) : -1;
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          const unsigned m2 = m & (m - 1);
          if (m2 == 0u) {  // best or runner-up not resolved from the list (can_rescan holds here)
            if (lane == 0) s_rescan = order[o];
            break;
          }
          if (lane == __ffs(m) - 1) taken.put(ci);
          if (lane == 0) {
            s_t1[o] = static_cast<unsigned char>(__ffs(m) - 1);
            s_t2[o] = static_cast<unsigned char>(__ffs(m2) - 1);
          }
          __syncwarp();  // the new entry of the taken set is visible to the next centre's probes
          ci = cn;
        }
        __syncwarp();
        for (int q = o0 + lane; q < o; q += 32) {
          const int j = order[q], t1 = s_t1[q], t2 = s_t2[q];
          reps[j] = cand_at(q, t1);
          r_d1[j] = dist_at(q, t1);
          r_d2[j] = dist_at(q, t2);
        }
      } else {
        for (; o < k2; ++o) {
          const bool ok = ci >= 0 && !taken.has(ci);
          // prefetch the next centre's candidates (independent of the taken set)
          const int64_t cn = (o + 1 < k2 && lane < T) ? cand_at(o + 1, lane) : -1;
          const unsigned m = __ballot_sync(0xffffffffu, ok);
          const int t1 = m ? __ffs(m) - 1 : -1;
          const unsigned m2 = m & (m - 1);
          const int t2 = m2 ? __ffs(m2) - 1 : -1;
          int64_t i1 = __shfl_sync(0xffffffffu, ci, t1 < 0 ? 0 : t1);
          if (t1 < 0) i1 = -1;
          if (t2 < 0 && can_rescan) {  // best or runner-up not resolved from the list
            if (lane == 0) s_rescan = order[o];
            break;
          }
          // multi-rank: D holds only this rank's points, no rescan here; the caller redoes the
          // pass with snap_dist_* (exact) when this flag is raised
          if (t2 < 0 && unresolved && lane == 0) *unresolved = 1;
          if (lane == 0) {
            const int j = order[o];
            float d1 = t1 >= 0 ? dist_at(o, t1) : FLT_MAX;
            if (i1 < 0) { set_status(ws, CABS_DEV_SNAP_EXHAUSTED); i1 = 0; d1 = 0.f; }
            taken.put(i1);
            reps[j] = i1;
            r_d1[j] = d1;
            r_d2[j] = t2 >= 0 ? dist_at(o, t2) : FLT_MAX;
          }
          __syncwarp();  // the new entry of the taken set is visible to the next centre's probes
          ci = cn;
        }
      }
      if (lane == 0) s_next = o;
    }
    __syncthreads();
    const int j = s_rescan;
#ifdef CABS_PROFILE_SNAP
    if (tid == 0) { atomicAdd(&g_snap_prof[1], static_cast<unsigned long long>(clock64() - tp0)); tp0 = clock64(); if (j >= 0) atomicAdd(&g_snap_prof[0], 1ull); }
#endif
    if (j < 0) break;
    // block-wide rescan of D[j, :] for the best and runner-up untaken points
    float b1 = FLT_MAX, b2 = FLT_MAX;
    int64_t i1 = INT64_MAX, i2 = INT64_MAX;
    const float* row = D + (int64_t)j * ldd;
    // 16-byte loads (four in flight per thread, 64 KB per CTA: one SM streams the row at a useful
    // rate); the taken set is probed only for an entry that would enter the thread's top two (the
    // same result: the others cannot)
    auto consider = [&](float v, int64_t p) {
      const int64_t gi = row_off + p;
      if (!lex_less(v, gi, b2, i2) || taken.has(gi)) return;
      if (lex_less(v, gi, b1, i1)) { b2 = b1; i2 = i1; b1 = v; i1 = gi; }
      else { b2 = v; i2 = gi; }
    };
    const int64_t head = N < 4 ? N : static_cast<int64_t>((4 - ((reinterpret_cast<uintptr_t>(row) >> 2) & 3)) & 3);
    if (tid < head) consider(__ldcg(row + tid), tid);
    const int64_t nv = (N - head) >> 2;  // whole float4 groups after the head
    const float4* rv = reinterpret_cast<const float4*>(row + head);
    constexpr int kRu = 4;
    for (int64_t v0 = tid; v0 < nv; v0 += kRu * (int64_t)blockDim.x) {
      float4 vb[kRu];
#pragma unroll
      for (int u = 0; u < kRu; ++u) {
        const int64_t v = v0 + (int64_t)u * blockDim.x;
        vb[u] = v < nv ? __ldcg(rv + v) : make_float4(FLT_MAX, FLT_MAX, FLT_MAX, FLT_MAX);
      }
#pragma unroll
      for (int u = 0; u < kRu; ++u) {
        const int64_t v = v0 + (int64_t)u * blockDim.x;
        if (v >= nv) continue;
        const int64_t p = head + 4 * v;
        consider(vb[u].x, p);
        consider(vb[u].y, p + 1);
        consider(vb[u].z, p + 2);
        consider(vb[u].w, p + 3);
      }
    }
    for (int64_t p = head + 4 * nv + tid; p < N; p += blockDim.x) consider(__ldcg(row + p), p);
    // reduce the (best, runner-up) pairs: warp butterflies, then the 8 warp results; the
    // lexicographic (distance, index) order is total, so the top two are unique and the
    // merge order does not matter
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ob1 = __shfl_xor_sync(0xffffffffu, b1, o), ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
      const int64_t oi1 = __shfl_xor_sync(0xffffffffu, i1, o), oi2 = __shfl_xor_sync(0xffffffffu, i2, o);
      if (lex_less(ob1, oi1, b1, i1)) {  // other best wins: runner-up = min(own best, other runner-up)
        if (lex_less(b1, i1, ob2, oi2)) { b2 = b1; i2 = i1; }
        else { b2 = ob2; i2 = oi2; }
        b1 = ob1; i1 = oi1;
      } else if (lex_less(ob1, oi1, b2, i2)) {
        b2 = ob1; i2 = oi1;
      }
    }
    const int wid = tid >> 5;
    if ((tid & 31) == 0) { rd[wid] = b1; ri[wid] = i1; rs[wid] = b2; ri2[wid] = i2; }
    __syncthreads();
    if (tid == 0) {
      float B1 = FLT_MAX, B2 = FLT_MAX;
      int64_t I1 = INT64_MAX, I2 = INT64_MAX;
      for (int t = 0; t < static_cast<int>(blockDim.x >> 5); ++t) {
        const float cands_d[2] = {rd[t], rs[t]};
        const int64_t cands_i[2] = {ri[t], ri2[t]};
        for (int q = 0; q < 2; ++q) {
          const float v = cands_d[q];
          const int64_t gi = cands_i[q];
          if (gi == INT64_MAX) continue;
          if (lex_less(v, gi, B1, I1)) { B2 = B1; I2 = I1; B1 = v; I1 = gi; }
          else if (lex_less(v, gi, B2, I2)) { B2 = v; I2 = gi; }
        }
      }
      if (I1 == INT64_MAX) { set_status(ws, CABS_DEV_SNAP_EXHAUSTED); I1 = 0; B1 = 0.f; }
      taken.put(I1);
      reps[j] = I1;
      r_d1[j] = B1;
      r_d2[j] = I2 == INT64_MAX ? FLT_MAX : B2;
      s_next = s_next + 1;
    }
    __syncthreads();
  }
  __syncthreads();
  for (int j = tid; j < k2; j += blockDim.x) {  // outputs of every centre, and the sorted representatives
    const int64_t v = reps[j];
    if (rep_of_centre) rep_of_centre[j] = v;
    if (gap) {
      const float d1 = r_d1[j], d2 = r_d2[j];
      gap[j] = (d2 == FLT_MAX) ? FLT_MAX : (d2 > 0.f ? (d2 - d1) / d2 : 0.f);
    }
    int rk = 0;
    for (int q = 0; q < k2; ++q) rk += reps[q] < v;
    reps_sorted[rk] = v;
  }
}

void snap_debug_counters(long long* out) {
#ifdef CABS_PROFILE_SNAP
  cudaMemcpyFromSymbol(out, g_snap_prof, sizeof(long long) * 4);
#else
  for (int i = 0; i < 4; ++i) out[i] = 0;
#endif
}

void launch_snap_dedupe(const float* cand_d, const int64_t* cand_i, int k2, int T, const double* cluster_w,
                        const float* D, int64_t ldd, int64_t N, int64_t row_off, bool can_rescan,
                        int64_t* rep_of_centre, float* gap, int64_t* reps_sorted, void* ws, cudaStream_t st,
                        int* unresolved) {
  constexpr size_t kCap = 160 * 1024;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(snap_dedupe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kCap));
    attr = true;
  }
  size_t cand = (((size_t)k2 * T * (sizeof(int64_t) + sizeof(float))) + 15) & ~size_t(15);
  const bool staged = cand <= kCap;
  if (!staged) cand = 0;
  const size_t bits = ((N + 127) / 128) * 16;  // one bit per point (16-byte multiple)
  const bool bitmap = can_rescan && N <= kBitmapMax && cand + bits <= kCap && !getenv("CABS_SNAP_HASH");
  const size_t bytes = cand + (bitmap ? bits : 0);
  note_launch();
  snap_dedupe_kernel<<<1, kDedupeThreads, bytes, st>>>(cand_d, cand_i, k2, T, cluster_w, D, ldd, N, row_off, can_rescan,
                                            rep_of_centre, gap, reps_sorted, ws, staged, bitmap, unresolved);
}

// ---------------------------------------------------------------- multi-rank exact greedy pass
// When the exchanged lists leave some centre's best or runner-up unresolved (T-1 or more of its
// T nearest points already taken), the greedy pass of readings Z13/Z14 is redone centre by
// centre over the whole distance matrix: every rank scans ITS rows of D[j, :] for its two
// nearest untaken points (snap_dist_scan + snap_dist_local), the ranks' pairs meet in one
// sum-allreduce of 4 doubles per rank (zeros elsewhere), and every rank takes the same winner
// (snap_dist_take).  k2 small collectives: slow, exact, and only taken when needed.
struct SnapDist {
  int* order;       // [k2] visiting order (-omega_j, j)
  int* count;       // [1] number of taken points
  int64_t* taken;   // [k2] taken global indices, ascending
  int64_t* reps;    // [k2] per centre
  float* d1;        // [k2]
  float* d2;        // [k2]
  double* slots;    // [4 nranks] (d1, i1, d2, i2) per rank, empty: (FLT_MAX, -1)
  float* bd;        // [2 G] per-block top two
  int64_t* bi;
};
constexpr int kSnapDistG = 64;  // scan blocks

size_t snap_dist_bytes(int k2, int nranks) {
  return (size_t)k2 * (4 + 8 + 8 + 4 + 4) + 64 + sizeof(double) * 4 * nranks + (size_t)2 * kSnapDistG * 12 + 256;
}

static SnapDist snap_dist_carve(void* buf, int k2, int nranks) {
  char* b = static_cast<char*>(buf);
  SnapDist s;
  s.slots = reinterpret_cast<double*>(b);  b += sizeof(double) * 4 * nranks;
  s.taken = reinterpret_cast<int64_t*>(b); b += sizeof(int64_t) * k2;
  s.reps = reinterpret_cast<int64_t*>(b);  b += sizeof(int64_t) * k2;
  s.bi = reinterpret_cast<int64_t*>(b);    b += sizeof(int64_t) * 2 * kSnapDistG;
  s.bd = reinterpret_cast<float*>(b);      b += sizeof(float) * 2 * kSnapDistG;
  s.d1 = reinterpret_cast<float*>(b);      b += sizeof(float) * k2;
  s.d2 = reinterpret_cast<float*>(b);      b += sizeof(float) * k2;
  s.order = reinterpret_cast<int*>(b);     b += sizeof(int) * k2;
  s.count = reinterpret_cast<int*>(b);
  return s;
}

__global__ void __launch_bounds__(256) snap_dist_init_kernel(const double* __restrict__ cluster_w, int k2, SnapDist s) {
  for (int j = threadIdx.x; j < k2; j += blockDim.x) {
    const double wj = cluster_w[j];
    int rk = 0;
    for (int q = 0; q < k2; ++q) {
      const double wq = cluster_w[q];
      rk += (wq > wj) || (wq == wj && q < j);
    }
    s.order[rk] = j;
  }
  if (threadIdx.x == 0) *s.count = 0;
}

// the (best, runner-up) pair update in lexicographic (d, idx) order
__device__ __forceinline__ void top2_push(float v, int64_t i, float& b1, int64_t& i1, float& b2, int64_t& i2) {
  if (lex_less(v, i, b1, i1)) { b2 = b1; i2 = i1; b1 = v; i1 = i; }
  else if (lex_less(v, i, b2, i2)) { b2 = v; i2 = i; }
}

__device__ void block_top2(float& b1, int64_t& i1, float& b2, int64_t& i2) {  // result valid in thread 0
  __shared__ float sd[16];
  __shared__ int64_t si[16];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ob1 = __shfl_xor_sync(0xffffffffu, b1, o), ob2 = __shfl_xor_sync(0xffffffffu, b2, o);
    const int64_t oi1 = __shfl_xor_sync(0xffffffffu, i1, o), oi2 = __shfl_xor_sync(0xffffffffu, i2, o);
    top2_push(ob1, oi1, b1, i1, b2, i2);
    top2_push(ob2, oi2, b1, i1, b2, i2);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { sd[2 * w] = b1; si[2 * w] = i1; sd[2 * w + 1] = b2; si[2 * w + 1] = i2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int e = 2; e < 2 * static_cast<int>(blockDim.x >> 5); ++e) top2_push(sd[e], si[e], b1, i1, b2, i2);
  }
}

__global__ void __launch_bounds__(256) snap_dist_scan_kernel(const float* __restrict__ D, int64_t ldd, int64_t N,
                                                             int64_t row_off, int o, SnapDist s) {
  __shared__ int64_t tk[CABS_KMAX];
  const int cnt = *s.count;
  for (int e = threadIdx.x; e < cnt; e += blockDim.x) tk[e] = s.taken[e];
  __syncthreads();
  const float* row = D + (int64_t)s.order[o] * ldd;
  float b1 = FLT_MAX, b2 = FLT_MAX;
  int64_t i1 = INT64_MAX, i2 = INT64_MAX;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < N; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t gi = row_off + p;
    int lo = 0, hi = cnt;  // binary search of the sorted taken list
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (tk[mid] < gi) lo = mid + 1; else hi = mid;
    }
    if (lo < cnt && tk[lo] == gi) continue;
    top2_push(row[p], gi, b1, i1, b2, i2);
  }
  block_top2(b1, i1, b2, i2);
  if (threadIdx.x == 0) {
    s.bd[2 * blockIdx.x] = b1; s.bi[2 * blockIdx.x] = i1;
    s.bd[2 * blockIdx.x + 1] = b2; s.bi[2 * blockIdx.x + 1] = i2;
  }
}

__global__ void __launch_bounds__(32) snap_dist_local_kernel(int G, int rank, int nranks, SnapDist s) {
  if (threadIdx.x != 0) return;
  float b1 = FLT_MAX, b2 = FLT_MAX;
  int64_t i1 = INT64_MAX, i2 = INT64_MAX;
  for (int e = 0; e < 2 * G; ++e) top2_push(s.bd[e], s.bi[e], b1, i1, b2, i2);
  for (int r = 0; r < nranks; ++r) {
    double* sl = s.slots + 4 * r;
    if (r == rank) {
      sl[0] = i1 == INT64_MAX ? static_cast<double>(FLT_MAX) : static_cast<double>(b1);
      sl[1] = i1 == INT64_MAX ? -1.0 : static_cast<double>(i1);
      sl[2] = i2 == INT64_MAX ? static_cast<double>(FLT_MAX) : static_cast<double>(b2);
      sl[3] = i2 == INT64_MAX ? -1.0 : static_cast<double>(i2);
    } else {
      sl[0] = sl[1] = sl[2] = sl[3] = 0.0;
    }
  }
}

__global__ void __launch_bounds__(32) snap_dist_take_kernel(int o, int nranks, SnapDist s, void* ws) {
  if (threadIdx.x != 0) return;
  float b1 = FLT_MAX, b2 = FLT_MAX;
  int64_t i1 = INT64_MAX, i2 = INT64_MAX;
  for (int e = 0; e < 2 * nranks; ++e) {
    const int64_t i = static_cast<int64_t>(s.slots[2 * e + 1]);
    if (i >= 0) top2_push(static_cast<float>(s.slots[2 * e]), i, b1, i1, b2, i2);
  }
  const int j = s.order[o];
  if (i1 == INT64_MAX) { set_status(ws, CABS_DEV_SNAP_EXHAUSTED); i1 = 0; b1 = 0.f; }
  s.reps[j] = i1;
  s.d1[j] = b1;
  s.d2[j] = i2 == INT64_MAX ? FLT_MAX : b2;
  int c = *s.count;  // sorted insertion
  while (c > 0 && s.taken[c - 1] > i1) { s.taken[c] = s.taken[c - 1]; --c; }
  s.taken[c] = i1;
  *s.count += 1;
}

__global__ void __launch_bounds__(256) snap_dist_finish_kernel(int k2, SnapDist s, int64_t* __restrict__ rep_of_centre,
                                                               float* __restrict__ gap, int64_t* __restrict__ reps_sorted) {
  for (int j = threadIdx.x; j < k2; j += blockDim.x) {  // the same outputs as snap_dedupe_kernel
    const int64_t v = s.reps[j];
    if (rep_of_centre) rep_of_centre[j] = v;
    if (gap) {
      const float d1 = s.d1[j], d2 = s.d2[j];
      gap[j] = (d2 == FLT_MAX) ? FLT_MAX : (d2 > 0.f ? (d2 - d1) / d2 : 0.f);
    }
    int rk = 0;
    for (int q = 0; q < k2; ++q) rk += s.reps[q] < v;
    reps_sorted[rk] = v;
  }
}

int snap_dist_run(const float* D, int64_t ldd, int64_t N, int64_t row_off, int k2, const double* cluster_w,
                  int rank, int nranks, void* buf, int64_t* rep_of_centre, float* gap, int64_t* reps_sorted,
                  void* ws, cudaStream_t st, int (*allreduce)(double*, int64_t, void*), void* ctx) {
  const SnapDist s = snap_dist_carve(buf, k2, nranks);
  int G = static_cast<int>(ceil_div(N > 0 ? N : 1, 1024));
  if (G > kSnapDistG) G = kSnapDistG;
  note_launch();
  snap_dist_init_kernel<<<1, 256, 0, st>>>(cluster_w, k2, s);
  for (int o = 0; o < k2; ++o) {
    note_launch();
    snap_dist_scan_kernel<<<G, 256, 0, st>>>(D, ldd, N, row_off, o, s);
    note_launch();
    snap_dist_local_kernel<<<1, 32, 0, st>>>(G, rank, nranks, s);
    if (cudaGetLastError() != cudaSuccess) return -1;
    if (allreduce && allreduce(s.slots, 4LL * nranks, ctx) != 0) return -2;
    note_launch();
    snap_dist_take_kernel<<<1, 32, 0, st>>>(o, nranks, s, ws);
  }
  note_launch();
  snap_dist_finish_kernel<<<1, 256, 0, st>>>(k2, s, rep_of_centre, gap, reps_sorted);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace cabsk
