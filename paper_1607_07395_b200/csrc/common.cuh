// common.cuh -- shared helpers of libcabs (workspace layout, status word, reductions).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/cabs.h"

namespace cabsk {

constexpr int kNumSM = 148;           // B200: 2 dies x 74 SMs
constexpr int kSnapT = 8;             // per-centre candidate list length in the snap
constexpr int kSnapTMulti = 32;       // ... when candidates are merged across ranks
constexpr int kSnapSeg = 8;           // point segments scanned in parallel per centre
constexpr int kAccGrid = 2 * kNumSM;  // k-means accumulation CTAs (per-CTA partials)
constexpr int kAssignGrid = 4 * kNumSM;
constexpr int kResGrid = 8 * kNumSM;  // persistent residual CTAs (upper bound)
constexpr int kNormTile = 64;         // points per embed-GEMM tile (norm partial rows)
constexpr int kKmItersCap = 256;      // Lloyd iterations the persistent kernel's scratch covers
constexpr int kOrthMaxBlocks = 148;   // Gram-partial CTAs per side (cabs_orthogonalize)
constexpr int kHardLocalRows = 2048;  // rows per CTA of the hard-threshold key + local top-k kernel

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// ---------------------------------------------------------------- workspace
struct Ws {
  size_t status, scal;
  size_t w64, a64, v64, sig64, uw32, vw32;
  size_t qr;  // SVD QR preconditioner: R scratch (K x K FP64) + pivots (K int)
  size_t norm_part, norms, scales;
  size_t km_w, km_scr, km_pobj, km_ptie, km_red, km_cnt;  // km_w, km_scr, km_cnt: two problems
  size_t km_scr_bytes;                                     // per problem
  size_t km_q;                                             // lloyd_prune: w ||x||^2 per point (int64), two problems
  size_t dist, cand_d, cand_i, cand_all;  // snap scratch of problem slot 0 ...
  size_t dist2, cand_d2, cand_i2, cand_all2;  // ... and slot 1 (cabs_select_pair)
  size_t hcand, idx;
  size_t cb, rb, wb;
  size_t res_part, res_split;  // res_split: G_hi, G_lo (TF32: n x round_up(ncomp, 32) each, <= 192; FP16: n x round_up(ncomp, 64) halves, <= 384)
  size_t hcand_side;
  size_t orth_part, orth;  // cabs_orthogonalize: Gram partials | gram, U_K, V_K, sigma, r, K, T_U, T_V
  size_t total;
  // dims
  int64_t K, Kp, m_loc, n_sl, Nmax, n, ldrb, npt;
};

inline Ws ws_layout(const cabs_plan& p) {
  Ws w{};
  w.K = p.kmax;
  w.Kp = round_up(w.K, 32);
  w.m_loc = p.row_end - p.row_begin;
  w.n_sl = p.col_end - p.col_begin;
  w.Nmax = w.m_loc > w.n_sl ? w.m_loc : w.n_sl;
  if (w.Nmax < 1) w.Nmax = 1;
  w.n = p.n;
  w.ldrb = round_up(p.n, 4);
  w.npt = ceil_div(w.Nmax, kNormTile);
  const int64_t K = w.K, Kp = w.Kp;
  const int nr = p.nranks > 0 ? p.nranks : 1;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  w.status = take(256);
  w.scal = take(4096);
  w.w64 = take(sizeof(double) * K * K);
  w.a64 = take(sizeof(double) * K * K);
  w.v64 = take(sizeof(double) * (K * K + K));  // (+ K: the QR preconditioner's reflector scales)
  // QR preconditioner: R scratch (K x K) + pivots (K int); for k > 128 (grid kernel) also the
  // double-buffered column copies [2][K][round_up(K, 32)], the per-CTA bests [2][128][2], R_jj
  // (K) and the barrier counter
  w.qr = take(sizeof(double) * K * K + sizeof(int) * K +
              (K > 128 ? sizeof(double) * (2 * K * Kp + 2 * 128 * 2 + K) + 256 : 0));
  w.sig64 = take(sizeof(double) * Kp);
  w.uw32 = take(sizeof(float) * K * Kp);
  w.vw32 = take(sizeof(float) * K * Kp);
  w.norm_part = take(sizeof(double) * 2 * w.npt * Kp);
  w.norms = take(sizeof(double) * 2 * Kp);
  w.scales = take(sizeof(float) * 8 * Kp);
  w.km_w = take(sizeof(float) * 2 * w.Nmax);
  // k-means scratch per problem: int64 sums [3][K*Kp + K (+1: 16-byte slots)] | grid barrier |
  // objective and near-tie partials [kKmItersCap][2 kNumSM] (the persistent kernel: up to two
  // CTAs per SM; the per-iteration path uses the first K*Kp + K sums)
  w.km_scr_bytes = (sizeof(long long) * 3 * ((size_t)K * Kp + K + 1) + 16 +
                    (sizeof(double) + sizeof(int)) * kKmItersCap * 2 * kNumSM + 255) & ~size_t(255);
  w.km_scr = take(2 * w.km_scr_bytes);
  w.km_pobj = take(sizeof(double) * kAssignGrid);
  w.km_ptie = take(sizeof(int) * kAssignGrid);
  w.km_red = take(sizeof(double) * 2 * (K * Kp + K + 2));  // two problems' payloads (fused pair)
  w.km_q = take(sizeof(long long) * 2 * w.Nmax);
  w.km_cnt = take(sizeof(int) * 64);
  w.dist = take(sizeof(float) * K * w.Nmax);
  w.cand_d = take(sizeof(float) * K * kSnapTMulti);
  w.cand_i = take(sizeof(int64_t) * K * kSnapTMulti);
  w.cand_all = take(sizeof(double) * 2 * nr * kSnapSeg * K * kSnapTMulti);
  w.dist2 = take(sizeof(float) * K * w.Nmax);
  w.cand_d2 = take(sizeof(float) * K * kSnapTMulti);
  w.cand_i2 = take(sizeof(int64_t) * K * kSnapTMulti);
  w.cand_all2 = take(sizeof(double) * 2 * nr * kSnapSeg * K * kSnapTMulti);
  // hard threshold: (key, index) candidates of every 2048-row CTA, both sides of a pair
  w.hcand_side = 2 * ceil_div(w.Nmax, kHardLocalRows) * K;  // doubles per side
  w.hcand = take(sizeof(double) * 2 * w.hcand_side);
  {  // cabs_orthogonalize (orth.cu): Gram partials of <= max(kOrthMaxBlocks, tile pairs) CTAs per side
    const int64_t nt = (K + 63) / 64, np = nt * (nt + 1) / 2;
    w.orth_part = take(sizeof(double) * 2 * (np > kOrthMaxBlocks ? np : kOrthMaxBlocks) * 64 * 64);
  }
  w.orth = take(sizeof(double) * (4 * K * K + K) + 256 + sizeof(float) * 3 * K * Kp);
  w.idx = take(sizeof(int64_t) * 8 * Kp);
  w.cb = take(sizeof(float) * (w.m_loc > 0 ? w.m_loc : 1) * Kp);
  w.rb = take(sizeof(float) * K * w.ldrb);
  w.wb = take(sizeof(float) * K * Kp);
  w.res_part = take(sizeof(double) * 2 * kResGrid);
  // G hi/lo (TF32: pitch round_up(K, 32) <= 192; FP16: round_up(K, 64) <= 384 halves) + max; G has n rows, or
  // m_loc rows when the block is column-major (cabs_source.transposed: the factors are exchanged)
  w.res_split = take(sizeof(float) * 2 * (size_t)(p.n > w.m_loc ? p.n : w.m_loc) * (Kp < 192 ? Kp : 192) + 256);
  w.total = off;
  return w;
}

template <typename T>
inline T* wsp(void* ws, size_t off) {
  return reinterpret_cast<T*>(static_cast<char*>(ws) + off);
}

// scalar slots inside ws.scal (ints)
enum ScalSlot : int { SCAL_R_PILOT = 0, SCAL_R_TMP = 1, SCAL_NRANKS = 2, SCAL_EXHAUST = 3, SCAL_EBAR = 4 /* [2] */,
                       SCAL_UNRES = 8 /* [2]: a multi-rank snap left a centre unresolved */ };

__device__ inline void set_status(void* ws, uint32_t bit) {
  atomicOr(reinterpret_cast<unsigned int*>(ws), bit);
}

// ---------------------------------------------------------------- warp helpers
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_sum_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// ---------------------------------------------------------------- grid barrier
// Sense-reversing barrier for persistent kernels launched cooperatively (all CTAs
// co-resident).  bar[0] = arrivals, bar[1] = generation; both zero before launch.
// Release/acquire at GPU scope; data exchanged across CTAs must be read through L2
// (ld.global.cg / atomics), since no L1 invalidation is performed.
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned& gen) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned nb = gridDim.x * gridDim.y * gridDim.z;
    if (atomicAdd(bar, 1u) == nb - 1) {
      atomicExch(bar, 0u);
      __threadfence();
      atomicExch(bar + 1, gen + 1);
    } else {
      while (ld_acquire_gpu(bar + 1) == gen) __nanosleep(32);
    }
  }
  ++gen;
  __syncthreads();
}

// (d, idx) lexicographic "less"
__device__ __forceinline__ bool lex_less(float da, int64_t ia, float db, int64_t ib) {
  return da < db || (da == db && ia < ib);
}

}  // namespace cabsk

// ---------------------------------------------------------------- error plumbing
void cabs_set_cuda_error(cudaError_t e, const char* where);
void cabs_set_error_msg(const char* msg);

#define CABS_LAUNCH_CHECK(where)                       \
  do {                                                 \
    cudaError_t e_ = cudaGetLastError();               \
    if (e_ != cudaSuccess) {                           \
      cabs_set_cuda_error(e_, where);                  \
      return CABS_ERR_CUDA;                            \
    }                                                  \
  } while (0)

#define CABS_CUDA_TRY(x)                               \
  do {                                                 \
    cudaError_t e_ = (x);                              \
    if (e_ != cudaSuccess) {                           \
      cabs_set_cuda_error(e_, #x);                     \
      return CABS_ERR_CUDA;                            \
    }                                                  \
  } while (0)

#define CABS_TRY(x)                                    \
  do {                                                 \
    int32_t s_ = (x);                                  \
    if (s_ != CABS_OK) return s_;                      \
  } while (0)
