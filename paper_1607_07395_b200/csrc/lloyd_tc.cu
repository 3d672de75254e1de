// lloyd_tc.cu -- the whole Lloyd loop of one or two k-means problems (rows and columns of
// CABS, Alg. 2 steps 6-7; Eq. 6) in ONE persistent kernel whose distance
// cross-term runs on the 5th-generation tensor cores.
//
// Per iteration and CTA (one CTA per SM, each running one problem over a contiguous slice of
// its points):
//  phase A (assign), warp-specialised over 128-point tiles:
//    warp 0     TMA producer: the tile's rows of X in 32-column boxes (4-deep ring)
//    warps 2-5  loaders (thread = point): each box -> TMEM as the FP16 hi/lo split of x * gs
//               (the MMA's A operand) and as exact FP32 (for the refine); ||x||^2
//    warp 1     MMA issuer (whole warp, elected lane): acc = (x gs) . (c gs) by
//               tcgen05.mma kind::f16, three products per 16-wide k step (Xh Ch + Xh Cl + Xl Ch)
//               -> TMEM accumulator (2 stages), N = k2 rounded up to 16
//    warps 6-9  epilogue (thread = point): expanded distances dd_j = ||c_j||^2 - 2 x.c_j, a
//               rigorous error bound e_j, the candidate set {j : dd_j - e_j <= (min_j dd_j +
//               e_j)(1 + 2.5e-5)} and, for every candidate, the DIRECT-DIFFERENCE FP32 distance
//               (dimensions ascending, one fmaf chain: the arithmetic of the FFMA kernels) ->
//               label (lowest j on ties), objective, near ties (and the near-tie log).  The
//               labels, the near-tie decisions and the objective terms are therefore those of
//               the FFMA path bit for bit; the tensor cores only prune the centres.
//  phase B (update): the CTA's points re-read from global memory in 128-point chunks, the
//    exact int64 fixed-point sums (km_fixed.cuh) accumulated by cluster-owning warps into a
//    dense per-CTA partial (no atomics), DSMEM reduction over the thread-block cluster and one
//    red.global.add.u64 per entry, a grid barrier per problem, then every CTA forms the next
//    centres from the global sums (an empty cluster keeps its centre).
// The phase-A operands (centre splits, X ring) and the phase-B buffers (partial, staging)
// share shared memory: the centres are rebuilt from the sums through registers.
#include <cooperative_groups.h>
#include <cuda_fp16.h>
#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "common.cuh"
#include "kernels.cuh"
#include "km_fixed.cuh"
#include "km_tile.cuh"
#include "tc_ptx.cuh"

namespace cg = cooperative_groups;

namespace cabsk {

constexpr int kKT = 384;        // 12 warps
constexpr int kKM = 128;        // points per tile (TMEM lanes)
constexpr int kXS = 3;          // X box ring depth
constexpr uint32_t kXBox = kKM * 128;  // 16 KB: 128 rows x 32 floats

#ifdef CABS_PROFILE_KTC
// global-timer stamps (ns) of the phase boundaries of CTA 0, per iteration (<= 64)
__device__ long long g_ktc_tl[64][8];
#define KTC_STAMP(i) do { if (blockIdx.x == 0 && tid == 0 && it < 64) { long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_ktc_tl[it][i] = t_; } } while (0)
#else
#define KTC_STAMP(i) do { } while (0)
#endif

#ifdef CABS_PROFILE_KTC
// per-tile stamps of iteration 2 in CTA 0: [tile][0 loader start, 1 x_ready, 2 MMA issued, 3 acc_full
// seen by the epilogue, 4 candidates ready (bar 1), 5 tile done (bar 2)]
__device__ long long g_ktc_tile[32][8];
#define KTC_TSTAMP(t, i) do { if (blockIdx.x == 0 && it == 2 && (t) < 32) { long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_ktc_tile[t][i] = t_; } } while (0)
// candidates refined per iteration (all CTAs, both problems): [it][0] points, [it][1] candidates
__device__ unsigned long long g_ktc_cand[64][2];
#define KTC_CAND(np_, nc_) do { if (it < 64) { atomicAdd(&g_ktc_cand[it][0], (unsigned long long)(np_)); \
    atomicAdd(&g_ktc_cand[it][1], (unsigned long long)(nc_)); } } while (0)
#else
#define KTC_CAND(np_, nc_) do { } while (0)
#define KTC_TSTAMP(t, i) do { } while (0)
#endif

void ktc_debug_timeline(long long* out, int n) {
#ifdef CABS_PROFILE_KTC
  const int m = n < 64 * 8 ? n : 64 * 8;
  cudaMemcpyFromSymbol(out, g_ktc_tl, sizeof(long long) * m);
  if (n >= 64 * 8 + 32 * 8) cudaMemcpyFromSymbol(out + 64 * 8, g_ktc_tile, sizeof(long long) * 32 * 8);
  if (n >= 64 * 8 + 32 * 8 + 64 * 2) cudaMemcpyFromSymbol(out + 64 * 8 + 32 * 8, g_ktc_cand, sizeof(long long) * 64 * 2);
#else
  for (int i = 0; i < n; ++i) out[i] = 0;
#endif
}

struct KtcProb {
  const float* X;
  int64_t ldx, N;
  int d, k2;
  const float* w;
  const unsigned* bounds;
  float* centres;
  int64_t ldc;
  int* labels;
  double* objective;
  int* near_ties;
  double* cluster_w;
  long long* fsum;  // [3][Eqp]
  double* pobj;     // [iters][Gq]
  int* ptie;        // [iters][Gq]
  int* tie_log;     // [1 + 5 cap] or null
  int tie_cap;
  int64_t row_off;  // global index of local point 0
};

struct KtcArgs {
  KtcProb pr[2];
  int nprob, iters, g0;
  unsigned* gbar[2];
  // shared-memory plan (identical for both problems: sized for the larger)
  int nc;          // MMA N: round_up(max k2, 16)
  int kp16;        // K padded to 64 (FP16 atoms)
  int capn;        // max points per CTA (labels kept for phase B)
  int xp;          // pitch (floats) of the FP32 tile and the FP32 centres: odd, >= max d (bank-conflict free)
  int sp;          // pitch of the phase-B staging rows: multiple of 4 (16-byte cp.async)
  uint32_t off_cbh, off_cbl, off_xr, off_xs, off_part, off_stg, off_c32, off_lab, off_c2, off_wd, off_x2, total;
};

__host__ __device__ inline uint32_t ktc_align(uint32_t x, uint32_t a) { return (x + a - 1) / a * a; }

// shared-memory plan: a region shared by phase A {centre hi, centre lo, X ring, FP32 tile} and
// phase B {partial, staging}; then the FP32 centres, the labels of the CTA's points, ||c||^2,
// 1/weight, ||x||^2 of the tile
inline void ktc_plan(KtcArgs& a, int dmax, int k2max, int64_t capn) {
  a.nc = static_cast<int>(round_up(k2max, 16));
  a.kp16 = static_cast<int>(round_up(dmax, 64));
  a.capn = static_cast<int>(capn);
  a.xp = dmax | 1;
  a.sp = static_cast<int>(round_up(dmax, 4));
  const uint32_t atoms = static_cast<uint32_t>(a.kp16 / 64);
  a.off_cbh = 0;
  a.off_cbl = atoms * a.nc * 128;
  a.off_xr = ktc_align(a.off_cbl + atoms * a.nc * 128, 1024);
  a.off_xs = a.off_xr + kXS * kXBox;
  const uint32_t endA = a.off_xs + sizeof(float) * kKM * a.xp;
  a.off_part = 0;
  const size_t E = ((size_t)k2max * dmax + k2max + 1) & ~size_t(1);
  a.off_stg = ktc_align(static_cast<uint32_t>(E * 8), 16);
  const uint32_t endB = a.off_stg + static_cast<uint32_t>(sizeof(float) * kKM * a.sp);
  uint32_t o = ktc_align(endA > endB ? endA : endB, 16);
  a.off_c32 = o;
  o = ktc_align(o + sizeof(float) * k2max * a.xp, 16);
  a.off_lab = o;
  o = ktc_align(o + sizeof(int) * static_cast<uint32_t>(capn), 16);
  a.off_c2 = o;
  o = ktc_align(o + sizeof(float) * a.nc, 16);
  a.off_wd = o;
  o = ktc_align(o + sizeof(double) * k2max, 16);
  a.off_x2 = o;
  o = ktc_align(o + sizeof(float) * 2 * kKM, 16);
  a.total = o;
}

__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
      "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15])
      : "memory");
}
__device__ __forceinline__ void tmem_st32f(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]),
      "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]),
      "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]),
      "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}
__device__ __forceinline__ void mma_f16_ts_k(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc));
}
__host__ __device__ constexpr uint32_t idesc_f16_k(int M, int N) {
  return (1u << 4) | (static_cast<uint32_t>(N >> 3) << 17) | (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t pack_h2_k(float a, float b, float& ra, float& rb) {
  // returns the packed FP16 pair (a, b) (element 0 in the low half); ra, rb = the exact remainders
  const __half ha = __float2half_rn(a), hb = __float2half_rn(b);
  ra = a - __half2float(ha);
  rb = b - __half2float(hb);
  return static_cast<uint32_t>(__half_as_ushort(ha)) | (static_cast<uint32_t>(__half_as_ushort(hb)) << 16);
}
__device__ __forceinline__ uint32_t pack_h2_only(float a, float b) {
  return static_cast<uint32_t>(__half_as_ushort(__float2half_rn(a))) |
         (static_cast<uint32_t>(__half_as_ushort(__float2half_rn(b))) << 16);
}
__device__ __forceinline__ float x_gscale(const unsigned* bounds) {
  const float xm = __uint_as_float(__ldcg(bounds));
  return xm > 0.f ? exp2f(static_cast<float>(13 - ilogbf(xm))) : 1.f;
}

// the FP16 hi / lo split of a centre row into the 128B-swizzled K-major B operand (atoms of 64
// elements; row j of atom a at a * nc * 128 + j * 128, 16-byte chunk c at (c ^ (j & 7)) * 16)
__device__ __forceinline__ void put_centre_h(uint8_t* cbh, uint8_t* cbl, int nc, int j, int i, float v) {
  const int a = i >> 6, e = i & 63;
  const uint32_t off = static_cast<uint32_t>(a * nc * 128 + j * 128 + ((((e >> 3) ^ (j & 7)) << 4) | ((e & 7) << 1)));
  const __half h = __float2half_rn(v);
  *reinterpret_cast<__half*>(cbh + off) = h;
  *reinterpret_cast<__half*>(cbl + off) = __float2half_rn(v - __half2float(h));
}

__global__ void __launch_bounds__(kKT, 1)
lloyd_tc_kernel(const __grid_constant__ CUtensorMap tmX0, const __grid_constant__ CUtensorMap tmX1, KtcArgs a) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-byte alignment by an offset into the __shared__ array (not by integer casts, which
  // would turn every access into a generic one)
  uint8_t* sm = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* cbh = sm + a.off_cbh;
  uint8_t* cbl = sm + a.off_cbl;
  uint8_t* xr = sm + a.off_xr;
  float* xs = reinterpret_cast<float*>(sm + a.off_xs);
  long long* part = reinterpret_cast<long long*>(sm + a.off_part);
  float* stg = reinterpret_cast<float*>(sm + a.off_stg);
  float* c32 = reinterpret_cast<float*>(sm + a.off_c32);
  int* lab_all = reinterpret_cast<int*>(sm + a.off_lab);
  float* c2 = reinterpret_cast<float*>(sm + a.off_c2);
  double* wd = reinterpret_cast<double*>(sm + a.off_wd);
  float* x2s = reinterpret_cast<float*>(sm + a.off_x2);
  __shared__ uint64_t xr_full[kXS], xr_empty[kXS], x_ready, acc_full, cand_ready, tile_done, s_mbar;
  __shared__ uint32_t cms[kKM * 4];  // candidate masks of the tile
  __shared__ uint32_t tmem_base;
  __shared__ double s_red[kKT / 32];
  __shared__ int s_tie[kKT / 32];
  __shared__ double s_wsc[kKM];
  __shared__ long long s_iw[kKM];

  cg::cluster_group cluster = cg::this_cluster();
  const int crank = static_cast<int>(cluster.block_rank()), csize = static_cast<int>(cluster.num_blocks());
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int G = gridDim.x;
  const int myq = (a.nprob > 1 && static_cast<int>(blockIdx.x) >= a.g0) ? 1 : 0;
  const int b = myq ? static_cast<int>(blockIdx.x) - a.g0 : static_cast<int>(blockIdx.x);
  const int Gb = a.nprob > 1 ? (myq ? G - a.g0 : a.g0) : G;
  const KtcProb& pr = a.pr[myq];
  const CUtensorMap* tmX = myq ? &tmX1 : &tmX0;
  const int d = pr.d, k2 = pr.k2, nc = a.nc;
  const int64_t pbeg = (pr.N * b) / Gb, pend = (pr.N * (b + 1)) / Gb, npts = pend - pbeg;
  const int ntiles = static_cast<int>(ceil_div(npts, kKM));
  const int nld = (d + 31) / 32;            // X boxes with data per tile
  const int nks = (d + 15) / 16;            // 16-wide k steps
  const int kp16 = a.kp16, nbx = kp16 / 32;  // 32-wide chunks of the FP16 operand (zeros past nld)
  const int64_t Eq = (int64_t)k2 * d + k2, Eqp = (Eq + 1) & ~int64_t(1);
  const int64_t ebeg = Eq * crank / csize, eend = Eq * (crank + 1) / csize;
  double scale, scale_w;
  fx_scales(pr.bounds, pr.N, scale, scale_w);
  const float gs = x_gscale(pr.bounds);
  const float ig2 = 1.f / (gs * gs);  // exact (power of two)
  // TMEM: accumulator [0, 128); X FP16 at 256: hi [0, kp16/2), lo [kp16/2, kp16)
  const uint32_t kXH = 256, kXL = 256 + static_cast<uint32_t>(kp16 / 2);
  const int xp = a.xp, sp = a.sp;

  if (tid == 0) {
    for (int s = 0; s < kXS; ++s) { tc::mbar_init(&xr_full[s], 1); tc::mbar_init(&xr_empty[s], 4); }
    tc::mbar_init(&x_ready, 4);
    tc::mbar_init(&acc_full, 1);
    tc::mbar_init(&cand_ready, 4);
    tc::mbar_init(&tile_done, 8);
    tc::mbar_init(&s_mbar, 1);
    tc::mbar_fence_init();
    tc::tma_prefetch(tmX);
  }
  if (warp == 1) tc::tmem_alloc(&tmem_base, 512);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = tmem_base;

  // centres of iteration 0 (the initialisation, global) -> FP32 copy
  for (int e = tid; e < k2 * d; e += kKT) {
    const int j = e / d, i = e - j * d;
    c32[j * xp + i] = __ldcg(pr.centres + (int64_t)j * pr.ldc + i);
  }
  __syncthreads();

  int64_t gtile = 0;   // tiles processed by this CTA so far (all iterations): the ring phases
  int64_t gchunk = 0;  // X boxes
  for (int it = 0; it < a.iters; ++it) {
    KTC_STAMP(0);
    // ------------------------------------------------------------ centres of this iteration
    if (it > 0) {
      // the previous iteration's exact sums reach every CTA of the cluster by multicast bulk
      // copies (one L2 read per cluster) into the partial buffer
      if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");
        tc::mbar_expect_tx(&s_mbar, static_cast<uint32_t>(Eqp * 8));
        const int64_t n16 = Eqp / 2;
        const int64_t q0 = n16 * crank / csize, q1 = n16 * (crank + 1) / csize;
        if (q1 > q0) {
          const long long* src = pr.fsum + (size_t)((it + 2) % 3) * Eqp + 2 * q0;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster "
              "[%0], [%1], %2, [%3], %4;" ::"r"(tc::smem_u32(part + 2 * q0)),
              "l"(src), "r"(static_cast<uint32_t>((q1 - q0) * 16)), "r"(tc::smem_u32(&s_mbar)),
              "h"(static_cast<uint16_t>((1u << csize) - 1u))
              : "memory");
        }
      }
      tc::mbar_wait(&s_mbar, static_cast<uint32_t>((it - 1) & 1));
      const int nsum = k2 * d;
      for (int j = tid; j < k2; j += kKT) {
        const long long wj = part[nsum + j];
        wd[j] = wj > 0 ? 1.0 / (static_cast<double>(wj) * (1.0 / scale_w)) : 0.0;
      }
      __syncthreads();
      // new centres into registers (the partial shares memory with the centre operand), then
      // into the FP32 copy; an empty cluster keeps its centre
      constexpr int kPer = 48;  // entries per thread: k2 d <= 128 * 128 / 384 < 43
      float nv[kPer];
      const double inv_scale = 1.0 / scale;
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = tid + u * kKT;
        nv[u] = 0.f;
        if (e < nsum) {
          const int j = e / d;
          const double rw = wd[j];
          nv[u] = rw > 0 ? static_cast<float>((static_cast<double>(part[e]) * inv_scale) * rw) : c32[j * xp + e - j * d];
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = tid + u * kKT;
        if (e < nsum) c32[(e / d) * xp + e % d] = nv[u];
      }
      // zero this CTA's share of the slot the next iteration accumulates into
      long long* fs_next = pr.fsum + (size_t)((it + 1) % 3) * Eqp;
      for (int64_t e = (int64_t)b * kKT + tid; e < Eq; e += (int64_t)Gb * kKT) fs_next[e] = 0;
      __syncthreads();
    }
    // FP16 hi/lo operand (zero rows past k2 and columns past d), ||c_j||^2 in FP32 (dims ascending)
    {
      const int lk = kp16 == 64 ? 6 : 7;  // kp16 in {64, 128}
      for (int e = tid; e < nc << lk; e += kKT) {
        const int i = e & (kp16 - 1), j = e >> lk;
        const float v = (j < k2 && i < d) ? c32[j * xp + i] * gs : 0.f;
        put_centre_h(cbh, cbl, nc, j, i, v);
      }
      for (int j = warp; j < nc; j += kKT / 32) {  // ||c_j||^2: lanes over dimensions, fixed-order tree
        float s2 = 0.f;
        if (j < k2)
          for (int i = lane; i < d; i += 32) s2 = fmaf(c32[j * xp + i], c32[j * xp + i], s2);
        s2 = warp_sum_f(s2);
        if (lane == 0) c2[j] = s2;
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic writes -> tensor-core reads
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    KTC_STAMP(1);

    // ------------------------------------------------------------ phase A: assignment
    double obj = 0.0;
    int ties = 0;
    if (warp == 0) {
      if (lane == 0) {  // TMA producer
        for (int t = 0; t < ntiles; ++t) {
          const int y = static_cast<int>(pbeg + (int64_t)t * kKM);
          for (int c = 0; c < nld; ++c) {
            const int64_t g = gchunk + (int64_t)t * nld + c;
            const int s = static_cast<int>(g % kXS);
            if (g >= kXS) tc::mbar_wait(&xr_empty[s], static_cast<uint32_t>(((g - kXS) / kXS) & 1));
            tc::mbar_expect_tx(&xr_full[s], kXBox);
            tc::tma_load_2d(xr + s * kXBox, tmX, 32 * c, y, &xr_full[s]);
          }
        }
      }
    } else if (warp == 1) {  // MMA issuer (whole warp; one elected lane issues)
      const uint32_t idesc = idesc_f16_k(kKM, nc);
      const uint64_t dbh = tc::desc_sw128(tc::smem_u32(cbh)), dbl = tc::desc_sw128(tc::smem_u32(cbl));
      const uint64_t atom16 = static_cast<uint64_t>(nc) * 128 >> 4;
      for (int t = 0; t < ntiles; ++t) {
        const int64_t g = gtile + t;
        tc::mbar_wait(&x_ready, static_cast<uint32_t>(g & 1));
        tc::fence_after_sync();
        if (tc::elect_one()) {
          for (int q = 0; q < nks; ++q) {
            const uint64_t boff = static_cast<uint64_t>(q >> 2) * atom16 + static_cast<uint64_t>((q & 3) * 2);
            const uint32_t ah = tmem + kXH + static_cast<uint32_t>(8 * q), al = tmem + kXL + static_cast<uint32_t>(8 * q);
            mma_f16_ts_k(tmem, ah, dbh + boff, idesc, q > 0 ? 1u : 0u);
            mma_f16_ts_k(tmem, ah, dbl + boff, idesc, 1u);
            mma_f16_ts_k(tmem, al, dbh + boff, idesc, 1u);
          }
          tc::mma_commit(&acc_full);
          KTC_TSTAMP(t, 2);
        }
        __syncwarp();
      }
    } else if (warp >= 2 && warp <= 9) {
      // per tile: warps 2-5 load it (TMEM FP16 split + FP32 rows in shared memory), the MMA runs,
      // warps 6-9 turn the accumulator into candidate masks, then warps 2-9 refine two threads per
      // point; named barriers 1 (candidates ready) and 2 (tile done) order the steps
      const bool loader = warp <= 5;
      const int qd = warp & 3;
      const uint32_t lrow = tmem + (static_cast<uint32_t>(qd * 32) << 16);
      const float tabs = 0.125f * ig2;  // absolute bound on the FP16 underflow terms
      const int tt = tid - 64;          // 0..255 within warps 2-9
      const int rp = tt >> 1, hp = tt & 1;  // refine: point rp, half hp of its candidates
      for (int t = 0; t < ntiles; ++t) {
        const int64_t g = gtile + t;
        if (loader) {
          const int r = qd * 32 + lane;
          if (tid == 64) KTC_TSTAMP(t, 0);
          float x2 = 0.f;
          for (int c = 0; c < nbx; ++c) {
            float v[32];
            if (c < nld) {
              const int64_t gc = gchunk + (int64_t)t * nld + c;
              const int sl = static_cast<int>(gc % kXS);
              tc::mbar_wait(&xr_full[sl], static_cast<uint32_t>((gc / kXS) & 1));
              const uint8_t* row = xr + sl * kXBox + r * 128;
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const float4 f = *reinterpret_cast<const float4*>(row + ((k ^ (r & 7)) << 4));
                v[4 * k] = f.x; v[4 * k + 1] = f.y; v[4 * k + 2] = f.z; v[4 * k + 3] = f.w;
              }
              __syncwarp();
              if (lane == 0) tc::mbar_arrive(&xr_empty[sl]);
              float* xrow = xs + r * xp + 32 * c;
#pragma unroll
              for (int k = 0; k < 32; ++k) {  // columns >= d of the box are the zero padding of X
                if (32 * c + k >= d) v[k] = 0.f;
                else xrow[k] = v[k];
                x2 = fmaf(v[k], v[k], x2);
              }
            } else {
#pragma unroll
              for (int k = 0; k < 32; ++k) v[k] = 0.f;
            }
            uint32_t hi[16], lo[16];
#pragma unroll
            for (int k = 0; k < 16; ++k) {
              float ra, rb;
              hi[k] = pack_h2_k(v[2 * k] * gs, v[2 * k + 1] * gs, ra, rb);
              lo[k] = pack_h2_only(ra, rb);
            }
            tmem_st16(lrow + kXH + static_cast<uint32_t>(16 * c), hi);
            tmem_st16(lrow + kXL + static_cast<uint32_t>(16 * c), lo);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
          x2s[r] = x2;
          tc::fence_before_sync();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&x_ready);
          if (tid == 64) KTC_TSTAMP(t, 1);
        } else {
          const int r = qd * 32 + lane;
          tc::mbar_wait(&acc_full, static_cast<uint32_t>(g & 1));
          if (tid == 192) KTC_TSTAMP(t, 3);
          tc::fence_after_sync();
          const float x2 = x2s[r];
          // one pass over the accumulator: a running smallest upper bound U* of the distance and
          // every centre whose lower bound is within (1 + 2.5e-5) U* at its turn -- a superset of
          // the candidates against the final U* (U* only decreases), which the refine then sorts out
          float umin = FLT_MAX;
          for (int cc = 0; cc < nc; cc += 32) {
            float v[32];
            tc::tmem_ld32(lrow + static_cast<uint32_t>(cc), v);
            float lo[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
              const int j = cc + k;
              const float cj = c2[j < k2 ? j : 0];
              const float e = 6.103515625e-05f * (x2 + cj) + tabs;  // 2^-14 (||x||^2 + ||c_j||^2) + underflow
              const float dd = fmaf(-2.f * ig2, v[k], cj) + x2;
              lo[k] = j < k2 ? dd - e : FLT_MAX;
              if (j < k2) umin = fminf(umin, dd + e);
            }
            const float thr = umin * (1.f + 2.5e-5f);
            uint32_t bits = 0u;
#pragma unroll
            for (int k = 0; k < 32; ++k) bits |= (lo[k] <= thr ? 1u : 0u) << k;
            cms[r * 4 + (cc >> 5)] = bits;
          }
          // drop the early marks the final bound excludes: a second look at the masked words only
          {
            const float thr = umin * (1.f + 2.5e-5f);
            for (int cc = 0; cc < nc; cc += 32) {
              float v[32];
              tc::tmem_ld32(lrow + static_cast<uint32_t>(cc), v);
              uint32_t bits = cms[r * 4 + (cc >> 5)], keep = 0u;
#pragma unroll
              for (int k = 0; k < 32; ++k) {
                if (bits & (1u << k)) {
                  const float cj = c2[cc + k];
                  const float e = 6.103515625e-05f * (x2 + cj) + tabs;
                  if (fmaf(-2.f * ig2, v[k], cj) + x2 - e <= thr) keep |= 1u << k;
                }
              }
              cms[r * 4 + (cc >> 5)] = keep;
            }
          }
          for (int w = (nc + 31) >> 5; w < 4; ++w) cms[r * 4 + w] = 0u;
#ifdef CABS_PROFILE_KTC
          {
            const bool in = (int64_t)t * kKM + r < npts;
            int cnt = in ? __popc(cms[r * 4]) + __popc(cms[r * 4 + 1]) + __popc(cms[r * 4 + 2]) + __popc(cms[r * 4 + 3]) : 0;
            int np_ = in;
            for (int o = 16; o > 0; o >>= 1) { cnt += __shfl_xor_sync(0xffffffffu, cnt, o); np_ += __shfl_xor_sync(0xffffffffu, np_, o); }
            if (lane == 0) KTC_CAND(np_, cnt);
          }
#endif
          tc::fence_before_sync();
        }
        // candidates of the tile ready (mbarrier: the 4 epilogue warps arrive, warps 2-9 wait)
        if (!loader) {
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&cand_ready);
        }
        tc::mbar_wait(&cand_ready, static_cast<uint32_t>(g & 1));
        if (tid == 64) KTC_TSTAMP(t, 4);
        // refine: the candidates' direct-difference FP32 distances (dimensions ascending, one fmaf
        // chain per centre: the FFMA kernels' arithmetic), four centres at a time (ILP); x and the
        // centres from shared memory (odd pitches: conflict-free).  Thread pair (2 rp, 2 rp + 1)
        // splits point rp's candidates alternately.
        float bd = FLT_MAX, sd = FLT_MAX;
        int bj = 0x7fffffff, sj = -1;
        {
          const float* xrow = xs + rp * xp;
          uint32_t rem[4] = {cms[rp * 4], cms[rp * 4 + 1], cms[rp * 4 + 2], cms[rp * 4 + 3]};
          int parity = 0;
          auto next = [&]() {
            for (;;) {
              int j = -1;
#pragma unroll
              for (int w = 0; w < 4; ++w)
                if (j < 0 && rem[w]) { j = 32 * w + __ffs(rem[w]) - 1; rem[w] &= rem[w] - 1; }
              if (j < 0) return -1;
              const bool mine = parity == hp;
              parity ^= 1;
              if (mine) return j;
            }
          };
          auto take = [&](float val, int j) {
            if (val < bd || (val == bd && j < bj)) { sd = bd; sj = bj; bd = val; bj = j; }
            else if (val < sd) { sd = val; sj = j; }
          };
          for (;;) {
            const int j0 = next();
            if (j0 < 0) break;
            const int j1 = next(), j2 = next(), j3 = next();
            const float* c0 = c32 + j0 * xp;
            const float* c1 = c32 + (j1 < 0 ? j0 : j1) * xp;
            const float* c2p = c32 + (j2 < 0 ? j0 : j2) * xp;
            const float* c3p = c32 + (j3 < 0 ? j0 : j3) * xp;
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 4
            for (int i = 0; i < d; ++i) {
              const float xv = xrow[i];
              const float f0 = xv - c0[i], f1 = xv - c1[i], f2 = xv - c2p[i], f3 = xv - c3p[i];
              a0 = fmaf(f0, f0, a0);
              a1 = fmaf(f1, f1, a1);
              a2 = fmaf(f2, f2, a2);
              a3 = fmaf(f3, f3, a3);
            }
            take(a0, j0);
            if (j1 >= 0) take(a1, j1);
            if (j2 >= 0) take(a2, j2);
            if (j3 >= 0) take(a3, j3);
          }
          // merge the pair (lanes 2q, 2q + 1): lowest j on ties
          const float obd = __shfl_xor_sync(0xffffffffu, bd, 1), osd = __shfl_xor_sync(0xffffffffu, sd, 1);
          const int obj = __shfl_xor_sync(0xffffffffu, bj, 1), osj = __shfl_xor_sync(0xffffffffu, sj, 1);
          take(obd, obj);
          if (osj >= 0) take(osd, osj);
        }
        const int64_t pl = (int64_t)t * kKM + rp;
        if (hp == 0 && pl < npts) {
          const int64_t p = pbeg + pl;
          lab_all[pl] = bj;
          pr.labels[p] = bj;
          obj += static_cast<double>(__ldg(pr.w + p)) * static_cast<double>(bd);
          const bool tie = (sd - bd) < kNearTie * sd;
          ties += tie;
          if (tie && pr.tie_log) km_log_tie(pr.tie_log, pr.tie_cap, it, pr.row_off + p, bj, sj, bd, sd);
        }
        // tile done: xs and the masks may be rewritten (every warp of 2-9 arrives and waits)
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&tile_done);
        tc::mbar_wait(&tile_done, static_cast<uint32_t>(g & 1));
        if (tid == 64) KTC_TSTAMP(t, 5);
      }
    }
    gtile += ntiles;
    gchunk += (int64_t)ntiles * nld;
    // ------------------------------------------------------------ phase B: exact sums
    tc::fence_before_sync();
    __syncthreads();  // phase A done (the partial overlays the centre operand and the X ring)
    tc::fence_after_sync();
    KTC_STAMP(2);
    for (int64_t e = tid; e < Eqp; e += kKT) part[e] = 0;
    __syncthreads();
    for (int64_t c0 = 0; c0 < npts; c0 += kKM) {
      const int np = static_cast<int>(npts - c0 < kKM ? npts - c0 : kKM);
      // stage the chunk's rows (16-byte cp.async: every copy in flight at once), w 2^S, llrint(w 2^Sw)
      {
        const int d4 = (d + 3) >> 2;
        for (int e = tid; e < np * d4; e += kKT) {
          const int pp = e / d4, i4 = e - pp * d4;
          const float* src = pr.X + (pbeg + c0 + pp) * pr.ldx + 4 * i4;  // ldx >= round_up(d, 4): in bounds
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::smem_u32(stg + pp * sp + 4 * i4)),
                       "l"(src)
                       : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      }
      for (int pp = tid; pp < kKM; pp += kKT) {
        const float w = pp < np ? __ldg(pr.w + pbeg + c0 + pp) : 0.f;
        s_wsc[pp] = static_cast<double>(w) * scale;
        s_iw[pp] = llrint(static_cast<double>(w) * scale_w);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      // balanced over the points (cluster sizes are skewed): warp w takes points [w np / 12, (w + 1) np
      // / 12), lanes over dimensions; every int64 product is added EXACTLY into the partial by two
      // native 32-bit shared-memory atomics (low word, then high word + the low word's carry): the
      // sum is an integer, so it does not depend on the order of the additions
      {
        const int nsum = k2 * d;
        unsigned* pw = reinterpret_cast<unsigned*>(part);
        const int pa = (np * warp) / (kKT / 32), pb = (np * (warp + 1)) / (kKT / 32);
        auto add64 = [&](int e, long long v) {
          const unsigned lo = static_cast<unsigned>(v);
          const unsigned old = atomicAdd(pw + 2 * e, lo);
          atomicAdd(reinterpret_cast<int*>(pw + 2 * e + 1), static_cast<int>(v >> 32) + ((old + lo) < old ? 1 : 0));
        };
        for (int pp = pa; pp < pb; pp += 4) {
          int jj[4];
          double ws[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int q = pp + u < pb ? pp + u : pa;
            jj[u] = pp + u < pb ? lab_all[c0 + q] : -1;
            ws[u] = s_wsc[q];
          }
          for (int i = lane; i < d; i += 32) {
            long long v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) v[u] = fx_prod_magic(ws[u], stg[(pp + u < pb ? pp + u : pa) * sp + i]);
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (jj[u] >= 0) add64(jj[u] * d + i, v[u]);
          }
          if (lane < 4) {
            long long iw = 0;
            int jw = -1;
#pragma unroll
            for (int u = 0; u < 4; ++u)
              if (u == lane && jj[u] >= 0) { iw = s_iw[pp + u]; jw = jj[u]; }
            if (jw >= 0) add64(nsum + jw, iw);
          }
        }
      }
      __syncthreads();
    }
    // objective / near ties of this CTA
    obj = warp_sum_d(obj);
    {
      int tt = ties;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tt += __shfl_xor_sync(0xffffffffu, tt, o);
      if (lane == 0) { s_red[warp] = obj; s_tie[warp] = tt; }
    }
    // cluster reduction of the dense partials (DSMEM), one global integer add per entry
    KTC_STAMP(3);
    cluster.sync();
    {
      long long* fs_cur = pr.fsum + (size_t)(it % 3) * Eqp;
      const long long* rp[8];
#pragma unroll
      for (int rr = 0; rr < 8; ++rr) rp[rr] = rr < csize ? cluster.map_shared_rank(part, rr) : part;
      for (int64_t e = ebeg + tid; e < eend; e += kKT) {
        long long s = 0;
#pragma unroll
        for (int rr = 0; rr < 8; ++rr) s += rr < csize ? rp[rr][e] : 0;
        if (s != 0) red_add_u64(fs_cur + e, s);
      }
    }
    if (tid == 0) {
      double sacc = 0;
      int qq = 0;
      for (int w = 0; w < kKT / 32; ++w) { sacc += s_red[w]; qq += s_tie[w]; }
      pr.pobj[(size_t)it * Gb + b] = sacc;
      pr.ptie[(size_t)it * Gb + b] = qq;
    }
    cluster.sync();  // the cluster's partials are read: the buffer may be overwritten
    KTC_STAMP(4);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      unsigned* bar = a.gbar[myq];
      atomicAdd(bar, 1u);
      const unsigned target = static_cast<unsigned>(Gb) * static_cast<unsigned>(it + 1);
      while (ld_acquire_gpu(bar) < target) __nanosleep(20);
    }
    __syncthreads();
    KTC_STAMP(5);
  }
  // ---------------- epilogue (CTA 0 of each problem): final centres, cluster weights, objective
  if (b == 0) {
    const int nsum = k2 * d;
    const double inv_scale = 1.0 / scale, inv_scale_w = 1.0 / scale_w;
    const long long* fs_last = pr.fsum + (size_t)((a.iters - 1) % 3) * Eqp;
    for (int e = tid; e < nsum; e += kKT) {
      const int j = e / d, i = e - j * d;
      const long long wj = __ldcg(fs_last + nsum + j);
      pr.centres[(int64_t)j * pr.ldc + i] =
          wj > 0 ? static_cast<float>((static_cast<double>(__ldcg(fs_last + e)) * inv_scale) *
                                      (1.0 / (static_cast<double>(wj) * inv_scale_w)))
                 : c32[j * xp + i];
    }
    for (int j = tid; j < k2; j += kKT) pr.cluster_w[j] = static_cast<double>(__ldcg(fs_last + nsum + j)) / scale_w;
    for (int t = tid; t < a.iters; t += kKT) {
      double s = 0;
      long long qq = 0;
      for (int g = 0; g < Gb; ++g) {
        s += __ldcg(pr.pobj + (size_t)t * Gb + g);
        qq += __ldcg(pr.ptie + (size_t)t * Gb + g);
      }
      pr.objective[t] = s;
      if (pr.near_ties) pr.near_ties[t] = static_cast<int>(qq);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 512);
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFnK)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFnK encoder_k() {
  static EncodeTiledFnK fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFnK>(p);
  }
  return fn;
}

static bool x_map(CUtensorMap* tm, const float* X, int64_t ldx, int64_t N) {
  EncodeTiledFnK enc = encoder_k();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(ldx), static_cast<cuuint64_t>(N)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * sizeof(float)};
  cuuint32_t box[2] = {32, kKM};
  cuuint32_t estr[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

constexpr size_t kKtcSmemCap = 220 * 1024;  // dynamic (the kernel also has ~3 KB of static shared memory)

// The tensor cores prune the centres, the candidates are then refined by FFMA: worth it once the
// FFMA kernel's per-point work k2 d is large (c3: k2 = d = 100 -> 5.3 vs 14.1 ms; c2: k2 = d = 50
// -> 0.91 vs 0.50 ms, measured with tools/prof_ktc.py).  CABS_KMEANS_TC=1 forces it wherever it
// applies, CABS_KMEANS_FFMA=1 disables it.
bool kmeans_tc_selected(int k2, int d) {
  if (getenv("CABS_KMEANS_FFMA")) return false;
  if (k2 < 1 || k2 > 128 || d < 1 || d > 128) return false;
  if (!getenv("CABS_KMEANS_TC") && k2 * d < 4096) return false;
  KtcArgs a{};
  ktc_plan(a, d, k2, 2048);
  return a.total + 1024 <= kKtcSmemCap && encoder_k() != nullptr;
}

bool launch_lloyd_tc(const LloydJob* jobs, int njobs, int iters, cudaStream_t st) {
  if (njobs < 1 || njobs > 2) return false;
  int dmax = 0, k2max = 0;
  for (int q = 0; q < njobs; ++q) {
    if (!kmeans_tc_selected(jobs[q].k2, jobs[q].d) || jobs[q].N <= 0) return false;
    if ((jobs[q].ldx % 4) != 0 || (reinterpret_cast<uintptr_t>(jobs[q].X) & 15) != 0) return false;
    dmax = jobs[q].d > dmax ? jobs[q].d : dmax;
    k2max = jobs[q].k2 > k2max ? jobs[q].k2 : k2max;
  }
  int dev = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kKT);
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  const double Ntot = static_cast<double>(jobs[0].N) + (njobs > 1 ? static_cast<double>(jobs[1].N) : 0.0);
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(lloyd_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(kKtcSmemCap)) != cudaSuccess)
      return false;
    attr = true;
  }
  KtcArgs a{};
  int csize = 0;
  int64_t Gq[2] = {0, 0}, Gt = 0;
  for (int c = 8; c >= 1 && csize == 0; c >>= 1) {
    const int64_t tot = (int64_t)nsm / c * c;
    if (tot < c * njobs) continue;
    int64_t g[2] = {tot, 0};
    if (njobs > 1) {
      g[0] = (int64_t)llround(static_cast<double>(tot) * static_cast<double>(jobs[0].N) / Ntot / c) * c;
      g[0] = g[0] < c ? c : (g[0] > tot - c ? tot - c : g[0]);
      g[1] = tot - g[0];
    }
    bool ok = true;
    int64_t capn = 0;
    for (int q = 0; q < njobs; ++q) {
      if (g[q] > jobs[q].N) ok = false;
      const int64_t per = ceil_div(jobs[q].N, g[q] > 0 ? g[q] : 1);
      capn = per > capn ? per : capn;
    }
    if (!ok) continue;
    KtcArgs t{};
    ktc_plan(t, dmax, k2max, round_up(capn, 4));
    if (t.total + 1024 > kKtcSmemCap) continue;
    at[0].val.clusterDim.x = static_cast<unsigned>(c);
    cfg.gridDim = dim3(static_cast<unsigned>(tot));
    cfg.dynamicSmemBytes = t.total + 1024;
    int ncl = 0;
    if (cudaOccupancyMaxActiveClusters(&ncl, lloyd_tc_kernel, &cfg) == cudaSuccess && (int64_t)ncl * c >= tot) {
      csize = c;
      Gt = tot;
      Gq[0] = g[0];
      Gq[1] = g[1];
      a = t;
    }
  }
  cudaGetLastError();
  if (csize == 0) {
    if (getenv("CABS_KMEANS_REQUIRE_TC")) fprintf(stderr, "lloyd_tc: no launch configuration\n");
    return false;
  }
  a.nprob = njobs;
  a.iters = iters;
  a.g0 = static_cast<int>(Gq[0]);
  CUtensorMap tm[2];
  for (int q = 0; q < njobs; ++q) {
    const LloydJob& j = jobs[q];
    if (!x_map(&tm[q], j.X, j.ldx, j.N)) return false;
    const size_t E = ((size_t)j.k2 * j.d + j.k2 + 1) & ~size_t(1);
    const size_t need = sizeof(long long) * 3 * E + 16 + (sizeof(double) + sizeof(int)) * iters * Gt;
    if (need > j.scratch_bytes) return false;
    char* base = static_cast<char*>(j.scratch);
    KtcProb& p = a.pr[q];
    p.X = j.X; p.ldx = j.ldx; p.N = j.N; p.d = j.d; p.k2 = j.k2; p.w = j.w; p.bounds = j.bounds;
    p.centres = j.centres; p.ldc = j.ldc; p.labels = j.labels; p.objective = j.objective;
    p.near_ties = j.near_ties; p.cluster_w = j.cluster_w;
    p.fsum = reinterpret_cast<long long*>(base);
    unsigned* gb = reinterpret_cast<unsigned*>(p.fsum + 3 * E);
    a.gbar[q] = gb;
    p.pobj = reinterpret_cast<double*>(gb + 4);
    p.ptie = reinterpret_cast<int*>(p.pobj + (size_t)iters * Gt);
    p.tie_log = j.tie_log;
    p.tie_cap = j.tie_cap;
    p.row_off = j.row_off;
    if (cudaMemsetAsync(base, 0, sizeof(long long) * 3 * E + 16, st) != cudaSuccess) return false;
  }
  if (njobs == 1) tm[1] = tm[0];
  cfg.gridDim = dim3(static_cast<unsigned>(Gt));
  cfg.dynamicSmemBytes = a.total + 1024;
  at[0].val.clusterDim.x = static_cast<unsigned>(csize);
  note_launch();
  return cudaLaunchKernelEx(&cfg, lloyd_tc_kernel, tm[0], tm[1], a) == cudaSuccess;
}

}  // namespace cabsk
