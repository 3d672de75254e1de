// residual_tc.cu -- S10 on the 5th-generation tensor cores: ||A - F diag(s) G^T||_F^2
// and ||A||_F^2 with the reconstruction produced tile by tile in TMEM by
// tcgen05.mma (kind::tf32, 3xTF32 split for FP32-level accuracy) and consumed by an
// epilogue that streams the matching A tile through shared memory (TMA), so
// A - F G^T is never materialised and A is read from HBM exactly once.
//
// Persistent, warp-specialised, one CTA per SM:
//   warp 0  TMA producer: F_hi/F_lo row band (resident while the band lasts),
//           G_hi/G_lo column tiles and A tiles, double-buffered (mbarrier ring)
//   warp 1  TMEM allocator + single-thread MMA issuer: per 128 x 64 tile and per
//           8-wide k step, D += Fh Gh^T + Fh Gl^T + Fl Gh^T into one of two TMEM
//           accumulators (64 columns each)
//   warps 2-5 epilogue: tcgen05.ld the accumulator row (lane = row), read the A row
//           from the 128B-swizzled smem tile, accumulate (a - a~)^2 and a^2 in FP32
//           per tile, FP64 across tiles; fixed-order block and grid reductions.
// Tile order is row-band major over a static contiguous tile range per CTA, so the
// result is bit-reproducible.  Requires ncomp <= 64 (two 32-float K atoms).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_ptx.cuh"

namespace cabsk {

constexpr int kTcBM = 128, kTcBN = 64, kTcKA = 2;  // K atoms of 32 floats (128 B)
constexpr int kTcThreads = 192;
constexpr uint32_t kFAtomBytes = kTcBM * 128;      // 16 KB
constexpr uint32_t kGAtomBytes = kTcBN * 128;      // 8 KB
constexpr uint32_t kABoxBytes = kTcBM * 128;       // 16 KB: 128 rows x 32 floats

struct TcSmem {
  // 1024-byte aligned operand tiles (128B swizzle atoms)
  uint8_t fh[kTcKA][kFAtomBytes];
  uint8_t fl[kTcKA][kFAtomBytes];
  uint8_t gh[2][kTcKA][kGAtomBytes];
  uint8_t gl[2][kTcKA][kGAtomBytes];
  uint8_t a[2][2][kABoxBytes];  // [stage][column half]
  uint64_t f_full, f_empty;
  uint64_t g_full[2], g_empty[2];
  uint64_t a_full[2], a_empty[2];
  uint64_t acc_full[2], acc_empty[2];
  uint32_t tmem_base;
  double red[2][4];
};

__global__ void __launch_bounds__(kTcThreads, 1)
residual_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmFh,
                   const __grid_constant__ CUtensorMap tmFl, const __grid_constant__ CUtensorMap tmGh,
                   const __grid_constant__ CUtensorMap tmGl, int64_t m, int64_t n, int ksteps,
                   double* __restrict__ part) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  TcSmem& S = *reinterpret_cast<TcSmem*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntr = ceil_div(m, kTcBM), ntc = ceil_div(n, kTcBN);
  const int64_t T = ntr * ntc;
  const int64_t t_beg = (T * blockIdx.x) / gridDim.x, t_end = (T * (blockIdx.x + 1)) / gridDim.x;
  const int katoms = ksteps > 4 ? 2 : 1;  // 8-wide k steps per 32-float atom = 4

  if (warp == 0 && lane == 0) {
    tc::tma_prefetch(&tmA); tc::tma_prefetch(&tmFh); tc::tma_prefetch(&tmFl);
    tc::tma_prefetch(&tmGh); tc::tma_prefetch(&tmGl);
    tc::mbar_init(&S.f_full, 1);
    tc::mbar_init(&S.f_empty, 1);
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&S.g_full[s], 1);
      tc::mbar_init(&S.g_empty[s], 1);
      tc::mbar_init(&S.a_full[s], 1);
      tc::mbar_init(&S.a_empty[s], 4);
      tc::mbar_init(&S.acc_full[s], 1);
      tc::mbar_init(&S.acc_empty[s], 4);
    }
    tc::mbar_fence_init();
  }
  if (warp == 1) tc::tmem_alloc(&S.tmem_base, 128);
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = S.tmem_base;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      int64_t prev_rb = -1;
      uint32_t nf = 0;
      for (int64_t t = t_beg, i = 0; t < t_end; ++t, ++i) {
        const int64_t rb = t / ntc, cb = t % ntc;
        const int s = static_cast<int>(i & 1);
        if (rb != prev_rb) {
          if (nf > 0) tc::mbar_wait(&S.f_empty, (nf - 1) & 1);
          tc::mbar_expect_tx(&S.f_full, 2 * katoms * kFAtomBytes);
          for (int a = 0; a < katoms; ++a) {
            tc::tma_load_2d(S.fh[a], &tmFh, a * 32, static_cast<int>(rb * kTcBM), &S.f_full);
            tc::tma_load_2d(S.fl[a], &tmFl, a * 32, static_cast<int>(rb * kTcBM), &S.f_full);
          }
          ++nf;
          prev_rb = rb;
        }
        if (i >= 2) tc::mbar_wait(&S.g_empty[s], ((i >> 1) - 1) & 1);
        tc::mbar_expect_tx(&S.g_full[s], 2 * katoms * kGAtomBytes);
        for (int a = 0; a < katoms; ++a) {
          tc::tma_load_2d(S.gh[s][a], &tmGh, a * 32, static_cast<int>(cb * kTcBN), &S.g_full[s]);
          tc::tma_load_2d(S.gl[s][a], &tmGl, a * 32, static_cast<int>(cb * kTcBN), &S.g_full[s]);
        }
        if (i >= 2) tc::mbar_wait(&S.a_empty[s], ((i >> 1) - 1) & 1);
        tc::mbar_expect_tx(&S.a_full[s], 2 * kABoxBytes);
        for (int h = 0; h < 2; ++h)
          tc::tma_load_2d(S.a[s][h], &tmA, static_cast<int>(cb * kTcBN + h * 32), static_cast<int>(rb * kTcBM),
                          &S.a_full[s]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(kTcBM, kTcBN);
      int64_t prev_rb = -1;
      uint32_t nf = 0;
      for (int64_t t = t_beg, i = 0; t < t_end; ++t, ++i) {
        const int64_t rb = t / ntc;
        const int s = static_cast<int>(i & 1);
        if (rb != prev_rb) {
          tc::mbar_wait(&S.f_full, nf & 1);
          ++nf;
          prev_rb = rb;
        }
        tc::mbar_wait(&S.g_full[s], (i >> 1) & 1);
        if (i >= 2) tc::mbar_wait(&S.acc_empty[s], ((i >> 1) - 1) & 1);
        tc::fence_after_sync();
        const uint32_t d = tmem + static_cast<uint32_t>(s * kTcBN);
        for (int kk = 0; kk < ksteps; ++kk) {
          const int a = kk >> 2;
          const uint32_t off = static_cast<uint32_t>((kk & 3) * 32);
          const uint64_t fh = tc::desc_sw128(tc::smem_u32(S.fh[a]) + off);
          const uint64_t fl = tc::desc_sw128(tc::smem_u32(S.fl[a]) + off);
          const uint64_t gh = tc::desc_sw128(tc::smem_u32(S.gh[s][a]) + off);
          const uint64_t gl = tc::desc_sw128(tc::smem_u32(S.gl[s][a]) + off);
          tc::mma_tf32(d, fh, gh, idesc, kk > 0 ? 1u : 0u);
          tc::mma_tf32(d, fh, gl, idesc, 1u);
          tc::mma_tf32(d, fl, gh, idesc, 1u);
        }
        tc::mma_commit(&S.g_empty[s]);
        tc::mma_commit(&S.acc_full[s]);
        const bool band_ends = (t + 1 == t_end) || ((t + 1) / ntc != rb);
        if (band_ends) tc::mma_commit(&S.f_empty);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue (warps 2-5)
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int row = q * 32 + lane;    // row within the 128-row tile
    double r2 = 0.0, a2 = 0.0;
    for (int64_t t = t_beg, i = 0; t < t_end; ++t, ++i) {
      const int s = static_cast<int>(i & 1);
      const uint32_t ph = static_cast<uint32_t>((i >> 1) & 1);
      tc::mbar_wait(&S.acc_full[s], ph);
      tc::fence_after_sync();
      tc::mbar_wait(&S.a_full[s], ph);
      float tr = 0.f, ta = 0.f;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        float v[32];
        tc::tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(s * kTcBN + h * 32), v);
        const uint8_t* arow = S.a[s][h] + row * 128;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 a4 = *reinterpret_cast<const float4*>(arow + ((c ^ (row & 7)) << 4));
          const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
          for (int x = 0; x < 4; ++x) {
            const float e = av[x] - v[c * 4 + x];
            tr = fmaf(e, e, tr);
            ta = fmaf(av[x], av[x], ta);
          }
        }
      }
      tc::fence_before_sync();
      __syncwarp();
      if (lane == 0) {
        tc::mbar_arrive(&S.acc_empty[s]);
        tc::mbar_arrive(&S.a_empty[s]);
      }
      r2 += static_cast<double>(tr);
      a2 += static_cast<double>(ta);
    }
    r2 = warp_sum_d(r2);
    a2 = warp_sum_d(a2);
    if (lane == 0) {
      S.red[0][q] = r2;
      S.red[1][q] = a2;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (warp == 1) {
    tc::fence_after_sync();
    tc::tmem_dealloc(tmem, 128);
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = ((S.red[0][0] + S.red[0][1]) + S.red[0][2]) + S.red[0][3];
    part[2 * blockIdx.x + 1] = ((S.red[1][0] + S.red[1][1]) + S.red[1][2]) + S.red[1][3];
  }
}

// Fh = tf32(F diag(s)), Fl = F diag(s) - Fh (exact), zero-padded to kp columns; same for G.
__global__ void split_tf32_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows, int ncomp,
                                  const float* __restrict__ s, float* __restrict__ hi, float* __restrict__ lo, int kp) {
  const int64_t total = rows * kp;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = e / kp;
    const int c = static_cast<int>(e % kp);
    float x = 0.f;
    if (c < ncomp) x = X[r * ldx + c] * (s ? s[c] : 1.f);
    const float h = tc::tf32_rna(x);
    hi[e] = h;
    lo[e] = x - h;
  }
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encoder() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2D fp32 tensor map: `cols` x `rows`, row pitch `ld` floats, box 32 x box_rows, 128B swizzle.
static bool make_map(CUtensorMap* tm, const float* base, int64_t cols, int64_t rows, int64_t ld, uint32_t box_rows) {
  EncodeTiledFn enc = encoder();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * sizeof(float)};
  cuuint32_t box[2] = {32, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return enc(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool residual_tc_supported(const float* A, int64_t lda, int64_t m_loc, int64_t n, int ncomp) {
  if (ncomp < 1 || ncomp > kTcKA * 32 || m_loc < 1 || n < 1) return false;
  if ((lda % 4) != 0 || (reinterpret_cast<uintptr_t>(A) & 15) != 0) return false;
  if (m_loc > 0x7fffffff || n > 0x7fffffff) return false;
  if (getenv("CABS_RESIDUAL_FFMA")) return false;
  return encoder() != nullptr;
}

int launch_residual_tc(const float* A, int64_t lda, int64_t m_loc, int64_t n, const float* F, int64_t ldf,
                       const float* s, const float* G, int64_t ldg, int ncomp, float* split, double* part, double* out,
                       cudaStream_t st) {
  const int kp = ncomp > 32 ? 64 : 32;
  float* fh = split;
  float* fl = fh + m_loc * kp;
  float* gh = fl + m_loc * kp;
  float* gl = gh + n * kp;
  note_launch();
  split_tf32_kernel<<<2 * kNumSM, 256, 0, st>>>(F, ldf, m_loc, ncomp, s, fh, fl, kp);
  note_launch();
  split_tf32_kernel<<<2 * kNumSM, 256, 0, st>>>(G, ldg, n, ncomp, nullptr, gh, gl, kp);
  CUtensorMap tA, tFh, tFl, tGh, tGl;
  if (!make_map(&tA, A, n, m_loc, lda, kTcBM) || !make_map(&tFh, fh, kp, m_loc, kp, kTcBM) ||
      !make_map(&tFl, fl, kp, m_loc, kp, kTcBM) || !make_map(&tGh, gh, kp, n, kp, kTcBN) ||
      !make_map(&tGl, gl, kp, n, kp, kTcBN))
    return -1;
  static bool attr = false;
  const size_t smem = sizeof(TcSmem) + 1024;
  if (!attr) {
    cudaFuncSetAttribute(residual_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    attr = true;
  }
  const int64_t T = ceil_div(m_loc, kTcBM) * ceil_div(n, kTcBN);
  int dev = 0, nsm = kNumSM;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int64_t g = T < nsm ? T : nsm;
  const int ksteps = static_cast<int>(ceil_div(ncomp, 8));
  note_launch();
  residual_tc_kernel<<<static_cast<unsigned>(g), kTcThreads, smem, st>>>(tA, tFh, tFl, tGh, tGl, m_loc, n, ksteps, part);
  launch_residual_final(part, static_cast<int>(g), out, st);
  return 0;
}

}  // namespace cabsk
