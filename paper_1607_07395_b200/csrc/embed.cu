// embed.cu -- S5: extrapolation products and the sketching routine's normalisation
// (P:227-232).  Y_c = C V_w, Y_r = R^T U_w; N_c, N_r = column 2-norms;
// P = Y_c diag(sqrt(s)/N_c), Q = Y_r diag(sqrt(s)/N_r)  (pilot embeddings)
// or U = Y_c N_c^-1, V = Y_r N_r^-1                    (sketch factors).
#include "common.cuh"
#include "kernels.cuh"

namespace cabsk {

constexpr int kGemmBM = 64, kGemmBN = 64, kGemmBK = 16;

// Y[p, c] = sum_i X(p, i) B[i, c];  X(p, i) = X[p*ldx + i] (row-major C) or
// X[i*ldx + p] (TRANS: rows of R, i.e. R^T).  FP32 FFMA, ascending i.  Epilogue:
// per-tile FP64 column sums of squares -> norm_part[tile, c] (fixed order).
#ifdef CABS_PROFILE_EMBED
__device__ long long g_emb_tl[2][8];
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define ETL(i) do { if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1)) \
                      g_emb_tl[blockIdx.x == 0 ? 0 : 1][i] = gtimer(); } while (0)
#else
#define ETL(i) do { } while (0)
#endif
struct __align__(16) GemmSmem {
  float Xs[64][kGemmBM + 4];
  float Bs[64][kGemmBN + 4];
  double red[16][kGemmBN];
};

template <bool TRANS>
__device__ __forceinline__ void gemm_tile(const float* __restrict__ X, int64_t ldx, int64_t N, int k,
                                          const float* __restrict__ B, int64_t ldb, int64_t bx, int by,
                                          float (&acc)[4][4], double* __restrict__ norm_part, int64_t ldn,
                                          GemmSmem& sm) {
  auto& Xs = sm.Xs;
  auto& Bs = sm.Bs;
  auto& red = sm.red;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t p0 = bx * kGemmBM;
  const int c0 = by * kGemmBN;
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;
  for (int i0 = 0; i0 < k; i0 += kGemmBK) {
    if (!TRANS) {
      const int pp = tid >> 2, ii = (tid & 3) * 4;
      const int64_t p = p0 + pp;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int i = i0 + ii + q;
        Xs[ii + q][pp] = (p < N && i < k) ? __ldg(X + p * ldx + i) : 0.f;
      }
    } else {
      const int ii = tid >> 4, pp = (tid & 15) * 4;
      const int i = i0 + ii;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t p = p0 + pp + q;
        Xs[ii][pp + q] = (p < N && i < k) ? __ldg(X + (int64_t)i * ldx + p) : 0.f;
      }
    }
    {
      const int ii = tid >> 4, cc = (tid & 15) * 4;
      const int i = i0 + ii;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int c = c0 + cc + q;
        Bs[ii][cc + q] = (i < k && c < k) ? __ldg(B + (int64_t)i * ldb + c) : 0.f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int ii = 0; ii < kGemmBK; ++ii) {
      float a[4], b[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        a[q] = Xs[ii][ty * 4 + q];
        b[q] = Bs[ii][tx * 4 + q];
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
  double ss[4] = {0, 0, 0, 0};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t p = p0 + ty * 4 + u;
    if (p >= N) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int c = c0 + tx * 4 + v;
      if (c < k) ss[v] += static_cast<double>(acc[u][v]) * static_cast<double>(acc[u][v]);
    }
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) red[ty][tx * 4 + v] = ss[v];
  __syncthreads();
  if (tid < kGemmBN) {
    double s2 = 0;
    for (int t = 0; t < 16; ++t) s2 += red[t][tid];
    const int c = c0 + tid;
    if (c < k) norm_part[bx * ldn + c] = s2;
  }
}

// k <= 64: the whole X tile (64 points x k) and B (k x 64) staged at once (every load in
// flight together, one barrier), then the same FP32 FFMA chain in ascending i.
template <bool TRANS>
__device__ __forceinline__ void gemm_tile_k64(const float* __restrict__ X, int64_t ldx, int64_t N, int k,
                                              const float* __restrict__ B, int64_t ldb, int64_t bx, int by,
                                              float (&acc)[4][4], double* __restrict__ norm_part, int64_t ldn,
                                              GemmSmem& sm) {
  auto& Xs = sm.Xs;
  auto& Bs = sm.Bs;
  auto& red = sm.red;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t p0 = bx * kGemmBM;
  const int c0 = by * kGemmBN;
  // float4 loads (ldx, ldb multiples of 4, 16-byte aligned bases: checked by the launcher)
  if (!TRANS) {  // X row-major: row p, dims i4..i4+3
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + 256 * q;  // 64 rows x 16 quads
      const int pp = e >> 4, i4 = (e & 15) * 4;
      const int64_t p = p0 + pp;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p < N && i4 < k) v = __ldg(reinterpret_cast<const float4*>(X + p * ldx + i4));
      Xs[i4][pp] = i4 < k ? v.x : 0.f;
      Xs[i4 + 1][pp] = i4 + 1 < k ? v.y : 0.f;
      Xs[i4 + 2][pp] = i4 + 2 < k ? v.z : 0.f;
      Xs[i4 + 3][pp] = i4 + 3 < k ? v.w : 0.f;
    }
  } else {  // X = R^T: row i of R, points pp..pp+3
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int e = tid + 256 * q;  // 64 dims x 16 quads of points
      const int ii = e >> 4, pp = (e & 15) * 4;
      const int64_t p = p0 + pp;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (ii < k) {
        if (p + 3 < N) {
          v = __ldg(reinterpret_cast<const float4*>(X + (int64_t)ii * ldx + p));
        } else {
          if (p < N) v.x = __ldg(X + (int64_t)ii * ldx + p);
          if (p + 1 < N) v.y = __ldg(X + (int64_t)ii * ldx + p + 1);
          if (p + 2 < N) v.z = __ldg(X + (int64_t)ii * ldx + p + 2);
        }
      }
      *reinterpret_cast<float4*>(&Xs[ii][pp]) = v;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int e = tid + 256 * q;
    const int ii = e >> 4, cc = (e & 15) * 4;
    const int c = c0 + cc;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (ii < k) {
      if (c + 3 < k) {
        v = __ldg(reinterpret_cast<const float4*>(B + (int64_t)ii * ldb + c));
      } else {
        if (c < k) v.x = __ldg(B + (int64_t)ii * ldb + c);
        if (c + 1 < k) v.y = __ldg(B + (int64_t)ii * ldb + c + 1);
        if (c + 2 < k) v.z = __ldg(B + (int64_t)ii * ldb + c + 2);
      }
    }
    *reinterpret_cast<float4*>(&Bs[ii][cc]) = v;
  }
  __syncthreads();
  ETL(6);
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) acc[u][v] = 0.f;
#pragma unroll 8
  for (int ii = 0; ii < k; ++ii) {
    float a[4], b[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a[q] = Xs[ii][ty * 4 + q];
      b[q] = Bs[ii][tx * 4 + q];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = fmaf(a[u], b[v], acc[u][v]);
  }
  double ss[4] = {0, 0, 0, 0};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t p = p0 + ty * 4 + u;
    if (p >= N) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int c = c0 + tx * 4 + v;
      if (c < k) ss[v] += static_cast<double>(acc[u][v]) * static_cast<double>(acc[u][v]);
    }
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) red[ty][tx * 4 + v] = ss[v];
  __syncthreads();
  if (tid < kGemmBN) {
    double s2 = 0;
    for (int t = 0; t < 16; ++t) s2 += red[t][tid];
    const int c = c0 + tid;
    if (c < k) norm_part[bx * ldn + c] = s2;
  }
}

template <bool TRANS>
__global__ void __launch_bounds__(256) embed_gemm_kernel(const float* __restrict__ X, int64_t ldx, int64_t N, int k,
                                                         const float* __restrict__ B, int64_t ldb,
                                                         float* __restrict__ Y, int64_t ldy,
                                                         double* __restrict__ norm_part, int64_t ldn) {
  __shared__ GemmSmem sm;
  float acc[4][4];
  gemm_tile<TRANS>(X, ldx, N, k, B, ldb, blockIdx.x, blockIdx.y, acc, norm_part, ldn, sm);
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int64_t p = (int64_t)blockIdx.x * kGemmBM + ty * 4 + u;
    if (p >= N) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int c = blockIdx.y * kGemmBN + tx * 4 + v;
      if (c < k) Y[p * ldy + c] = acc[u][v];
    }
  }
}

// norms2[c] = sum_t part[t, c] in fixed order (FP64).
__global__ void __launch_bounds__(256) reduce_cols_kernel(const double* __restrict__ part, int64_t ntiles, int64_t ldp,
                                                          int k, double* __restrict__ out) {
  __shared__ double red[256];
  const int c = blockIdx.x;
  double s = 0;
  for (int64_t t = threadIdx.x; t < ntiles; t += blockDim.x) s += part[t * ldp + c];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[c] = red[0];
}

int launch_embed_products(int64_t m_loc, int64_t n_sl, int k, const float* C, int64_t ldc, const float* R_slice,
                          int64_t ldr, float* Yc, int64_t ldyc, float* Yr, int64_t ldyr, void* ws, const Ws& L,
                          cudaStream_t st, cudaStream_t st2) {
  // st2 (optional): Y_r's product and norm reduction run there, concurrently with Y_c's
  if (!st2) st2 = st;
  double* part = wsp<double>(ws, L.norm_part);
  double* norms = wsp<double>(ws, L.norms);
  const int gy = static_cast<int>(ceil_div(k, kGemmBN));
  // Y_c = C V_w
  if (m_loc > 0) {
    dim3 g(static_cast<unsigned>(ceil_div(m_loc, kGemmBM)), gy);
    note_launch();
    embed_gemm_kernel<false><<<g, 256, 0, st>>>(C, ldc, m_loc, k, wsp<float>(ws, L.vw32), L.Kp, Yc, ldyc, part, L.Kp);
    note_launch();
    reduce_cols_kernel<<<k, 256, 0, st>>>(part, ceil_div(m_loc, kGemmBM), L.Kp, k, norms);
  } else {
    cudaMemsetAsync(norms, 0, sizeof(double) * k, st);
  }
  // Y_r = R^T U_w over this rank's column slice
  double* part_r = part + L.npt * L.Kp;
  if (n_sl > 0) {
    dim3 g(static_cast<unsigned>(ceil_div(n_sl, kGemmBM)), gy);
    note_launch();
    embed_gemm_kernel<true><<<g, 256, 0, st2>>>(R_slice, ldr, n_sl, k, wsp<float>(ws, L.uw32), L.Kp, Yr, ldyr, part_r,
                                                L.Kp);
    note_launch();
    reduce_cols_kernel<<<k, 256, 0, st2>>>(part_r, ceil_div(n_sl, kGemmBM), L.Kp, k, norms + L.Kp);
  } else {
    cudaMemsetAsync(norms + L.Kp, 0, sizeof(double) * k, st2);
  }
  return 0;
}

// Scales of the sketching routine.  keep_c = c < r && N_c,c > 0 && N_r,c > 0.
// kind 0 (embed):  alpha = sqrt(s)/N_c, beta = sqrt(s)/N_r
// kind 1 (sketch): alpha = 1/N_c,       beta = 1/N_r,  s_out = s
// s = sigma sqrt(m n)/k (STABILIZED) or N_c N_r / sigma (PSEUDO_SKELETON, Eq. 2).
// One thread per component; newpos = exclusive prefix count of kept components (block scan).
// flags[0] = r_eff, flags[1] = 1 when the kept components are exactly 0..r_eff-1 (no compaction).
__global__ void __launch_bounds__(1024) embed_finalize_kernel(int k, const double* __restrict__ sig,
                                                              const int* __restrict__ r_in,
                                                              const double* __restrict__ nc2,
                                                              const double* __restrict__ nr2, int mode, double m,
                                                              double n, double ksamp, int kind,
                                                              double* __restrict__ alpha, double* __restrict__ beta,
                                                              int* __restrict__ newpos, float* __restrict__ s_out,
                                                              int* __restrict__ r_out, int* __restrict__ r_out2,
                                                              int* __restrict__ flags) {
  __shared__ int warp_cnt[32];
  __shared__ int s_total, s_hole;
  const int c = threadIdx.x, lane = c & 31, warp = c >> 5;
  const int r = *r_in;
  bool keep = false;
  double s = 0, a = 0, bb = 0;
  if (c < k) {
    const double Nc = sqrt(nc2[c]), Nr = sqrt(nr2[c]);
    keep = c < r && Nc > 0 && Nr > 0;
    if (keep) {
      s = (mode == CABS_STABILIZED) ? sig[c] * sqrt(m * n) / ksamp : Nc * Nr / sig[c];
      if (kind == 0) {
        const double rs = sqrt(s);
        a = rs / Nc;
        bb = rs / Nr;
      } else {
        a = 1.0 / Nc;
        bb = 1.0 / Nr;
      }
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) warp_cnt[warp] = __popc(bal);
  if (c == 0) s_hole = 0;
  __syncthreads();
  if (c == 0) {
    int t = 0;
    for (int w = 0; w < 32; ++w) { const int x = warp_cnt[w]; warp_cnt[w] = t; t += x; }
    s_total = t;
  }
  __syncthreads();
  const int pos = warp_cnt[warp] + __popc(bal & ((1u << lane) - 1u));
  if (c < k) {
    newpos[c] = keep ? pos : -1;
    alpha[c] = a;
    beta[c] = bb;
    if (keep && pos != c) atomicOr(&s_hole, 1);
  }
  __syncthreads();
  const int reff = s_total;
  if (c < k && s_out) s_out[c] = 0.f;
  __syncthreads();
  if (keep && s_out) s_out[pos] = static_cast<float>(s);
  if (c == 0) {
    if (r_out) *r_out = reff;
    if (r_out2) *r_out2 = reff;
    flags[0] = reff;
    flags[1] = s_hole ? 0 : 1;
  }
}

// Element-wise fast path (kept components are 0..r_eff-1): Y[p, c] *= scale[c], zero c >= r_eff.
__global__ void __launch_bounds__(256) scale_ident_kernel(float* __restrict__ Y, int64_t ldy, int64_t N, int k,
                                                          const double* __restrict__ scale,
                                                          const int* __restrict__ flags) {
  if (flags[1] == 0) return;  // compaction needed: scale_compact_kernel does it
  const int reff = flags[0];
  const int64_t total = N * k;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = e / k;
    const int c = static_cast<int>(e - p * k);
    float* y = Y + p * ldy + c;
    *y = c < reff ? static_cast<float>(static_cast<double>(*y) * scale[c]) : 0.f;
  }
}

// In-place compaction (a dropped component inside [0, r)): row[newpos[c]] = row[c] * scale[c]
// for kept c, zeros in [r_eff, k).  Rare; one warp per row.
__global__ void __launch_bounds__(256) scale_compact_kernel(float* __restrict__ Y, int64_t ldy, int64_t N, int k,
                                                            const double* __restrict__ scale,
                                                            const int* __restrict__ newpos,
                                                            const int* __restrict__ flags) {
  if (flags[1] != 0) return;  // identity layout: handled element-wise by scale_ident_kernel
  __shared__ double s_scale[CABS_KMAX];
  __shared__ int s_pos[CABS_KMAX];
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    s_scale[c] = scale[c];
    s_pos[c] = newpos[c];
  }
  __syncthreads();
  const int reff = flags[0];
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  constexpr int kPer = CABS_KMAX / 32;
  for (int64_t p = warp; p < N; p += nw) {
    float* row = Y + p * ldy;
    float v[kPer];
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int c = lane + 32 * q;
      v[q] = c < k ? row[c] : 0.f;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int c = lane + 32 * q;
      if (c < k && c >= reff) row[c] = 0.f;
    }
    __syncwarp();
#pragma unroll
    for (int q = 0; q < kPer; ++q) {
      const int c = lane + 32 * q;
      if (c < k && s_pos[c] >= 0) row[s_pos[c]] = static_cast<float>(static_cast<double>(v[q]) * s_scale[c]);
    }
    __syncwarp();
  }
}

int launch_embed_finalize(int k, int mode, double m, double n, double ksamp, int kind, float* s_out, int* r_user,
                          void* ws, const Ws& L, cudaStream_t st) {
  double* sc = wsp<double>(ws, L.scales);
  int* newpos = reinterpret_cast<int*>(sc + 2 * L.Kp);
  int* flags = newpos + L.Kp;
  const double* norms = wsp<double>(ws, L.norms);
  int* scal = wsp<int>(ws, L.scal);
  note_launch();
  embed_finalize_kernel<<<1, 1024, 0, st>>>(k, wsp<double>(ws, L.sig64), scal + SCAL_R_TMP, norms, norms + L.Kp, mode,
                                            m, n, ksamp, kind, sc, sc + L.Kp, newpos, s_out, scal + SCAL_R_TMP,
                                            r_user, flags);
  return 0;
}

int launch_scale_compact(float* Y, int64_t ldy, int64_t N, int k, int which, void* ws, const Ws& L, cudaStream_t st) {
  if (N <= 0) return 0;
  double* sc = wsp<double>(ws, L.scales);
  int* newpos = reinterpret_cast<int*>(sc + 2 * L.Kp);
  int* flags = newpos + L.Kp;
  int64_t blocks = ceil_div(N * k, 256 * 4);
  if (blocks > 8 * kNumSM) blocks = 8 * kNumSM;
  if (blocks < 1) blocks = 1;
  note_launch();
  scale_ident_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(Y, ldy, N, k, sc + which * L.Kp, flags);
  blocks = ceil_div(N, 8);
  if (blocks > 8 * kNumSM) blocks = 8 * kNumSM;
  note_launch();
  scale_compact_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(Y, ldy, N, k, sc + which * L.Kp, newpos, flags);
  return 0;
}

// ---------------------------------------------------------------- single-GPU fused S5
// ONE cooperative launch for both products and the normalisation: GEMM tiles of Y_c = C V_w
// and Y_r = R^T U_w (accumulators stay in registers) | grid barrier | column norms from the
// tile partials (fixed order, as reduce_cols_kernel) | grid barrier | every CTA forms the
// scales and the compaction map (as embed_finalize_kernel) and writes its tile of P, Q (or
// U, V) scaled, compacted and zero-padded -- no memsets, no second pass over Y.
struct EmbedFused {
  const float* X[2];
  int64_t ldx[2], N[2];
  const float* B[2];
  int64_t ldb;
  float* Y[2];
  int64_t ldy[2];
  int k, gy;
  int64_t tiles0;
  double* part[2];
  double* norms;
  int64_t Kp;
  const double* sig;
  const int* r_in;
  int mode, kind;
  double m, n, ksamp;
  double* alpha;
  double* beta;
  int* newpos;
  float* s_out;
  int* r_out;
  int* r_out2;
  int* flags;
  unsigned* bar;
};

__global__ void __launch_bounds__(256) embed_fused_kernel(EmbedFused a) {
  __shared__ double s_scale[256];
  __shared__ int s_pos[256];
  __shared__ int warp_cnt[8];
  __shared__ int s_total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, tx = tid & 15, ty = tid >> 4;
  const int k = a.k;
  const int side = static_cast<int64_t>(blockIdx.x) < a.tiles0 ? 0 : 1;
  const int64_t tl = side ? static_cast<int64_t>(blockIdx.x) - a.tiles0 : static_cast<int64_t>(blockIdx.x);
  const int64_t bx = tl / a.gy;
  const int by = static_cast<int>(tl - bx * a.gy);
  ETL(0);
  const int r = *a.r_in;  // read before CTA 0 rewrites the slot (after the second barrier)
  float acc[4][4];
  __shared__ GemmSmem sm;
  if (k <= 64) {
    if (side == 0) gemm_tile_k64<false>(a.X[0], a.ldx[0], a.N[0], k, a.B[0], a.ldb, bx, by, acc, a.part[0], a.Kp, sm);
    else gemm_tile_k64<true>(a.X[1], a.ldx[1], a.N[1], k, a.B[1], a.ldb, bx, by, acc, a.part[1], a.Kp, sm);
  } else {
    if (side == 0) gemm_tile<false>(a.X[0], a.ldx[0], a.N[0], k, a.B[0], a.ldb, bx, by, acc, a.part[0], a.Kp, sm);
    else gemm_tile<true>(a.X[1], a.ldx[1], a.N[1], k, a.B[1], a.ldb, bx, by, acc, a.part[1], a.Kp, sm);
  }
  unsigned gen = 0;
  ETL(1);
  grid_barrier(a.bar, gen);
  ETL(2);
  double* s_red = &sm.red[0][0];  // the tile is done with it
  for (int cc = blockIdx.x; cc < 2 * k; cc += gridDim.x) {  // column norms, fixed order
    const int sd = cc / k, c = cc - sd * k;
    const int64_t ntiles = ceil_div(a.N[sd], kGemmBM);
    double acc2 = 0;
    for (int64_t t = tid; t < ntiles; t += blockDim.x) acc2 += __ldcg(a.part[sd] + t * a.Kp + c);
    s_red[tid] = acc2;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
      if (tid < w) s_red[tid] += s_red[tid + w];
      __syncthreads();
    }
    if (tid == 0) a.norms[sd * a.Kp + c] = s_red[0];
    __syncthreads();
  }
  ETL(3);
  grid_barrier(a.bar, gen);
  ETL(4);
  // scales of the sketching routine (embed_finalize_kernel), component c = tid
  bool keep = false;
  double sv = 0, al = 0, be = 0;
  if (tid < k) {
    const double Nc = sqrt(__ldcg(a.norms + tid)), Nr = sqrt(__ldcg(a.norms + a.Kp + tid));
    keep = tid < r && Nc > 0 && Nr > 0;
    if (keep) {
      const double sg = __ldcg(a.sig + tid);
      sv = (a.mode == CABS_STABILIZED) ? sg * sqrt(a.m * a.n) / a.ksamp : Nc * Nr / sg;
      if (a.kind == 0) {
        const double rs = sqrt(sv);
        al = rs / Nc;
        be = rs / Nr;
      } else {
        al = 1.0 / Nc;
        be = 1.0 / Nr;
      }
    }
  }
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if (lane == 0) warp_cnt[warp] = __popc(bal);
  __syncthreads();
  if (tid == 0) {
    int t = 0;
    for (int w = 0; w < 8; ++w) { const int x = warp_cnt[w]; warp_cnt[w] = t; t += x; }
    s_total = t;
  }
  __syncthreads();
  const int pos = warp_cnt[warp] + __popc(bal & ((1u << lane) - 1u));
  s_scale[tid] = side ? be : al;
  s_pos[tid] = keep ? pos : -1;
  __syncthreads();
  const int reff = s_total;
  if (blockIdx.x == 0) {
    if (tid < k) {
      a.newpos[tid] = keep ? pos : -1;
      a.alpha[tid] = al;
      a.beta[tid] = be;
      if (a.s_out) a.s_out[tid] = 0.f;
    }
    __syncthreads();
    if (keep && a.s_out) a.s_out[pos] = static_cast<float>(sv);
    if (tid == 0) {
      if (a.r_out) *a.r_out = reff;
      if (a.r_out2) *a.r_out2 = reff;
      a.flags[0] = reff;
      a.flags[1] = 1;
    }
  }
  // this tile of the output: kept columns scaled into their compacted positions, zeros in
  // [r_eff, ldy) (the last column tile covers the padding up to ldy)
  float* Y = a.Y[side];
  const int64_t ldy = a.ldy[side], N = a.N[side];
  const int c0 = by * kGemmBN;
  if (a.gy == 1 && ldy <= kGemmBN + 4 && (ldy & 3) == 0) {
    // whole rows in this tile: stage the compacted, scaled rows in shared memory, then write
    // each row [0, ldy) with coalesced 16-byte stores
    __syncthreads();
    float (*T)[kGemmBM + 4] = sm.Xs;  // [row][col]
    for (int e = tid; e < kGemmBM * (kGemmBN + 4); e += blockDim.x) (&T[0][0])[e] = 0.f;
    __syncthreads();
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int c = tx * 4 + v;
        if (c < k && s_pos[c] >= 0) T[ty * 4 + u][s_pos[c]] = static_cast<float>(static_cast<double>(acc[u][v]) * s_scale[c]);
      }
    __syncthreads();
    const int q4 = static_cast<int>(ldy >> 2);
    for (int e = tid; e < kGemmBM * q4; e += blockDim.x) {
      const int row = e / q4, c4 = (e - row * q4) * 4;
      const int64_t p = bx * kGemmBM + row;
      if (p < N) *reinterpret_cast<float4*>(Y + p * ldy + c4) = *reinterpret_cast<const float4*>(&T[row][c4]);
    }
  } else {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t p = bx * kGemmBM + ty * 4 + u;
      if (p >= N) continue;
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        const int c = c0 + tx * 4 + v;
        if (c < k && s_pos[c] >= 0)
          Y[p * ldy + s_pos[c]] = static_cast<float>(static_cast<double>(acc[u][v]) * s_scale[c]);
      }
    }
    const int q0 = c0 > reff ? c0 : reff;
    const int64_t q1 = by == a.gy - 1 ? ldy : c0 + kGemmBN;
    for (int64_t q = q0 + tx; q < q1; q += 16)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t p = bx * kGemmBM + ty * 4 + u;
        if (p < N) Y[p * ldy + q] = 0.f;
      }
  }
  ETL(5);
}
void embed_debug_timeline(long long* out) {
#ifdef CABS_PROFILE_EMBED
  cudaMemcpyFromSymbol(out, g_emb_tl, sizeof(long long) * 16);
#else
  for (int i = 0; i < 16; ++i) out[i] = 0;
#endif
}

bool launch_embed_fused(int64_t m_loc, int64_t n_sl, int k, const float* C, int64_t ldc, const float* R_slice,
                        int64_t ldr, float* Y1, int64_t ld1, float* Y2, int64_t ld2, int mode, double m, double n,
                        double ksamp, int kind, float* s_out, int* r_user, void* ws, const Ws& L, cudaStream_t st) {
  if (k > 256 || m_loc < 1 || n_sl < 1) return false;
  if ((ldc & 3) || (ldr & 3) || (L.Kp & 3) || (reinterpret_cast<uintptr_t>(C) & 15) ||
      (reinterpret_cast<uintptr_t>(R_slice) & 15) || (reinterpret_cast<uintptr_t>(Y1) & 15) ||
      (reinterpret_cast<uintptr_t>(Y2) & 15))
    return false;
  const int gy = static_cast<int>(ceil_div(k, kGemmBN));
  const int64_t tiles0 = ceil_div(m_loc, kGemmBM) * gy, tiles1 = ceil_div(n_sl, kGemmBM) * gy;
  const int64_t G = tiles0 + tiles1;
  int dev = 0, nsm = 0, per = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, embed_fused_kernel, 256, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (G > (int64_t)per * nsm || G > 0x7fffffff) return false;
  EmbedFused a{};
  a.X[0] = C; a.ldx[0] = ldc; a.N[0] = m_loc;
  a.X[1] = R_slice; a.ldx[1] = ldr; a.N[1] = n_sl;
  a.B[0] = wsp<float>(ws, L.vw32); a.B[1] = wsp<float>(ws, L.uw32); a.ldb = L.Kp;
  a.Y[0] = Y1; a.ldy[0] = ld1; a.Y[1] = Y2; a.ldy[1] = ld2;
  a.k = k; a.gy = gy; a.tiles0 = tiles0;
  double* part = wsp<double>(ws, L.norm_part);
  a.part[0] = part; a.part[1] = part + L.npt * L.Kp;
  a.norms = wsp<double>(ws, L.norms); a.Kp = L.Kp;
  double* sc = wsp<double>(ws, L.scales);
  int* scal = wsp<int>(ws, L.scal);
  a.sig = wsp<double>(ws, L.sig64); a.r_in = scal + SCAL_R_TMP;
  a.mode = mode; a.kind = kind; a.m = m; a.n = n; a.ksamp = ksamp;
  a.alpha = sc; a.beta = sc + L.Kp;
  a.newpos = reinterpret_cast<int*>(sc + 2 * L.Kp);
  a.flags = a.newpos + L.Kp;
  a.s_out = s_out; a.r_out = scal + SCAL_R_TMP; a.r_out2 = r_user;
  a.bar = reinterpret_cast<unsigned*>(scal + SCAL_EBAR);
  if (cudaMemsetAsync(a.bar, 0, 2 * sizeof(unsigned), st) != cudaSuccess) return false;
  void* args[] = {&a};
  note_launch();
  return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(embed_fused_kernel), dim3(static_cast<unsigned>(G)),
                                     dim3(256), args, 0, st) == cudaSuccess;
}

}  // namespace cabsk
