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
template <bool TRANS>
__global__ void __launch_bounds__(256) embed_gemm_kernel(const float* __restrict__ X, int64_t ldx, int64_t N, int k,
                                                         const float* __restrict__ B, int64_t ldb,
                                                         float* __restrict__ Y, int64_t ldy,
                                                         double* __restrict__ norm_part, int64_t ldn) {
  __shared__ float Xs[kGemmBK][kGemmBM + 4];
  __shared__ float Bs[kGemmBK][kGemmBN + 4];
  __shared__ double red[16][kGemmBN];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int64_t p0 = (int64_t)blockIdx.x * kGemmBM;
  const int c0 = blockIdx.y * kGemmBN;
  float acc[4][4] = {};
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
      if (c < k) {
        Y[p * ldy + c] = acc[u][v];
        ss[v] += static_cast<double>(acc[u][v]) * static_cast<double>(acc[u][v]);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < 4; ++v) red[ty][tx * 4 + v] = ss[v];
  __syncthreads();
  if (tid < kGemmBN) {
    double s = 0;
    for (int t = 0; t < 16; ++t) s += red[t][tid];
    const int c = c0 + tid;
    if (c < k) norm_part[(int64_t)blockIdx.x * ldn + c] = s;
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
                          cudaStream_t st) {
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
    embed_gemm_kernel<true><<<g, 256, 0, st>>>(R_slice, ldr, n_sl, k, wsp<float>(ws, L.uw32), L.Kp, Yr, ldyr, part_r,
                                               L.Kp);
    note_launch();
    reduce_cols_kernel<<<k, 256, 0, st>>>(part_r, ceil_div(n_sl, kGemmBM), L.Kp, k, norms + L.Kp);
  } else {
    cudaMemsetAsync(norms + L.Kp, 0, sizeof(double) * k, st);
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

}  // namespace cabsk
