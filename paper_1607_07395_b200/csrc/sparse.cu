// sparse.cu -- a sparse source A ("For sparse matrices",
// Table 1; cabs.h CABS_SOURCE_CSR_F32): the gathers of Alg. 2 from
// the rank's row block in CSR (rows) and CSC (columns), and the P:313 error without forming
// A - F S G^T:
//   ||A - F S G^T||^2 = ||A||^2 - 2 sum_{nonzeros} a_ij (F S G^T)_ij + sum_kl (F^T F)_kl s_k s_l (G^T G)_kl
// (the Gram products come from the FP64 Gram kernels of orth.cu).  Gathers are exact copies
// (every entry is either a stored value or 0), identical to the dense gathers of the densified
// matrix.
#include <float.h>

#include "common.cuh"
#include "kernels.cuh"

namespace cabsk {

constexpr int kSpT = 256;

// R[a, :] = A(I[a], :) for the sampled rows this rank owns: the row is zeroed, then its
// nonzeros scattered (one CTA per sampled row).  Rows owned elsewhere are left untouched (the
// caller's allreduce completes them, as for a dense source).
__global__ void __launch_bounds__(kSpT) csr_rows_kernel(CsrSrc a, int64_t row_begin, int64_t row_end,
                                                        const int64_t* __restrict__ I, int64_t n, float* R, int64_t ldr) {
  const int b = blockIdx.x;
  const int64_t i = I[b];
  if (i < row_begin || i >= row_end) return;
  float* dst = R + b * ldr;
  for (int64_t c = threadIdx.x; c < n; c += kSpT) dst[c] = 0.f;
  __syncthreads();
  const int64_t lo = a.row_ptr[i - row_begin], hi = a.row_ptr[i - row_begin + 1];
  for (int64_t e = lo + threadIdx.x; e < hi; e += kSpT) dst[__ldg(a.col_idx + e)] = __ldg(a.row_val + e);
}

// C[r, c] = 0 for the rank's rows r and c < k (16-byte stores where the row allows)
__global__ void __launch_bounds__(kSpT) zero_cols_kernel(int64_t m_loc, int k, float* C, int64_t ldc) {
  const int64_t total = m_loc * k;
  for (int64_t e = blockIdx.x * (int64_t)kSpT + threadIdx.x; e < total; e += (int64_t)gridDim.x * kSpT) {
    const int64_t r = e / k;
    C[r * ldc + (e - r * k)] = 0.f;
  }
}

// C[r, c] = A(r, J[c]): column J[c]'s nonzeros (CSC) scattered into column c of C; one warp per
// sampled column.  An index outside [0, n) contributes nothing (validate_idx reports it).
__global__ void __launch_bounds__(kSpT) csc_cols_kernel(CsrSrc a, int64_t n, const int64_t* __restrict__ J, int k,
                                                        float* C, int64_t ldc) {
  const int c = static_cast<int>((blockIdx.x * (int64_t)kSpT + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (c >= k) return;
  const int64_t j = J[c];
  if (j < 0 || j >= n) return;
  const int64_t lo = a.col_ptr[j], hi = a.col_ptr[j + 1];
  for (int64_t e = lo + lane; e < hi; e += 32) C[static_cast<int64_t>(__ldg(a.row_idx + e)) * ldc + c] = __ldg(a.col_val + e);
}

// W[a, c] = A(I[a], J[c]) straight from the CSR rows (single rank): the row's nonzero columns are
// matched against J (staged in shared memory; J need not be sorted).  One CTA per sampled row.
__global__ void __launch_bounds__(kSpT) csr_w_kernel(CsrSrc a, int64_t row_begin, int64_t row_end,
                                                     const int64_t* __restrict__ I, const int64_t* __restrict__ J,
                                                     int k, float* W, int64_t ldw) {
  extern __shared__ int64_t sJ[];
  const int b = blockIdx.x;
  for (int c = threadIdx.x; c < k; c += kSpT) {
    sJ[c] = J[c];
    W[b * ldw + c] = 0.f;
  }
  __syncthreads();
  const int64_t i = I[b];
  if (i < row_begin || i >= row_end) return;
  const int64_t lo = a.row_ptr[i - row_begin], hi = a.row_ptr[i - row_begin + 1];
  for (int64_t e = lo + threadIdx.x; e < hi; e += kSpT) {
    const int64_t col = __ldg(a.col_idx + e);
    const float v = __ldg(a.row_val + e);
    for (int c = 0; c < k; ++c)
      if (sJ[c] == col) W[b * ldw + c] = v;
  }
}

void launch_csr_rows(const CsrSrc& a, int64_t row_begin, int64_t row_end, const int64_t* I, int k, int64_t n, float* R,
                     int64_t ldr, cudaStream_t st) {
  note_launch();
  csr_rows_kernel<<<k, kSpT, 0, st>>>(a, row_begin, row_end, I, n, R, ldr);
}

void launch_csc_cols(const CsrSrc& a, int64_t m_loc, int64_t n, const int64_t* J, int k, float* C, int64_t ldc,
                     cudaStream_t st) {
  if (m_loc <= 0) return;
  int64_t blocks = ceil_div(m_loc * k, kSpT);
  if (blocks > 8 * kNumSM) blocks = 8 * kNumSM;
  note_launch();
  zero_cols_kernel<<<static_cast<unsigned>(blocks), kSpT, 0, st>>>(m_loc, k, C, ldc);
  note_launch();
  csc_cols_kernel<<<static_cast<unsigned>(ceil_div(32LL * k, kSpT)), kSpT, 0, st>>>(a, n, J, k, C, ldc);
}

void launch_csr_w(const CsrSrc& a, int64_t row_begin, int64_t row_end, const int64_t* I, const int64_t* J, int k,
                  float* W, int64_t ldw, cudaStream_t st) {
  note_launch();
  csr_w_kernel<<<k, kSpT, sizeof(int64_t) * k, st>>>(a, row_begin, row_end, I, J, k, W, ldw);
}

// ---------------------------------------------------------------- residual
// Per CTA (fixed row partition, warps over rows in a fixed order): sum over the nonzeros of a^2
// and of a (F S G^T)_ij.  The warp's F_i diag(s) is staged in shared memory; groups of 8 lanes
// take one nonzero each (4 per warp at a time), the group's lanes read contiguous 16-byte chunks
// of the G row (coalesced) and the partial dot products meet by 3 shuffles.  FP32 products, FP64
// accumulation of a (.) per nonzero.
constexpr int kSpResMaxK = 512;
__global__ void __launch_bounds__(kSpT) sparse_res_nnz_kernel(CsrSrc a, int64_t m_loc, const float* __restrict__ F,
                                                              int64_t ldf, const float* __restrict__ s,
                                                              const float* __restrict__ G, int64_t ldg, int ncomp,
                                                              double* part) {
  __shared__ __align__(16) float fs[kSpT / 32][kSpResMaxK];
  __shared__ double r0[kSpT / 32], r1[kSpT / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
  const int64_t per = ceil_div(m_loc, gridDim.x);
  const int64_t rb = blockIdx.x * per, re = rb + per < m_loc ? rb + per : m_loc;
  const bool vec = (ldg & 3) == 0 && (reinterpret_cast<uintptr_t>(G) & 15) == 0;
  const int nc4 = (ncomp + 3) >> 2;
  double a2 = 0.0, cr = 0.0;
  float* f = fs[warp];
  for (int64_t i = rb + warp; i < re; i += kSpT / 32) {
    __syncwarp();
    for (int c = lane; c < 4 * nc4; c += 32) f[c] = c < ncomp ? __ldg(F + i * ldf + c) * (s ? __ldg(s + c) : 1.f) : 0.f;
    __syncwarp();
    const int64_t lo = a.row_ptr[i], hi = a.row_ptr[i + 1];
    for (int64_t e0 = lo; e0 < hi; e0 += 4) {
      const int64_t e = e0 + grp;
      const bool on = e < hi;
      const float v = on ? __ldg(a.row_val + e) : 0.f;
      const float* g = G + static_cast<int64_t>(on ? __ldg(a.col_idx + e) : 0) * ldg;
      float t = 0.f;
      if (vec) {
        for (int c4 = gl; c4 < nc4; c4 += 8) {
          float4 gv = __ldg(reinterpret_cast<const float4*>(g) + c4);
          if (4 * c4 + 3 >= ncomp) {  // the tail of the row: G's padding need not be zero
            if (4 * c4 + 1 >= ncomp) gv.y = 0.f;
            if (4 * c4 + 2 >= ncomp) gv.z = 0.f;
            gv.w = 0.f;
          }
          const float4 fv = *reinterpret_cast<const float4*>(f + 4 * c4);
          t = fmaf(fv.x, gv.x, t);
          t = fmaf(fv.y, gv.y, t);
          t = fmaf(fv.z, gv.z, t);
          t = fmaf(fv.w, gv.w, t);
        }
      } else {
        for (int c = gl; c < ncomp; c += 8) t = fmaf(f[c], __ldg(g + c), t);
      }
      t += __shfl_xor_sync(0xffffffffu, t, 1);
      t += __shfl_xor_sync(0xffffffffu, t, 2);
      t += __shfl_xor_sync(0xffffffffu, t, 4);
      if (on && gl == 0) {
        a2 = fma(static_cast<double>(v), static_cast<double>(v), a2);
        cr = fma(static_cast<double>(v), static_cast<double>(t), cr);
      }
    }
  }
  a2 = warp_sum_d(a2);
  cr = warp_sum_d(cr);
  if (lane == 0) { r0[warp] = a2; r1[warp] = cr; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w = 0; w < kSpT / 32; ++w) { x += r0[w]; y += r1[w]; }
    part[2 * blockIdx.x] = x;
    part[2 * blockIdx.x + 1] = y;
  }
}

// out = (a2 - 2 cross + sum_kl GU_kl s_k s_l GV_kl, a2); one CTA, fixed order
__global__ void __launch_bounds__(kSpT) sparse_res_final_kernel(const double* __restrict__ part, int nb,
                                                                const double* __restrict__ gram, int r,  // 0: no B
                                                                const float* __restrict__ s, double* out) {
  __shared__ double sa[kSpT], sc[kSpT], sg[kSpT];
  double x = 0.0, y = 0.0, z = 0.0;
  for (int b = threadIdx.x; b < nb; b += kSpT) { x += part[2 * b]; y += part[2 * b + 1]; }
  const double* GU = gram;
  const double* GV = gram + static_cast<int64_t>(r) * r;
  for (int64_t e = threadIdx.x; e < static_cast<int64_t>(r) * r; e += kSpT) {
    const int k = static_cast<int>(e / r), l = static_cast<int>(e % r);
    const double sk = s ? static_cast<double>(s[k]) : 1.0, sl = s ? static_cast<double>(s[l]) : 1.0;
    z = fma(GU[e] * sk * sl, GV[e], z);
  }
  sa[threadIdx.x] = x;
  sc[threadIdx.x] = y;
  sg[threadIdx.x] = z;
  __syncthreads();
  for (int w = kSpT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      sa[threadIdx.x] += sa[threadIdx.x + w];
      sc[threadIdx.x] += sc[threadIdx.x + w];
      sg[threadIdx.x] += sg[threadIdx.x + w];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = sa[0] - 2.0 * sc[0] + sg[0];
    out[1] = sa[0];
  }
}

bool sparse_residual_supported(int ncomp) { return ncomp >= 0 && ncomp <= kSpResMaxK; }

void launch_residual_sparse(const CsrSrc& a, int64_t m_loc, int64_t n, const float* F, int64_t ldf, const float* s,
                            const float* G, int64_t ldg, int ncomp, OrthArgs& ga, double* part, double* out,
                            cudaStream_t st) {
  // many rows in flight: each warp's step is two dependent L2 round trips (index, then G row)
  int64_t nb = ceil_div(m_loc > 0 ? m_loc : 1, 16);
  if (nb > kResGrid) nb = kResGrid;
  note_launch();
  sparse_res_nnz_kernel<<<static_cast<unsigned>(nb), kSpT, 0, st>>>(a, m_loc, F, ldf, s, G, ldg, ncomp, part);
  // F^T F over the rank's rows, G^T G over all n rows (FP64 products of FP32 entries: exact)
  ga.U = F; ga.ldu = ldf; ga.nu = m_loc;
  ga.V = G; ga.ldv = ldg; ga.nv = n;
  ga.r = ncomp > 0 ? ncomp : 1;
  ga.s = nullptr;
  ga.nblk = orth_gram_blocks(m_loc, n, ga.r);
  launch_orth_gram(ga, st);
  note_launch();
  sparse_res_final_kernel<<<1, kSpT, 0, st>>>(part, static_cast<int>(nb), ga.gram, ncomp, s, out);
  (void)n;
}

}  // namespace cabsk
