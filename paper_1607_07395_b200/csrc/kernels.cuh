// kernels.cuh -- host launchers of libcabs kernels (internal; the public ABI is include/cabs.h).
#pragma once
#include "common.cuh"

namespace cabsk {

// host-side count of kernel launches issued by this library (cabs_launch_count)
void note_launch();

// sample_gather.cu
int launch_floyd2(int64_t N0, int32_t k0, uint32_t tag0, int64_t* out0, int64_t N1, int32_t k1, uint32_t tag1,
                  int64_t* out1, uint64_t seed, cudaStream_t st);
void launch_philox_blocks(uint64_t seed, uint32_t tag, uint64_t start, int64_t count, uint32_t* out, cudaStream_t st);
void launch_validate_idx(const int64_t* idx, int32_t k, int64_t N, void* ws, cudaStream_t st);
void launch_validate_idx2(const int64_t* idx0, int64_t N0, const int64_t* idx1, int64_t N1, int32_t k, void* ws,
                          cudaStream_t st);
void launch_fill_neg_zero(float* p, int64_t n, cudaStream_t st);
void launch_gather_rows(const float* A, int64_t lda, int64_t row_begin, int64_t row_end, const int64_t* I, int32_t k,
                        int64_t n, float* R, int64_t ldr, void* ws, cudaStream_t st);
void launch_gather_cols(const float* A, int64_t lda, int64_t m_loc, int64_t n, const int64_t* J, int32_t k, float* C, int64_t ldc,
                        void* ws, cudaStream_t st);
void launch_gather_w(const float* R, int64_t ldr, int64_t n, const int64_t* J, int32_t k, float* W, int64_t ldw, cudaStream_t st);
void launch_gather_w_direct(const float* A, int64_t lda, int64_t row_begin, int64_t m_loc, int64_t n,
                            const int64_t* I, const int64_t* J, int32_t k, float* W, int64_t ldw, cudaStream_t st);
// the same gathers from a column-major block At = A^T (n x m_loc, ldt): cabs_source.transposed
void launch_gather_cols_t(const float* At, int64_t ldt, int64_t m_loc, int64_t n, const int64_t* J, int32_t k,
                          float* C, int64_t ldc, void* ws, cudaStream_t st);
void launch_gather_rows_t(const float* At, int64_t ldt, int64_t row_begin, int64_t row_end, const int64_t* I,
                          int32_t k, int64_t n, float* R, int64_t ldr, void* ws, cudaStream_t st);
void launch_gather_w_t(const float* At, int64_t ldt, int64_t row_begin, int64_t m_loc, int64_t n, const int64_t* I,
                       const int64_t* J, int32_t k, float* W, int64_t ldw, cudaStream_t st);

// svd.cu
int launch_svd(int k, const float* W, int64_t ldw, double tol, void* ws, const Ws& L, double* sigma_user, double* Uw64,
               double* Vw64, int* r_user, cudaStream_t st);

// svd_cluster.cu: k in (1, 320] on a cluster of ceil(k / 32) CTAs (false: not launched)
// QR-preconditioner buffers in the workspace (svd.cu fills them from the layout): Xt (K x K),
// Hv (K x K + K), Rg (K x K), piv (K), extra = the grid kernel's scratch (k > 128)
struct SvdQrBufs {
  double* Xt;
  double* Hv;
  double* Rg;
  int* piv;
  double* extra;
  int64_t K;
};
bool launch_svd_cluster(int k, const float* W, int64_t ldw, double tol, double* sig, double* Uw64, double* Vw64,
                        float* uw32, float* vw32, int64_t ld32, int* r_ws, int* r_user, void* ws, cudaStream_t st,
                        const struct SvdQrBufs* qb = nullptr);

// embed.cu
int launch_embed_products(int64_t m_loc, int64_t n_sl, int k, const float* C, int64_t ldc, const float* R_slice,
                          int64_t ldr, float* Yc, int64_t ldyc, float* Yr, int64_t ldyr, void* ws, const Ws& L,
                          cudaStream_t st,
                          cudaStream_t st2 = nullptr);
int launch_embed_finalize(int k, int mode, double m, double n, double ksamp, int kind, float* s_out, int* r_user,
                          void* ws, const Ws& L, cudaStream_t st);
int launch_scale_compact(float* Y, int64_t ldy, int64_t N, int k, int which, void* ws, const Ws& L, cudaStream_t st);
bool launch_embed_fused(int64_t m_loc, int64_t n_sl, int k, const float* C, int64_t ldc, const float* R_slice,
                        int64_t ldr, float* Y1, int64_t ld1, float* Y2, int64_t ld2, int mode, double m, double n,
                        double ksamp, int kind, float* s_out, int* r_user, void* ws, const Ws& L, cudaStream_t st);

// kmeans.cu
struct KmWeightJob {
  const float* X;
  int64_t ldx, N;
  int d;
  float* w;
  int* cnt;
  unsigned* bounds;
};
struct KmInitJob {
  const float* X;
  int64_t ldx, n_loc, row_off;
  int d, k2;
  const int64_t* idx;
  const float* init_c;
  int64_t ldic;
  float* centres;
  int64_t ldc;
};
void launch_km_weights2(const KmWeightJob& j0, const KmWeightJob* j1, int kind, float p, cudaStream_t st);
void launch_km_init2(const KmInitJob& j0, const KmInitJob* j1, cudaStream_t st);
void launch_km_weights(const float* X, int64_t ldx, int64_t N, int d, int kind, float p, float* w, int* cnt,
                       unsigned* bounds, cudaStream_t st);
void launch_km_init(const float* X, int64_t ldx, int64_t n_loc, int64_t row_off, int d, int k2, const int64_t* idx,
                    const float* init_c, int64_t ldic, float* centres, int64_t ldc, cudaStream_t st);
void launch_km_assign(const float* X, int64_t ldx, int64_t N, int d, const float* centres, int64_t ldc, int k2,
                      const float* w, int* labels, double* pobj, int* ptie, int* grid_out, cudaStream_t st,
                      int* tie_log = nullptr, int tie_cap = 0, int it = 0, int64_t row_off = 0);
void launch_km_distmat(const float* X, int64_t ldx, int64_t N, int d, const float* centres, int64_t ldc, int k2,
                       float* D, int64_t ldd, cudaStream_t st);
void launch_km_accum(const float* X, int64_t ldx, int64_t N, int d, const int* labels, const float* w,
                     const unsigned* bounds, long long* fsum, long long* fw, cudaStream_t st);
void launch_km_reduce(long long* fsum, long long* fw, const unsigned* bounds, int64_t N, int k2, int d,
                      const double* pobj, const int* ptie, int Gobj, double* red, cudaStream_t st);
void launch_km_finalize(const double* red, int k2, int d, float* centres, int64_t ldc, double* objective,
                        int* near_ties, double* cluster_w, int t, cudaStream_t st);

// lloyd.cu (single-GPU persistent Lloyd loop of one or two problems; false -> use the
// per-iteration kernels)
struct LloydJob {
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
  void* scratch;
  size_t scratch_bytes;
  int* tie_log;      // near-tie log or null (km_tile.cuh: km_log_tie)
  int tie_cap;
  int64_t row_off;   // global index of local point 0
  float* ebuf;       // lloyd_prune: per-point per-centre bound buffer (N x round_up(k2, 4)) or null
  size_t ebuf_bytes;
  long long* qbuf;   // lloyd_prune: N int64 (w ||x||^2 in fixed point) or null
};
bool launch_lloyd_persistent(const LloydJob* jobs, int njobs, int iters, long long* prof, cudaStream_t st);
// lloyd_tc.cu: the same loop with the distance cross-term on the tensor cores (d, k2 <= 128);
// the jobs' near-tie logs as km_log_tie.  False -> not applicable.
void ktc_debug_timeline(long long* out, int n);
bool launch_lloyd_tc(const LloydJob* jobs, int njobs, int iters, cudaStream_t st);
// lloyd_ex.cu: the same loop with the candidates pruned exactly by the triangle inequality
// against the centre-centre distances (d, k2 <= 128, shared-memory plan permitting)
bool kmeans_prune_selected(int k2, int d);
bool launch_lloyd_prune(const LloydJob* jobs, int njobs, int iters, cudaStream_t st);
void lex_debug_timeline(long long* out, int n);
void lloyd_debug_timeline(long long* out, int n);
void embed_debug_timeline(long long* out);
void snap_debug_counters(long long* out);

// select.cu
void launch_snap_topT(const float* D, int64_t ldd, int64_t N, int k2, int64_t row_off, int T, int nseg, int slot0,
                      double* all, cudaStream_t st);
void launch_snap_merge(const double* all, int k2, int T, int nlists, float* cand_d, int64_t* cand_i, cudaStream_t st);
void launch_snap_dedupe(const float* cand_d, const int64_t* cand_i, int k2, int T, const double* cluster_w,
                        const float* D, int64_t ldd, int64_t N, int64_t row_off, bool can_rescan,
                        int64_t* rep_of_centre, float* gap, int64_t* reps_sorted, void* ws, cudaStream_t st,
                        int* unresolved = nullptr);
// multi-rank exact greedy pass (select.cu): scratch of snap_dist_bytes at buf; allreduce(buf, n, ctx)
// sums n doubles over the ranks on st
size_t snap_dist_bytes(int k2, int nranks);
int snap_dist_run(const float* D, int64_t ldd, int64_t N, int64_t row_off, int k2, const double* cluster_w,
                  int rank, int nranks, void* buf, int64_t* rep_of_centre, float* gap, int64_t* reps_sorted,
                  void* ws, cudaStream_t st, int (*allreduce)(double*, int64_t, void*), void* ctx);

// hard.cu -- one side (rows or columns) of the hard-threshold selection; up to two per launch
struct HardSide {
  const float* X;      // keys kernel: N x d embedding (ldx)
  int64_t ldx, N;      // N: points (keys kernel) / candidates (top-k kernel)
  int d;
  double* key;         // keys kernel output; top-k input key[l * ks]
  int64_t ks;
  const double* cidx;  // top-k: candidate indices at cidx[l * ks], or NULL (index = off + l)
  int64_t off;
  int64_t* out;        // top-k: winners ascending (or NULL)
  double* slot;        // top-k: (key, index) pairs of the winners, (-1, -1) padding (or NULL)
  int k;               // top-k: winners wanted (min(k, N) taken)
  int mode;            // local kernel: 0 = key ||X_l||^2 (variant (f)); 1 = leverage ES key
  uint64_t seed;       // mode 1: Philox seed / tag of the per-point uniforms
  uint32_t tag;
};
struct HardArgs {
  HardSide s[2];
  int nb0;  // local kernel: blocks of side 0 (set by the launcher)
};
int64_t hard_local_blocks(int64_t N);
void launch_hard_local(const HardArgs& a, int nside, double* cand, int64_t side_stride, void* ws, cudaStream_t st);
void launch_hard_topk(const HardArgs& a, int nside, cudaStream_t st);

// orth.cu -- orthogonalization of a sketch (Supp. 3), r <= kmax
struct OrthArgs {
  const float* U;  // nu x r (ldu), this rank's rows
  int64_t ldu, nu;
  const float* V;  // nv x r (ldv), this rank's column slice
  int64_t ldv, nv;
  int r;
  const float* s;  // float[r] or NULL (ones)
  double* part;    // [2][nblk][tile pairs][64*64] Gram partials
  int nblk;
  double* gram;    // [2][r*r]: G_U, G_V -> R_U, R_V (ld r)
  float* K;        // r x kp core (FP32, input of the Jacobi SVD)
  int64_t kp;
  double* UK;      // r x r (ld r), from the SVD; T_U in place
  double* VK;
  double* sig;     // SVD singular values
  int* r_svd;      // SVD rank
  float* TU;       // r x kp
  float* TV;
  float* s_out;    // float[r]
  int* r_out;      // or NULL
  float* Uo;
  int64_t lduo;
  float* Vo;
  int64_t ldvo;
};
int orth_gram_blocks(int64_t nu, int64_t nv, int r);
void launch_orth_gram(OrthArgs& a, cudaStream_t st);
void launch_orth_core(const OrthArgs& a, void* ws, cudaStream_t st);
void launch_orth_finish(const OrthArgs& a, cudaStream_t st);
void launch_orth_apply_u(const OrthArgs& a, cudaStream_t st);

// cur.cu -- BR-CUR / Sketch-CUR middle matrix and the validation rank sweep
void launch_pick_cols(const float* src, int64_t lds, int nr, const int64_t* cols, int nc, int pad, float* out,
                      int64_t ldo, double* out64, cudaStream_t st);
void launch_pick_rows(const float* X, int64_t ldx, const int64_t* rows, int nr, int ncol, int pad, float* out,
                      int64_t ldo, double* out64, cudaStream_t st);
void launch_transpose(const float* R, int64_t ldr, int k, int64_t n, float* G, int64_t ldg, cudaStream_t st);
void launch_zero_rows(float* X, int64_t ldx, int nr, int npad, int ncol, cudaStream_t st);
void launch_cur_middle(int k1, int k2, const double* U1, const double* V1, const double* sig1, const double* U2,
                       const double* V2, const double* sig2, double tol, const double* M, double* d1, double* d2,
                       double* X1, double* Y, double* X2, double* Ustar, cudaStream_t st);
void launch_f32_of(const double* X, int rows, int cols, float* Y, int64_t ldy, int pad, cudaStream_t st);
void launch_sweep(const double* B, int hr, int hc, const double* VH, const double* UH, const float* s,
                  const double* gram, int r, double* W1, double* err, cudaStream_t st);

// sparse.cu -- CSR / CSC source (cabs.h CABS_SOURCE_CSR_F32), this rank's row block
struct CsrSrc {
  const int64_t* row_ptr;  // m_loc + 1
  const int32_t* col_idx;
  const float* row_val;
  const int64_t* col_ptr;  // n + 1
  const int32_t* row_idx;  // local row indices
  const float* col_val;
};
void launch_csr_rows(const CsrSrc& a, int64_t row_begin, int64_t row_end, const int64_t* I, int k, int64_t n, float* R,
                     int64_t ldr, cudaStream_t st);
void launch_csc_cols(const CsrSrc& a, int64_t m_loc, int64_t n, const int64_t* J, int k, float* C, int64_t ldc,
                     cudaStream_t st);
void launch_csr_w(const CsrSrc& a, int64_t row_begin, int64_t row_end, const int64_t* I, const int64_t* J, int k,
                  float* W, int64_t ldw, cudaStream_t st);
bool sparse_residual_supported(int ncomp);
void launch_residual_sparse(const CsrSrc& a, int64_t m_loc, int64_t n, const float* F, int64_t ldf, const float* s,
                            const float* G, int64_t ldg, int ncomp, OrthArgs& ga, double* part, double* out,
                            cudaStream_t st);

// residual.cu
int launch_residual(const float* A, int64_t lda, int64_t m_loc, int64_t n, const float* F, int64_t ldf, const float* s,
                    const float* G, int64_t ldg, int ncomp, double* part, double* out, cudaStream_t st);

void launch_residual_final(const double* part, int G, double* out, cudaStream_t st);

// residual_tc.cu (tcgen05 3xTF32 path; ncomp <= 192)
void residual_debug_counters(long long* out, int n);
int residual_tc_kmax();
bool residual_tc_covers(int ncomp);
// lloyd_tc.cu: whether cabs_kmeans(_pair) takes the tensor-core distance path for (k2, d)
bool kmeans_tc_selected(int k2, int d);
bool residual_tc_supported(const float* A, int64_t lda, int64_t m_loc, int64_t n, int ncomp);
int launch_residual_tc(const float* A, int64_t lda, int64_t m_loc, int64_t n, const float* F, int64_t ldf,
                       const float* s, const float* G, int64_t ldg, int ncomp, float* split, double* part, double* out,
                       cudaStream_t st);

// rbf.cu: the implicit RBF source (reading Z23) and the sampled residual (Z17 / Z23)
struct RbfSrc {
  const float* x;  // m x ldx (all points)
  const float* y;  // n x ldy
  int64_t ldx, ldy;
  int d;
  float g;  // 1 / (2 sigma^2)
};
struct SampArgs {
  const float* A;  // dense source (rbf.x == nullptr): the rank's rows
  int64_t lda;
  int transposed;  // dense: A(i, j) at A + j*lda + (i - row_begin) (cabs_source.transposed)
  RbfSrc rbf;      // implicit source when rbf.x != nullptr
  uint64_t m, n, thr_m, thr_n;
  int64_t row_begin, row_end;
  const float* F;  // m_loc x ncomp (ldf)
  int64_t ldf;
  const float* s;  // ncomp or null
  const float* G;  // n x ncomp (ldg)
  int64_t ldg;
  int ncomp;
  int64_t T;
  uint64_t seed;
};
void launch_rbf_rows(const RbfSrc& s, const int64_t* I, int k, int64_t n, float* R, int64_t ldr, cudaStream_t st);
void launch_rbf_cols(const RbfSrc& s, int64_t row_begin, int64_t m_loc, const int64_t* J, int k, float* C,
                     int64_t ldc, cudaStream_t st);
void launch_rbf_w(const RbfSrc& s, const int64_t* I, const int64_t* J, int k, float* W, int64_t ldw,
                  cudaStream_t st);
void launch_residual_pairs(uint64_t seed, uint64_t t0, int64_t T, int64_t m, int64_t n, int64_t* oi, int64_t* oj,
                           cudaStream_t st);
void launch_residual_sampled(const SampArgs& a, double* part, double* out, cudaStream_t st);
int residual_sampled_part_doubles();

}  // namespace cabsk
