/*
 * cabs.h -- C ABI of libcabs.so, the B200 (sm_100a) hot path of Cascaded
 * Bilateral Sampling (CABS, arXiv 1607.07395).
 *
 * Citation keys: P:n = PAPER.md line n (the paper), S:n = SPEC.md line n.
 *
 * The method (Algorithm 2):
 *   1. pilot sampling  : k1 uniform rows I and columns J; C = A(:,J), R = A(I,:),
 *                        W = A(I,J)
 *   2. pilot sketching : [U,S,V] = sketching(C,R,W); P = U S^1/2, Q = V S^1/2
 *   3. follow-up       : weighted k-means on P and on Q, each centre snapped to
 *                        its closest in-sample point -> Ibar, Jbar
 *   4. follow-up sketch: [Ubar,Sbar,Vbar] = sketching(Cbar,Rbar,Wbar)
 *   5. evaluation      : ||A - Ubar Sbar Vbar^T||_F
 * The `sketching` routine is the paper's stabilized variant of the pseudo-skeleton
 * (P:222-232); the plain pseudo-skeleton A ~ C W^+ R (Eq. 2) is a mode.
 *
 * Conventions (all entry points)
 * ------------------------------
 * - Memory: every pointer argument is DEVICE memory allocated by the caller,
 *   unless the parameter comment says "host".  The library never allocates
 *   device memory; it uses the caller's workspace `ws` of at least
 *   cabs_workspace_bytes(plan) bytes (256-byte aligned).
 * - Layout: dense matrices are row-major float32 with an explicit leading
 *   dimension (elements).  Index arrays are int64, sorted ascending on output.
 *   Factor buffers (C, P, Q, U, V, F, G, centres) must have ld >= k; columns
 *   [r, ld) are written as zeros, so ld = cabs_padded_ld(k) is recommended.
 * - Execution: asynchronous, stream-ordered on `stream` (a cudaStream_t; NULL =
 *   legacy default stream).  No host synchronisation inside the hot path except
 *   where a comment says so.  Reentrant across distinct (workspace, stream) pairs.
 * - Errors: argument checks are synchronous and return a cabs_status.  Data-
 *   dependent errors (non-finite input S:21/S:71, out-of-range or duplicate
 *   supplied index S:62/S:66, snap exhaustion) set bits of a device status word
 *   in `ws`, read with cabs_device_status().  A rank-0 sketch is not an error
 *   (S:245): it yields r = 0.  No C++ exception crosses this ABI.
 * - Multi-GPU: one process per GPU; A is split into contiguous row blocks and the
 *   column-side embedding into contiguous column slices (cabs_plan).  Collectives
 *   are delegated to the caller through cabs_comm (sum-allreduce callbacks,
 *   stream-ordered).  comm == NULL or nranks == 1 means single GPU.
 */
#ifndef CABS_H_
#define CABS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CABS_VERSION_MAJOR 0
#define CABS_VERSION_MINOR 1
#define CABS_KMAX 1024 /* largest supported k1, k2 */

typedef enum {
  CABS_OK = 0,
  CABS_ERR_INVALID_ARG = 1, /* k < 1, k > min(m,n), iters < 1, bad mode/ld */
  CABS_ERR_RANGE = 2,       /* supplied index out of range / duplicated */
  CABS_ERR_DEGENERATE = 3,  /* ||A||_F = 0 where a relative error is asked */
  CABS_ERR_CUDA = 4,        /* CUDA runtime failure; see cabs_last_error_string() */
  CABS_ERR_COMM = 5,        /* a cabs_comm callback returned nonzero */
  CABS_ERR_WORKSPACE = 6    /* ws NULL or smaller than cabs_workspace_bytes() */
} cabs_status;

/* Device status word bits (cabs_device_status). */
#define CABS_DEV_NONFINITE 0x1u      /* a gathered entry of A was NaN/Inf */
#define CABS_DEV_RANGE 0x2u          /* supplied index out of range */
#define CABS_DEV_DUPLICATE 0x4u      /* supplied indices not distinct */
#define CABS_DEV_SNAP_EXHAUSTED 0x8u /* multi-GPU snap ran out of candidates */
#define CABS_DEV_TOO_FEW_POINTS 0x10u /* fewer than k2 points with nonzero weight */
#define CABS_DEV_SVD_NOCONV 0x20u    /* Jacobi SVD hit its sweep cap */
#define CABS_DEV_ORTH_RANK 0x40u     /* cabs_orthogonalize: a factor is rank-deficient (Cholesky pivot <= 0) */

typedef enum {
  CABS_STABILIZED = 0,     /* the paper's routine: U = C V_w N_c^-1, V = R^T U_w N_r^-1,
                              S = Sigma_w sqrt(mn)/k */
  CABS_PSEUDO_SKELETON = 1 /* Eq. 2: same factors, S = N_c N_r Sigma_w^-1 so that
                              U S V^T = C W_r^+ R exactly */
} cabs_mode;

typedef enum {
  CABS_WEIGHT_CONST = 0, /* Upsilon = 1 (dense matrices) */
  CABS_WEIGHT_POWER = 1  /* Upsilon(x) = x^p (Eq. 6) */
} cabs_weight_kind;

/* Partition of the global m x n problem for this rank (host struct). */
typedef struct cabs_plan {
  int64_t m, n;                 /* global matrix dims */
  int64_t row_begin, row_end;   /* rows of A held by this rank (P rows follow them) */
  int64_t col_begin, col_end;   /* columns whose embedding rows (Q, V) this rank owns */
  int32_t kmax;                 /* max(k1, k2) used with this workspace, <= CABS_KMAX */
  int32_t rank, nranks;
} cabs_plan;

/* Source of the matrix A (host struct).  A zero-initialised struct with a / lda set is dense.
 *
 * CABS_SOURCE_DENSE_F32: row i of the rank's block is at a + (i - row_begin)*lda (device,
 *   (row_end - row_begin) x n, row-major, lda >= n).  With transposed = 1 the same
 *   block is held column-major instead: A(i, j) is at a + j*lda + (i - row_begin), i.e. `a` is
 *   the n x (row_end - row_begin) row-major array A^T, lda >= row_end - row_begin.  Every entry
 *   point computes exactly what it computes for the row-major copy (same I, J, C, R, W, P, Q,
 *   representatives, U, s, V -- the gathers are exact copies, so everything downstream of them
 *   is bit-identical; only the residual's summation order differs): the column gather becomes
 *   contiguous reads and the row gather the one-element-per-sector one, k (n + m/8) sectors
 *   instead of k (m + n/8), fewer whenever m > n.  The residual runs the same kernels on A^T
 *   with F and G exchanged (||A - F S G^T||_F = ||A^T - G S F^T||_F).
 * CABS_SOURCE_RBF_F32: the implicit matrix of BASELINE.json configs[4] (reading Z23),
 *   A_ij = exp(-|x_i - y_j|^2 * inv_two_sigma2), generated on access in FP32 (direct
 *   differences summed over the d coordinates in order, exp via ex2.approx) -- PAPER.md P:24
 *   "never knowing the remaining entries".  x: device, ALL m points (m x ldx, replicated on
 *   every rank); y: device, all n points (n x ldy); 1 <= d <= 64; inv_two_sigma2 = 1/(2 sigma^2) > 0.
 *   No gather crosses ranks; cabs_residual needs n_samples > 0 for this kind.
 * CABS_SOURCE_CSR_F32: a sparse A ("For sparse matrices", Table 1
 *   P:301-302): the rank's row block in CSR (row gathers, W) and in CSC (column gathers), both
 *   supplied by the caller (the library does not convert).  Entries not stored are 0; gathers
 *   are exact copies, identical to the dense gathers of the densified matrix.  Rows sampled on
 *   other ranks arrive through the allreduce, as for a dense source.  cabs_residual (exact)
 *   evaluates ||A||^2 - 2 sum_nnz a_ij (F S G^T)_ij + sum_kl (F^T F)_kl s_k s_l (G^T G)_kl
 *   (ncomp <= 512) without forming A - F S G^T; no index or value checks beyond the dims. */
#define CABS_SOURCE_DENSE_F32 0
#define CABS_SOURCE_RBF_F32 1
#define CABS_SOURCE_CSR_F32 2
typedef struct cabs_source {
  const float* a;         /* dense: device, (row_end - row_begin) x n, row-major */
  int64_t lda;            /* dense: >= n */
  int32_t kind;           /* CABS_SOURCE_* */
  int32_t d;              /* RBF: point dimension */
  const float* x;         /* RBF: m x ldx */
  const float* y;         /* RBF: n x ldy */
  int64_t ldx, ldy;       /* RBF: >= d */
  float inv_two_sigma2;   /* RBF */
  /* CSR: the rank's row block twice, device arrays (row indices local to the block) */
  const int64_t* row_ptr; /* CSR: int64[m_loc + 1], row_ptr[0] = 0 */
  const int32_t* col_idx; /* CSR: int32[nnz], strictly increasing within a row */
  const float* row_val;   /* CSR: float[nnz] */
  const int64_t* col_ptr; /* CSC of the same block: int64[n + 1] */
  const int32_t* row_idx; /* CSC: int32[nnz], local rows, strictly increasing within a column */
  const float* col_val;   /* CSC: float[nnz] */
  int32_t transposed;     /* dense only: 0 = row-major block, 1 = column-major block (see above);
                             any other value, or 1 with another kind -> INVALID_ARG */
  int32_t host_resident;  /* dense only: 1 = `a` is pinned host memory mapped into the device address
                             space (cudaHostAlloc / cudaHostRegister; same address under UVA) instead of
                             device memory: nothing is copied, the gathers read exactly the sampled rows
                             and columns over the interconnect ("never knowing the remaining
                             entries", P:29 matrices that do not fit in memory), results bit-identical
                             to the device-resident block; the exact residual then reads all of A over
                             the interconnect with plain loads (no TMA) -- use n_samples > 0 instead.
                             Any value but 0 / 1, or 1 with another kind -> INVALID_ARG */
  const float* at;        /* dense only, optional (NULL = absent): the SAME block held column-major as
                             well, A(i, j) at at + j*ldat + (i - row_begin) (the n x m_loc row-major
                             array A^T, as for transposed = 1; same memory space as `a`).  When given,
                             the column gathers read `at` and the row gathers read `a`, so both are
                             contiguous copies: 4 k (m + n) bytes per gather pair instead of one 32-byte
                             sector per element (the sparse kind's CSR + CSC pair is the same
                             idea).  The two copies must hold the same values (not checked); results
                             are then bit-identical to the single-layout run.  Requires transposed = 0
                             and ldat >= row_end - row_begin, else INVALID_ARG */
  int64_t ldat;
} cabs_source;

/* Collectives supplied by the caller (host struct).  Each callback sums `count`
 * elements of the device buffer `buf` in place across all ranks, ordered on
 * `stream`, and returns 0 on success. */
typedef struct cabs_comm {
  int32_t rank, nranks;
  int32_t (*allreduce_f64)(double* buf, int64_t count, void* ctx, void* stream);
  int32_t (*allreduce_f32)(float* buf, int64_t count, void* ctx, void* stream);
  void* ctx;
} cabs_comm;

/* ---------------------------------------------------------------- utilities */
const char* cabs_status_string(int32_t status);
const char* cabs_last_error_string(void);
void cabs_version(int32_t* major, int32_t* minor);
/* Recommended leading dimension for k-column factor buffers: k rounded up to 32. */
int64_t cabs_padded_ld(int32_t k);
/* Workspace bytes needed by every entry point for this plan. */
size_t cabs_workspace_bytes(const cabs_plan* plan);
/* Zero the device status word (stream-ordered). */
int32_t cabs_clear_status(void* ws, void* stream);
/* Number of kernel launches this library has issued in this process (host-side counter;
 * benchmarks report the delta over a timed region as their launch count). */
int64_t cabs_launch_count(void);
/* Which kernel family an entry point dispatches to for these sizes (host query, no launch):
 * op CABS_OP_KMEANS (k = k2, d = embedding width): CABS_PATH_PRUNE (persistent Lloyd kernel
 * whose candidates are pruned exactly by the triangle inequality against the centre-centre
 * distances, then FP32 direct differences), CABS_PATH_FFMA (FP32 direct differences against
 * every centre) or CABS_PATH_TC (tcgen05 FP16-split cross-term + FP32 refine); all three take
 * bit-identical decisions;
 * op CABS_OP_RESIDUAL (k = ncomp, d ignored): CABS_PATH_FFMA or CABS_PATH_TC.  Returns -1 for
 * an unknown op.  Benchmarks use it to label the roofline of the kernel that actually ran. */
#define CABS_OP_KMEANS 0
#define CABS_OP_RESIDUAL 1
#define CABS_PATH_FFMA 0
#define CABS_PATH_TC 1
#define CABS_PATH_PRUNE 2
int32_t cabs_kernel_path(int32_t op, int32_t k, int32_t d);
/* Synchronises `stream`, then copies the device status word to host *flags. */
int32_t cabs_device_status(const void* ws, void* stream, uint32_t* flags);

/* ---------------------------------------------------------------- S1-S3 pilot
 * Algorithm 2 step 1: I = Floyd(m, k, seed, tag 1), J = Floyd(n, k, seed,
 * tag 2) with the Philox4x32-10 / Lemire / Floyd generator of DESIGN.md "RNG";
 * both sorted ascending.  C = A(:,J) for this rank's rows (m_loc x k, ldc);
 * R = A(I,:) as k x n (ldr >= n), complete on every rank after the comm step;
 * W = A(I,J) (k x k, ldw >= k).  Gathers are bit-exact copies.
 * I, J: device int64[k].  Errors: k < 1 or k > min(m, n) -> INVALID_ARG. */
int32_t cabs_pilot(const cabs_plan* plan, const cabs_source* src, int32_t k, uint64_t seed,
                   int64_t* I, int64_t* J, float* C, int64_t ldc, float* R, int64_t ldr,
                   float* W, int64_t ldw, void* ws, size_t ws_bytes, const cabs_comm* comm,
                   void* stream);

/* ---------------------------------------------------------------- S4-S5 embed
 * Algorithm 2 step 2 using the sketching routine:
 * W = U_w Sigma_w V_w^T (FP64 one-sided Jacobi; sigma descending; truncated to
 * sigma_i > tol*sigma_1; canonical signs: largest-|.| entry of each U_w column
 * positive), Y_c = C V_w, Y_r = R^T U_w, N_c/N_r their column norms, components
 * with zero norm dropped; s_i = sigma_i sqrt(mn)/k (STABILIZED) or
 * N_c,i N_r,i / sigma_i (PSEUDO_SKELETON); P = Y_c diag(sqrt(s)/N_c) (m_loc x k,
 * ldp), Q = Y_r diag(sqrt(s)/N_r) for columns [col_begin, col_end) (ldq).
 * Outputs: s (float[k], zeros past r), r (device int32), sigma (optional, device
 * double[k], singular values of W before truncation, NULL to skip).
 * k = number of sampled rows = sampled columns (Z3). */
int32_t cabs_embed(const cabs_plan* plan, int32_t k, const float* C, int64_t ldc,
                   const float* R, int64_t ldr, const float* W, int64_t ldw, int32_t mode,
                   double tol, float* P, int64_t ldp, float* Q, int64_t ldq, float* s,
                   int32_t* r, double* sigma, void* ws, size_t ws_bytes,
                   const cabs_comm* comm, void* stream);

/* S1-S5 in one call: exactly cabs_pilot followed by cabs_embed on its outputs (same
 * arguments, same results).  On one GPU the SVD of W = A(I,J) (gathered first, straight
 * from A) runs on the library's side stream while C and R are gathered on `stream`, so the
 * two 2-SM and HBM-bound steps overlap; with a communicator it is the two calls in order. */
int32_t cabs_pilot_embed(const cabs_plan* plan, const cabs_source* src, int32_t k, uint64_t seed,
                         int64_t* I, int64_t* J, float* C, int64_t ldc, float* R, int64_t ldr,
                         float* W, int64_t ldw, int32_t mode, double tol, float* P, int64_t ldp,
                         float* Q, int64_t ldq, float* s, int32_t* r, double* sigma, void* ws,
                         size_t ws_bytes, const cabs_comm* comm, void* stream);

/* ---------------------------------------------------------------- S6-S7 k-means
 * Weighted Lloyd k-means (Eq. 6; c iterations) on the rows of
 * X (n_loc local rows of n_glob, global index = row_off + local, d columns, ldx).
 * Weights w_l = Upsilon(||X_l||) (weight_kind, weight_p).  Init: centres =
 * X[init_idx] if init_idx != NULL (device int64[k2], global indices), else
 * init_centres (device k2 x ldc) if != NULL, else X[Floyd(n_glob, k2, seed, tag)].
 * Each iteration t: s(l) = argmin_j ||X_l - c_j||^2 (direct differences, FP32,
 * lowest j on ties), objective[t] = sum_l w_l min_j d (FP64); every cluster with
 * positive weight moves to its weighted mean, an empty one keeps its centre.
 * Outputs: centres (k2 x ldc, after the last update), labels (int32[n_loc], last
 * assignment), cluster_w (double[k2], weights of the last assignment),
 * objective (double[iters]), near_ties (int32[iters] or NULL: points whose
 * FP32 relative gap (d2-d1)/d2 < 1e-5, north_star near-tie rule), tie_log (int32[1 + 5
 * tie_log_cap] or NULL: the near-tie log the north_star asks for -- tie_log[0] = number of
 * near ties seen (all iterations, this rank's points), then per entry (iteration, global point
 * index, nearest centre, runner-up centre, relative gap as FP32 bits); entries beyond
 * tie_log_cap are counted but not stored; order of entries unspecified). */
int32_t cabs_kmeans(const cabs_plan* plan, const float* X, int64_t ldx, int64_t n_loc,
                    int64_t n_glob, int64_t row_off, int32_t d, int32_t k2, int32_t iters,
                    int32_t weight_kind, float weight_p, uint64_t seed, int32_t tag,
                    const int64_t* init_idx, const float* init_centres, float* centres,
                    int64_t ldc, int32_t* labels, double* cluster_w, double* objective,
                    int32_t* near_ties, int32_t* tie_log, int32_t tie_log_cap, void* ws,
                    size_t ws_bytes, const cabs_comm* comm, void* stream);

/* One k-means problem of cabs_kmeans_pair: the arguments of cabs_kmeans that differ
 * between the row side (X = P, rows of A) and the column side (X = Q, columns of A). */
typedef struct cabs_km_problem {
  const float* X;               /* device n_loc x ldx */
  int64_t ldx, n_loc, n_glob, row_off;
  int32_t d, k2, tag;           /* tag: Philox stream of the Floyd initialisation */
  const int64_t* init_idx;      /* device int64[k2] or NULL */
  const float* init_centres;    /* device k2 x ldc or NULL */
  float* centres;               /* device k2 x ldc (out) */
  int64_t ldc;
  int32_t* labels;              /* device int32[n_loc] (out) */
  double* cluster_w;            /* device double[k2] (out) */
  double* objective;            /* device double[iters] (out) */
  int32_t* near_ties;           /* device int32[iters] (out) or NULL */
  int32_t* tie_log;             /* device int32[1 + 5 tie_log_cap] (out) or NULL: see cabs_kmeans */
  int32_t tie_log_cap;
} cabs_km_problem;

/* Alg. 2 steps 6-7 for BOTH sides at once: exactly cabs_kmeans(a) and cabs_kmeans(b) with
 * the shared iters / weight / seed arguments (same results, bit for bit: the sums are exact
 * integers), run by ONE persistent kernel on a single GPU whose grid barrier and cluster
 * reductions serve both problems each iteration.  Multi-rank (comm with nranks > 1) runs
 * the two problems one after the other.  Errors as cabs_kmeans; nothing is written when an
 * argument check fails. */
int32_t cabs_kmeans_pair(const cabs_plan* plan, const cabs_km_problem* a, const cabs_km_problem* b,
                         int32_t iters, int32_t weight_kind, float weight_p, uint64_t seed, void* ws,
                         size_t ws_bytes, const cabs_comm* comm, void* stream);

/* ---------------------------------------------------------------- S8 select
 * Snap ("any k-means clustering center will be replaced with its closest
 * in-sample point"): centres visited in order (-cluster_w[j], j), each taking its
 * nearest not-yet-taken point over all n_glob points (FP32 direct differences;
 * ties -> lowest index).  Outputs: reps (int64[k2], sorted ascending: the
 * follow-up index set), rep_of_centre (int64[k2] or NULL), gap (float[k2] or
 * NULL: relative gap between the best and runner-up untaken point). */
int32_t cabs_select(const cabs_plan* plan, const float* X, int64_t ldx, int64_t n_loc,
                    int64_t n_glob, int64_t row_off, int32_t d, const float* centres,
                    int64_t ldc, int32_t k2, const double* cluster_w, int64_t* reps,
                    int64_t* rep_of_centre, float* gap, void* ws, size_t ws_bytes,
                    const cabs_comm* comm, void* stream);

/* One snap problem of cabs_select_pair: the arguments of cabs_select. */
typedef struct cabs_sel_problem {
  const float* X;               /* device n_loc x ldx (the embedding the k-means ran on) */
  int64_t ldx, n_loc, n_glob, row_off;
  int32_t d;
  const float* centres;         /* device k2 x ldc */
  int64_t ldc;
  int32_t k2;
  const double* cluster_w;      /* device double[k2] */
  int64_t* reps;                /* device int64[k2] (out, ascending) */
  int64_t* rep_of_centre;       /* device int64[k2] (out) or NULL */
  float* gap;                   /* device float[k2] (out) or NULL */
} cabs_sel_problem;

/* Alg. 2 step 8 for BOTH sides: exactly cabs_select(a) and cabs_select(b) (same results),
 * on a single GPU run concurrently -- b on a library-owned side stream forked from and
 * joined back into `stream` -- with separate scratch.  Multi-rank runs them one after the
 * other on `stream`.  Errors as cabs_select. */
int32_t cabs_select_pair(const cabs_plan* plan, const cabs_sel_problem* a, const cabs_sel_problem* b,
                         void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream);

/* ---------------------------------------------------------------- S8' hard threshold
 * The paper's follow-up variant (f) ("top-k samples with largest weighting
 * coefficients (Equation eq:wkmeans)"), replacing S6-S8: the k2 points of
 * the embedding X (n_loc local rows of n_glob, global index = row_off + local, d columns,
 * ldx) with the largest Upsilon(||X_l||).  Upsilon is monotone, so the key is ||X_l||^2,
 * the FP64 sum of the exact squares of the FP32 entries in column order (Z26);
 * ties -> lowest global index.  Outputs: reps (device int64[k2], ascending: the follow-up
 * index set), keys (device double[n_loc] or NULL: the local keys).  Multi-rank: one
 * sum-allreduce of 2 * nranks * k2 doubles; every rank receives the same reps.
 * Errors: k2 < 1, k2 > kmax or k2 > n_glob, bad dims -> INVALID_ARG; a non-finite key sets
 * CABS_DEV_NONFINITE (NaN keys rank below every finite key). */
int32_t cabs_hard_select(const cabs_plan* plan, const float* X, int64_t ldx, int64_t n_loc,
                         int64_t n_glob, int64_t row_off, int32_t d, int32_t k2, int64_t* reps,
                         double* keys, void* ws, size_t ws_bytes, const cabs_comm* comm,
                         void* stream);

/* One side of cabs_hard_select_pair: the arguments of cabs_hard_select. */
typedef struct cabs_hard_problem {
  const float* X;               /* device n_loc x ldx */
  int64_t ldx, n_loc, n_glob, row_off;
  int32_t d, k2;
  int64_t* reps;                /* device int64[k2] (out, ascending) */
  double* keys;                 /* device double[n_loc] (out) or NULL */
} cabs_hard_problem;

/* Variant (f) for BOTH sides: exactly cabs_hard_select(a) and cabs_hard_select(b) (same
 * results); on a single GPU the two sides share one key launch and one top-k launch (one
 * CTA per side).  Multi-rank runs them one after the other.  Errors as cabs_hard_select. */
int32_t cabs_hard_select_pair(const cabs_plan* plan, const cabs_hard_problem* a,
                              const cabs_hard_problem* b, void* ws, size_t ws_bytes,
                              const cabs_comm* comm, void* stream);

/* ---------------------------------------------------------------- variant (e): leverage
 * Orthogonalization of a sketch (Supp. section 3): given A ~ U diag(s) V^T
 * (U: this rank's m_loc x r rows, ldu; V: this rank's column slice, n_sl x r, ldv; s:
 * device float[r] or NULL = ones), writes the thin SVD of that product, A ~ Uo diag(so)
 * Vo^T with orthonormal Uo, Vo (the paper's (U0 U1, S1, V1), unique up to signs; canonical
 * signs as Z5), so descending, components with so_j <= 1e-12 so_1 dropped (zero columns,
 * r_out = kept count).  Computed as Gram matrices (one allreduce of 2 r^2 doubles across
 * ranks), FP64 Cholesky, the FP64 Jacobi SVD of the r x r core, and one pass over U and V.
 * Errors: r < 1 or r > kmax, ld < r -> INVALID_ARG; all-zero columns (the zero
 * padding beyond a truncated rank) drop out; a numerically rank-deficient U or V (negative
 * Cholesky pivot) sets CABS_DEV_ORTH_RANK.  sigma: device double[r] or NULL.  Uo may not alias U. */
int32_t cabs_orthogonalize(const cabs_plan* plan, int32_t r, const float* U, int64_t ldu,
                           const float* s, const float* V, int64_t ldv, float* Uo, int64_t lduo,
                           float* so, float* Vo, int64_t ldvo, int32_t* r_out, double* sigma,
                           void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream);

/* ---------------------------------------------------------------- NEXT-4 baselines
 * BR-CUR, Algorithm 1, on the same gathers: C = A(:, Ibc) (m_loc x k1), R = A(Ibr, :)
 * (k1 x n), C_bar = A(Itr, Ibc), R_bar = A(Ibr, Itc), M = A(Itr, Itc), U* = C_bar^+ M R_bar^+
 * (step 4's minimum-norm least-squares solution; pseudo-inverses from the FP64 Jacobi SVD of the
 * zero-padded k2 x k2 matrices, singular values <= tol * sigma_1 dropped).  Outputs the
 * reconstruction A ~ F G^T as F = C U* (m_loc x k1, ldf) and G = R^T (n x k1, ldg), ready for
 * cabs_residual(F, NULL, G, k1); Umid (device double[k1 * k1] row-major, or NULL) = U*.
 * Sketch-CUR is this call with Itr, Itc drawn uniformly and independently of the base
 * (P:312 (a): three times as many; cabs_uniform_indices with tags 8 / 9).  Ibr, Ibc: k1 indices,
 * Itr, Itc: k2 indices (device int64; distinct, in range).  Single rank.  Errors: k1 < 1,
 * k2 < k1, k2 > min(m, n, kmax), ld < k1, nranks > 1 -> INVALID_ARG. */
int32_t cabs_br_cur(const cabs_plan* plan, const cabs_source* src, int32_t k1, const int64_t* Ibr,
                    const int64_t* Ibc, int32_t k2, const int64_t* Itr, const int64_t* Itc, double tol,
                    float* F, int64_t ldf, float* G, int64_t ldg, double* Umid, void* ws,
                    size_t ws_bytes, const cabs_comm* comm, void* stream);

/* The rank sweep on a validation block ("approximation error varies with the number
 * of singular vectors used", "use a validation set to choose the optimal number"):
 * errs[rho] = ||A(Hr, Hc) - U(Hr, :rho) diag(s[:rho]) V(Hc, :rho)^T||_F^2 for rho = 0..r (device
 * double[r + 1]), from the exact entries of the hr x hc block and the expansion through the r x r
 * Gram products (FP64).  U: m_loc x r (ldu), V: all n rows (ldv), s: device float[r]; Hr, Hc:
 * device int64 (the caller keeps them disjoint from the sketch's own indices).  The rank
 * chosen is the argmin over rho >= 1 (lowest on ties).  Single rank; 1 <= hr, hc, r <= kmax. */
int32_t cabs_holdout_errors(const cabs_plan* plan, const cabs_source* src, const int64_t* Hr,
                            int32_t hr, const int64_t* Hc, int32_t hc, const float* U, int64_t ldu,
                            const float* s, const float* V, int64_t ldv, int32_t r, double* errs,
                            void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream);

/* Leverage-score follow-up (P:312 variant (e); Z27): k2 distinct
 * points of the orthonormal factor F (n_loc local rows of n_glob, global index = row_off +
 * local, r columns, ldf) drawn without replacement with probability proportional to the
 * scores l = ||F_l||^2 / r: the k2 largest Efraimidis-Spirakis keys l / (-log u_l), u_l the
 * per-point Philox uniform of (seed, tag, global index); ties ->
 * lowest index; reps ascending; keys (double[n_loc] or NULL) receives the keys.  Errors and
 * multi-rank behaviour as cabs_hard_select. */
int32_t cabs_leverage_select(const cabs_plan* plan, const float* F, int64_t ldf, int64_t n_loc,
                             int64_t n_glob, int64_t row_off, int32_t r, int32_t k2, uint64_t seed,
                             uint32_t tag, int64_t* reps, double* keys, void* ws, size_t ws_bytes,
                             const cabs_comm* comm, void* stream);

/* Both sides at once (a: rows with tag_a, b: columns with tag_b; the d field of each
 * problem is its r): one key launch and one merge launch on a single GPU. */
int32_t cabs_leverage_select_pair(const cabs_plan* plan, const cabs_hard_problem* a,
                                  const cabs_hard_problem* b, uint64_t seed, uint32_t tag_a,
                                  uint32_t tag_b, void* ws, size_t ws_bytes, const cabs_comm* comm,
                                  void* stream);

/* ---------------------------------------------------------------- S9 sketch
 * Follow-up sketching, or a sketch from any given index sets:
 * gathers Cbar = A(:,Ic), Rbar = A(Ir,:), Wbar = A(Ir,Ic) (Ir, Ic: device int64[k],
 * distinct, in range; else status bits RANGE/DUPLICATE), then the sketching
 * routine as in cabs_embed with output U = Y_c N_c^-1 (m_loc x k, ldu),
 * V = Y_r N_r^-1 (columns [col_begin, col_end), ldv), s (float[k]), r (int32).
 * A ~ U diag(s) V^T. */
int32_t cabs_sketch(const cabs_plan* plan, const cabs_source* src, const int64_t* Ir,
                    const int64_t* Ic, int32_t k, int32_t mode, double tol, float* U,
                    int64_t ldu, float* s, float* V, int64_t ldv, int32_t* r, double* sigma,
                    void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream);

/* ---------------------------------------------------------------- S10 residual
 * Evaluation ("error ||A - A~||_F/||A||_F"): out[0] = sum_ij (A - F diag(s)
 * G^T)_ij^2 and out[1] = sum_ij A_ij^2 over the global matrix (FP64, reduced over
 * ranks).  F: this rank's m_loc x ncomp (ldf); G: all n rows x ncomp (ldg);
 * s: float[ncomp] or NULL (= ones).  The reconstruction is never materialised.
 * n_samples = 0: the exact sums over all entries (dense source only).  n_samples = T > 0: the
 * unbiased estimates (m n / T) sum_t (A_{i_t j_t} - F_{i_t} diag(s) G_{j_t}^T)^2 and
 * (m n / T) sum_t A_{i_t j_t}^2 over T i.i.d. uniform positions from the Philox stream of
 * `seed`, tag 5 (BASELINE.json configs[4] "residual estimated on a seeded 1e9-entry uniform
 * subset"; readings Z17 / Z23; cabs_residual_pairs returns the same positions); every rank
 * draws all T positions and adds the ones whose row it owns.
 * out: device double[2]. */
int32_t cabs_residual(const cabs_plan* plan, const cabs_source* src, const float* F,
                      int64_t ldf, const float* s, const float* G, int64_t ldg, int32_t ncomp,
                      int64_t n_samples, uint64_t seed, double* out, void* ws, size_t ws_bytes,
                      const cabs_comm* comm, void* stream);

/* ---------------------------------------------------------------- test hooks
 * Building blocks exposed for step-level parity tests (same kernels as above). */
/* Philox4x32-10 blocks: out[4*b + i] = Philox(ctr=(start+b lo, hi, tag, 0), key=seed)[i]. */
int32_t cabs_philox_blocks(uint64_t seed, uint32_t tag, uint64_t start, int64_t count,
                           uint32_t* out, void* stream);
/* Positions of sampled-residual pairs t0 .. t0+T-1 (the stream cabs_residual draws when
 * n_samples > 0): device int64 i[T], j[T]. */
int32_t cabs_residual_pairs(uint64_t seed, uint64_t t0, int64_t T, int64_t m, int64_t n, int64_t* i, int64_t* j,
                            void* stream);
/* Floyd sample of k distinct values in [0, N), sorted (the generator of cabs_pilot). */
int32_t cabs_uniform_indices(int64_t N, int32_t k, uint64_t seed, uint32_t tag, int64_t* out,
                             void* stream);
/* Diagnostic counters of profiling builds: out[0..16) per-role cycle sums of the tensor-core
 * residual kernel's CTA 0 (-DCABS_PROFILE_RES); out[16 + 16 b + i] the global-timer stamps
 * (ns) of phase boundary i of iteration 10 in CTA b of the persistent Lloyd kernel
 * (-DCABS_PROFILE_LLOYD, b < 320).  Host out[n]; zeros in normal builds.  Synchronises the
 * device. */
int32_t cabs_debug_counters(int64_t* out, int32_t n);
/* FP64 Jacobi SVD of W (k x k, ldw): sigma (double[k], descending, all k), Uw, Vw
 * (double k x k row-major, column i = i-th singular vector, canonical signs,
 * columns >= r zeroed), r (int32: count of sigma_i > tol*sigma_1). */
int32_t cabs_svd(const cabs_plan* plan, int32_t k, const float* W, int64_t ldw, double tol,
                 double* sigma, double* Uw, double* Vw, int32_t* r, void* ws, size_t ws_bytes,
                 void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CABS_H_ */
