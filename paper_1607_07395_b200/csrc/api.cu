// api.cu -- the extern "C" boundary of libcabs.so (declared and documented in include/cabs.h).
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>

#include "common.cuh"
#include "kernels.cuh"

using namespace cabsk;

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

namespace cabsk {
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace cabsk

void cabs_set_cuda_error(cudaError_t e, const char* where) {
  snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
}
void cabs_set_error_msg(const char* msg) { snprintf(g_err, sizeof(g_err), "%s", msg); }

static int32_t arg_error(const char* msg) {
  cabs_set_error_msg(msg);
  return CABS_ERR_INVALID_ARG;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

static int32_t check_plan(const cabs_plan* p) {
  if (!p) return arg_error("plan is NULL");
  if (p->m < 1 || p->n < 1) return arg_error("plan: m, n must be >= 1");
  if (p->row_begin < 0 || p->row_end < p->row_begin || p->row_end > p->m) return arg_error("plan: bad row range");
  if (p->col_begin < 0 || p->col_end < p->col_begin || p->col_end > p->n) return arg_error("plan: bad column range");
  if (p->kmax < 1 || p->kmax > CABS_KMAX) return arg_error("plan: kmax out of [1, CABS_KMAX]");
  if (p->nranks < 1 || p->rank < 0 || p->rank >= p->nranks) return arg_error("plan: bad rank/nranks");
  return CABS_OK;
}

static int32_t check_ws(const cabs_plan* p, void* ws, size_t bytes, Ws* L) {
  *L = ws_layout(*p);
  if (!ws || bytes < L->total) {
    cabs_set_error_msg("workspace missing or smaller than cabs_workspace_bytes()");
    return CABS_ERR_WORKSPACE;
  }
  return CABS_OK;
}

static bool multi(const cabs_comm* c) { return c && c->nranks > 1; }

static int32_t comm_f64(const cabs_comm* c, double* buf, int64_t count, void* stream) {
  if (!multi(c)) return CABS_OK;
  if (!c->allreduce_f64 || c->allreduce_f64(buf, count, c->ctx, stream) != 0) {
    cabs_set_error_msg("allreduce_f64 callback failed");
    return CABS_ERR_COMM;
  }
  return CABS_OK;
}
static int32_t comm_f32(const cabs_comm* c, float* buf, int64_t count, void* stream) {
  if (!multi(c)) return CABS_OK;
  if (!c->allreduce_f32 || c->allreduce_f32(buf, count, c->ctx, stream) != 0) {
    cabs_set_error_msg("allreduce_f32 callback failed");
    return CABS_ERR_COMM;
  }
  return CABS_OK;
}

extern "C" {

const char* cabs_status_string(int32_t s) {
  switch (s) {
    case CABS_OK: return "ok";
    case CABS_ERR_INVALID_ARG: return "invalid argument";
    case CABS_ERR_RANGE: return "index out of range or duplicated";
    case CABS_ERR_DEGENERATE: return "degenerate input (||A||_F = 0)";
    case CABS_ERR_CUDA: return "CUDA error";
    case CABS_ERR_COMM: return "communication callback failed";
    case CABS_ERR_WORKSPACE: return "workspace too small";
    default: return "unknown status";
  }
}

const char* cabs_last_error_string(void) { return g_err; }

int32_t cabs_debug_counters(int64_t* out, int32_t n) {
  if (!out || n < 0) return CABS_ERR_INVALID_ARG;
  cudaDeviceSynchronize();
  residual_debug_counters(reinterpret_cast<long long*>(out), n < 16 ? n : 16);
#ifdef CABS_PROFILE_EMBED
  if (n >= 16) embed_debug_timeline(reinterpret_cast<long long*>(out));
#endif
#ifdef CABS_PROFILE_SNAP
  if (n >= 4) snap_debug_counters(reinterpret_cast<long long*>(out));
#endif
#if defined(CABS_PROFILE_KTC)
  if (n > 16) ktc_debug_timeline(reinterpret_cast<long long*>(out) + 16, n - 16);
#elif defined(CABS_PROFILE_LEX)
  if (n > 16) lex_debug_timeline(reinterpret_cast<long long*>(out) + 16, n - 16);
#else
  if (n > 16) lloyd_debug_timeline(reinterpret_cast<long long*>(out) + 16, n - 16);
#endif
  return CABS_OK;
}

int64_t cabs_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

int32_t cabs_kernel_path(int32_t op, int32_t k, int32_t d) {
  if (op == CABS_OP_KMEANS)
    return kmeans_prune_selected(k, d) ? CABS_PATH_PRUNE : kmeans_tc_selected(k, d) ? CABS_PATH_TC : CABS_PATH_FFMA;
  if (op == CABS_OP_RESIDUAL) return residual_tc_covers(k) ? CABS_PATH_TC
                                                                                                         : CABS_PATH_FFMA;
  return -1;
}

void cabs_version(int32_t* major, int32_t* minor) {
  if (major) *major = CABS_VERSION_MAJOR;
  if (minor) *minor = CABS_VERSION_MINOR;
}

int64_t cabs_padded_ld(int32_t k) { return round_up(k < 1 ? 1 : k, 32); }

size_t cabs_workspace_bytes(const cabs_plan* plan) {
  if (check_plan(plan) != CABS_OK) return 0;
  return ws_layout(*plan).total;
}

int32_t cabs_clear_status(void* ws, void* stream) {
  if (!ws) return CABS_ERR_WORKSPACE;
  CABS_CUDA_TRY(cudaMemsetAsync(ws, 0, 256, S(stream)));
  return CABS_OK;
}

int32_t cabs_device_status(const void* ws, void* stream, uint32_t* flags) {
  if (!ws || !flags) return CABS_ERR_INVALID_ARG;
  CABS_CUDA_TRY(cudaStreamSynchronize(S(stream)));
  CABS_CUDA_TRY(cudaMemcpy(flags, ws, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return CABS_OK;
}

// ---------------------------------------------------------------- test hooks
int32_t cabs_philox_blocks(uint64_t seed, uint32_t tag, uint64_t start, int64_t count, uint32_t* out, void* stream) {
  if (count < 0 || (count > 0 && !out)) return arg_error("philox_blocks: bad count/out");
  launch_philox_blocks(seed, tag, start, count, out, S(stream));
  CABS_LAUNCH_CHECK("philox_blocks");
  return CABS_OK;
}

int32_t cabs_uniform_indices(int64_t N, int32_t k, uint64_t seed, uint32_t tag, int64_t* out, void* stream) {
  if (k < 0 || k > CABS_KMAX || k > N || N >= 0xFFFFFFFFll) return arg_error("uniform_indices: need 0 <= k <= min(N, KMAX)");
  if (k == 0) return CABS_OK;
  launch_floyd2(N, k, tag, out, 0, 0, 0, nullptr, seed, S(stream));
  CABS_LAUNCH_CHECK("floyd");
  return CABS_OK;
}

int32_t cabs_svd(const cabs_plan* plan, int32_t k, const float* W, int64_t ldw, double tol, double* sigma, double* Uw,
                 double* Vw, int32_t* r, void* ws, size_t ws_bytes, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  if (k < 1 || k > plan->kmax || ldw < k || !W) return arg_error("svd: bad k/ldw");
  launch_svd(k, W, ldw, tol, ws, L, sigma, Uw, Vw, r, S(stream));
  CABS_LAUNCH_CHECK("svd");
  return CABS_OK;
}

// A library-owned non-blocking side stream per device (and fork/join events) for the
// second problem of the *_pair entry points.
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
// Per host thread (thread_local): a caller's event record + stream wait cannot interleave with
// another thread's, so distinct (workspace, stream) pairs stay reentrant across threads.
static int32_t side_stream(SideStream** out) {
  static thread_local SideStream side[64];
  int dev = 0;
  CABS_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return arg_error("device index out of range");
  SideStream& ss = side[dev];
  if (!ss.s) {
    CABS_CUDA_TRY(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
    CABS_CUDA_TRY(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    CABS_CUDA_TRY(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
  }
  *out = &ss;
  return CABS_OK;
}

// ---------------------------------------------------------------- sources
static bool is_rbf(const cabs_source* s) { return s->kind == CABS_SOURCE_RBF_F32; }
static bool is_csr(const cabs_source* s) { return s->kind == CABS_SOURCE_CSR_F32; }
static CsrSrc csr_of(const cabs_source* s) {
  return CsrSrc{s->row_ptr, s->col_idx, s->row_val, s->col_ptr, s->row_idx, s->col_val};
}
static RbfSrc rbf_of(const cabs_source* s) {
  return RbfSrc{s->x, s->y, s->ldx, s->ldy, s->d, s->inv_two_sigma2};
}
static int32_t check_source(const cabs_plan& p, const cabs_source* src, const char* what) {
  if (!src) return arg_error(what);
  if (src->transposed != 0 && (src->transposed != 1 || src->kind != CABS_SOURCE_DENSE_F32)) return arg_error(what);
  if (src->host_resident != 0 && (src->host_resident != 1 || src->kind != CABS_SOURCE_DENSE_F32)) return arg_error(what);
  if (src->at && (src->kind != CABS_SOURCE_DENSE_F32 || src->transposed || src->ldat < p.row_end - p.row_begin))
    return arg_error(what);
  if (src->kind == CABS_SOURCE_DENSE_F32) {
    // row-major block: lda >= n; column-major block (transposed): lda >= m_loc
    if ((p.row_end > p.row_begin && !src->a) || src->lda < (src->transposed ? p.row_end - p.row_begin : p.n))
      return arg_error(what);
    return CABS_OK;
  }
  if (src->kind == CABS_SOURCE_RBF_F32) {
    if (!src->x || !src->y || src->d < 1 || src->d > 64 || src->ldx < src->d || src->ldy < src->d ||
        !(src->inv_two_sigma2 > 0.f))
      return arg_error(what);
    return CABS_OK;
  }
  if (src->kind == CABS_SOURCE_CSR_F32) {
    if (!src->row_ptr || !src->col_ptr || p.n >= 0x7FFFFFFFll || p.row_end - p.row_begin >= 0x7FFFFFFFll)
      return arg_error(what);
    return CABS_OK;
  }
  return arg_error(what);
}
// C = A(rows of this rank, J)
static void src_cols(const cabs_plan& p, const cabs_source* src, const int64_t* J, int k, float* C, int64_t ldc,
                     void* ws, cudaStream_t st) {
  const int64_t m_loc = p.row_end - p.row_begin;
  if (is_rbf(src)) launch_rbf_cols(rbf_of(src), p.row_begin, m_loc, J, k, C, ldc, st);
  else if (is_csr(src)) launch_csc_cols(csr_of(src), m_loc, p.n, J, k, C, ldc, st);
  else if (src->at) launch_gather_cols_t(src->at, src->ldat, m_loc, p.n, J, k, C, ldc, ws, st);  // second, column-major copy
  else if (src->transposed) launch_gather_cols_t(src->a, src->lda, m_loc, p.n, J, k, C, ldc, ws, st);
  else launch_gather_cols(src->a, src->lda, m_loc, p.n, J, k, C, ldc, ws, st);
}
// R = A(I, :): dense -- the rows this rank owns (others: completed by the caller's allreduce);
// implicit -- every row, on every rank
static void src_rows(const cabs_plan& p, const cabs_source* src, const int64_t* I, int k, float* R, int64_t ldr,
                     void* ws, cudaStream_t st) {
  if (is_rbf(src)) launch_rbf_rows(rbf_of(src), I, k, p.n, R, ldr, st);
  else if (is_csr(src)) launch_csr_rows(csr_of(src), p.row_begin, p.row_end, I, k, p.n, R, ldr, st);
  else if (src->transposed) launch_gather_rows_t(src->a, src->lda, p.row_begin, p.row_end, I, k, p.n, R, ldr, ws, st);
  else launch_gather_rows(src->a, src->lda, p.row_begin, p.row_end, I, k, p.n, R, ldr, ws, st);
}
// W = A(I, J) straight from the source (single rank, or implicit)
static void src_w(const cabs_plan& p, const cabs_source* src, const int64_t* I, const int64_t* J, int k, float* W,
                  int64_t ldw, cudaStream_t st) {
  if (is_rbf(src)) launch_rbf_w(rbf_of(src), I, J, k, W, ldw, st);
  else if (is_csr(src)) launch_csr_w(csr_of(src), p.row_begin, p.row_end, I, J, k, W, ldw, st);
  else if (src->transposed) launch_gather_w_t(src->a, src->lda, p.row_begin, p.row_end - p.row_begin, p.n, I, J, k, W, ldw, st);
  else launch_gather_w_direct(src->a, src->lda, p.row_begin, p.row_end - p.row_begin, p.n, I, J, k, W, ldw, st);
}
// rows of R are exchanged only for a dense source on several ranks
static bool rows_need_comm(const cabs_source* src, const cabs_comm* comm) { return multi(comm) && !is_rbf(src); }

// ---------------------------------------------------------------- S1-S3
int32_t cabs_pilot(const cabs_plan* plan, const cabs_source* src, int32_t k, uint64_t seed, int64_t* I, int64_t* J,
                   float* C, int64_t ldc, float* R, int64_t ldr, float* W, int64_t ldw, void* ws, size_t ws_bytes,
                   const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_plan& p = *plan;
  if (k < 1 || k > p.kmax || k > p.m || k > p.n) return arg_error("pilot: need 1 <= k <= min(m, n, kmax)");
  CABS_TRY(check_source(p, src, "pilot: bad source"));
  if (!I || !J || !C || !R || !W || ldc < k || ldr < p.n || ldw < k) return arg_error("pilot: bad output buffers");
  if (p.m >= 0xFFFFFFFFll || p.n >= 0xFFFFFFFFll) return arg_error("pilot: dims must be < 2^32 - 1");
  cudaStream_t st = S(stream);
  launch_floyd2(p.m, k, 1u, I, p.n, k, 2u, J, seed, st);  // tags ROWS_PILOT = 1, COLS_PILOT = 2
  CABS_LAUNCH_CHECK("floyd");
  src_cols(p, src, J, k, C, ldc, ws, st);
  CABS_LAUNCH_CHECK("gather_cols");
  const bool xr = rows_need_comm(src, comm);
  if (xr) launch_fill_neg_zero(R, ldr * (int64_t)k, st);  // -0.0: the allreduce is then bit-exact
  src_rows(p, src, I, k, R, ldr, ws, st);
  CABS_LAUNCH_CHECK("gather_rows");
  if (xr) CABS_TRY(comm_f32(comm, R, ldr * (int64_t)k, stream));
  launch_gather_w(R, ldr, p.n, J, k, W, ldw, st);
  CABS_LAUNCH_CHECK("gather_w");
  return CABS_OK;
}

// shared S4-S5 core: kind 0 = pilot embeddings (P, Q), kind 1 = sketch factors (U, V)
static int32_t embed_core(const cabs_plan& p, const Ws& L, int32_t k, const float* C, int64_t ldc, const float* R,
                          int64_t ldr, const float* W, int64_t ldw, int32_t mode, double tol, float* Y1, int64_t ld1,
                          float* Y2, int64_t ld2, float* s, int32_t* r, double* sigma, int kind, void* ws,
                          const cabs_comm* comm, void* stream, bool svd_done = false) {
  cudaStream_t st = S(stream);
  const int64_t m_loc = p.row_end - p.row_begin, n_sl = p.col_end - p.col_begin;
  if (!svd_done) {
    launch_svd(k, W, ldw, tol, ws, L, sigma, nullptr, nullptr, nullptr, st);
    CABS_LAUNCH_CHECK("svd");
  }
  if (!multi(comm) && !getenv("CABS_EMBED_UNFUSED") &&
      launch_embed_fused(m_loc, n_sl, k, C, ldc, R + p.col_begin, ldr, Y1, ld1, Y2, ld2, mode,
                         static_cast<double>(p.m), static_cast<double>(p.n), static_cast<double>(k), kind, s, r, ws,
                         L, st)) {
    CABS_LAUNCH_CHECK("embed_fused");
    return CABS_OK;
  }
  // the two products (Y_c = C V_w here, Y_r = R^T U_w on the side stream) run concurrently
  SideStream* ss = nullptr;
  CABS_TRY(side_stream(&ss));
  CABS_CUDA_TRY(cudaEventRecord(ss->fork, st));
  CABS_CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
  if (m_loc > 0) CABS_CUDA_TRY(cudaMemsetAsync(Y1, 0, sizeof(float) * ld1 * m_loc, st));
  if (n_sl > 0) CABS_CUDA_TRY(cudaMemsetAsync(Y2, 0, sizeof(float) * ld2 * n_sl, ss->s));
  launch_embed_products(m_loc, n_sl, k, C, ldc, R + p.col_begin, ldr, Y1, ld1, Y2, ld2, ws, L, st, ss->s);
  CABS_LAUNCH_CHECK("embed_products");
  CABS_CUDA_TRY(cudaEventRecord(ss->join, ss->s));
  CABS_CUDA_TRY(cudaStreamWaitEvent(st, ss->join, 0));
  double* norms = wsp<double>(ws, L.norms);
  if (multi(comm)) {
    // one message carries both norm vectors: [N_c^2 (Kp) | N_r^2 (Kp)]
    CABS_TRY(comm_f64(comm, norms, 2 * L.Kp, stream));
  }
  launch_embed_finalize(k, mode, static_cast<double>(p.m), static_cast<double>(p.n), static_cast<double>(k), kind, s, r,
                        ws, L, st);
  CABS_LAUNCH_CHECK("embed_finalize");
  launch_scale_compact(Y1, ld1, m_loc, k, 0, ws, L, st);
  launch_scale_compact(Y2, ld2, n_sl, k, 1, ws, L, st);
  CABS_LAUNCH_CHECK("scale_compact");
  return CABS_OK;
}

int32_t cabs_embed(const cabs_plan* plan, int32_t k, const float* C, int64_t ldc, const float* R, int64_t ldr,
                   const float* W, int64_t ldw, int32_t mode, double tol, float* P, int64_t ldp, float* Q, int64_t ldq,
                   float* s, int32_t* r, double* sigma, void* ws, size_t ws_bytes, const cabs_comm* comm,
                   void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  if (k < 1 || k > plan->kmax) return arg_error("embed: bad k");
  if (mode != CABS_STABILIZED && mode != CABS_PSEUDO_SKELETON) return arg_error("embed: bad mode");
  if (!C || !R || !W || !P || !Q || !s || ldc < k || ldr < plan->n || ldw < k || ldp < k || ldq < k)
    return arg_error("embed: bad buffers");
  return embed_core(*plan, L, k, C, ldc, R, ldr, W, ldw, mode, tol, P, ldp, Q, ldq, s, r, sigma, 0, ws, comm, stream);
}

int32_t cabs_pilot_embed(const cabs_plan* plan, const cabs_source* src, int32_t k, uint64_t seed, int64_t* I,
                         int64_t* J, float* C, int64_t ldc, float* R, int64_t ldr, float* W, int64_t ldw, int32_t mode,
                         double tol, float* P, int64_t ldp, float* Q, int64_t ldq, float* s, int32_t* r,
                         double* sigma, void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream) {
  if (multi(comm)) {
    CABS_TRY(cabs_pilot(plan, src, k, seed, I, J, C, ldc, R, ldr, W, ldw, ws, ws_bytes, comm, stream));
    return cabs_embed(plan, k, C, ldc, R, ldr, W, ldw, mode, tol, P, ldp, Q, ldq, s, r, sigma, ws, ws_bytes, comm,
                      stream);
  }
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_plan& p = *plan;
  if (k < 1 || k > p.kmax || k > p.m || k > p.n) return arg_error("pilot: need 1 <= k <= min(m, n, kmax)");
  CABS_TRY(check_source(p, src, "pilot: bad source"));
  if (!I || !J || !C || !R || !W || ldc < k || ldr < p.n || ldw < k) return arg_error("pilot: bad output buffers");
  if (p.m >= 0xFFFFFFFFll || p.n >= 0xFFFFFFFFll) return arg_error("pilot: dims must be < 2^32 - 1");
  if (mode != CABS_STABILIZED && mode != CABS_PSEUDO_SKELETON) return arg_error("embed: bad mode");
  if (!P || !Q || !s || ldp < k || ldq < k) return arg_error("embed: bad buffers");
  cudaStream_t st = S(stream);
  launch_floyd2(p.m, k, 1u, I, p.n, k, 2u, J, seed, st);  // tags ROWS_PILOT = 1, COLS_PILOT = 2
  CABS_LAUNCH_CHECK("floyd");
  // W = A(I, J) first, its SVD on the side stream while C and R are gathered here
  src_w(p, src, I, J, k, W, ldw, st);
  CABS_LAUNCH_CHECK("gather_w_direct");
  SideStream* ss = nullptr;
  CABS_TRY(side_stream(&ss));
  CABS_CUDA_TRY(cudaEventRecord(ss->fork, st));
  CABS_CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
  launch_svd(k, W, ldw, tol, ws, L, sigma, nullptr, nullptr, nullptr, ss->s);
  CABS_LAUNCH_CHECK("svd");
  src_cols(p, src, J, k, C, ldc, ws, st);
  src_rows(p, src, I, k, R, ldr, ws, st);
  CABS_LAUNCH_CHECK("pilot gathers");
  CABS_CUDA_TRY(cudaEventRecord(ss->join, ss->s));
  CABS_CUDA_TRY(cudaStreamWaitEvent(st, ss->join, 0));
  return embed_core(p, L, k, C, ldc, R, ldr, W, ldw, mode, tol, P, ldp, Q, ldq, s, r, sigma, 0, ws, comm, stream,
                    true);
}

int32_t cabs_sketch(const cabs_plan* plan, const cabs_source* src, const int64_t* Ir, const int64_t* Ic, int32_t k,
                    int32_t mode, double tol, float* U, int64_t ldu, float* s, float* V, int64_t ldv, int32_t* r,
                    double* sigma, void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_plan& p = *plan;
  if (k < 1 || k > p.kmax || k > p.m || k > p.n) return arg_error("sketch: need 1 <= k <= min(m, n, kmax)");
  if (mode != CABS_STABILIZED && mode != CABS_PSEUDO_SKELETON) return arg_error("sketch: bad mode");
  CABS_TRY(check_source(p, src, "sketch: bad source"));
  if (!Ir || !Ic || !U || !V || !s || ldu < k || ldv < k) return arg_error("sketch: bad buffers");
  cudaStream_t st = S(stream);
  float* Cb = wsp<float>(ws, L.cb);
  float* Rb = wsp<float>(ws, L.rb);
  float* Wb = wsp<float>(ws, L.wb);
  if (!multi(comm)) {
    // single GPU: W = A(Ir, Ic) and its SVD (2 SMs) on the side stream, the index check and
    // the large C and R gathers on the caller's stream meanwhile, then join
    SideStream* ss = nullptr;
    CABS_TRY(side_stream(&ss));
    CABS_CUDA_TRY(cudaEventRecord(ss->fork, st));
    CABS_CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
    src_w(p, src, Ir, Ic, k, Wb, L.Kp, ss->s);
    CABS_LAUNCH_CHECK("gather_w_direct");
    launch_svd(k, Wb, L.Kp, tol, ws, L, sigma, nullptr, nullptr, nullptr, ss->s);
    CABS_LAUNCH_CHECK("svd");
    launch_validate_idx2(Ir, p.m, Ic, p.n, k, ws, st);
    src_cols(p, src, Ic, k, Cb, L.Kp, ws, st);
    src_rows(p, src, Ir, k, Rb, L.ldrb, ws, st);
    CABS_LAUNCH_CHECK("sketch gathers");
    CABS_CUDA_TRY(cudaEventRecord(ss->join, ss->s));
    CABS_CUDA_TRY(cudaStreamWaitEvent(st, ss->join, 0));
    return embed_core(p, L, k, Cb, L.Kp, Rb, L.ldrb, Wb, L.Kp, mode, tol, U, ldu, V, ldv, s, r, sigma, 1, ws, comm,
                      stream, true);
  }
  launch_validate_idx2(Ir, p.m, Ic, p.n, k, ws, st);
  src_cols(p, src, Ic, k, Cb, L.Kp, ws, st);
  const bool xr = rows_need_comm(src, comm);
  if (xr) launch_fill_neg_zero(Rb, L.ldrb * (int64_t)k, st);
  src_rows(p, src, Ir, k, Rb, L.ldrb, ws, st);
  CABS_LAUNCH_CHECK("sketch gathers");
  if (xr) CABS_TRY(comm_f32(comm, Rb, L.ldrb * (int64_t)k, stream));
  launch_gather_w(Rb, L.ldrb, p.n, Ic, k, Wb, L.Kp, st);
  CABS_LAUNCH_CHECK("gather_w");
  return embed_core(p, L, k, Cb, L.Kp, Rb, L.ldrb, Wb, L.Kp, mode, tol, U, ldu, V, ldv, s, r, sigma, 1, ws, comm,
                    stream);
}

// ---------------------------------------------------------------- S6-S7
static int32_t km_check(const cabs_plan* plan, const Ws& L, const cabs_km_problem& p, int32_t iters,
                        int32_t weight_kind) {
  if (p.k2 < 1 || p.k2 > plan->kmax || p.k2 > p.n_glob) return arg_error("kmeans: need 1 <= k2 <= min(n_glob, kmax)");
  if (iters < 1) return arg_error("kmeans: iters must be >= 1");
  if (p.d < 1 || p.d > L.Kp || p.ldx < p.d || p.ldc < p.d || p.n_loc < 0 || p.n_loc > L.Nmax)
    return arg_error("kmeans: bad dims");
  if (weight_kind != CABS_WEIGHT_CONST && weight_kind != CABS_WEIGHT_POWER) return arg_error("kmeans: bad weight");
  if (!p.centres || (p.n_loc > 0 && (!p.X || !p.labels)) || !p.cluster_w || !p.objective)
    return arg_error("kmeans: bad buffers");
  return CABS_OK;
}

// workspace of problem slot q (0 or 1)
struct KmSlot {
  float* w;
  int* cnt;
  unsigned* bounds;
  int64_t* idx;
  void* scr;
  size_t scr_bytes;
  float* ebuf;  // the snap distance buffer of the slot (free during the k-means)
  size_t ebuf_bytes;
  long long* qbuf;
};
static KmSlot km_slot(void* ws, const Ws& L, int q) {
  KmSlot k;
  k.ebuf = wsp<float>(ws, q ? L.dist2 : L.dist);
  k.qbuf = wsp<long long>(ws, L.km_q) + (size_t)q * L.Nmax;
  k.ebuf_bytes = sizeof(float) * (size_t)L.K * (size_t)L.Nmax;
  k.w = wsp<float>(ws, L.km_w) + (size_t)q * L.Nmax;
  k.cnt = wsp<int>(ws, L.km_cnt) + 16 * q;
  k.bounds = reinterpret_cast<unsigned*>(k.cnt + 2);
  k.idx = wsp<int64_t>(ws, L.idx) + (size_t)(4 * q) * L.Kp;
  k.scr = static_cast<char*>(wsp<char>(ws, L.km_scr)) + (size_t)q * L.km_scr_bytes;
  k.scr_bytes = L.km_scr_bytes;
  return k;
}

// weights w_l = Upsilon(||X_l||) and the fixed-point bounds; initial centres (replicated)
static int32_t km_prepare(const cabs_km_problem& p, int32_t weight_kind, float weight_p, uint64_t seed,
                          const KmSlot& k, const cabs_comm* comm, void* stream) {
  cudaStream_t st = S(stream);
  CABS_CUDA_TRY(cudaMemsetAsync(k.cnt, 0, sizeof(int) * 4, st));
  launch_km_weights(p.X, p.ldx, p.n_loc, p.d, weight_kind, weight_p, k.w, k.cnt, k.bounds, st);
  CABS_LAUNCH_CHECK("km_weights");
  const int64_t* idx = p.init_idx;
  if (!p.init_idx && !p.init_centres) {
    launch_floyd2(p.n_glob, p.k2, static_cast<uint32_t>(p.tag), k.idx, 0, 0, 0, nullptr, seed, st);
    CABS_LAUNCH_CHECK("floyd init");
    idx = k.idx;
  }
  launch_km_init(p.X, p.ldx, p.n_loc, p.row_off, p.d, p.k2, p.init_centres ? nullptr : idx, p.init_centres, p.ldc,
                 p.centres, p.ldc, st);
  CABS_LAUNCH_CHECK("km_init");
  if (!p.init_centres) CABS_TRY(comm_f32(comm, p.centres, p.ldc * (int64_t)p.k2, stream));
  return CABS_OK;
}

static LloydJob km_job(const cabs_km_problem& p, const KmSlot& k) {
  LloydJob j;
  j.X = p.X; j.ldx = p.ldx; j.N = p.n_loc; j.d = p.d; j.k2 = p.k2; j.w = k.w; j.bounds = k.bounds;
  j.centres = p.centres; j.ldc = p.ldc; j.labels = p.labels; j.objective = p.objective; j.near_ties = p.near_ties;
  j.cluster_w = p.cluster_w; j.scratch = k.scr; j.scratch_bytes = k.scr_bytes;
  j.tie_log = p.tie_log; j.tie_cap = p.tie_log_cap; j.row_off = p.row_off;
  j.ebuf = k.ebuf; j.ebuf_bytes = k.ebuf_bytes; j.qbuf = k.qbuf;
  return j;
}

static bool km_persistent_allowed(const cabs_comm* comm) {
  const char* path = getenv("CABS_KMEANS_PATH");  // "loop" forces the per-iteration kernels (tests)
  return !(path && strcmp(path, "loop") == 0) && !multi(comm);
}

// per-iteration kernels (multi-rank, or when the persistent kernel does not apply) for np <= 2
// problems: each iteration reduces every problem's sums into its part of ONE payload, so a
// pair costs one collective per iteration, not two
static int32_t km_loop(const cabs_km_problem* const* pp, const KmSlot* const* kk, int np, int32_t iters, void* ws,
                       const Ws& L, const cabs_comm* comm, void* stream) {
  cudaStream_t st = S(stream);
  double* red[2];
  int64_t payload[2], total = 0;
  for (int q = 0; q < np; ++q) {
    const cabs_km_problem& p = *pp[q];
    red[q] = wsp<double>(ws, L.km_red) + total;
    payload[q] = (int64_t)p.k2 * p.d + p.k2 + 2;
    total += payload[q];
    long long* fsum = static_cast<long long*>(kk[q]->scr);  // exact int64 sums (km_fixed.cuh), re-zeroed by km_reduce
    CABS_CUDA_TRY(cudaMemsetAsync(fsum, 0, sizeof(long long) * ((int64_t)p.k2 * p.d + p.k2), st));
  }
  for (int t = 0; t < iters; ++t) {
    for (int q = 0; q < np; ++q) {
      const cabs_km_problem& p = *pp[q];
      const KmSlot& k = *kk[q];
      const int k2 = p.k2, d = p.d;
      long long* fsum = static_cast<long long*>(k.scr);
      long long* fwt = fsum + (int64_t)k2 * d;
      int ga = 1;
      if (p.n_loc > 0) {
        launch_km_assign(p.X, p.ldx, p.n_loc, d, p.centres, p.ldc, k2, k.w, p.labels, wsp<double>(ws, L.km_pobj),
                         wsp<int>(ws, L.km_ptie), &ga, st, p.tie_log, p.tie_log_cap, t, p.row_off);
        launch_km_accum(p.X, p.ldx, p.n_loc, d, p.labels, k.w, k.bounds, fsum, fwt, st);
        CABS_LAUNCH_CHECK("km_assign/accum");
        launch_km_reduce(fsum, fwt, k.bounds, p.n_loc, k2, d, wsp<double>(ws, L.km_pobj), wsp<int>(ws, L.km_ptie),
                         ga, red[q], st);
      } else {
        CABS_CUDA_TRY(cudaMemsetAsync(red[q], 0, sizeof(double) * payload[q], st));
      }
      CABS_LAUNCH_CHECK("km_reduce");
    }
    CABS_TRY(comm_f64(comm, red[0], total, stream));  // ONE fused message per iteration
    for (int q = 0; q < np; ++q) {
      const cabs_km_problem& p = *pp[q];
      launch_km_finalize(red[q], p.k2, p.d, p.centres, p.ldc, p.objective, p.near_ties, p.cluster_w, t, st);
      CABS_LAUNCH_CHECK("km_finalize");
    }
  }
  return CABS_OK;
}

int32_t cabs_kmeans(const cabs_plan* plan, const float* X, int64_t ldx, int64_t n_loc, int64_t n_glob, int64_t row_off,
                    int32_t d, int32_t k2, int32_t iters, int32_t weight_kind, float weight_p, uint64_t seed,
                    int32_t tag, const int64_t* init_idx, const float* init_centres, float* centres, int64_t ldc,
                    int32_t* labels, double* cluster_w, double* objective, int32_t* near_ties, int32_t* tie_log,
                    int32_t tie_log_cap, void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_km_problem p{X, ldx, n_loc, n_glob, row_off, d, k2, tag, init_idx, init_centres, centres, ldc,
                          labels, cluster_w, objective, near_ties, tie_log, tie_log_cap};
  CABS_TRY(km_check(plan, L, p, iters, weight_kind));
  if (tie_log) CABS_CUDA_TRY(cudaMemsetAsync(tie_log, 0, sizeof(int32_t), S(stream)));
  const KmSlot k = km_slot(ws, L, 0);
  CABS_TRY(km_prepare(p, weight_kind, weight_p, seed, k, comm, stream));
  if (km_persistent_allowed(comm) && n_loc > 0) {
    const LloydJob j = km_job(p, k);
    if (kmeans_prune_selected(k2, d)) {
      if (launch_lloyd_prune(&j, 1, iters, S(stream))) {
        CABS_LAUNCH_CHECK("lloyd_prune");
        return CABS_OK;
      }
      cudaGetLastError();
    }
    if (kmeans_tc_selected(k2, d)) {
      if (launch_lloyd_tc(&j, 1, iters, S(stream))) {
        CABS_LAUNCH_CHECK("lloyd_tc");
        return CABS_OK;
      }
      if (getenv("CABS_KMEANS_REQUIRE_TC")) return arg_error("kmeans: tensor-core kernel not launched");
    }
    cudaGetLastError();
    if (launch_lloyd_persistent(&j, 1, iters, reinterpret_cast<long long*>(ws) + 8, S(stream))) {
      CABS_LAUNCH_CHECK("lloyd_persistent");
      return CABS_OK;
    }
  }
  cudaGetLastError();  // a refused cooperative launch is not an error: use the per-iteration kernels
  const cabs_km_problem* pp = &p;
  const KmSlot* kp = &k;
  return km_loop(&pp, &kp, 1, iters, ws, L, comm, stream);
}

int32_t cabs_kmeans_pair(const cabs_plan* plan, const cabs_km_problem* a, const cabs_km_problem* b, int32_t iters,
                         int32_t weight_kind, float weight_p, uint64_t seed, void* ws, size_t ws_bytes,
                         const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  if (!a || !b) return arg_error("kmeans_pair: null problem");
  CABS_TRY(km_check(plan, L, *a, iters, weight_kind));
  CABS_TRY(km_check(plan, L, *b, iters, weight_kind));
  if (a->tie_log) CABS_CUDA_TRY(cudaMemsetAsync(a->tie_log, 0, sizeof(int32_t), S(stream)));
  if (b->tie_log) CABS_CUDA_TRY(cudaMemsetAsync(b->tie_log, 0, sizeof(int32_t), S(stream)));
  const KmSlot ka = km_slot(ws, L, 0), kb = km_slot(ws, L, 1);
  if (!multi(comm)) {
    // both sides' weights, Floyd initialisations and initial centres in one launch each; the
    // weights (independent of the initialisation) run on the side stream meanwhile
    cudaStream_t st = S(stream);
    SideStream* ss = nullptr;
    CABS_TRY(side_stream(&ss));
    CABS_CUDA_TRY(cudaEventRecord(ss->fork, st));
    CABS_CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
    CABS_CUDA_TRY(cudaMemsetAsync(ka.cnt, 0, sizeof(int) * 20, ss->s));  // slot 0 [0, 4), slot 1 [16, 20)
    const KmWeightJob wa{a->X, a->ldx, a->n_loc, a->d, ka.w, ka.cnt, ka.bounds};
    const KmWeightJob wb{b->X, b->ldx, b->n_loc, b->d, kb.w, kb.cnt, kb.bounds};
    launch_km_weights2(wa, &wb, weight_kind, weight_p, ss->s);
    CABS_LAUNCH_CHECK("km_weights");
    CABS_CUDA_TRY(cudaEventRecord(ss->join, ss->s));
    const bool fa = !a->init_idx && !a->init_centres, fb = !b->init_idx && !b->init_centres;
    if (fa || fb) {
      launch_floyd2(a->n_glob, fa ? a->k2 : 0, static_cast<uint32_t>(a->tag), fa ? ka.idx : nullptr, b->n_glob,
                    fb ? b->k2 : 0, static_cast<uint32_t>(b->tag), fb ? kb.idx : nullptr, seed, st);
      CABS_LAUNCH_CHECK("floyd init");
    }
    const KmInitJob ia{a->X, a->ldx, a->n_loc, a->row_off, a->d, a->k2, fa ? ka.idx : a->init_idx,
                       a->init_centres, a->ldc, a->centres, a->ldc};  // init_centres takes precedence
    const KmInitJob ib{b->X, b->ldx, b->n_loc, b->row_off, b->d, b->k2, fb ? kb.idx : b->init_idx,
                       b->init_centres, b->ldc, b->centres, b->ldc};
    launch_km_init2(ia, &ib, st);
    CABS_LAUNCH_CHECK("km_init");
    CABS_CUDA_TRY(cudaStreamWaitEvent(st, ss->join, 0));
  } else {
    CABS_TRY(km_prepare(*a, weight_kind, weight_p, seed, ka, comm, stream));
    CABS_TRY(km_prepare(*b, weight_kind, weight_p, seed, kb, comm, stream));
  }
  if (km_persistent_allowed(comm) && a->n_loc > 0 && b->n_loc > 0) {
    const LloydJob j[2] = {km_job(*a, ka), km_job(*b, kb)};
    if (kmeans_prune_selected(a->k2, a->d) && kmeans_prune_selected(b->k2, b->d)) {
      if (launch_lloyd_prune(j, 2, iters, S(stream))) {
        CABS_LAUNCH_CHECK("lloyd_prune");
        return CABS_OK;
      }
      cudaGetLastError();
    }
    if (kmeans_tc_selected(a->k2, a->d) && kmeans_tc_selected(b->k2, b->d)) {
      if (launch_lloyd_tc(j, 2, iters, S(stream))) {
        CABS_LAUNCH_CHECK("lloyd_tc");
        return CABS_OK;
      }
      if (getenv("CABS_KMEANS_REQUIRE_TC")) return arg_error("kmeans_pair: tensor-core kernel not launched");
    }
    cudaGetLastError();
    if (launch_lloyd_persistent(j, 2, iters, reinterpret_cast<long long*>(ws) + 8, S(stream))) {
      CABS_LAUNCH_CHECK("lloyd_persistent");
      return CABS_OK;
    }
  }
  cudaGetLastError();
  const cabs_km_problem* pp[2] = {a, b};
  const KmSlot* kk[2] = {&ka, &kb};
  if (multi(comm)) return km_loop(pp, kk, 2, iters, ws, L, comm, stream);  // one fused payload per iteration
  // one problem at a time (each may still take the single-problem persistent kernel)
  for (int q = 0; q < 2; ++q) {
    bool done = false;
    if (km_persistent_allowed(comm) && pp[q]->n_loc > 0) {
      const LloydJob j = km_job(*pp[q], *kk[q]);
      done = launch_lloyd_persistent(&j, 1, iters, reinterpret_cast<long long*>(ws) + 8, S(stream));
      if (done) CABS_LAUNCH_CHECK("lloyd_persistent");
    }
    cudaGetLastError();
    if (!done) CABS_TRY(km_loop(&pp[q], &kk[q], 1, iters, ws, L, comm, stream));
  }
  return CABS_OK;
}

// ---------------------------------------------------------------- S8
static int32_t sel_check(const cabs_plan* plan, const Ws& L, const cabs_sel_problem& p) {
  if (p.k2 < 1 || p.k2 > plan->kmax || p.k2 > p.n_glob) return arg_error("select: bad k2");
  if (p.d < 1 || p.ldx < p.d || p.ldc < p.d || p.n_loc < 0 || p.n_loc > L.Nmax) return arg_error("select: bad dims");
  if (!p.centres || !p.cluster_w || !p.reps || (p.n_loc > 0 && !p.X)) return arg_error("select: bad buffers");
  return CABS_OK;
}

// snap of one problem with the scratch of slot q
struct SnapComm {
  const cabs_comm* comm;
  void* stream;
};
static int snap_allreduce(double* buf, int64_t n, void* ctx) {
  const SnapComm* c = static_cast<const SnapComm*>(ctx);
  return comm_f64(c->comm, buf, n, c->stream) == CABS_OK ? 0 : -1;
}

static int32_t sel_run(const cabs_sel_problem& p, int q, void* ws, const Ws& L, const cabs_comm* comm, void* stream) {
  cudaStream_t st = S(stream);
  float* D = wsp<float>(ws, q ? L.dist2 : L.dist);
  float* cd = wsp<float>(ws, q ? L.cand_d2 : L.cand_d);
  int64_t* ci = wsp<int64_t>(ws, q ? L.cand_i2 : L.cand_i);
  double* all = wsp<double>(ws, q ? L.cand_all2 : L.cand_all);
  const bool mr = multi(comm);
  const int T = mr ? kSnapTMulti : kSnapT;
  const int nr = mr ? comm->nranks : 1, rank = mr ? comm->rank : 0;
  launch_km_distmat(p.X, p.ldx, p.n_loc, p.d, p.centres, p.ldc, p.k2, D, L.Nmax, st);
  // per-centre top-T over S point segments in parallel; lists packed as doubles so that
  // other ranks' slots (zeros here) are completed by ONE sum-allreduce, then merged.  Multi-rank:
  // S = kSnapSeg on every rank (slot offsets must agree), and a rank without points still
  // writes its (FLT_MAX, -1) sentinels (topT of an empty range)
  int Sg = kSnapSeg;
  if (!mr) {
    Sg = static_cast<int>(ceil_div(p.n_loc > 0 ? p.n_loc : 1, 4096));
    if (Sg > kSnapSeg) Sg = kSnapSeg;
  }
  const int64_t nall = 2LL * nr * Sg * p.k2 * T;
  if (mr) CABS_CUDA_TRY(cudaMemsetAsync(all, 0, sizeof(double) * nall, st));
  if (p.n_loc > 0 || mr) launch_snap_topT(D, L.Nmax, p.n_loc, p.k2, p.row_off, T, Sg, rank * Sg, all, st);
  CABS_LAUNCH_CHECK("snap distmat/topT");
  CABS_TRY(comm_f64(comm, all, nall, stream));
  launch_snap_merge(all, p.k2, T, nr * Sg, cd, ci, st);
  CABS_LAUNCH_CHECK("snap_merge");
  int* unres = wsp<int>(ws, L.scal) + SCAL_UNRES + q;
  if (mr) CABS_CUDA_TRY(cudaMemsetAsync(unres, 0, sizeof(int), st));
  launch_snap_dedupe(cd, ci, p.k2, T, p.cluster_w, D, L.Nmax, p.n_loc, p.row_off, !mr, p.rep_of_centre, p.gap,
                     p.reps, ws, st, mr ? unres : nullptr);
  CABS_LAUNCH_CHECK("snap_dedupe");
  // multi-rank: a centre whose best or runner-up the exchanged lists did not resolve (every rank
  // sees the same merged lists, so all ranks agree) -> the exact pass over the ranks' rows of D
  bool redo = getenv("CABS_SNAP_FORCE_DIST") != nullptr;
  if (mr && !redo) {
    int h = 0;
    CABS_CUDA_TRY(cudaMemcpyAsync(&h, unres, sizeof(int), cudaMemcpyDeviceToHost, st));
    CABS_CUDA_TRY(cudaStreamSynchronize(st));
    redo = h != 0;
  }
  if (redo) {
    // scratch: the candidate array (>= 4096 K bytes, > snap_dist_bytes for any k2 <= K)
    if (sizeof(double) * 2 * nr * kSnapSeg * L.K * kSnapTMulti < snap_dist_bytes(p.k2, nr))
      return arg_error("select: snap scratch too small");
    SnapComm sc{comm, stream};
    const int rc = snap_dist_run(D, L.Nmax, p.n_loc, p.row_off, p.k2, p.cluster_w, rank, nr, all, p.rep_of_centre,
                                 p.gap, p.reps, ws, st, snap_allreduce, &sc);
    if (rc == -2) return CABS_ERR_COMM;
    CABS_LAUNCH_CHECK("snap_dist");
  }
  return CABS_OK;
}

int32_t cabs_select(const cabs_plan* plan, const float* X, int64_t ldx, int64_t n_loc, int64_t n_glob, int64_t row_off,
                    int32_t d, const float* centres, int64_t ldc, int32_t k2, const double* cluster_w, int64_t* reps,
                    int64_t* rep_of_centre, float* gap, void* ws, size_t ws_bytes, const cabs_comm* comm,
                    void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_sel_problem p{X, ldx, n_loc, n_glob, row_off, d, centres, ldc, k2, cluster_w, reps, rep_of_centre, gap};
  CABS_TRY(sel_check(plan, L, p));
  return sel_run(p, 0, ws, L, comm, stream);
}

int32_t cabs_select_pair(const cabs_plan* plan, const cabs_sel_problem* a, const cabs_sel_problem* b, void* ws,
                         size_t ws_bytes, const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  if (!a || !b) return arg_error("select_pair: null problem");
  CABS_TRY(sel_check(plan, L, *a));
  CABS_TRY(sel_check(plan, L, *b));
  if (multi(comm)) {  // the collectives run on the caller's stream: one problem after the other
    CABS_TRY(sel_run(*a, 0, ws, L, comm, stream));
    return sel_run(*b, 1, ws, L, comm, stream);
  }
  SideStream* ss = nullptr;
  CABS_TRY(side_stream(&ss));
  cudaStream_t st = S(stream);
  CABS_CUDA_TRY(cudaEventRecord(ss->fork, st));
  CABS_CUDA_TRY(cudaStreamWaitEvent(ss->s, ss->fork, 0));
  const int32_t ra = sel_run(*a, 0, ws, L, comm, stream);
  const int32_t rb = sel_run(*b, 1, ws, L, comm, ss->s);
  CABS_CUDA_TRY(cudaEventRecord(ss->join, ss->s));
  CABS_CUDA_TRY(cudaStreamWaitEvent(st, ss->join, 0));
  return ra != CABS_OK ? ra : rb;
}

// ---------------------------------------------------------------- S8' hard threshold (P:312 (f))
static int32_t hard_check(const cabs_plan* plan, const Ws& L, const cabs_hard_problem& p) {
  if (p.k2 < 1 || p.k2 > plan->kmax || p.k2 > p.n_glob) return arg_error("hard_select: bad k2");
  if (p.d < 1 || p.ldx < p.d || p.n_loc < 0 || p.n_loc > L.Nmax || p.row_off < 0 || p.row_off + p.n_loc > p.n_glob)
    return arg_error("hard_select: bad dims");
  if (!p.reps || (p.n_loc > 0 && !p.X)) return arg_error("hard_select: bad buffers");
  return CABS_OK;
}

static cabsk::HardSide hard_side(const cabs_hard_problem& p) {
  cabsk::HardSide h{};
  h.X = p.X;
  h.ldx = p.ldx;
  h.N = p.n_loc;
  h.d = p.d;
  h.key = p.keys;  // NULL: keys are not stored
  h.ks = 1;
  h.off = p.row_off;
  h.k = p.k2;
  return h;
}

// top-k over the (key, index) candidate pairs at c (n candidates)
static cabsk::HardSide hard_merge_side(double* c, int64_t n, int k, int64_t* out, double* slot) {
  cabsk::HardSide h{};
  h.key = c;
  h.ks = 2;
  h.cidx = c + 1;
  h.N = n;
  h.k = k;
  h.out = out;
  h.slot = slot;
  return h;
}

// nprob problems (1 or 2); single GPU: one key + local top-k launch and one merge launch
static int32_t hard_run(const cabs_hard_problem* const* pr, int nprob, void* ws, const Ws& L, const cabs_comm* comm,
                        void* stream, int mode = 0, uint64_t seed = 0, const uint32_t* tags = nullptr) {
  cudaStream_t st = S(stream);
  auto keyed = [&](cabsk::HardSide h, int q) {  // the key of the local kernel: (f) or leverage (e)
    h.mode = mode;
    h.seed = seed;
    h.tag = tags ? tags[q] : 0u;
    return h;
  };
  double* cand = wsp<double>(ws, L.hcand);
  if (!multi(comm)) {
    cabsk::HardArgs a{}, m{};
    for (int q = 0; q < nprob; ++q) {
      const cabs_hard_problem& p = *pr[q];
      a.s[q] = keyed(hard_side(p), q);
      m.s[q] = hard_merge_side(cand + q * L.hcand_side, hard_local_blocks(p.n_loc) * p.k2, p.k2, p.reps, nullptr);
    }
    launch_hard_local(a, nprob, cand, L.hcand_side, ws, st);
    launch_hard_topk(m, nprob, st);
    CABS_LAUNCH_CHECK("hard_select");
    return CABS_OK;
  }
  // multi-rank, one problem after the other: this rank's winners go to its slot of a zeroed
  // [nranks][k2] (key, index) buffer, one sum-allreduce, then the top-k2 of those candidates
  double* all = wsp<double>(ws, L.cand_all);
  for (int q = 0; q < nprob; ++q) {
    const cabs_hard_problem& p = *pr[q];
    const int64_t nall = 2LL * comm->nranks * p.k2;
    CABS_CUDA_TRY(cudaMemsetAsync(all, 0, sizeof(double) * nall, st));
    cabsk::HardArgs a{}, m{}, f{};
    a.s[0] = keyed(hard_side(p), q);
    m.s[0] = hard_merge_side(cand, hard_local_blocks(p.n_loc) * p.k2, p.k2, nullptr, all + 2LL * comm->rank * p.k2);
    launch_hard_local(a, 1, cand, L.hcand_side, ws, st);
    launch_hard_topk(m, 1, st);
    CABS_LAUNCH_CHECK("hard_select local");
    CABS_TRY(comm_f64(comm, all, nall, stream));
    f.s[0] = hard_merge_side(all, (int64_t)comm->nranks * p.k2, p.k2, p.reps, nullptr);
    launch_hard_topk(f, 1, st);
    CABS_LAUNCH_CHECK("hard_select merge");
  }
  return CABS_OK;
}

int32_t cabs_hard_select(const cabs_plan* plan, const float* X, int64_t ldx, int64_t n_loc, int64_t n_glob,
                         int64_t row_off, int32_t d, int32_t k2, int64_t* reps, double* keys, void* ws,
                         size_t ws_bytes, const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_hard_problem p{X, ldx, n_loc, n_glob, row_off, d, k2, reps, keys};
  CABS_TRY(hard_check(plan, L, p));
  const cabs_hard_problem* pr[1] = {&p};
  return hard_run(pr, 1, ws, L, comm, stream);
}

int32_t cabs_hard_select_pair(const cabs_plan* plan, const cabs_hard_problem* a, const cabs_hard_problem* b, void* ws,
                              size_t ws_bytes, const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  if (!a || !b) return arg_error("hard_select_pair: null problem");
  CABS_TRY(hard_check(plan, L, *a));
  CABS_TRY(hard_check(plan, L, *b));
  const cabs_hard_problem* pr[2] = {a, b};
  return hard_run(pr, 2, ws, L, comm, stream);
}

// ---------------------------------------------------------------- variant (e): Supp. 3 + leverage
int32_t cabs_orthogonalize(const cabs_plan* plan, int32_t r, const float* U, int64_t ldu, const float* s,
                           const float* V, int64_t ldv, float* Uo, int64_t lduo, float* so, float* Vo, int64_t ldvo,
                           int32_t* r_out, double* sigma, void* ws, size_t ws_bytes, const cabs_comm* comm,
                           void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_plan& p = *plan;
  const int64_t m_loc = p.row_end - p.row_begin, n_sl = p.col_end - p.col_begin;
  if (r < 1 || r > p.kmax) return arg_error("orthogonalize: need 1 <= r <= kmax");
  if (ldu < r || ldv < r || lduo < r || ldvo < r) return arg_error("orthogonalize: bad leading dimensions");
  if ((m_loc > 0 && (!U || !Uo)) || (n_sl > 0 && (!V || !Vo)) || !so) return arg_error("orthogonalize: bad buffers");
  cudaStream_t st = S(stream);
  unsigned char* o = static_cast<unsigned char*>(ws) + L.orth;
  cabsk::OrthArgs a{};
  a.U = U; a.ldu = ldu; a.nu = m_loc;
  a.V = V; a.ldv = ldv; a.nv = n_sl;
  a.r = r; a.s = s;
  a.part = wsp<double>(ws, L.orth_part);
  a.nblk = orth_gram_blocks(m_loc, n_sl, r);
  // [gram: 2 r^2 | U_K: r^2 | V_K: r^2 | sigma: r | r_svd] FP64, then K, T_U, T_V (r x Kp FP32)
  const size_t rr = static_cast<size_t>(r) * r;
  a.gram = reinterpret_cast<double*>(o);
  a.UK = a.gram + 2 * rr;
  a.VK = a.UK + rr;
  a.sig = sigma ? sigma : a.VK + rr;
  a.r_svd = reinterpret_cast<int*>(a.VK + rr + r);
  a.kp = L.Kp;
  a.K = reinterpret_cast<float*>(o + sizeof(double) * (4 * rr + r) + 256);
  a.TU = a.K + static_cast<size_t>(r) * L.Kp;
  a.TV = a.TU + static_cast<size_t>(r) * L.Kp;
  a.s_out = so; a.r_out = r_out;
  a.Uo = Uo; a.lduo = lduo; a.Vo = Vo; a.ldvo = ldvo;
  launch_orth_gram(a, st);
  CABS_LAUNCH_CHECK("orth_gram");
  CABS_TRY(comm_f64(comm, a.gram, static_cast<int64_t>(2) * r * r, stream));
  launch_orth_core(a, ws, st);
  CABS_LAUNCH_CHECK("orth_core");
  launch_svd(r, a.K, a.kp, 1e-12, ws, L, a.sig, a.UK, a.VK, a.r_svd, st);
  CABS_LAUNCH_CHECK("orth_svd");
  launch_orth_finish(a, st);
  CABS_LAUNCH_CHECK("orth_finish");
  return CABS_OK;
}

// ---------------------------------------------------------------- NEXT-4: BR-CUR / Sketch-CUR, rank sweep
int32_t cabs_br_cur(const cabs_plan* plan, const cabs_source* src, int32_t k1, const int64_t* Ibr, const int64_t* Ibc,
                    int32_t k2, const int64_t* Itr, const int64_t* Itc, double tol, float* F, int64_t ldf, float* G,
                    int64_t ldg, double* Umid, void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_plan& p = *plan;
  if (multi(comm) || p.nranks > 1) return arg_error("br_cur: single rank only");
  CABS_TRY(check_source(p, src, "br_cur: bad source"));
  if (k1 < 1 || k2 < k1 || k2 > p.kmax || k2 > p.m || k2 > p.n) return arg_error("br_cur: need 1 <= k1 <= k2 <= min(m, n, kmax)");
  if (!Ibr || !Ibc || !Itr || !Itc || !F || !G || ldf < k1 || ldg < k1) return arg_error("br_cur: bad buffers");
  cudaStream_t st = S(stream);
  const int64_t m_loc = p.row_end - p.row_begin;
  float* Cb = wsp<float>(ws, L.cb);
  float* Rb = wsp<float>(ws, L.rb);
  float* Wb = wsp<float>(ws, L.wb);
  const size_t KK = (size_t)L.K * L.K;
  double* o = reinterpret_cast<double*>(static_cast<unsigned char*>(ws) + L.orth);
  double *U1 = o, *V1 = o + KK, *U2 = o + 2 * KK, *V2 = o + 3 * KK, *sig1 = o + 4 * KK, *sig2 = sig1 + L.K;
  double* M = wsp<double>(ws, L.w64);
  double* tmp = wsp<double>(ws, L.orth_part);  // d1, d2, X1, Y, X2, U* (after the SVDs)
  if (sizeof(double) * (2.0 * k2 + 3.0 * k1 * k2 + 1.0 * k1 * k1) > static_cast<double>(L.orth - L.orth_part))
    return arg_error("br_cur: k1, k2 too large for the workspace");
  double *d1 = tmp, *d2 = d1 + k2, *X1 = d2 + k2, *Y = X1 + (size_t)k1 * k2, *X2 = Y + (size_t)k1 * k2;
  double* Ust = X2 + (size_t)k2 * k1;
  // steps 1-2 (Alg. 1): C = A(:, I^b_c); R = A(I^b_r, :) -> G = R^T and R_bar = R(:, I^t_c) padded to k2 x k2
  src_cols(p, src, Ibc, k1, Cb, L.Kp, ws, st);
  src_rows(p, src, Ibr, k1, Rb, L.ldrb, ws, st);
  CABS_LAUNCH_CHECK("br_cur gathers");
  launch_transpose(Rb, L.ldrb, k1, p.n, G, ldg, st);
  launch_pick_cols(Rb, L.ldrb, k1, Itc, k2, k2, Wb, L.Kp, nullptr, st);
  launch_zero_rows(Wb, L.Kp, k1, k2, k2, st);
  launch_svd(k2, Wb, L.Kp, tol, ws, L, sig2, U2, V2, nullptr, st);
  CABS_LAUNCH_CHECK("br_cur svd R_bar");
  // steps 2-3: the target rows A(I^t_r, :) -> C_bar = (.)(:, I^b_c) padded, M = (.)(:, I^t_c)
  src_rows(p, src, Itr, k2, Rb, L.ldrb, ws, st);
  launch_pick_cols(Rb, L.ldrb, k2, Ibc, k1, k2, Wb, L.Kp, nullptr, st);
  launch_pick_cols(Rb, L.ldrb, k2, Itc, k2, k2, nullptr, 0, M, st);
  CABS_LAUNCH_CHECK("br_cur targets");
  launch_svd(k2, Wb, L.Kp, tol, ws, L, sig1, U1, V1, nullptr, st);
  CABS_LAUNCH_CHECK("br_cur svd C_bar");
  // step 4: U* = C_bar^+ M R_bar^+ (FP64); step 5: F = C U*, A ~ F G^T
  launch_cur_middle(k1, k2, U1, V1, sig1, U2, V2, sig2, tol, M, d1, d2, X1, Y, X2, Ust, st);
  float* Uf = wsp<float>(ws, L.uw32);
  launch_f32_of(Ust, k1, k1, Uf, L.Kp, static_cast<int>(L.Kp), st);
  cabsk::OrthArgs a{};
  a.U = Cb; a.ldu = L.Kp; a.nu = m_loc; a.r = k1; a.TU = Uf; a.kp = L.Kp; a.Uo = F; a.lduo = ldf;
  launch_orth_apply_u(a, st);
  CABS_LAUNCH_CHECK("br_cur middle");
  if (Umid) CABS_CUDA_TRY(cudaMemcpyAsync(Umid, Ust, sizeof(double) * k1 * k1, cudaMemcpyDeviceToDevice, st));
  return CABS_OK;
}

int32_t cabs_holdout_errors(const cabs_plan* plan, const cabs_source* src, const int64_t* Hr, int32_t hr,
                            const int64_t* Hc, int32_t hc, const float* U, int64_t ldu, const float* s, const float* V,
                            int64_t ldv, int32_t r, double* errs, void* ws, size_t ws_bytes, const cabs_comm* comm,
                            void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_plan& p = *plan;
  if (multi(comm) || p.nranks > 1) return arg_error("holdout_errors: single rank only");
  CABS_TRY(check_source(p, src, "holdout_errors: bad source"));
  if (hr < 1 || hc < 1 || hr > p.kmax || hc > p.kmax || r < 1 || r > p.kmax) return arg_error("holdout_errors: bad sizes");
  if (!Hr || !Hc || !U || !V || !s || !errs || ldu < r || ldv < r) return arg_error("holdout_errors: bad buffers");
  cudaStream_t st = S(stream);
  float* Rb = wsp<float>(ws, L.rb);
  double* B = wsp<double>(ws, L.w64);
  float* Uh = wsp<float>(ws, L.uw32);
  float* Vh = wsp<float>(ws, L.vw32);
  double* Uh64 = wsp<double>(ws, L.a64);
  double* Vh64 = wsp<double>(ws, L.v64);
  // the validation block B = A(Hr, Hc) (FP64 copy of exact entries), U_H = U(Hr, :r), V_H = V(Hc, :r)
  src_rows(p, src, Hr, hr, Rb, L.ldrb, ws, st);
  launch_pick_cols(Rb, L.ldrb, hr, Hc, hc, hc, nullptr, 0, B, st);
  launch_pick_rows(U, ldu, Hr, hr, r, static_cast<int>(L.Kp), Uh, L.Kp, Uh64, st);
  launch_pick_rows(V, ldv, Hc, hc, r, static_cast<int>(L.Kp), Vh, L.Kp, Vh64, st);
  CABS_LAUNCH_CHECK("holdout gathers");
  cabsk::OrthArgs a{};
  a.U = Uh; a.ldu = L.Kp; a.nu = hr; a.V = Vh; a.ldv = L.Kp; a.nv = hc; a.r = r;
  a.part = wsp<double>(ws, L.orth_part);
  a.nblk = orth_gram_blocks(hr, hc, r);
  a.gram = reinterpret_cast<double*>(static_cast<unsigned char*>(ws) + L.orth);
  launch_orth_gram(a, st);  // U_H^T U_H, V_H^T V_H (exact FP64 products)
  launch_sweep(B, hr, hc, Vh64, Uh64, s, a.gram, r, a.part, errs, st);
  CABS_LAUNCH_CHECK("holdout sweep");
  return CABS_OK;
}

static int32_t lev_run(const cabs_plan* plan, const cabs_hard_problem* const* pr, const uint32_t* tags, int nprob,
                       uint64_t seed, void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  for (int q = 0; q < nprob; ++q) {
    if (!pr[q]) return arg_error("leverage_select: null problem");
    CABS_TRY(hard_check(plan, L, *pr[q]));
  }
  return hard_run(pr, nprob, ws, L, comm, stream, 1, seed, tags);
}

int32_t cabs_leverage_select(const cabs_plan* plan, const float* F, int64_t ldf, int64_t n_loc, int64_t n_glob,
                             int64_t row_off, int32_t r, int32_t k2, uint64_t seed, uint32_t tag, int64_t* reps,
                             double* keys, void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream) {
  const cabs_hard_problem p{F, ldf, n_loc, n_glob, row_off, r, k2, reps, keys};
  const cabs_hard_problem* pr[1] = {&p};
  return lev_run(plan, pr, &tag, 1, seed, ws, ws_bytes, comm, stream);
}

int32_t cabs_leverage_select_pair(const cabs_plan* plan, const cabs_hard_problem* a, const cabs_hard_problem* b,
                                  uint64_t seed, uint32_t tag_a, uint32_t tag_b, void* ws, size_t ws_bytes,
                                  const cabs_comm* comm, void* stream) {
  const cabs_hard_problem* pr[2] = {a, b};
  const uint32_t tags[2] = {tag_a, tag_b};
  return lev_run(plan, pr, tags, 2, seed, ws, ws_bytes, comm, stream);
}

// ---------------------------------------------------------------- S10
int32_t cabs_residual(const cabs_plan* plan, const cabs_source* src, const float* F, int64_t ldf, const float* s,
                      const float* G, int64_t ldg, int32_t ncomp, int64_t n_samples, uint64_t seed, double* out,
                      void* ws, size_t ws_bytes, const cabs_comm* comm, void* stream) {
  CABS_TRY(check_plan(plan));
  Ws L;
  CABS_TRY(check_ws(plan, ws, ws_bytes, &L));
  const cabs_plan& p = *plan;
  CABS_TRY(check_source(p, src, "residual: bad source"));
  if (!F || !G || !out || ncomp < 0 || ncomp > CABS_KMAX || ldf < ncomp || ldg < ncomp || n_samples < 0)
    return arg_error("residual: bad arguments");
  const int64_t m_loc = p.row_end - p.row_begin;
  if (n_samples > 0 && is_csr(src)) return arg_error("residual: the sampled estimate needs a dense or implicit source");
  if (n_samples > 0) {  // the sampled estimate (readings Z17 / Z23)
    if (p.m > (1ll << 32) || p.n > (1ll << 32)) return arg_error("residual: sampled dims must be <= 2^32");
    SampArgs a{};
    if (is_rbf(src)) a.rbf = rbf_of(src);
    else { a.A = src->a; a.lda = src->lda; a.transposed = src->transposed; }
    a.m = static_cast<uint64_t>(p.m);
    a.n = static_cast<uint64_t>(p.n);
    a.row_begin = p.row_begin;
    a.row_end = p.row_end;
    a.F = F; a.ldf = ldf; a.s = s; a.G = G; a.ldg = ldg; a.ncomp = ncomp;
    a.T = n_samples;
    a.seed = seed;
    launch_residual_sampled(a, wsp<double>(ws, L.res_part), out, S(stream));
    CABS_LAUNCH_CHECK("residual_sampled");
    CABS_TRY(comm_f64(comm, out, 2, stream));
    return CABS_OK;
  }
  if (is_rbf(src)) return arg_error("residual: the implicit source needs n_samples > 0");
  if (is_csr(src)) {
    if (!sparse_residual_supported(ncomp)) return arg_error("residual: sparse source needs ncomp <= 512");
    cabsk::OrthArgs ga{};
    ga.part = wsp<double>(ws, L.orth_part);
    ga.gram = reinterpret_cast<double*>(static_cast<unsigned char*>(ws) + L.orth);
    launch_residual_sparse(csr_of(src), m_loc, p.n, F, ldf, s, G, ldg, ncomp, ga, wsp<double>(ws, L.res_part), out,
                           S(stream));
    CABS_LAUNCH_CHECK("residual_sparse");
    CABS_TRY(comm_f64(comm, out, 2, stream));
    return CABS_OK;
  }
  // a column-major block is the row-major n x m_loc matrix A^T: ||A - F S G^T|| = ||A^T - G S F^T||,
  // so the same kernels run with the factors exchanged (res_split holds max(n, m_loc) rows)
  const bool tr = src->transposed != 0;
  const int64_t ra = tr ? p.n : m_loc, ca = tr ? m_loc : p.n;
  const float* Fa = tr ? G : F;
  const float* Ga = tr ? F : G;
  const int64_t ldfa = tr ? ldg : ldf, ldga = tr ? ldf : ldg;
  // a host-resident block (pinned, mapped) is read with plain loads over the interconnect, not by TMA
  if (!src->host_resident && residual_tc_supported(src->a, src->lda, ra, ca, ncomp)) {
    if (launch_residual_tc(src->a, src->lda, ra, ca, Fa, ldfa, s, Ga, ldga, ncomp, wsp<float>(ws, L.res_split),
                           wsp<double>(ws, L.res_part), out, S(stream)) != 0) {
      cabs_set_error_msg("residual: tensor map encoding failed");
      return CABS_ERR_CUDA;
    }
  } else {
    launch_residual(src->a, src->lda, ra, ca, Fa, ldfa, s, Ga, ldga, ncomp, wsp<double>(ws, L.res_part), out,
                    S(stream));
  }
  CABS_LAUNCH_CHECK("residual");
  CABS_TRY(comm_f64(comm, out, 2, stream));
  return CABS_OK;
}

int32_t cabs_residual_pairs(uint64_t seed, uint64_t t0, int64_t T, int64_t m, int64_t n, int64_t* i, int64_t* j,
                            void* stream) {
  if (T < 0 || m < 1 || n < 1 || m > (1ll << 32) || n > (1ll << 32) || (T > 0 && (!i || !j)))
    return arg_error("residual_pairs: bad arguments");
  launch_residual_pairs(seed, t0, T, m, n, i, j, S(stream));
  CABS_LAUNCH_CHECK("residual_pairs");
  return CABS_OK;
}

}  // extern "C"
