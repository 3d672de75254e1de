"""ctypes binding of libcabs.so -- argument marshalling only.

Every function here has the name of the C entry point it wraps (include/cabs.h)
and does nothing but convert torch tensors to (pointer, leading dimension) pairs,
call the library and raise on a non-zero status.  Every step of the CABS path
runs in the CUDA kernels of libcabs.so; there is no CPU fallback: if the library
is missing this module raises at import of the first call.
"""
from __future__ import annotations

import ctypes
import os

import torch

from . import build as _build

_LIB = None

c_i32, c_i64, c_u32, c_u64, c_f32, c_f64 = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32,
                                              ctypes.c_uint64, ctypes.c_float, ctypes.c_double)
c_vp, c_sz = ctypes.c_void_p, ctypes.c_size_t

STABILIZED = 0
PSEUDO_SKELETON = 1
WEIGHT_CONST = 0
WEIGHT_POWER = 1
KMAX = 1024

DEV_NONFINITE = 0x1
DEV_RANGE = 0x2
DEV_DUPLICATE = 0x4
DEV_SNAP_EXHAUSTED = 0x8
DEV_TOO_FEW_POINTS = 0x10
DEV_SVD_NOCONV = 0x20

TAG_PILOT_ROWS, TAG_PILOT_COLS, TAG_INIT_ROWS, TAG_INIT_COLS = 1, 2, 3, 4
TAG_LEVERAGE_ROWS, TAG_LEVERAGE_COLS = 6, 7
OP_KMEANS, OP_RESIDUAL, PATH_FFMA, PATH_TC, PATH_PRUNE = 0, 1, 0, 1, 2
ORTH_RMAX = 1024  # cabs_orthogonalize: largest supported r (= CABS_KMAX)


class CabsError(RuntimeError):
    pass


class Plan(ctypes.Structure):
    _fields_ = [("m", c_i64), ("n", c_i64), ("row_begin", c_i64), ("row_end", c_i64),
                ("col_begin", c_i64), ("col_end", c_i64), ("kmax", c_i32), ("rank", c_i32),
                ("nranks", c_i32)]

    @property
    def m_loc(self):
        return self.row_end - self.row_begin

    @property
    def n_sl(self):
        return self.col_end - self.col_begin


SOURCE_DENSE_F32 = 0
SOURCE_RBF_F32 = 1
SOURCE_CSR_F32 = 2


class Source(ctypes.Structure):
    _fields_ = [("a", c_vp), ("lda", c_i64), ("kind", c_i32), ("d", c_i32), ("x", c_vp), ("y", c_vp),
                ("ldx", c_i64), ("ldy", c_i64), ("inv_two_sigma2", c_f32),
                ("row_ptr", c_vp), ("col_idx", c_vp), ("row_val", c_vp), ("col_ptr", c_vp),
                ("row_idx", c_vp), ("col_val", c_vp), ("transposed", c_i32), ("host_resident", c_i32),
                ("at", c_vp), ("ldat", c_i64)]


class TransposedDense:
    """A dense row block held column-major (cabs.h: CABS_SOURCE_DENSE_F32 with transposed = 1, SURVEY
    H1): `At` is the device float32 tensor A^T of this rank's block, shape (n, m_loc), row-major with
    stride(0) >= m_loc.  Same results as the row-major block; the column gather reads contiguously."""

    def __init__(self, At):
        if At.dtype != torch.float32 or not At.is_cuda or At.dim() != 2 or (At.shape[1] > 1 and At.stride(1) != 1):
            raise TypeError("TransposedDense: a 2-D float32 CUDA tensor with unit column stride")
        self.At = At
        self.shape = (At.shape[1], At.shape[0])
        self.device = At.device


class HostDense:
    """A dense row-major row block that stays in pinned (page-locked, device-mapped) HOST memory
    (cabs.h: cabs_source.host_resident): the gathers read only the sampled rows and columns over the
    interconnect, the paper's linear access taken literally ("matrices which won't fit in
    the main memory").  A: pinned CPU float32 tensor (m_loc, n); At (optional): the same block held
    column-major too, a pinned (n, m_loc) tensor (cabs_source.at: contiguous column gathers); device:
    the CUDA device the kernels run on.  Results are those of the device-resident copy, bit for bit."""

    def __init__(self, A, device, At=None):
        for t in (A,) + ((At,) if At is not None else ()):
            if t.dtype != torch.float32 or t.is_cuda or not t.is_pinned() or t.dim() != 2 or t.stride(1) != 1:
                raise TypeError("HostDense: pinned 2-D float32 CPU tensors with unit column stride")
        if At is not None and tuple(At.shape) != (A.shape[1], A.shape[0]):
            raise ValueError("HostDense: At must be (n, m_loc)")
        self.A, self.At = A, At
        self.shape = tuple(A.shape)
        self.device = torch.device(device)


class DualDense:
    """A device-resident dense block in both layouts (cabs.h: cabs_source.a + cabs_source.at): A (m_loc, n)
    row-major and At (n, m_loc) = A^T row-major, the same values; row and column gathers both contiguous."""

    def __init__(self, A, At):
        for t in (A, At):
            if t.dtype != torch.float32 or not t.is_cuda or t.dim() != 2 or t.stride(1) != 1:
                raise TypeError("DualDense: 2-D float32 CUDA tensors with unit column stride")
        if tuple(At.shape) != (A.shape[1], A.shape[0]):
            raise ValueError("DualDense: At must be (n, m_loc)")
        self.A, self.At = A, At
        self.shape = tuple(A.shape)
        self.device = A.device


class RbfSource:
    """The implicit RBF matrix of BASELINE.json configs[4]: A_ij = exp(-|x_i - y_j|^2 / (2 sigma^2)),
    generated on access by the library (cabs.h CABS_SOURCE_RBF_F32).  x: device float32 (m, d) with
    ALL m points, y: device float32 (n, d); the tensors must outlive the calls."""

    def __init__(self, x, y, sigma):
        assert x.dtype == y.dtype == torch.float32 and x.is_cuda and y.is_cuda and x.shape[1] == y.shape[1]
        self.x, self.y = x.contiguous(), y.contiguous()
        self.sigma = float(sigma)
        self.inv_two_sigma2 = 1.0 / (2.0 * self.sigma * self.sigma)
        self.shape = (x.shape[0], y.shape[0])
        self.device = x.device


class CsrSource:
    """A sparse row block (cabs.h CABS_SOURCE_CSR_F32): CSR (row_ptr int64[m_loc+1],
    col_idx int32, row_val float32) and CSC of the same block (col_ptr int64[n+1], row_idx int32 local
    rows, col_val float32), device tensors that must outlive the calls.  shape = (m_loc, n)."""

    def __init__(self, row_ptr, col_idx, row_val, col_ptr, row_idx, col_val, n):
        for t, dt in ((row_ptr, torch.int64), (col_idx, torch.int32), (row_val, torch.float32),
                      (col_ptr, torch.int64), (row_idx, torch.int32), (col_val, torch.float32)):
            if t.dtype != dt or not t.is_contiguous():
                raise TypeError("CsrSource: int64 pointers, int32 indices, float32 values, contiguous")
        self.row_ptr, self.col_idx, self.row_val = row_ptr, col_idx, row_val
        self.col_ptr, self.row_idx, self.col_val = col_ptr, row_idx, col_val
        self.shape = (row_ptr.numel() - 1, int(n))
        self.device = row_ptr.device

    @property
    def nnz(self):
        return int(self.col_idx.numel())


def _source(A):
    """cabs_source for a dense row block (a torch tensor), an RbfSource or a CsrSource."""
    if isinstance(A, CsrSource):
        return Source(None, 0, SOURCE_CSR_F32, 0, None, None, 0, 0, 0.0, A.row_ptr.data_ptr(), A.col_idx.data_ptr(),
                      A.row_val.data_ptr(), A.col_ptr.data_ptr(), A.row_idx.data_ptr(), A.col_val.data_ptr())
    if isinstance(A, RbfSource):
        return Source(None, 0, SOURCE_RBF_F32, A.x.shape[1], A.x.data_ptr(), A.y.data_ptr(), A.x.stride(0),
                      A.y.stride(0), A.inv_two_sigma2)
    if isinstance(A, (HostDense, DualDense)):
        src = Source(A.A.data_ptr(), _ld(A.A), SOURCE_DENSE_F32, 0, None, None, 0, 0, 0.0)
        src.host_resident = 1 if isinstance(A, HostDense) else 0
        if A.At is not None:
            src.at, src.ldat = A.At.data_ptr(), _ld(A.At)
        return src
    if isinstance(A, TransposedDense):
        src = Source(A.At.data_ptr(), _ld(A.At), SOURCE_DENSE_F32, 0, None, None, 0, 0, 0.0)
        src.transposed = 1
        return src
    return Source(A.data_ptr(), _ld(A), SOURCE_DENSE_F32, 0, None, None, 0, 0, 0.0)


ALLREDUCE_FN = ctypes.CFUNCTYPE(c_i32, c_vp, c_i64, c_vp, c_vp)


class Comm(ctypes.Structure):
    _fields_ = [("rank", c_i32), ("nranks", c_i32), ("allreduce_f64", ALLREDUCE_FN),
                ("allreduce_f32", ALLREDUCE_FN), ("ctx", c_vp)]


class KmProblem(ctypes.Structure):
    """cabs_km_problem: one side (rows or columns) of cabs_kmeans_pair."""
    _fields_ = [("X", c_vp), ("ldx", c_i64), ("n_loc", c_i64), ("n_glob", c_i64), ("row_off", c_i64),
                ("d", c_i32), ("k2", c_i32), ("tag", c_i32), ("init_idx", c_vp), ("init_centres", c_vp),
                ("centres", c_vp), ("ldc", c_i64), ("labels", c_vp), ("cluster_w", c_vp), ("objective", c_vp),
                ("near_ties", c_vp), ("tie_log", c_vp), ("tie_log_cap", c_i32)]


class SelProblem(ctypes.Structure):
    """cabs_sel_problem: one side (rows or columns) of cabs_select_pair."""
    _fields_ = [("X", c_vp), ("ldx", c_i64), ("n_loc", c_i64), ("n_glob", c_i64), ("row_off", c_i64),
                ("d", c_i32), ("centres", c_vp), ("ldc", c_i64), ("k2", c_i32), ("cluster_w", c_vp),
                ("reps", c_vp), ("rep_of_centre", c_vp), ("gap", c_vp)]


class HardProblem(ctypes.Structure):
    """cabs_hard_problem: one side (rows or columns) of cabs_hard_select_pair."""
    _fields_ = [("X", c_vp), ("ldx", c_i64), ("n_loc", c_i64), ("n_glob", c_i64), ("row_off", c_i64),
                ("d", c_i32), ("k2", c_i32), ("reps", c_vp), ("keys", c_vp)]


_SIGS = {
    "cabs_status_string": (ctypes.c_char_p, [c_i32]),
    "cabs_last_error_string": (ctypes.c_char_p, []),
    "cabs_version": (None, [ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]),
    "cabs_padded_ld": (c_i64, [c_i32]),
    "cabs_launch_count": (c_i64, []),
    "cabs_kernel_path": (c_i32, [c_i32, c_i32, c_i32]),
    "cabs_debug_counters": (c_i32, [ctypes.POINTER(c_i64), c_i32]),
    "cabs_workspace_bytes": (c_sz, [ctypes.POINTER(Plan)]),
    "cabs_clear_status": (c_i32, [c_vp, c_vp]),
    "cabs_device_status": (c_i32, [c_vp, c_vp, ctypes.POINTER(c_u32)]),
    "cabs_pilot": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(Source), c_i32, c_u64, c_vp, c_vp,
                           c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_pilot_embed": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(Source), c_i32, c_u64, c_vp, c_vp,
                                 c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i32, c_f64, c_vp, c_i64, c_vp, c_i64,
                                 c_vp, c_vp, c_vp, c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_embed": (c_i32, [ctypes.POINTER(Plan), c_i32, c_vp, c_i64, c_vp, c_i64, c_vp, c_i64, c_i32,
                           c_f64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_sz,
                           ctypes.POINTER(Comm), c_vp]),
    "cabs_kmeans": (c_i32, [ctypes.POINTER(Plan), c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_i32,
                            c_i32, c_f32, c_u64, c_i32, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_vp,
                            c_vp, c_i32, c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_kmeans_pair": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(KmProblem), ctypes.POINTER(KmProblem), c_i32,
                                 c_i32, c_f32, c_u64, c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_select": (c_i32, [ctypes.POINTER(Plan), c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_vp, c_i64,
                            c_i32, c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_select_pair": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(SelProblem), ctypes.POINTER(SelProblem), c_vp,
                                 c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_hard_select": (c_i32, [ctypes.POINTER(Plan), c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_vp,
                                 c_vp, c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_hard_select_pair": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(HardProblem),
                                      ctypes.POINTER(HardProblem), c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_br_cur": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(Source), c_i32, c_vp, c_vp, c_i32, c_vp, c_vp,
                            ctypes.c_double, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp, ctypes.c_size_t, c_vp, c_vp]),
    "cabs_holdout_errors": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(Source), c_vp, c_i32, c_vp, c_i32, c_vp,
                                    c_i64, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp, ctypes.c_size_t, c_vp, c_vp]),
    "cabs_orthogonalize": (c_i32, [ctypes.POINTER(Plan), c_i32, c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_i64, c_vp,
                                   c_vp, c_i64, c_vp, c_vp, c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_leverage_select": (c_i32, [ctypes.POINTER(Plan), c_vp, c_i64, c_i64, c_i64, c_i64, c_i32, c_i32, c_u64,
                                     c_u32, c_vp, c_vp, c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_leverage_select_pair": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(HardProblem),
                                          ctypes.POINTER(HardProblem), c_u64, c_u32, c_u32, c_vp, c_sz,
                                          ctypes.POINTER(Comm), c_vp]),
    "cabs_sketch": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(Source), c_vp, c_vp, c_i32, c_i32, c_f64,
                            c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp, c_sz,
                            ctypes.POINTER(Comm), c_vp]),
    "cabs_residual": (c_i32, [ctypes.POINTER(Plan), ctypes.POINTER(Source), c_vp, c_i64, c_vp, c_vp, c_i64,
                              c_i32, c_i64, c_u64, c_vp, c_vp, c_sz, ctypes.POINTER(Comm), c_vp]),
    "cabs_philox_blocks": (c_i32, [c_u64, c_u32, c_u64, c_i64, c_vp, c_vp]),
    "cabs_uniform_indices": (c_i32, [c_i64, c_i32, c_u64, c_u32, c_vp, c_vp]),
    "cabs_residual_pairs": (c_i32, [c_u64, c_u64, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "cabs_svd": (c_i32, [ctypes.POINTER(Plan), c_i32, c_vp, c_i64, c_f64, c_vp, c_vp, c_vp, c_vp, c_vp,
                         c_sz, c_vp]),
}


def lib_path() -> str:
    return _build.LIB


def load(build_if_stale: bool = False):
    """Load libcabs.so (in-tree).  Raises if it is missing: there is no fallback."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if build_if_stale:
        _build.build()
    path = lib_path()
    if not os.path.exists(path):
        raise CabsError(f"libcabs.so not found at {path}: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(path)
    for name, (res, args) in _SIGS.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _LIB = L
    return L


def exported_symbols():
    return list(_SIGS)


def _check(status: int, what: str):
    if status != 0:
        L = load()
        raise CabsError(f"{what}: {L.cabs_status_string(status).decode()} "
                        f"({L.cabs_last_error_string().decode()})")


def _p(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _ld(t):
    if t.dim() == 1:
        return t.shape[0]
    assert t.stride(1) == 1, "row-major tensors only"
    return t.stride(0)


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _comm(comm):
    return None if comm is None else ctypes.byref(comm.c)


# ---------------------------------------------------------------- utilities
def cabs_padded_ld(k: int) -> int:
    return int(load().cabs_padded_ld(int(k)))


def cabs_workspace_bytes(plan: Plan) -> int:
    n = int(load().cabs_workspace_bytes(ctypes.byref(plan)))
    if n == 0:
        raise CabsError("invalid plan")
    return n


def cabs_debug_counters(n=16):
    buf = (c_i64 * n)()
    _check(load().cabs_debug_counters(buf, n), "cabs_debug_counters")
    return list(buf)


def cabs_launch_count() -> int:
    return int(load().cabs_launch_count())


def cabs_kernel_path(op: int, k: int, d: int = 0) -> int:
    return int(load().cabs_kernel_path(op, k, d))


def cabs_kmeans_path(k2: int, d: int) -> str:
    """'prune', 'tc' or 'ffma': the k-means kernel cabs_kmeans(_pair) runs for (k2, d)."""
    return {PATH_PRUNE: "prune", PATH_TC: "tc"}.get(cabs_kernel_path(OP_KMEANS, k2, d), "ffma")


def cabs_residual_path(ncomp: int) -> str:
    return "tc" if cabs_kernel_path(OP_RESIDUAL, ncomp) == PATH_TC else "ffma"


def cabs_version():
    a, b = c_i32(), c_i32()
    load().cabs_version(ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def cabs_clear_status(ws, stream=None):
    _check(load().cabs_clear_status(_p(ws), _stream(stream)), "cabs_clear_status")


def cabs_device_status(ws, stream=None) -> int:
    f = c_u32()
    _check(load().cabs_device_status(_p(ws), _stream(stream), ctypes.byref(f)), "cabs_device_status")
    return f.value


# ---------------------------------------------------------------- entry points
def cabs_pilot(plan, A, k, seed, I, J, C, R, W, ws, comm=None, stream=None):
    src = _source(A)
    _check(load().cabs_pilot(ctypes.byref(plan), ctypes.byref(src), int(k), int(seed), _p(I), _p(J),
                             _p(C), _ld(C), _p(R), _ld(R), _p(W), _ld(W), _p(ws), ws.numel(),
                             _comm(comm), _stream(stream)), "cabs_pilot")


def cabs_pilot_embed(plan, A, k, seed, I, J, C, R, W, mode, tol, P, Q, s, r, ws, sigma=None, comm=None,
                     stream=None):
    src = _source(A)
    _check(load().cabs_pilot_embed(ctypes.byref(plan), ctypes.byref(src), int(k), int(seed), _p(I), _p(J),
                                   _p(C), _ld(C), _p(R), _ld(R), _p(W), _ld(W), int(mode), float(tol),
                                   _p(P), _ld(P), _p(Q), _ld(Q), _p(s), _p(r), _p(sigma), _p(ws), ws.numel(),
                                   _comm(comm), _stream(stream)), "cabs_pilot_embed")


def cabs_embed(plan, k, C, R, W, mode, tol, P, Q, s, r, ws, sigma=None, comm=None, stream=None):
    _check(load().cabs_embed(ctypes.byref(plan), int(k), _p(C), _ld(C), _p(R), _ld(R), _p(W), _ld(W),
                             int(mode), float(tol), _p(P), _ld(P), _p(Q), _ld(Q), _p(s), _p(r),
                             _p(sigma), _p(ws), ws.numel(), _comm(comm), _stream(stream)), "cabs_embed")


def cabs_kmeans(plan, X, n_loc, n_glob, row_off, d, k2, iters, weight_kind, weight_p, seed, tag,
                centres, labels, cluster_w, objective, ws, near_ties=None, init_idx=None,
                init_centres=None, comm=None, stream=None, tie_log=None):
    _check(load().cabs_kmeans(ctypes.byref(plan), _p(X), _ld(X), int(n_loc), int(n_glob), int(row_off),
                              int(d), int(k2), int(iters), int(weight_kind), float(weight_p), int(seed),
                              int(tag), _p(init_idx), _p(init_centres), _p(centres), _ld(centres),
                              _p(labels), _p(cluster_w), _p(objective), _p(near_ties), _p(tie_log),
                              tie_log_cap(tie_log), _p(ws), ws.numel(), _comm(comm), _stream(stream)), "cabs_kmeans")


def tie_log_cap(tie_log):
    """Entries a near-tie log buffer holds (int32[1 + 5 cap])."""
    return 0 if tie_log is None else (tie_log.numel() - 1) // 5


def new_tie_log(cap, device):
    return torch.zeros(1 + 5 * cap, dtype=torch.int32, device=device)


def read_tie_log(tie_log):
    """Host list of (iteration, point, nearest centre, runner-up centre, relative gap) and the
    total count of near ties seen (which may exceed the stored entries)."""
    import struct
    v = tie_log.cpu().tolist()
    n = min(v[0], tie_log_cap(tie_log))
    out = []
    for q in range(n):
        it, p, j1, j2, gb = v[1 + 5 * q:6 + 5 * q]
        out.append((it, p, j1, j2, struct.unpack("<f", struct.pack("<i", gb))[0]))
    return sorted(out), v[0]


def km_problem(X, n_loc, n_glob, row_off, d, k2, tag, centres, labels, cluster_w, objective, near_ties=None,
               init_idx=None, init_centres=None, tie_log=None):
    """Describe one side of cabs_kmeans_pair (tensors must outlive the call)."""
    def ptr(t):
        return None if t is None else t.data_ptr()
    return KmProblem(ptr(X), _ld(X), int(n_loc), int(n_glob), int(row_off), int(d), int(k2), int(tag), ptr(init_idx),
                     ptr(init_centres), ptr(centres), _ld(centres), ptr(labels), ptr(cluster_w), ptr(objective),
                     ptr(near_ties), ptr(tie_log), tie_log_cap(tie_log))


def cabs_kmeans_pair(plan, a, b, iters, weight_kind, weight_p, seed, ws, comm=None, stream=None):
    _check(load().cabs_kmeans_pair(ctypes.byref(plan), ctypes.byref(a), ctypes.byref(b), int(iters),
                                   int(weight_kind), float(weight_p), int(seed), _p(ws), ws.numel(), _comm(comm),
                                   _stream(stream)), "cabs_kmeans_pair")


def cabs_select(plan, X, n_loc, n_glob, row_off, d, centres, k2, cluster_w, reps, ws,
                rep_of_centre=None, gap=None, comm=None, stream=None):
    _check(load().cabs_select(ctypes.byref(plan), _p(X), _ld(X), int(n_loc), int(n_glob), int(row_off),
                              int(d), _p(centres), _ld(centres), int(k2), _p(cluster_w), _p(reps),
                              _p(rep_of_centre), _p(gap), _p(ws), ws.numel(), _comm(comm),
                              _stream(stream)), "cabs_select")


def sel_problem(X, n_loc, n_glob, row_off, d, centres, k2, cluster_w, reps, rep_of_centre=None, gap=None):
    """Describe one side of cabs_select_pair (tensors must outlive the call)."""
    def ptr(t):
        return None if t is None else t.data_ptr()
    return SelProblem(ptr(X), _ld(X), int(n_loc), int(n_glob), int(row_off), int(d), ptr(centres), _ld(centres),
                      int(k2), ptr(cluster_w), ptr(reps), ptr(rep_of_centre), ptr(gap))


def cabs_select_pair(plan, a, b, ws, comm=None, stream=None):
    _check(load().cabs_select_pair(ctypes.byref(plan), ctypes.byref(a), ctypes.byref(b), _p(ws), ws.numel(),
                                   _comm(comm), _stream(stream)), "cabs_select_pair")


def cabs_hard_select(plan, X, n_loc, n_glob, row_off, d, k2, reps, ws, keys=None, comm=None, stream=None):
    _check(load().cabs_hard_select(ctypes.byref(plan), _p(X), _ld(X), int(n_loc), int(n_glob), int(row_off),
                                   int(d), int(k2), _p(reps), _p(keys), _p(ws), ws.numel(), _comm(comm),
                                   _stream(stream)), "cabs_hard_select")


def hard_problem(X, n_loc, n_glob, row_off, d, k2, reps, keys=None):
    """Describe one side of cabs_hard_select_pair (tensors must outlive the call)."""
    def ptr(t):
        return None if t is None else t.data_ptr()
    return HardProblem(ptr(X), _ld(X), int(n_loc), int(n_glob), int(row_off), int(d), int(k2), ptr(reps), ptr(keys))


def cabs_hard_select_pair(plan, a, b, ws, comm=None, stream=None):
    _check(load().cabs_hard_select_pair(ctypes.byref(plan), ctypes.byref(a), ctypes.byref(b), _p(ws), ws.numel(),
                                        _comm(comm), _stream(stream)), "cabs_hard_select_pair")


def cabs_orthogonalize(plan, r, U, s, V, Uo, so, Vo, ws, r_out=None, sigma=None, comm=None, stream=None):
    _check(load().cabs_orthogonalize(ctypes.byref(plan), int(r), _p(U), _ld(U), _p(s), _p(V), _ld(V), _p(Uo), _ld(Uo),
                                     _p(so), _p(Vo), _ld(Vo), _p(r_out), _p(sigma), _p(ws), ws.numel(), _comm(comm),
                                     _stream(stream)), "cabs_orthogonalize")


def cabs_leverage_select(plan, F, n_loc, n_glob, row_off, r, k2, seed, tag, reps, ws, keys=None, comm=None,
                         stream=None):
    _check(load().cabs_leverage_select(ctypes.byref(plan), _p(F), _ld(F), int(n_loc), int(n_glob), int(row_off),
                                       int(r), int(k2), int(seed), int(tag), _p(reps), _p(keys), _p(ws), ws.numel(),
                                       _comm(comm), _stream(stream)), "cabs_leverage_select")


def cabs_leverage_select_pair(plan, a, b, seed, tag_a, tag_b, ws, comm=None, stream=None):
    _check(load().cabs_leverage_select_pair(ctypes.byref(plan), ctypes.byref(a), ctypes.byref(b), int(seed),
                                            int(tag_a), int(tag_b), _p(ws), ws.numel(), _comm(comm),
                                            _stream(stream)), "cabs_leverage_select_pair")


def cabs_sketch(plan, A, Ir, Ic, k, mode, tol, U, s, V, r, ws, sigma=None, comm=None, stream=None):
    src = _source(A)
    _check(load().cabs_sketch(ctypes.byref(plan), ctypes.byref(src), _p(Ir), _p(Ic), int(k), int(mode),
                              float(tol), _p(U), _ld(U), _p(s), _p(V), _ld(V), _p(r), _p(sigma), _p(ws),
                              ws.numel(), _comm(comm), _stream(stream)), "cabs_sketch")


def cabs_residual(plan, A, F, s, G, ncomp, out, ws, comm=None, stream=None, n_samples=0, seed=0):
    """n_samples = 0: exact sums (dense A); n_samples > 0: the sampled estimate (cabs.h)."""
    src = _source(A)
    _check(load().cabs_residual(ctypes.byref(plan), ctypes.byref(src), _p(F), _ld(F), _p(s), _p(G),
                                _ld(G), int(ncomp), int(n_samples), int(seed), _p(out), _p(ws), ws.numel(),
                                _comm(comm), _stream(stream)), "cabs_residual")


def cabs_residual_pairs(seed, t0, T, m, n, i, j, stream=None):
    _check(load().cabs_residual_pairs(int(seed), int(t0), int(T), int(m), int(n), _p(i), _p(j), _stream(stream)),
           "cabs_residual_pairs")


# ---------------------------------------------------------------- test hooks
def cabs_philox_blocks(seed, tag, start, count, out, stream=None):
    _check(load().cabs_philox_blocks(int(seed), int(tag), int(start), int(count), _p(out), _stream(stream)),
           "cabs_philox_blocks")


def cabs_uniform_indices(N, k, seed, tag, out, stream=None):
    _check(load().cabs_uniform_indices(int(N), int(k), int(seed), int(tag), _p(out), _stream(stream)),
           "cabs_uniform_indices")


def cabs_svd(plan, k, W, tol, sigma, Uw, Vw, r, ws, stream=None):
    _check(load().cabs_svd(ctypes.byref(plan), int(k), _p(W), _ld(W), float(tol), _p(sigma), _p(Uw),
                           _p(Vw), _p(r), _p(ws), ws.numel(), _stream(stream)), "cabs_svd")


def cabs_br_cur(plan, A, k1, Ibr, Ibc, k2, Itr, Itc, F, G, ws, tol=1e-12, Umid=None, comm=None, stream=None):
    """BR-CUR (Algorithm 1): A ~ F G^T with F = C U*, G = R^T (cabs.h cabs_br_cur)."""
    src = _source(A)
    _check(load().cabs_br_cur(ctypes.byref(plan), ctypes.byref(src), int(k1), _p(Ibr), _p(Ibc), int(k2), _p(Itr),
                              _p(Itc), float(tol), _p(F), _ld(F), _p(G), _ld(G), _p(Umid), _p(ws), ws.numel(),
                              _comm(comm), _stream(stream)), "cabs_br_cur")


def cabs_holdout_errors(plan, A, Hr, Hc, U, s, V, r, errs, ws, comm=None, stream=None):
    """Rank sweep on the validation block A(Hr, Hc): errs[rho], rho = 0..r (cabs.h cabs_holdout_errors)."""
    src = _source(A)
    _check(load().cabs_holdout_errors(ctypes.byref(plan), ctypes.byref(src), _p(Hr), int(Hr.numel()), _p(Hc),
                                      int(Hc.numel()), _p(U), _ld(U), _p(s), _p(V), _ld(V), int(r), _p(errs), _p(ws),
                                      ws.numel(), _comm(comm), _stream(stream)), "cabs_holdout_errors")
