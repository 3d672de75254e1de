"""GPU parity of the leverage-score follow-up (P:312 variant (e)): the
orthogonalization (Supp. section 3) against the oracle's literal two-SVD recipe, the
Efraimidis-Spirakis keys and the sampled index sets against the oracle (Z27: a swap is
excused only at a boundary whose oracle keys are within a relative 1e-12, the `log` ulp),
and the end-to-end variant."""
import math

import numpy as np
import pytest
import torch

from oracle import cabs as O
from oracle import rng
from tests.helpers import NEAR_TIE, align_signs, rel_fro

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1607_07395_b200.cabs")
LOG_TIE = 1e-12


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    C.load()
    return torch.device("cuda:0")


def _pad(dev, X, ld):
    t = torch.zeros((max(X.shape[0], 1), ld), device=dev)
    t[:X.shape[0], :X.shape[1]] = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(dev)
    return t


def _separated_factors(g, m, n, r):
    """U, s, V with U diag(s) V^T = X diag(sig) Y^T, X, Y orthonormal and sig geometric (relative
    gaps 1%: the singular vectors are well determined at any r), U = X B for a well-conditioned
    random B, so U^T U is a full (non-identity) Gram matrix."""
    X = np.linalg.qr(g.standard_normal((m, r)))[0]
    Y = np.linalg.qr(g.standard_normal((n, r)))[0]
    sig = 3.0 * 0.99 ** np.arange(r)
    B = np.eye(r) + 0.3 * g.standard_normal((r, r)) / np.sqrt(r)
    s = g.uniform(0.5, 2.0, r)
    U = X @ B
    V = (Y * sig) @ np.linalg.inv(B).T / s
    return U.astype(np.float32), s.astype(np.float32), V.astype(np.float32)


@pytest.mark.parametrize("m,n,r,zero_cols", [(1000, 700, 20, 0), (20000, 10000, 50, 0), (777, 333, 64, 0),
                                             (100, 50, 1, 0), (3000, 2000, 10, 3), (5000, 3000, 100, 0),
                                             (100000, 50000, 100, 0), (4000, 2500, 200, 7), (3000, 2000, 300, 0),
                                             (2000, 1000, 230, 0)])
def test_orthogonalize_matches_oracle(dev, m, n, r, zero_cols):
    """r <= 64 with Gaussian factors; r >= 100 with well-separated singular values (r = 230, 300
    take the global-memory Cholesky)."""
    from paper_1607_07395_b200.dist import make_plan
    g = np.random.default_rng(m + r)
    if r < 100:
        U = g.standard_normal((m, r)).astype(np.float32)
        V = g.standard_normal((n, r)).astype(np.float32)
        s = g.uniform(0.2, 3.0, r).astype(np.float32)
    else:
        U, s, V = _separated_factors(g, m, n, r)
    if zero_cols:
        U[:, r - zero_cols:] = 0
        V[:, r - zero_cols:] = 0
    plan = make_plan(m, n, max(64, r))
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(r)
    Ut, Vt = _pad(dev, U, ld), _pad(dev, V, ld)
    Uo, Vo = torch.full((m, ld), 7.0, device=dev), torch.full((n, ld), 7.0, device=dev)
    so = torch.zeros(r, device=dev)
    ro = torch.zeros(1, dtype=torch.int32, device=dev)
    C.cabs_orthogonalize(plan, r, Ut, torch.from_numpy(s).to(dev), Vt, Uo, so, Vo, ws, r_out=ro)
    torch.cuda.synchronize()
    ref_U, ref_s, ref_V = O.orthogonalize(U[:, :r - zero_cols] if zero_cols else U, s[:r - zero_cols] if zero_cols
                                          else s, V[:, :r - zero_cols] if zero_cols else V)
    rk = int(ro.item())
    assert rk == ref_s.size
    so_h = so.cpu().numpy().astype(np.float64)
    assert np.allclose(so_h[:rk], ref_s, rtol=2e-5)
    assert np.all(so_h[rk:] == 0)
    Uh, Vh = Uo.cpu().numpy().astype(np.float64), Vo.cpu().numpy().astype(np.float64)
    assert np.all(Uh[:, rk:] == 0) and np.all(Vh[:, rk:] == 0)  # padding written as zeros
    # well-separated singular values: the vectors are unique up to sign
    assert rel_fro(align_signs(Uh[:, :rk], ref_U), ref_U) < 1e-4
    assert rel_fro(align_signs(Vh[:, :rk], ref_V), ref_V) < 1e-4
    assert np.abs(Uh[:, :rk].T @ Uh[:, :rk] - np.eye(rk)).max() < 1e-5
    assert np.abs(Vh[:, :rk].T @ Vh[:, :rk] - np.eye(rk)).max() < 1e-5


def _oracle_keys(F, seed, tag, off=0):
    r = F.shape[1]
    u = rng.uniform01(seed, tag, np.arange(off, off + F.shape[0]))
    return (O.row_sq_norms(F) / r) / -np.log(u)


def _same_or_log_tie(got, want, keys, k):
    if got == want:
        return True
    ks = np.sort(keys)[::-1]
    return k < ks.size and (ks[k - 1] - ks[k]) / ks[k - 1] < LOG_TIE


@pytest.mark.parametrize("N,r,k2,off", [(50, 5, 5, 0), (1000, 20, 50, 0), (20000, 50, 50, 17), (100003, 30, 200, 0),
                                        (3000, 8, 1000, 5)])
def test_leverage_keys_and_sample(dev, N, r, k2, off):
    from paper_1607_07395_b200.dist import make_plan
    g = np.random.default_rng(N)
    F, _ = np.linalg.qr(g.standard_normal((N, r)))
    F = F.astype(np.float32)
    n_glob = N + off
    plan = make_plan(n_glob, n_glob, 1024)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    Ft = _pad(dev, F, C.cabs_padded_ld(r))
    reps = torch.zeros(k2, dtype=torch.int64, device=dev)
    keys = torch.zeros(N, dtype=torch.float64, device=dev)
    C.cabs_leverage_select(plan, Ft, N, n_glob, off, r, k2, 11, C.TAG_LEVERAGE_ROWS, reps, ws, keys=keys)
    torch.cuda.synchronize()
    want_keys = _oracle_keys(F, 11, rng.TAG_LEVERAGE_ROWS, off)
    got_keys = keys.cpu().numpy()
    assert np.allclose(got_keys, want_keys, rtol=1e-15, atol=0)  # log: last-ulp differences only
    want = (O.hard_threshold_select(want_keys, k2) + off).tolist()
    assert _same_or_log_tie(reps.cpu().tolist(), want, want_keys, k2)


def test_leverage_pair_and_spec_example(dev):
    from paper_1607_07395_b200.dist import make_plan
    plan = make_plan(6, 6, 64)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    F = np.zeros((6, 2), np.float32)
    F[0, 0] = F[1, 1] = 1.0  # rows e1, e2 -> {0, 1}
    Ft = _pad(dev, F, 32)
    ra, rb = torch.zeros(2, dtype=torch.int64, device=dev), torch.zeros(2, dtype=torch.int64, device=dev)
    a = C.hard_problem(Ft, 6, 6, 0, 2, 2, ra)
    b = C.hard_problem(Ft, 6, 6, 0, 2, 2, rb)
    C.cabs_leverage_select_pair(plan, a, b, 5, C.TAG_LEVERAGE_ROWS, C.TAG_LEVERAGE_COLS, ws)
    torch.cuda.synchronize()
    assert ra.cpu().tolist() == [0, 1] and rb.cpu().tolist() == [0, 1]


@pytest.mark.parametrize("name,m,n,k,seed", [("c1", 2000, 1500, 20, 0), ("c2", 4000, 2000, 50, 1),
                                             ("c3", 8000, 4000, 100, 2)])
def test_e2e_leverage_followup(dev, name, m, n, k, seed):
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    from workloads import CONFIGS, make_A, scaled
    cfg = scaled(CONFIGS[name], m, n, k1=k, k2=k, iters=5, seed=seed)
    A_t = make_A(cfg, device=dev)
    A = A_t.cpu().numpy()
    pipe = CabsPipeline(A_t, m, n, CabsConfig(k, k, 5, seed=seed, followup="leverage"))
    pipe.run()
    g = pipe.results()
    ref = O.cabs_run(A, k, k, 5, seed=seed, followup="leverage")
    r_o = int(pipe.ro.item())
    Uo_ref, so_ref, Vo_ref = O.orthogonalize(ref.pilot.U, ref.pilot.s, ref.pilot.V)
    assert r_o == so_ref.size
    Uo = pipe.Uo.cpu().numpy()[:, :r_o].astype(np.float64)
    assert rel_fro(align_signs(Uo, Uo_ref), Uo_ref) < 1e-3
    assert np.allclose(pipe.so.cpu().numpy()[:r_o], so_ref, rtol=1e-4)
    # the GPU's decision on its own orthogonal factor is the oracle's up to the log ulp
    for side, F_g, got, tag in (("rows", Uo, g["Ib"], rng.TAG_LEVERAGE_ROWS),
                                ("cols", pipe.Vo.cpu().numpy()[:, :r_o].astype(np.float64), g["Jb"],
                                 rng.TAG_LEVERAGE_COLS)):
        kf = _oracle_keys(F_g.astype(np.float32).astype(np.float64), seed, tag)
        assert _same_or_log_tie(got.numpy().tolist(), O.hard_threshold_select(kf, k).tolist(), kf, k), side
    # against the FP64 oracle: equal unless the FP32 factor moved a boundary key by < NEAR_TIE
    for got, want, F_ref, tag in ((g["Ib"], ref.Ibar, Uo_ref, rng.TAG_LEVERAGE_ROWS),
                                  (g["Jb"], ref.Jbar, Vo_ref, rng.TAG_LEVERAGE_COLS)):
        if not np.array_equal(got.numpy(), want):
            ks = np.sort(_oracle_keys(F_ref, seed, tag))[::-1]
            assert (ks[k - 1] - ks[k]) / ks[k - 1] < NEAR_TIE
    if np.array_equal(g["Ib"].numpy(), ref.Ibar) and np.array_equal(g["Jb"].numpy(), ref.Jbar):
        a = math.sqrt(ref.a_sq)
        rg, ro = math.sqrt(max(g["resid_sq"], 0)), math.sqrt(ref.resid_sq)
        assert abs(rg - ro) <= 1e-4 * ro + 1e-6 * a, (rg, ro)


def test_orthogonalize_two_ranks_match_one(dev):
    """Row-sharded U and column-sliced V on two ranks (host-rendezvous allreduce, see
    test_gpu_hard): every rank's rows of Uo / Vo equal the single-rank result."""
    import threading
    from paper_1607_07395_b200.dist import make_plan
    from tests.test_gpu_hard import _HostRendezvousComm
    g = np.random.default_rng(21)
    m, n, r = 3001, 1999, 12
    U = g.standard_normal((m, r)).astype(np.float32)
    V = g.standard_normal((n, r)).astype(np.float32)
    s = torch.from_numpy(g.uniform(0.5, 2.0, r).astype(np.float32)).to(dev)
    ld = C.cabs_padded_ld(r)
    plan1 = make_plan(m, n, 64)
    ws1 = torch.zeros(C.cabs_workspace_bytes(plan1), dtype=torch.uint8, device=dev)
    Uo1, Vo1, so1 = torch.zeros((m, ld), device=dev), torch.zeros((n, ld), device=dev), torch.zeros(r, device=dev)
    C.cabs_orthogonalize(plan1, r, _pad(dev, U, ld), s, _pad(dev, V, ld), Uo1, so1, Vo1, ws1)
    torch.cuda.synchronize()
    rc = _HostRendezvousComm(2, dev)
    out, errs = [None, None], []

    def rank_main(k):
        try:
            p = make_plan(m, n, 64, k, 2)
            ws = torch.zeros(C.cabs_workspace_bytes(p), dtype=torch.uint8, device=dev)
            Ul, Vl = _pad(dev, U[p.row_begin:p.row_end], ld), _pad(dev, V[p.col_begin:p.col_end], ld)
            Uo, Vo = torch.zeros((max(p.m_loc, 1), ld), device=dev), torch.zeros((max(p.n_sl, 1), ld), device=dev)
            so = torch.zeros(r, device=dev)
            st = torch.cuda.Stream(device=dev)
            st.wait_stream(torch.cuda.current_stream(dev))  # inputs were written on the thread's default stream
            with torch.cuda.stream(st):
                C.cabs_orthogonalize(p, r, Ul, s, Vl, Uo, so, Vo, ws, comm=rc.comms[k], stream=st)
            st.synchronize()
            out[k] = (p, Uo.cpu(), Vo.cpu(), so.cpu())
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=rank_main, args=(k,)) for k in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    for p, Uo, Vo, so in out:
        assert torch.allclose(so, so1.cpu(), rtol=1e-6)
        # the Gram sums differ only in association across ranks: agreement to FP32 rounding
        assert torch.allclose(Uo[:p.m_loc], Uo1.cpu()[p.row_begin:p.row_end], atol=1e-5)
        assert torch.allclose(Vo[:p.n_sl], Vo1.cpu()[p.col_begin:p.col_end], atol=1e-5)
