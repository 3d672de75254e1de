"""Multi-rank paths on ONE GPU: ranks are host threads with their own streams, joined by the
host-rendezvous comm (tests/rendezvous.py), so no kernel ever waits on another rank's kernel.

P15: the whole CabsPipeline at nranks = 2 against nranks = 1 on the same A
(uneven row split, and a split that leaves one rank without rows): pilot indices bit-exact, the
k-means labels and representatives bit-exact except at points either run logs as near ties,
embeddings and follow-up factors within 1e-5, the residual within 1e-6 ||A||_F^2.

The snap's multi-rank candidate exchange: equal to the single-rank snap, including the exact
distributed greedy pass a rank falls back to when the exchanged lists run out (duplicate-heavy
inputs), checked against the FP64 oracle's snap.
"""
import numpy as np
import pytest
import torch

from oracle import cabs as O
from tests.helpers import NEAR_TIE, align_signs, rel_fro
from tests.rendezvous import HostRendezvousComm, run_ranks

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1607_07395_b200.cabs")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    C.load()
    return torch.device("cuda:0")


def _A(m, n, seed, dev):
    """A = G1 diag(1/i) G2^T + 0.01 N (the c1 recipe) at another size, FP32."""
    g = np.random.default_rng(seed)
    r = 24
    A = (g.standard_normal((m, r)) / np.arange(1, r + 1)) @ g.standard_normal((r, n)) + 0.01 * g.standard_normal((m, n))
    return torch.from_numpy(A.astype(np.float32)).to(dev)


def _pipelines(A, cfg, nranks, align, dev):
    from paper_1607_07395_b200.dist import make_plan
    from paper_1607_07395_b200.pipeline import CabsPipeline
    m, n = A.shape
    rc = HostRendezvousComm(nranks, dev)

    def rank(r):
        plan = make_plan(m, n, max(cfg.k1, cfg.k2), r, nranks, align)
        st = torch.cuda.Stream(device=dev)
        st.wait_stream(torch.cuda.current_stream(dev))  # inputs were written on the thread's default stream
        with torch.cuda.stream(st):
            A_loc = A[plan.row_begin:plan.row_end].contiguous()
            pipe = CabsPipeline(A_loc, m, n, cfg, r, nranks, comm=rc.comms[r], plan=plan)
            pipe.run()
        st.synchronize()
        with torch.cuda.stream(st):
            return plan, pipe.results()

    return run_ranks(nranks, rank), rc


def _tie_points(res_list, side):
    pts = set()
    for g in res_list:
        entries, count = g["tie_log_r" if side == "rows" else "tie_log_c"]
        pts |= {int(e[1]) for e in entries}
    return pts


@pytest.mark.parametrize("m,n,k1,k2,iters,align", [
    (8193, 3001, 40, 60, 6, 1),     # uneven rows (4097 / 4096) and columns (1501 / 1500)
    (3000, 2500, 30, 50, 5, 4096),  # rank 1 owns no rows
    (4100, 2051, 20, 20, 4, 1),     # FFMA k-means / snap at k2 = 20
])
def test_pipeline_two_ranks_match_one(dev, m, n, k1, k2, iters, align):
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    A = _A(m, n, m + n, dev)
    cfg = CabsConfig(k1, k2, iters, seed=3)
    one = CabsPipeline(A, m, n, cfg)
    one.run()
    g1 = one.results()
    outs, rc = _pipelines(A, cfg, 2, align, dev)
    plans = [p for p, _ in outs]
    gs = [g for _, g in outs]
    if align > 1:
        assert plans[1].m_loc == 0
    # S1-S3: indices bit-exact; the gathered pilot rows (sum-allreduce over -0.0 fills) too
    for g in gs:
        assert torch.equal(g["I"], g1["I"]) and torch.equal(g["J"], g1["J"])
        assert torch.equal(g["R"], g1["R"]) and torch.equal(g["W"], g1["W"])
        assert g["r1"] == g1["r1"]
    r1 = g1["r1"]
    cat_rows = lambda key: torch.cat([g[key][:p.m_loc] for p, g in zip(plans, gs)])  # noqa: E731
    cat_cols = lambda key: torch.cat([g[key][:p.n_sl] for p, g in zip(plans, gs)])  # noqa: E731
    P1, Q1 = g1["P"].numpy()[:, :r1], g1["Q"].numpy()[:, :r1]
    assert rel_fro(align_signs(cat_rows("P").numpy()[:, :r1], P1), P1) < 1e-5
    assert rel_fro(align_signs(cat_cols("Q").numpy()[:, :r1], Q1), Q1) < 1e-5
    # S6-S8: labels / representatives bit-exact except at logged near ties
    diverged = False
    for side, cat, lab, reps, rep_of, gap in (("rows", cat_rows, "lab_r", "Ib", "rep_r", "gap_r"),
                                              ("cols", cat_cols, "lab_c", "Jb", "rep_c", "gap_c")):
        l2 = cat(lab).numpy()
        l1 = g1[lab].numpy()[:l2.shape[0]]
        bad = set(np.nonzero(l2 != l1)[0].tolist())
        if bad:
            ties = _tie_points([g1] + gs, side)
            assert bad <= ties, f"{side}: label differences outside the near-tie logs: {sorted(bad - ties)[:10]}"
            diverged = True
            continue
        for g in gs:
            assert rel_fro(g["cen_r" if side == "rows" else "cen_c"].numpy(),
                           g1["cen_r" if side == "rows" else "cen_c"].numpy()) < 1e-5
            if not torch.equal(g[rep_of], g1[rep_of]):
                j = int(np.nonzero(g[rep_of].numpy() != g1[rep_of].numpy())[0][0])
                assert float(g1[gap][j]) < NEAR_TIE, (side, j)
                diverged = True
            else:
                assert torch.equal(g[reps], g1[reps])
    if diverged:
        pytest.skip("trajectories parted at a logged near tie (checked above)")
    # S9-S10: follow-up factors and residual
    r2 = g1["r2"]
    for g in gs:
        assert g["r2"] == r2
        assert abs(g["a_sq"] - g1["a_sq"]) <= 1e-9 * g1["a_sq"]  # FP32 tile partials, another split
        assert abs(g["resid_sq"] - g1["resid_sq"]) <= 1e-6 * g1["a_sq"]
        assert rel_fro(g["s2"].numpy()[:r2], g1["s2"].numpy()[:r2]) < 1e-5
    U1, V1 = g1["U"].numpy()[:, :r2], g1["V"].numpy()[:, :r2]
    assert rel_fro(align_signs(cat_rows("U").numpy()[:, :r2], U1), U1) < 1e-5
    assert rel_fro(align_signs(cat_cols("V").numpy()[:, :r2], V1), V1) < 1e-5
    assert all(c > 0 for c in rc.calls)


def _select_ranks(dev, X, cen, cw, k2, nranks, align=1):
    from paper_1607_07395_b200.dist import make_plan
    N, d = X.shape
    ld = C.cabs_padded_ld(d)
    rc = HostRendezvousComm(nranks, dev)
    cen_t = torch.zeros((k2, ld), device=dev)
    cen_t[:, :d] = torch.from_numpy(cen.astype(np.float32)).to(dev)
    cw_t = torch.from_numpy(cw).to(dev)

    def rank(r):
        plan = make_plan(N, N, max(d, k2), r, nranks, align)
        ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
        Xl = torch.zeros((max(plan.m_loc, 1), ld), device=dev)
        Xl[:plan.m_loc, :d] = torch.from_numpy(X[plan.row_begin:plan.row_end]).to(dev)
        reps = torch.zeros(k2, dtype=torch.int64, device=dev)
        roc = torch.zeros(k2, dtype=torch.int64, device=dev)
        gap = torch.zeros(k2, device=dev)
        st = torch.cuda.Stream(device=dev)
        st.wait_stream(torch.cuda.current_stream(dev))  # inputs were written on the thread's default stream
        with torch.cuda.stream(st):
            C.cabs_select(plan, Xl, plan.m_loc, N, plan.row_begin, d, cen_t, k2, cw_t, reps, ws,
                          rep_of_centre=roc, gap=gap, comm=rc.comms[r] if nranks > 1 else None, stream=st)
        st.synchronize()
        return reps.cpu().numpy(), roc.cpu().numpy(), gap.cpu().numpy()

    return run_ranks(nranks, rank)


@pytest.mark.parametrize("force", [False, True])
@pytest.mark.parametrize("N,d,k2,dup", [(6000, 12, 50, False), (3001, 5, 120, True), (700, 3, 300, True)])
def test_select_multi_rank_matches_single_and_oracle(dev, monkeypatch, N, d, k2, dup, force):
    """dup: every point is one of 4 values, so each centre's exchanged top-32 list is the same
    32 points and runs out after 31 centres: the ranks must take the exact distributed pass."""
    g = np.random.default_rng(N + k2)
    if dup:
        base = g.standard_normal((4, d)).astype(np.float32)
        X = base[g.integers(0, 4, N)]
        cen = base[g.integers(0, 4, k2)].astype(np.float64) + 1e-3 * g.standard_normal((k2, d))
    else:
        X = g.standard_normal((N, d)).astype(np.float32)
        cen = X[g.choice(N, k2, replace=False)].astype(np.float64) + 0.05 * g.standard_normal((k2, d))
    cen = cen.astype(np.float32).astype(np.float64)
    cw = g.integers(0, 30, k2).astype(np.float64)
    if force:
        monkeypatch.setenv("CABS_SNAP_FORCE_DIST", "1")
    one = _select_ranks(dev, X, cen, cw, k2, 1)[0]
    two = _select_ranks(dev, X, cen, cw, k2, 2)
    for reps, roc, gap in two:
        assert np.array_equal(reps, one[0]) and np.array_equal(roc, one[1])
        assert np.array_equal(gap, one[2])
    ref = O.snap(X, cen, cw)
    got = one[1]
    for j in ref.order:  # first disagreement with the FP64 oracle, in visiting order: a near tie
        if got[j] != ref.rep_of_centre[j]:
            assert ref.gap[j] < NEAR_TIE, (j, got[j], ref.rep_of_centre[j], ref.gap[j])
            break
    assert np.unique(got).size == k2


def test_select_rank_without_points(dev):
    """A rank owning no points still writes its sentinel slots: the result equals one rank's."""
    g = np.random.default_rng(5)
    N, d, k2 = 3000, 8, 40
    X = g.standard_normal((N, d)).astype(np.float32)
    cen = X[g.choice(N, k2, replace=False)].astype(np.float64)
    cw = g.integers(0, 30, k2).astype(np.float64)
    one = _select_ranks(dev, X, cen, cw, k2, 1)[0]
    two = _select_ranks(dev, X, cen, cw, k2, 2, align=4096)
    for reps, roc, gap in two:
        assert np.array_equal(reps, one[0]) and np.array_equal(roc, one[1])


def test_sketch_out_of_range_index_sets_status(dev):
    """a caller-supplied out-of-range column index reads nothing and raises
    CABS_DEV_RANGE in the status word (no illegal address)."""
    from paper_1607_07395_b200.dist import make_plan
    m, n, k = 600, 500, 16
    A = _A(m, n, 1, dev)
    plan = make_plan(m, n, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(k)
    Ir = torch.arange(0, 2 * k, 2, dtype=torch.int64, device=dev)
    Ic = torch.arange(0, 2 * k, 2, dtype=torch.int64, device=dev)
    Ic[5] = n + 1000
    Ic[7] = -3
    U, V = torch.zeros((m, ld), device=dev), torch.zeros((n, ld), device=dev)
    s, r = torch.zeros(k, device=dev), torch.zeros(1, dtype=torch.int32, device=dev)
    C.cabs_clear_status(ws)
    try:
        C.cabs_sketch(plan, A, Ir, Ic, k, C.STABILIZED, 1e-12, U, s, V, r, ws)
    except C.CabsError:
        pass
    torch.cuda.synchronize()
    assert C.cabs_device_status(ws) & C.DEV_RANGE


def test_pipeline_rbf_two_ranks_match_one(dev):
    """The implicit source on two ranks: every rank generates its own rows (no row exchange);
    the pipeline with the sampled residual equals the single-rank one (P15)."""
    from paper_1607_07395_b200.dist import make_plan
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    from workloads import CONFIGS, make_rbf, scaled
    m, n, k = 9001, 5003, 40
    x, y, sigma = make_rbf(scaled(CONFIGS["c5"], m, n))
    src = C.RbfSource(x.to(dev), y.to(dev), sigma)
    cfg = CabsConfig(k, k, 4, seed=1, residual_samples=1 << 20)
    one = CabsPipeline(src, m, n, cfg)
    one.run()
    g1 = one.results()
    rc = HostRendezvousComm(2, dev)

    def rank(r):
        plan = make_plan(m, n, k, r, 2)
        st = torch.cuda.Stream(device=dev)
        st.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(st):
            pipe = CabsPipeline(src, m, n, cfg, r, 2, comm=rc.comms[r], plan=plan)
            pipe.run()
        st.synchronize()
        with torch.cuda.stream(st):
            return plan, pipe.results()

    outs = run_ranks(2, rank)
    for plan, g in outs:
        assert torch.equal(g["I"], g1["I"]) and torch.equal(g["J"], g1["J"])
        assert torch.equal(g["R"], g1["R"]) and torch.equal(g["W"], g1["W"])
    cat = lambda key, rows: torch.cat([g[key][:(p.m_loc if rows else p.n_sl)] for p, g in outs])  # noqa: E731
    r1 = g1["r1"]
    P1 = g1["P"].numpy()[:, :r1]
    assert rel_fro(align_signs(cat("P", True).numpy()[:, :r1], P1), P1) < 1e-5
    same = all(torch.equal(g["Ib"], g1["Ib"]) and torch.equal(g["Jb"], g1["Jb"]) for _, g in outs)
    if not same:
        ties = _tie_points([g1] + [g for _, g in outs], "rows") | _tie_points([g1] + [g for _, g in outs], "cols")
        assert ties, "representatives differ without any logged near tie"
        pytest.skip("trajectories parted at a logged near tie")
    for _, g in outs:
        assert abs(g["resid_sq"] - g1["resid_sq"]) <= 1e-6 * g1["a_sq"]
        assert abs(g["a_sq"] - g1["a_sq"]) <= 1e-9 * g1["a_sq"]
