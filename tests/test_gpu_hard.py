"""GPU parity of the hard-threshold follow-up (P:312 variant (f); DESIGN.md
Z26) through the C ABI: the keys ||X_l||^2 are bit-identical to the oracle's (same FP64
operations in the same order on exact squares), the selected index sets are identical
(integer decisions on identical keys), and the end-to-end variant matches the FP64
oracle's Algorithm 2 with step 3 replaced."""
import math

import numpy as np
import pytest
import torch

from oracle import cabs as O
from tests.helpers import NEAR_TIE, align_signs, rel_fro

pytestmark = pytest.mark.gpu

C = pytest.importorskip("paper_1607_07395_b200.cabs")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    C.load()
    return torch.device("cuda:0")


def _select(dev, X, k2, n_glob=None, row_off=0, kmax=None):
    from paper_1607_07395_b200.dist import make_plan
    N, d = X.shape
    n_glob = N if n_glob is None else n_glob
    plan = make_plan(max(n_glob, 1), max(n_glob, 1), kmax or max(k2, d))
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(d)
    Xt = torch.zeros((max(N, 1), ld), device=dev)
    Xt[:N, :d] = torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)).to(dev)
    reps = torch.full((k2,), -7, dtype=torch.int64, device=dev)
    keys = torch.zeros(max(N, 1), dtype=torch.float64, device=dev)
    C.cabs_hard_select(plan, Xt, N, n_glob, row_off, d, k2, reps, ws, keys=keys)
    torch.cuda.synchronize()
    return reps.cpu().numpy(), keys.cpu().numpy()[:N]


@pytest.mark.parametrize("N,d,k2", [(1, 1, 1), (50, 7, 5), (1000, 50, 50), (1023, 33, 64), (1025, 64, 1),
                                    (20000, 50, 50), (100003, 21, 200), (25600, 8, 30), (25601, 8, 30), (3000, 100, 3000 // 4)])
def test_keys_and_selection_match_oracle(dev, N, d, k2):
    g = np.random.default_rng(N + d)
    X = (g.standard_normal((N, d)) * g.uniform(0.1, 3.0, size=(N, 1))).astype(np.float32)
    reps, keys = _select(dev, X, k2, kmax=max(k2, d, 64))
    want_keys = O.row_sq_norms(X)
    assert np.array_equal(keys, want_keys)  # bit-identical
    assert reps.tolist() == O.hard_threshold_followup(X, k2).tolist()


def test_ties_go_to_lowest_index(dev):
    g = np.random.default_rng(5)
    base = g.standard_normal((40, 9)).astype(np.float32)
    X = base[g.integers(0, 40, size=3000)]  # 3000 rows, only 40 distinct keys: big tie groups
    X[::7] = -X[::7]  # sign flips keep the key
    for k2 in (1, 13, 75, 76, 500, 1023, 1024):
        reps, keys = _select(dev, X, k2, kmax=max(k2, 64))
        assert reps.tolist() == O.hard_threshold_followup(X, k2).tolist(), k2
    Xb = np.tile(X, (12, 1))  # 36000 rows: the uncached (streaming) top-k kernel
    for k2 in (7, 1000):
        reps, _ = _select(dev, Xb, k2, kmax=1024)
        assert reps.tolist() == O.hard_threshold_followup(Xb, k2).tolist(), k2
    reps, _ = _select(dev, np.ones((500, 3), np.float32), 37, kmax=64)  # every key equal
    assert reps.tolist() == list(range(37))


def test_keys_differing_in_last_bits(dev):
    """Keys that share every high digit force all eight radix passes."""
    N = 4096
    x = (1.0 + np.arange(N, dtype=np.float64) * 2.0 ** -23)[np.random.default_rng(1).permutation(N)]
    X = x.astype(np.float32)[:, None]
    for k2 in (1, 100, 1000):
        reps, keys = _select(dev, X, k2, kmax=1024)
        assert np.array_equal(keys, O.row_sq_norms(X))
        assert reps.tolist() == O.hard_threshold_followup(X, k2).tolist()


def test_zero_rows_and_row_offset(dev):
    X = np.zeros((300, 4), np.float32)
    X[[5, 100, 299]] = 1.0
    reps, _ = _select(dev, X, 5, n_glob=1000, row_off=600, kmax=64)
    assert reps.tolist() == [600, 601, 605, 700, 899]  # the three nonzero rows, then zeros by index


def test_bad_arguments(dev):
    from paper_1607_07395_b200.dist import make_plan
    plan = make_plan(100, 100, 16)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    X = torch.zeros((100, 32), device=dev)
    reps = torch.zeros(16, dtype=torch.int64, device=dev)
    for k2 in (0, 17, 101):
        with pytest.raises(C.CabsError):
            C.cabs_hard_select(plan, X, 100, 100, 0, 8, k2, reps, ws)
    with pytest.raises(C.CabsError):
        C.cabs_hard_select(plan, X, 100, 100, 50, 8, 4, reps, ws)  # rows past n_glob


def _key_gap(X, k):
    """Relative gap between the k-th and (k+1)-th largest FP64 key (a near tie excuses a swap)."""
    ks = np.sort(O.row_sq_norms(X))[::-1]
    if k >= ks.size:
        return math.inf
    return (ks[k - 1] - ks[k]) / ks[k - 1] if ks[k - 1] > 0 else 0.0


@pytest.mark.parametrize("name,m,n,k,seed", [("c1", 2000, 1500, 20, 0), ("c2", 4000, 2000, 50, 1),
                                             ("c3", 4000, 2000, 100, 2)])
def test_e2e_hard_followup(dev, name, m, n, k, seed):
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    from workloads import CONFIGS, make_A, scaled
    cfg = scaled(CONFIGS[name], m, n, k1=k, k2=k, iters=5, seed=seed)
    A_t = make_A(cfg, device=dev)
    A = A_t.cpu().numpy()
    pipe = CabsPipeline(A_t, m, n, CabsConfig(k, k, 5, seed=seed, followup="hard"))
    pipe.run()
    g = pipe.results()
    r1 = g["r1"]
    P_g, Q_g = g["P"].numpy()[:, :r1], g["Q"].numpy()[:, :r1]
    # the GPU's decision on its own FP32 embedding is exact
    assert g["Ib"].numpy().tolist() == O.hard_threshold_followup(P_g, k).tolist()
    assert g["Jb"].numpy().tolist() == O.hard_threshold_followup(Q_g, k).tolist()
    ref = O.cabs_run(A, k, k, 5, seed=seed, followup="hard")
    assert rel_fro(align_signs(P_g, ref.P), ref.P) < 1e-4
    same_r = np.array_equal(g["Ib"].numpy(), ref.Ibar)
    same_c = np.array_equal(g["Jb"].numpy(), ref.Jbar)
    assert same_r or _key_gap(ref.P, k) < NEAR_TIE
    assert same_c or _key_gap(ref.Q, k) < NEAR_TIE
    if same_r and same_c:
        a = math.sqrt(ref.a_sq)
        rg, ro = math.sqrt(max(g["resid_sq"], 0)), math.sqrt(ref.resid_sq)
        assert abs(rg - ro) <= 1e-4 * ro + 1e-6 * a, (rg, ro)
        assert g["r2"] == ref.follow.r


def test_pair_equals_two_singles(dev):
    from paper_1607_07395_b200.dist import make_plan
    g = np.random.default_rng(11)
    Na, Nb, d, k2 = 20000, 9000, 50, 50
    plan = make_plan(Na, Nb, 64)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(d)
    Xa = torch.zeros((Na, ld), device=dev); Xa[:, :d] = torch.from_numpy(g.standard_normal((Na, d)).astype(np.float32))
    Xb = torch.zeros((Nb, ld), device=dev); Xb[:, :d] = torch.from_numpy(g.standard_normal((Nb, d)).astype(np.float32))
    ra, rb = torch.zeros(k2, dtype=torch.int64, device=dev), torch.zeros(k2 - 7, dtype=torch.int64, device=dev)
    ka, kb = torch.zeros(Na, dtype=torch.float64, device=dev), torch.zeros(Nb, dtype=torch.float64, device=dev)
    pa = C.hard_problem(Xa, Na, Na, 0, d, k2, ra, keys=ka)
    pb = C.hard_problem(Xb, Nb, Nb, 0, d, k2 - 7, rb, keys=kb)
    C.cabs_hard_select_pair(plan, pa, pb, ws)
    sa, sb = torch.zeros_like(ra), torch.zeros_like(rb)
    C.cabs_hard_select(plan, Xa, Na, Na, 0, d, k2, sa, ws)
    C.cabs_hard_select(plan, Xb, Nb, Nb, 0, d, k2 - 7, sb, ws)
    torch.cuda.synchronize()
    assert torch.equal(ra, sa) and torch.equal(rb, sb)
    assert ra.cpu().tolist() == O.hard_threshold_followup(Xa[:, :d].cpu().numpy(), k2).tolist()
    assert np.array_equal(kb.cpu().numpy(), O.row_sq_norms(Xb[:, :d].cpu().numpy()))


from tests.rendezvous import HostRendezvousComm as _HostRendezvousComm  # noqa: E402


@pytest.mark.parametrize("m,k2", [(5000, 50), (30, 20), (2049, 1)])
def test_multi_rank_merge_matches_single(dev, m, k2):
    import threading
    from paper_1607_07395_b200.dist import make_plan
    g = np.random.default_rng(m)
    d = 9
    X = g.standard_normal((m, d)).astype(np.float32)
    X[g.integers(0, m, size=m // 3)] = X[0]  # ties across the rank boundary
    want = O.hard_threshold_followup(X, k2).tolist()
    rc = _HostRendezvousComm(2, dev)
    got, errs = [None, None], []

    def rank_main(r):
        try:
            plan = make_plan(m, m, 64, r, 2)
            ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
            Xl = torch.zeros((max(plan.m_loc, 1), C.cabs_padded_ld(d)), device=dev)
            Xl[:plan.m_loc, :d] = torch.from_numpy(X[plan.row_begin:plan.row_end]).to(dev)
            reps = torch.zeros(k2, dtype=torch.int64, device=dev)
            st = torch.cuda.Stream(device=dev)
            st.wait_stream(torch.cuda.current_stream(dev))  # inputs were written on the thread's default stream
            with torch.cuda.stream(st):
                C.cabs_hard_select(plan, Xl, plan.m_loc, m, plan.row_begin, d, k2, reps, ws, comm=rc.comms[r],
                                   stream=st)
            st.synchronize()
            got[r] = reps.cpu().tolist()
        except Exception as e:  # noqa: BLE001
            errs.append(repr(e))

    th = [threading.Thread(target=rank_main, args=(r,)) for r in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=120)
    assert not errs, errs
    assert got[0] == want and got[1] == want
