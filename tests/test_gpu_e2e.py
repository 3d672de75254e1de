"""GPU end-to-end parity: Algorithm 2 + residual through the C ABI vs the FP64
oracle on the same seeded A.

Pilot indices are bit-exact; representative indices are bit-exact unless a near
tie (oracle gap < 1e-5) occurred on that side, which is logged; factors within
1e-4; residual |r_gpu - r_or| <= 1e-4 r_or + 1e-6 ||A||_F (STABILIZED)."""
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


def _run(A_t, m, n, k1, k2, iters, seed=0, mode=0, with_residual=True, **kw):
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    pipe = CabsPipeline(A_t, m, n, CabsConfig(k1, k2, iters, seed=seed, mode=mode, **kw))
    pipe.run(with_residual=with_residual)
    return pipe, pipe.results()


def _side_ok(g_reps, g_lab, ref_snap, ref_km, log, side):
    """Representatives must match unless the oracle saw a near tie on that side."""
    if np.array_equal(g_reps, ref_snap.reps_sorted):
        return True
    near = [float(np.min(gp)) for gp in ref_km.gaps] + [float(np.min(ref_snap.gap))]
    log.append((side, "reps differ", float(min(near))))
    return min(near) < NEAR_TIE


def _check_e2e(g, ref, A, log, mode=O.STABILIZED):
    assert np.array_equal(g["I"].numpy(), ref.I) and np.array_equal(g["J"].numpy(), ref.J)
    r1 = g["r1"]
    assert r1 == ref.pilot.r
    assert rel_fro(align_signs(g["P"].numpy()[:, :r1], ref.P), ref.P) < 1e-4
    assert rel_fro(align_signs(g["Q"].numpy()[:, :r1], ref.Q), ref.Q) < 1e-4
    ok_r = _side_ok(g["Ib"].numpy(), g["lab_r"].numpy(), ref.snap_rows, ref.km_rows, log, "rows")
    ok_c = _side_ok(g["Jb"].numpy(), g["lab_c"].numpy(), ref.snap_cols, ref.km_cols, log, "cols")
    assert ok_r and ok_c, f"representatives differ without a near tie: {log}"
    same = np.array_equal(g["Ib"].numpy(), ref.Ibar) and np.array_equal(g["Jb"].numpy(), ref.Jbar)
    a = math.sqrt(ref.a_sq)
    assert abs(math.sqrt(g["a_sq"]) - a) <= 1e-6 * a
    if same:
        r2 = g["r2"]
        assert r2 == ref.follow.r
        fu = ref.follow
        assert rel_fro(align_signs(g["U"].numpy()[:, :r2], fu.U), fu.U) < 1e-4
        assert rel_fro(align_signs(g["V"].numpy()[:, :r2], fu.V), fu.V) < 1e-4
        rg, ro = math.sqrt(max(g["resid_sq"], 0)), math.sqrt(ref.resid_sq)
        assert abs(rg - ro) <= 1e-4 * ro + 1e-6 * a, (rg, ro)
    else:  # trajectories legitimately diverged after a logged near tie: objectives agree
        for side, o_g, km in (("rows", g["obj_r"], ref.km_rows), ("cols", g["obj_c"], ref.km_cols)):
            assert abs(o_g[-1].item() - km.objective[-1]) <= 1e-4 * km.objective[-1] + 1e-9, side


def test_e2e_config1(dev):
    from workloads import CONFIGS, make_A
    cfg = CONFIGS["c1"]
    A_t = make_A(cfg, device=dev)
    A = A_t.cpu().numpy()
    pipe, g = _run(A_t, cfg.m, cfg.n, cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed)
    ref = O.cabs_run(A, cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed)
    log = []
    _check_e2e(g, ref, A, log)
    print("near-tie log:", log, "gpu near ties rows/cols:", g["tie_r"].tolist(), g["tie_c"].tolist())


@pytest.mark.parametrize("name,m,n,k,iters,seed", [("c2", 4000, 2000, 50, 20, 0), ("c3", 4000, 2000, 100, 8, 0),
                                                   ("c1", 1000, 700, 20, 10, 3), ("c4", 2000, 1000, 60, 6, 1)])
def test_e2e_scaled_configs(dev, name, m, n, k, iters, seed):
    from workloads import CONFIGS, make_A, scaled
    cfg = scaled(CONFIGS[name], m, n, k1=k, k2=k, iters=iters, seed=seed)
    A_t = make_A(cfg, device=dev)
    A = A_t.cpu().numpy()
    pipe, g = _run(A_t, m, n, k, k, iters, seed=seed)
    ref = O.cabs_run(A, k, k, iters, seed=seed)
    log = []
    _check_e2e(g, ref, A, log)
    print(name, "near-tie log:", log)


def test_e2e_pseudo_skeleton_mode(dev):
    from workloads import CONFIGS, make_A, scaled
    cfg = scaled(CONFIGS["c1"], 1500, 1000, k1=20, k2=20, iters=5)
    A_t = make_A(cfg, device=dev)
    A = A_t.cpu().numpy()
    pipe, g = _run(A_t, cfg.m, cfg.n, 20, 20, 5, mode=C.PSEUDO_SKELETON)
    ref = O.cabs_run(A, 20, 20, 5, mode=O.PSEUDO_SKELETON)
    assert np.array_equal(g["I"].numpy(), ref.I)
    if np.array_equal(g["Ib"].numpy(), ref.Ibar) and np.array_equal(g["Jb"].numpy(), ref.Jbar):
        a = math.sqrt(ref.a_sq)
        rg, ro = math.sqrt(g["resid_sq"]), math.sqrt(ref.resid_sq)
        Wb = A[np.ix_(ref.Ibar, ref.Jbar)].astype(np.float64)
        kappa = np.linalg.cond(Wb)
        assert abs(rg - ro) <= 1e-4 * ro + 10 * kappa * 2.0 ** -24 * a


def test_e2e_exact_recovery_p14(dev):
    """P14 on the GPU: block-replicated A, one pilot sample per block, one init per group ->
    representatives are the lowest index of each group and the residual is at the FP32 floor."""
    k, rows_per, cols_per = 6, 40, 30
    g = np.random.default_rng(3)
    B = g.standard_normal((k, k))
    rl = np.repeat(np.arange(k), rows_per)[g.permutation(k * rows_per)]
    cl = np.repeat(np.arange(k), cols_per)[g.permutation(k * cols_per)]
    A = B[np.ix_(rl, cl)].astype(np.float32)
    m, n = A.shape
    from paper_1607_07395_b200.dist import make_plan
    plan = make_plan(m, n, k)
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    A_t = torch.from_numpy(A).to(dev)
    I = torch.tensor(np.sort([np.where(rl == b)[0][-1] for b in range(k)]), device=dev)
    J = torch.tensor(np.sort([np.where(cl == b)[0][-1] for b in range(k)]), device=dev)
    ld = C.cabs_padded_ld(k)
    U = torch.zeros((m, ld), device=dev); V = torch.zeros((n, ld), device=dev)
    s = torch.zeros(k, device=dev); r = torch.zeros(1, dtype=torch.int32, device=dev)
    C.cabs_sketch(plan, A_t, I, J, k, C.STABILIZED, 1e-12, U, s, V, r, ws)
    P = torch.zeros((m, ld), device=dev); P[:, :k] = U[:, :k] * torch.sqrt(s)
    Q = torch.zeros((n, ld), device=dev); Q[:, :k] = V[:, :k] * torch.sqrt(s)
    reps = []
    for X, N, lab_of in ((P, m, rl), (Q, n, cl)):
        init = torch.tensor([np.where(lab_of == b)[0][1] for b in range(k)], device=dev)
        cen = torch.zeros((k, ld), device=dev)
        lab = torch.zeros(N, dtype=torch.int32, device=dev)
        cw = torch.zeros(k, dtype=torch.float64, device=dev)
        obj = torch.zeros(4, dtype=torch.float64, device=dev)
        C.cabs_kmeans(plan, X, N, N, 0, k, k, 4, C.WEIGHT_CONST, 2.0, 0, 3, cen, lab, cw, obj, ws, init_idx=init)
        rp = torch.zeros(k, dtype=torch.int64, device=dev)
        C.cabs_select(plan, X, N, N, 0, k, cen, k, cw, rp, ws)
        reps.append(rp)
        exp = np.sort([np.where(lab_of == b)[0][0] for b in range(k)])
        assert np.array_equal(rp.cpu().numpy(), exp)
    for mode in (C.STABILIZED, C.PSEUDO_SKELETON):
        C.cabs_sketch(plan, A_t, reps[0], reps[1], k, mode, 1e-12, U, s, V, r, ws)
        out = torch.zeros(2, dtype=torch.float64, device=dev)
        C.cabs_residual(plan, A_t, U, s, V, k, out, ws)
        rel = math.sqrt(out[0].item() / out[1].item())
        assert rel < 1e-5, (mode, rel)


def test_e2e_linear_access_nan_poison(dev):
    """P12 on the GPU: poisoning every entry outside the touched rows/columns changes nothing."""
    from workloads import CONFIGS, make_A, scaled
    cfg = scaled(CONFIGS["c1"], 1200, 900, k1=16, k2=16, iters=5)
    A_t = make_A(cfg, device=dev)
    pipe, g = _run(A_t, cfg.m, cfg.n, 16, 16, 5, with_residual=False)
    rows = np.union1d(g["I"].numpy(), g["Ib"].numpy())
    cols = np.union1d(g["J"].numpy(), g["Jb"].numpy())
    Ap = torch.full_like(A_t, float("nan"))
    rt, ct = torch.from_numpy(rows).to(dev), torch.from_numpy(cols).to(dev)
    Ap[rt, :] = A_t[rt, :]
    Ap[:, ct] = A_t[:, ct]
    pipe2, g2 = _run(Ap, cfg.m, cfg.n, 16, 16, 5, with_residual=False)
    for key in ("I", "J", "Ib", "Jb", "U", "V", "s2", "P", "Q"):
        assert torch.equal(g[key], g2[key]), key
    assert C.cabs_device_status(pipe2.ws) == 0


def test_e2e_deterministic(dev):
    from workloads import CONFIGS, make_A, scaled
    cfg = scaled(CONFIGS["c2"], 3000, 2000, k1=40, k2=40, iters=10)
    A_t = make_A(cfg, device=dev)
    _, g1 = _run(A_t, cfg.m, cfg.n, 40, 40, 10)
    _, g2 = _run(A_t, cfg.m, cfg.n, 40, 40, 10)
    for key in g1:
        if isinstance(g1[key], torch.Tensor):
            assert torch.equal(g1[key], g2[key]), key
        else:
            assert g1[key] == g2[key], key


def test_e2e_cuda_graph_replay_matches_eager(dev):
    """The whole hot path captured as one CUDA graph (bench.py's timed step) replays to the
    same results as the stream-ordered run, bit for bit, also on new data written in place."""
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    from workloads import CONFIGS, make_A, scaled
    cfg = scaled(CONFIGS["c2"], 3000, 2000, k1=40, k2=40, iters=8)
    A_t = make_A(cfg, device=dev)
    pipe = CabsPipeline(A_t, cfg.m, cfg.n, CabsConfig(40, 40, 8, seed=cfg.seed))
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pipe.run()
        ref = pipe.results()
        graph, launches = pipe.capture(stream=s)
    torch.cuda.synchronize()
    assert launches > 10
    pipe.out.zero_()
    pipe.U.zero_()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        graph.replay()
    torch.cuda.synchronize()
    got = pipe.results()
    for key in ref:
        if isinstance(ref[key], torch.Tensor):
            assert torch.equal(got[key], ref[key]), key
        else:
            assert got[key] == ref[key], key
    # new data in the same buffer: the replay recomputes (compare against an eager run)
    A2 = make_A(scaled(CONFIGS["c2"], 3000, 2000, k1=40, k2=40, iters=8, seed=cfg.seed + 1), device=dev)
    pipe.A.copy_(A2)
    s.wait_stream(torch.cuda.current_stream())  # the copy is on the default stream
    with torch.cuda.stream(s):
        graph.replay()
    torch.cuda.synchronize()
    got2 = pipe.results()
    _, ref2 = _run(A2, cfg.m, cfg.n, 40, 40, 8, seed=cfg.seed)
    bad = [k for k in ref2 if (not torch.equal(got2[k], ref2[k]) if isinstance(ref2[k], torch.Tensor)
                               else got2[k] != ref2[k])]
    assert not bad, bad
