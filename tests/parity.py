"""End-to-end GPU-vs-oracle parity with first-divergence logic (test-only; also used by
__graft_entry__.smoke()).

DESIGN.md section 5 / SURVEY.md 8(c-iv) step 3: pilot indices are bit-exact; the k-means
labels and the representatives are bit-exact until the FIRST place where the GPU and the FP64
oracle differ, and that place must be a near tie of the oracle (relative gap < 1e-5): a label
flip at the first iteration whose labels differ (every flipped point a near tie there), or, if
every iteration agrees, the first centre in the snap's visiting order that picks another point.
After a legitimate flip the trajectories may part, so the follow-up is then checked
teacher-forced: cabs_sketch and cabs_residual on the ORACLE's follow-up indices must match the
oracle's follow-up factors and residual -- always, divergence or not.  Without any divergence
the pipeline's own follow-up indices, factors and residual must match the oracle's as well.

The GPU's per-iteration labels come from re-running cabs_kmeans with iters = 1..c (the kernels
are deterministic and cabs_kmeans_pair equals two single calls bit for bit).
"""
from __future__ import annotations

import json
import math

import numpy as np
import torch

NEAR_TIE = 1e-5


def rel_fro(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def align_signs(X, Xref):
    X = np.array(X, np.float64, copy=True)
    for c in range(min(X.shape[1], Xref.shape[1])):
        if np.dot(X[:, c], Xref[:, c]) < 0:
            X[:, c] = -X[:, c]
    return X


def _gpu_labels_per_iteration(C, X_dev, N, d, k2, iters, seed, tag, weight_kind=0, weight_p=2.0):
    from paper_1607_07395_b200.dist import make_plan
    dev = X_dev.device
    plan = make_plan(N, N, max(d, k2))
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = X_dev.shape[1]
    out = []
    for t in range(1, iters + 1):
        cen = torch.zeros((k2, ld), device=dev)
        lab = torch.zeros(N, dtype=torch.int32, device=dev)
        cw = torch.zeros(k2, dtype=torch.float64, device=dev)
        obj = torch.zeros(t, dtype=torch.float64, device=dev)
        C.cabs_kmeans(plan, X_dev, N, N, 0, d, k2, t, weight_kind, weight_p, seed, tag, cen, lab, cw, obj, ws)
        out.append(lab.cpu().numpy().astype(np.int64))
    return out


def check_e2e(C, O, A_host, g, ref, pipe, log_path=None, factor_tol=1e-4, n_samples=0):
    """Returns the divergence log; raises AssertionError on any parity failure.  A_host: the
    oracle's matrix (dense array or oracle RbfSource); n_samples > 0: the residual is the
    sampled estimate on the same Philox pairs on both sides (c5)."""
    cfg = pipe.cfg
    m, n = A_host.shape
    k1, k2, iters = cfg.k1, cfg.k2, cfg.iters
    log = {"divergence": {}, "gpu_tie_log": {}, "teacher_forced": {}}
    # ---- S1-S5: pilot indices exact, embeddings within tolerance
    assert np.array_equal(g["I"].numpy(), ref.I) and np.array_equal(g["J"].numpy(), ref.J), "pilot indices"
    r1 = g["r1"]
    assert r1 == ref.pilot.r, ("pilot rank", r1, ref.pilot.r)
    assert rel_fro(align_signs(g["P"].numpy()[:, :r1], ref.P), ref.P) < factor_tol, "P"
    assert rel_fro(align_signs(g["Q"].numpy()[:, :r1], ref.Q), ref.Q) < factor_tol, "Q"
    # ---- S6-S8: first divergence per side
    diverged = {}
    for side, X, km, sn, reps_key, rep_of_key, tag in (
            ("rows", pipe.P, ref.km_rows, ref.snap_rows, "Ib", "rep_r", 3),
            ("cols", pipe.Q, ref.km_cols, ref.snap_cols, "Jb", "rep_c", 4)):
        N = X.shape[0]
        labs = _gpu_labels_per_iteration(C, X, N, r1, k2, iters, cfg.seed, tag, cfg.weight_kind, cfg.weight_p)
        first = None
        for t in range(iters):
            bad = np.nonzero(labs[t] != km.labels_hist[t])[0]
            if bad.size:
                gaps = km.gaps[t][bad]
                first = {"where": "kmeans", "iteration": t, "points": bad[:20].tolist(),
                         "oracle_gaps": gaps[:20].tolist(), "count": int(bad.size)}
                assert np.all(gaps < NEAR_TIE), f"{side}: label flip without a near tie at iteration {t}: {first}"
                break
        if first is None:
            # same trajectory: centres, weights, objective, then the snap in visiting order
            cen = g["cen_r" if side == "rows" else "cen_c"].numpy()[:, :r1]
            assert rel_fro(cen, km.centres) < 1e-5, f"{side}: centres"
            cw = g["cw_r" if side == "rows" else "cw_c"].numpy()
            assert np.allclose(cw, km.cluster_w, rtol=1e-6), f"{side}: cluster weights"
            ob = g["obj_r" if side == "rows" else "obj_c"].numpy()
            assert np.allclose(ob, km.objective, rtol=1e-4, atol=1e-7 * km.objective[0]), f"{side}: objective"
            g_rep = g[rep_of_key].numpy()
            for j in sn.order:
                if g_rep[j] != sn.rep_of_centre[j]:
                    first = {"where": "snap", "centre": int(j), "oracle_rep": int(sn.rep_of_centre[j]),
                             "gpu_rep": int(g_rep[j]), "oracle_gap": float(sn.gap[j])}
                    assert sn.gap[j] < NEAR_TIE, f"{side}: snap divergence without a near tie: {first}"
                    break
            if first is None:
                assert np.array_equal(g[reps_key].numpy(), sn.reps_sorted), f"{side}: representatives"
        diverged[side] = first
        log["divergence"][side] = first
        # the GPU's own near-tie log: every logged point (before any divergence) is close to a tie
        # for the oracle too (FP32 vs FP64 relative gaps differ by ~d 2^-24)
        entries, count = g["tie_log_r" if side == "rows" else "tie_log_c"]
        limit = iters if first is None or first["where"] == "snap" else first["iteration"]
        checked = []
        for (it, p, j1, j2, gap) in entries:
            if it < limit:
                og = float(km.gaps[it][p])
                checked.append((it, p, j1, j2, gap, og))
                assert og < 1e-4, f"{side}: GPU near tie at ({it}, {p}) with oracle gap {og}"
        log["gpu_tie_log"][side] = {"count": count, "entries": [list(e) for e in checked[:200]]}
    # ---- S9-S10 teacher-forced on the oracle's follow-up indices
    from paper_1607_07395_b200.dist import make_plan
    dev = pipe.A.device
    plan = make_plan(m, n, max(k1, k2))
    ws = torch.zeros(C.cabs_workspace_bytes(plan), dtype=torch.uint8, device=dev)
    ld = C.cabs_padded_ld(k2)
    U = torch.zeros((m, ld), device=dev)
    V = torch.zeros((n, ld), device=dev)
    s = torch.zeros(k2, device=dev)
    r = torch.zeros(1, dtype=torch.int32, device=dev)
    Ir = torch.from_numpy(ref.Ibar).to(dev)
    Ic = torch.from_numpy(ref.Jbar).to(dev)
    C.cabs_sketch(plan, pipe.A, Ir, Ic, k2, cfg.mode, cfg.tol, U, s, V, r, ws)
    out = torch.zeros(2, dtype=torch.float64, device=dev)
    r2 = int(r.item())
    C.cabs_residual(plan, pipe.A, U, s, V, r2, out, ws, n_samples=n_samples, seed=cfg.seed)
    fu = ref.follow
    assert r2 == fu.r, ("follow-up rank", r2, fu.r)
    eU = rel_fro(align_signs(U.cpu().numpy()[:, :r2], fu.U), fu.U)
    eV = rel_fro(align_signs(V.cpu().numpy()[:, :r2], fu.V), fu.V)
    es = rel_fro(s.cpu().numpy()[:r2], fu.s)
    a = math.sqrt(ref.a_sq)
    rg, ro = math.sqrt(max(out[0].item(), 0.0)), math.sqrt(ref.resid_sq)
    log["teacher_forced"] = {"U": eU, "V": eV, "s": es, "r_gpu": rg, "r_oracle": ro}
    assert max(eU, eV, es) < factor_tol, log["teacher_forced"]
    assert abs(out[1].item() - ref.a_sq) <= 1e-6 * ref.a_sq
    if cfg.mode == 0:
        assert abs(rg - ro) <= 1e-4 * ro + 1e-6 * a, log["teacher_forced"]
    # ---- without divergence the pipeline's own follow-up equals the oracle's
    if diverged["rows"] is None and diverged["cols"] is None:
        assert g["r2"] == fu.r
        assert rel_fro(align_signs(g["U"].numpy()[:, :fu.r], fu.U), fu.U) < factor_tol
        assert rel_fro(align_signs(g["V"].numpy()[:, :fu.r], fu.V), fu.V) < factor_tol
        rgp = math.sqrt(max(g["resid_sq"], 0.0))
        if cfg.mode == 0:
            assert abs(rgp - ro) <= 1e-4 * ro + 1e-6 * a, (rgp, ro)
    if log_path is not None:
        with open(log_path, "w") as f:
            json.dump(log, f, indent=1)
    return log
