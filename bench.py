#!/usr/bin/env python
"""Benchmark of the CABS hot path (S1-S10) on B200 -- prints ONE JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one pass of the whole hot path -- pilot sampling + gathers, pilot
sketch + embeddings, weighted Lloyd k-means on both sides, snap, follow-up
gathers + sketch, and the fused residual -- over the synthetic matrix of
BASELINE.json configs[2] (c3, 100000 x 50000 = 20 GB, k1 = k2 = 100, 25 Lloyd iterations:
the largest configuration that fits one GPU; c4 is a 2/4/8-GPU config) held in HBM.  Timing: W untimed warm-ups, then K steps, each bracketed by a
barrier + cuda.synchronize on both sides and timed with CUDA events on the
launching stream; the L2 is flushed (256 MiB write) before every timed step;
max over ranks.  N > 1: one process per GPU (torchrun), A row-sharded, NCCL.

`--impl reference` times the FP64 CPU oracle (the deliberately slow reference of
this tier) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from workloads import (CHUNK, CONFIGS, SPARSE_CONFIGS, SPARSE_DENSITY, Generator, csr_to_csc,  # noqa: E402
                       make_rbf, make_sparse)

METRIC = "CABS sketch wall time & k-means pts/s at 1/2/4/8 GPU; HBM GB/s vs peak"
UNIT = "rows+cols/s"
BASE_CFG = {1: "c3"}  # BASELINE.json configs[2]: the largest single-GPU configuration
CFG_INDEX = {"c1": 0, "c2": 1, "c3": 2, "c4": 3, "c5": 4}
ALL_CONFIGS = {**CONFIGS, **SPARSE_CONFIGS}


def workload_name(cfg):
    if cfg.name in CFG_INDEX:
        return f"{cfg.name} = BASELINE.json configs[{CFG_INDEX[cfg.name]}]: {cfg.note}"
    return f"{cfg.name} = SURVEY NEXT-3 sparse source (not a BASELINE config): {cfg.note}"


def sparse_block(cfg, r0, r1, dev):
    """The sparse_lowrank matrix of a sparse config (built on the device) -> this rank's rows
    [r0, r1) as CSR + CSC device tensors (library input, not part of the timed step)."""
    ip, ix, v = make_sparse(cfg, SPARSE_DENSITY[cfg.name], device=dev)
    lo, hi = int(ip[r0]), int(ip[r1])
    bip = (ip[r0:r1 + 1] - lo).contiguous()
    bix, bv = ix[lo:hi].contiguous(), v[lo:hi].contiguous()
    cp, ri, cv = csr_to_csc(bip, bix, bv, cfg.n)
    return (bip, bix, bv, cp, ri, cv), (ip, ix, v)
LIN_SAMPLES = 10 ** 6    # sampled-error pairs of the host-resident (linear access) end-to-end line
C5_SAMPLES = 10 ** 9     # BASELINE.json configs[4]: "residual estimated on a seeded 1e9-entry uniform subset"
ORACLE_RBF_SAMPLES = 1 << 20  # the oracle's bounded c5 sample: pairs of its leading block


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def traffic_of(traffic, key):
    t = traffic.get(key)
    return t.get("dram_bytes_per_launch") if isinstance(t, dict) else None


def m_loc_rows(plan):
    return plan.row_end - plan.row_begin


def n_loc_cols(plan):
    return plan.col_end - plan.col_begin


def load_traffic():
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


class ClockSampler:
    """Samples SM clock and clock-event reasons with NVML during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def setup_dist(n_gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def allreduce_max(x, world):
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------- reference arm (the oracle)
def oracle_sample(cfg):
    """The bounded sample of a config the oracle is timed on (10-30 s of host CPU per step):
    the leading ms x ns block of the same matrix, same k1, k2 and Lloyd iterations."""
    ms, ns = {"c1": (2000, 1500), "c2": (8000, 4000), "c3": (6000, 3000), "c4": (6000, 3000),
              "c5": (6000, 4000), "s1": (6000, 9000), "s2": (5000, 12000)}[cfg.name]
    return min(ms, cfg.m), min(ns, cfg.n)


def oracle_source(cfg, ms, ns):
    """The oracle's matrix for the bounded sample: the leading ms x ns block (dense), or the implicit
    source on the first ms / ns points (c5), with the residual sample size the oracle runs."""
    from oracle import cabs as O
    if cfg.kind == "rbf_mixture":
        x, y, sigma = make_rbf(cfg)
        return O.RbfSource(x[:ms].numpy(), y[:ns].numpy(), sigma), ORACLE_RBF_SAMPLES
    if cfg.kind == "sparse_lowrank":
        return oracle_sparse_block(make_sparse(cfg, SPARSE_DENSITY[cfg.name]), ms, ns), 0
    return Generator(cfg, device="cpu").rows(0, ms)[:, :ns].numpy().copy(), 0


def oracle_sparse_block(csr, ms, ns):
    """The leading ms x ns block of a CSR matrix as the oracle's CsrSource."""
    from oracle import cabs as O
    ip, ix, v = (t.cpu().numpy() for t in csr)
    rows = np.repeat(np.arange(ms), np.diff(ip[:ms + 1]))
    sel = ix[:ip[ms]] < ns
    r, c, val = rows[sel], ix[:ip[ms]][sel], v[:ip[ms]][sel]
    bip = np.zeros(ms + 1, np.int64)
    bip[1:] = np.cumsum(np.bincount(r, minlength=ms))
    return O.CsrSource(bip, c, val, (ms, ns))


def run_reference(args, cfg):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import cabs as O
    from workloads import Generator
    cores = len(os.sched_getaffinity(0))
    ms, ns = oracle_sample(cfg)
    A, T = oracle_source(cfg, ms, ns)
    wk = O.WEIGHT_POWER if cfg.kind == "sparse_lowrank" else O.WEIGHT_CONST
    k1, k2 = min(cfg.k1, ms, ns), min(cfg.k2, ms, ns)
    times = []
    for i in range(args.warmup + args.steps):
        if i < args.warmup:  # warm-up: a small run (page-in, BLAS init)
            O.cabs_run(A, min(k1, 20), min(k2, 20), 2, seed=cfg.seed, n_samples=min(T, 4096), weight_kind=wk)
            continue
        t0 = time.perf_counter()
        O.cabs_run(A, k1, k2, cfg.iters, seed=cfg.seed, n_samples=T, weight_kind=wk)
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    v = (ms + ns) / t
    sample = (f"leading {ms} x {ns} block of {cfg.name} (same recipe, k1={k1}, k2={k2}, {cfg.iters} Lloyd "
              f"iterations{f', residual on {T} sampled entries' if T else ''}), full S1-S10 of the FP64 NumPy "
              f"oracle per step")
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(cfg),
                       "m": cfg.m, "n": cfg.n, "k1": cfg.k1, "k2": cfg.k2, "iters": cfg.iters},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def oracle_cpu_baseline(cfg, A_host):
    """The oracle as it stands, on the host cores, on a bounded sample of the workload."""
    from oracle import cabs as O
    cores = len(os.sched_getaffinity(0))
    ms, ns = oracle_sample(cfg)
    if A_host is None:  # implicit or sparse source
        A, T = oracle_source(cfg, ms, ns)
    else:
        A, T = np.ascontiguousarray(A_host[:ms, :ns]), 0
    k1, k2 = min(cfg.k1, ms, ns), min(cfg.k2, ms, ns)
    wk = O.WEIGHT_POWER if cfg.kind == "sparse_lowrank" else O.WEIGHT_CONST
    t0 = time.perf_counter()
    O.cabs_run(A, k1, k2, cfg.iters, seed=cfg.seed, n_samples=T, weight_kind=wk)
    t = time.perf_counter() - t0
    return {"value": (ms + ns) / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"leading {ms} x {ns} block of {cfg.name} (k1={k1}, k2={k2}, {cfg.iters} Lloyd iterations"
                      f"{f', residual on {T} sampled entries' if T else ''}), one full S1-S10 step of the FP64 "
                      f"NumPy oracle ({t:.1f} s)"}


def parity_block(cfg, A_host, pipe, res, plan, dev, row_sample=2048):
    """Full-size parity of this bench run against the FP64 oracle, teacher-forced where the full
    oracle would take minutes.  Every comparison is on the SAME A:
      S1  pilot indices bit-exact (oracle Philox/Lemire/Floyd);  S2/S3 gathers bit-exact;
      S4-S5  the oracle's sketch of the gathered C, R, W -> r exact, P, Q within 1e-4;
      S7  every GPU centre = weighted mean of its GPU cluster (FP64 on the GPU's embedding), 1e-5;
      S6  objective non-increasing (1e-6 relative);
      S8  the oracle's snap of the GPU's final centres on the GPU's embedding -> representatives
          bit-exact, or the first divergence in visiting order is a near tie (gap < 1e-5);
      S9  the oracle's sketch from the GPU's follow-up indices -> r exact, U, V, s within 1e-4;
      S10 the GPU residual of a sampled row block vs the oracle's on the same rows and factors."""
    from oracle import cabs as O
    from oracle import rng
    from paper_1607_07395_b200 import cabs as C
    from paper_1607_07395_b200.dist import make_plan
    out = {"kind": "full-size, teacher-forced per step (the full FP64 Lloyd loop on 1.5e5 points is minutes)"}
    t0 = time.perf_counter()
    m, n, k1, k2 = cfg.m, cfg.n, cfg.k1, cfg.k2
    I, J = res["I"].numpy(), res["J"].numpy()
    out["S1_pilot_indices_exact"] = bool(np.array_equal(I, rng.floyd(m, k1, cfg.seed, rng.TAG_PILOT_ROWS)) and
                                         np.array_equal(J, rng.floyd(n, k1, cfg.seed, rng.TAG_PILOT_COLS)))
    Cg, Rg, Wg = res["C"].numpy()[:, :k1], res["R"].numpy()[:, :n], res["W"].numpy()[:, :k1]
    Co, Ro, Wo = O.gather(A_host, I, J)
    out["S2_S3_gathers_exact"] = bool(np.array_equal(Cg, Co) and np.array_equal(Rg, Ro) and np.array_equal(Wg, Wo))

    def fro(a, b):
        nb = np.linalg.norm(b)
        return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))

    def aligned(X, Xr):
        X = np.array(X, np.float64, copy=True)
        for c in range(min(X.shape[1], Xr.shape[1])):
            if np.dot(X[:, c], Xr[:, c]) < 0:
                X[:, c] = -X[:, c]
        return X

    sk = O.sketch(Co, Ro, Wo, m, n, k1)
    Po, Qo = O.embeddings(sk)
    r1 = res["r1"]
    Pg = res["P"].numpy()[:, :r1].astype(np.float64)
    Qg = res["Q"].numpy()[:, :r1].astype(np.float64)
    e_p = fro(aligned(Pg, Po), Po) if r1 == sk.r else float("inf")
    e_q = fro(aligned(Qg, Qo), Qo) if r1 == sk.r else float("inf")
    out["S4_S5"] = {"r_gpu": r1, "r_oracle": int(sk.r), "P_rel_fro": e_p, "Q_rel_fro": e_q,
                    "ok": bool(r1 == sk.r and e_p < 1e-4 and e_q < 1e-4)}
    s78 = {}
    for side, X, cen, lab, cw, obj, reps, rep_of in (
            ("rows", Pg, res["cen_r"], res["lab_r"], res["cw_r"], res["obj_r"], res["Ib"], res["rep_r"]),
            ("cols", Qg, res["cen_c"], res["lab_c"], res["cw_c"], res["obj_c"], res["Jb"], res["rep_c"])):
        cen = cen.numpy()[:, :r1].astype(np.float64)
        lab = lab.numpy()[:X.shape[0]].astype(np.int64)
        cwv = cw.numpy()
        sums = np.zeros_like(cen)
        np.add.at(sums, lab, X)
        cnt = np.bincount(lab, minlength=k2).astype(np.float64)
        nz = cnt > 0
        e_c = fro(cen[nz], sums[nz] / cnt[nz, None])
        ob = obj.numpy()
        mono = bool(np.all(ob[1:] <= ob[:-1] * (1 + 1e-6) + 1e-30))
        sn = O.snap(X, cen, cwv)
        g_rep = rep_of.numpy()
        first = None
        for j in sn.order:
            if g_rep[j] != sn.rep_of_centre[j]:
                first = int(j)
                break
        ok_snap = first is None or float(sn.gap[first]) < 1e-5
        s78[side] = {"centres_vs_cluster_means_rel": e_c, "objective_monotone": mono,
                     "reps_exact": bool(np.array_equal(np.sort(g_rep), reps.numpy()) and first is None),
                     "first_divergence": None if first is None else
                     {"centre": first, "oracle_rep": int(sn.rep_of_centre[first]), "gpu_rep": int(g_rep[first]),
                      "oracle_gap": float(sn.gap[first])},
                     "near_ties_gpu": int(res["tie_r" if side == "rows" else "tie_c"].sum()),
                     "ok": bool(e_c < 1e-5 and mono and ok_snap)}
    out["S6_S8"] = s78
    Ib, Jb = res["Ib"].numpy(), res["Jb"].numpy()
    Cb, Rb, Wb = O.gather(A_host, Ib, Jb)
    fu = O.sketch(Cb, Rb, Wb, m, n, k2)
    r2 = res["r2"]
    Ug = res["U"].numpy()[:, :r2].astype(np.float64)
    Vg = res["V"].numpy()[:, :r2].astype(np.float64)
    sg = res["s2"].numpy()[:r2].astype(np.float64)
    ok9 = r2 == fu.r
    e_u = fro(aligned(Ug, fu.U), fu.U) if ok9 else float("inf")
    e_v = fro(aligned(Vg, fu.V), fu.V) if ok9 else float("inf")
    e_s = fro(sg, fu.s) if ok9 else float("inf")
    out["S9"] = {"r_gpu": r2, "r_oracle": int(fu.r), "U_rel_fro": e_u, "V_rel_fro": e_v, "s_rel": e_s,
                 "ok": bool(ok9 and max(e_u, e_v, e_s) < 1e-4)}
    # S10 on a row sample: the GPU's residual of rows [r0, r0 + row_sample) vs the oracle's
    rs = min(row_sample, m)
    r0 = (m - rs) // 2
    sub = make_plan(rs, n, max(k1, k2))
    ws = torch.zeros(C.cabs_workspace_bytes(sub), dtype=torch.uint8, device=dev)
    o = torch.zeros(2, dtype=torch.float64, device=dev)
    C.cabs_residual(sub, pipe.A[r0:r0 + rs], pipe.U[r0:r0 + rs], pipe.s2, pipe.G, r2, o, ws)
    og = o.cpu().numpy()
    ro2, ao2 = O.residual(A_host[r0:r0 + rs], Ug[r0:r0 + rs], Vg, sg)
    rg, ro, ao = math.sqrt(max(og[0], 0)), math.sqrt(ro2), math.sqrt(ao2)
    out["S10_row_sample"] = {"rows": [r0, r0 + rs], "r_gpu": rg, "r_oracle": ro, "a_gpu": math.sqrt(og[1]),
                             "a_oracle": ao, "ok": bool(abs(rg - ro) <= 1e-4 * ro + 1e-6 * ao and
                                                        abs(og[1] - ao2) <= 1e-6 * ao2)}
    out["ok"] = bool(out["S1_pilot_indices_exact"] and out["S2_S3_gathers_exact"] and out["S4_S5"]["ok"] and
                     all(v["ok"] for v in s78.values()) and out["S9"]["ok"] and out["S10_row_sample"]["ok"])
    out["oracle_s"] = time.perf_counter() - t0
    return out


def parity_block_rbf(cfg, x, y, sigma, pipe, res, plan, dev, sample=2048, pairs=1 << 20):
    """Full-size c5 parity on samples the oracle computes one by one: S1 indices bit-exact; the
    generated gathers (a sample of rows of C, of columns of R, all of W) within 2e-6 of the FP64
    entries; S7 centres = cluster means, S6 objective monotone; S10 the GPU's sampled residual on
    the first `pairs` positions vs the oracle's on the same positions with the GPU's factors."""
    from oracle import cabs as O
    from oracle import rng
    from paper_1607_07395_b200 import cabs as C
    out = {"kind": "full-size c5, per-step checks on sampled outputs (the oracle cannot form the 2e6 x 1e6 "
                   "matrix; the whole pipeline is compared with the oracle at reduced sizes in tests/test_gpu_rbf.py)"}
    t0 = time.perf_counter()
    m, n, k1, k2 = cfg.m, cfg.n, cfg.k1, cfg.k2
    osrc = O.RbfSource(x.numpy(), y.numpy(), sigma)
    I, J = res["I"].numpy(), res["J"].numpy()
    out["S1_pilot_indices_exact"] = bool(np.array_equal(I, rng.floyd(m, k1, cfg.seed, rng.TAG_PILOT_ROWS)) and
                                         np.array_equal(J, rng.floyd(n, k1, cfg.seed, rng.TAG_PILOT_COLS)))
    g = np.random.default_rng(0)
    rows = np.sort(g.choice(m, sample, replace=False))
    cols = np.sort(g.choice(n, sample, replace=False))
    e_c = float(np.abs(res["C"].numpy()[rows, :k1] - osrc.entries(rows, J)).max())
    e_r = float(np.abs(res["R"].numpy()[:, cols] - osrc.entries(I, cols)).max())
    e_w = float(np.abs(res["W"].numpy()[:, :k1] - osrc.entries(I, J)).max())
    out["S2_S3_generated_gathers"] = {"C_rows_sampled": sample, "R_cols_sampled": sample, "max_abs_err":
                                      max(e_c, e_r, e_w), "ok": bool(max(e_c, e_r, e_w) < 2e-6)}
    r1 = res["r1"]
    s7 = {}
    for side, X, cen, lab, obj in (("rows", res["P"], res["cen_r"], res["lab_r"], res["obj_r"]),
                                   ("cols", res["Q"], res["cen_c"], res["lab_c"], res["obj_c"])):
        Xn = X.numpy()[:, :r1].astype(np.float64)
        c = cen.numpy()[:, :r1].astype(np.float64)
        lb = lab.numpy()[:Xn.shape[0]].astype(np.int64)
        sums = np.zeros_like(c)
        np.add.at(sums, lb, Xn)
        cnt = np.bincount(lb, minlength=k2).astype(np.float64)
        nz = cnt > 0
        err = float(np.linalg.norm(c[nz] - sums[nz] / cnt[nz, None]) / np.linalg.norm(c[nz]))
        ob = obj.numpy()
        mono = bool(np.all(ob[1:] <= ob[:-1] * (1 + 1e-6) + 1e-30))
        s7[side] = {"centres_vs_cluster_means_rel": err, "objective_monotone": mono, "ok": bool(err < 1e-5 and mono)}
    out["S6_S7"] = s7
    r2 = res["r2"]
    ws = pipe.ws
    o = torch.zeros(2, dtype=torch.float64, device=dev)
    C.cabs_residual(plan, pipe.A, pipe.U, pipe.s2, pipe.G, r2, o, ws, n_samples=pairs, seed=cfg.seed)
    og = o.cpu().numpy()
    pi, pj = rng.residual_pairs(cfg.seed, pairs, m, n)
    iu, inv = np.unique(pi, return_inverse=True)
    Fu = pipe.U[torch.from_numpy(iu).to(dev), :r2].cpu().numpy()
    ro2, ao2 = O.residual_sampled(osrc, Fu, res["V"].numpy()[:, :r2], pi, pj, res["s2"].numpy()[:r2], f_rows=inv)
    rg, ro, ao = math.sqrt(max(og[0], 0)), math.sqrt(ro2), math.sqrt(ao2)
    out["S10_sampled"] = {"pairs": pairs, "r_gpu": rg, "r_oracle": ro, "a_gpu": math.sqrt(og[1]), "a_oracle": ao,
                          "ok": bool(abs(rg - ro) <= 1e-4 * ro + 1e-6 * ao and abs(og[1] - ao2) <= 1e-6 * ao2)}
    out["ok"] = bool(out["S1_pilot_indices_exact"] and out["S2_S3_generated_gathers"]["ok"] and
                     all(v["ok"] for v in s7.values()) and out["S10_sampled"]["ok"])
    out["oracle_s"] = time.perf_counter() - t0
    return out


# ---------------------------------------------------------------------- our arm
def parity_block_sparse(cfg, csr, pipe, res):
    """Full-size sparse parity against the FP64 oracle's CsrSource of the SAME
    matrix: S1 indices bit-exact; S2/S3 the gathered R and W bit-exact, a sample of C's rows bit-
    exact; S10 the oracle's split residual (residual_sparse) on the GPU's follow-up factors vs the
    GPU's (1e-6 of ||A||^2 + ||F S G^T||^2).  The whole pipeline is compared with the oracle at
    reduced sizes in tests/test_gpu_sparse.py."""
    from oracle import cabs as O
    from oracle import rng
    t0 = time.perf_counter()
    ip, ix, v = (t.cpu().numpy() for t in csr)
    osrc = O.CsrSource(ip, ix, v, (cfg.m, cfg.n))
    out = {"kind": "full-size sparse, per-step checks (oracle CsrSource of the same nonzeros)"}
    I = rng.floyd(cfg.m, cfg.k1, cfg.seed, rng.TAG_PILOT_ROWS)
    J = rng.floyd(cfg.n, cfg.k1, cfg.seed, rng.TAG_PILOT_COLS)
    out["S1_pilot_indices_exact"] = bool(np.array_equal(res["I"].numpy(), I) and np.array_equal(res["J"].numpy(), J))
    Rg = res["R"].numpy()[:, :cfg.n]
    Wg = res["W"].numpy()[:, :cfg.k1]
    rows = np.arange(0, cfg.m, max(1, cfg.m // 2048))
    Cg = res["C"].numpy()[rows][:, :cfg.k1]
    out["S2_S3_gathers_exact"] = bool(np.array_equal(Rg, osrc.entries(I, np.arange(cfg.n)))
                                      and np.array_equal(Wg, osrc.entries(I, J))
                                      and np.array_equal(Cg, osrc.entries(rows, J)))
    r2 = res["r2"]
    U, V, s = res["U"].numpy()[:, :r2], res["V"].numpy()[:, :r2], res["s2"].numpy()[:r2]
    rr, ra = O.residual_sparse(osrc, U, V, s)
    b2 = float(np.sum((U.astype(np.float64).T @ U) * np.outer(s, s) * (V.astype(np.float64).T @ V)))
    out["S10"] = {"gpu_resid_sq": res["resid_sq"], "oracle_resid_sq": rr, "gpu_a_sq": res["a_sq"], "oracle_a_sq": ra,
                  "ok": bool(abs(res["resid_sq"] - rr) <= 1e-6 * (ra + b2) and abs(res["a_sq"] - ra) <= 1e-9 * ra)}
    out["ok"] = bool(out["S1_pilot_indices_exact"] and out["S2_S3_gathers_exact"] and out["S10"]["ok"])
    out["oracle_s"] = time.perf_counter() - t0
    return out


def time_sketch_cur(args, cfg, A, flush, samples):
    """The paper's Sketch-CUR baseline (P:115, P:312 (a): target rate 3x the base rate; SURVEY
    NEXT-4) on the same matrix and kernels: base = the pilot's uniform k1 rows / columns, 3 k1
    uniform targets, BR-CUR (Algorithm 1), the P:313 error."""
    from paper_1607_07395_b200.pipeline import SketchCurRun
    run = SketchCurRun(A, cfg.m, cfg.n, cfg.k1, mult=3, seed=cfg.seed, residual_samples=samples)
    for _ in range(max(args.warmup, 2)):
        run.run()
    ts = []
    for _ in range(min(args.steps, 3)):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        run.run(with_residual=False)
        e1.record()
        from paper_1607_07395_b200 import cabs as C
        C.cabs_residual(run.plan, run.A, run.F, None, run.G, run.k1, run.out, run.ws, n_samples=samples, seed=cfg.seed)
        e2.record()
        torch.cuda.synchronize()
        ts.append((e0.elapsed_time(e1), e1.elapsed_time(e2)))
    sk = statistics.mean(t[0] for t in ts)
    rs = statistics.mean(t[1] for t in ts)
    return {"followup": "P:312 (a) Sketch-CUR: BR-CUR (Alg. 1, cabs_br_cur) with 3 k1 uniform targets",
            "value": (cfg.m + cfg.n) / ((sk + rs) / 1e3), "unit": UNIT, "ms_per_step": sk + rs,
            "breakdown_ms": {"br_cur": sk, "residual": rs},
            "rel_err": math.sqrt(max(run.out[0].item(), 0) / run.out[1].item())}


def time_rank_sweep(pipe, h=None):
    """The validation rank sweep on the timed pipeline's follow-up sketch:
    the holdout errors for every rank and the chosen one."""
    from paper_1607_07395_b200.pipeline import rank_sweep
    h = h or min(2 * pipe.cfg.k2, pipe.plan.kmax)
    rank_sweep(pipe, h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e, rank, Hr, Hc = rank_sweep(pipe, h)
    dt = 1e3 * (time.perf_counter() - t0)
    return {"desc": "P:232 validation set: holdout errors for rho = 0..r (cabs_holdout_errors), argmin",
            "holdout": [int(Hr.numel()), int(Hc.numel())], "ms_wall": dt, "rank_chosen": rank,
            "r": int(e.numel() - 1), "rel_err_at_chosen": math.sqrt(float(e[rank] / e[0])),
            "rel_err_at_r": math.sqrt(float(e[-1] / e[0]))}


def time_variant(args, cfg, A, plan, rank, world, comm, flush, stream, followup, desc):
    """One of the paper's follow-up variants on the same matrix, timed like the main step."""
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    samples = C5_SAMPLES if cfg.kind == "rbf_mixture" else 0
    wk = 1 if cfg.kind == "sparse_lowrank" else 0  # WEIGHT_POWER for sparse inputs
    vp = CabsPipeline(A, cfg.m, cfg.n, CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed, followup=followup,
                                                  residual_samples=samples, weight_kind=wk), rank, world, comm=comm,
                      plan=plan)
    for _ in range(args.warmup):
        vp.run()
    per = {}
    for _ in range(min(args.steps, 3)):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        vp.run(timed=True)
        for k_, v in vp.step_ms().items():
            per.setdefault(k_, []).append(v)
    graph = None
    if world == 1 and not args.eager:
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            vp.run()
            graph, _ = vp.capture(stream=cap)
        stream.wait_stream(cap)
        torch.cuda.synchronize()
    ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        graph.replay() if graph is not None else vp.run()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier(world)
        ms.append(e0.elapsed_time(e1))
    t = allreduce_max(sum(ms), world) / args.steps
    res = vp.results()
    return {"followup": desc, "value": (cfg.m + cfg.n) / (t / 1e3), "unit": UNIT, "ms_per_step": t,
            "breakdown_ms": {k_: allreduce_max(statistics.mean(v), world) for k_, v in per.items()},
            "rel_err_followup": math.sqrt(max(res["resid_sq"], 0) / res["a_sq"])}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=BASE_CFG[1])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-size oracle parity block")
    ap.add_argument("--no-variants", action="store_true", help="skip the variant (f) timing")
    ap.add_argument("--eager", action="store_true", help="time stream-ordered launches instead of the CUDA graph")
    args = ap.parse_args()
    cfg = ALL_CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)

    from paper_1607_07395_b200 import cabs as C
    from paper_1607_07395_b200.dist import TorchComm, make_plan
    from paper_1607_07395_b200.pipeline import STEPS, CabsConfig, CabsPipeline

    world, rank, local = setup_dist(args.gpus)
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    C.load()
    plan = make_plan(cfg.m, cfg.n, max(cfg.k1, cfg.k2), rank, world, align=CHUNK)
    rbf = cfg.kind == "rbf_mixture"
    sparse = cfg.kind == "sparse_lowrank"
    if rbf:  # implicit source: the points on every rank, entries generated on access
        xh, yh, sigma = make_rbf(cfg)
        A = C.RbfSource(xh.to(dev), yh.to(dev), sigma)
    elif sparse:  # this rank's row block as CSR + CSC
        sp_arrays, sp_full = sparse_block(cfg, plan.row_begin, plan.row_end, dev)
        A = C.CsrSource(*sp_arrays, cfg.n)
    else:
        gen = Generator(cfg, device=dev)
        A = gen.rows(plan.row_begin, plan.row_end)
        del gen
    torch.cuda.empty_cache()
    comm = TorchComm(dev) if world > 1 else None
    samples = C5_SAMPLES if rbf else 0
    # sparse inputs: the power weighting Upsilon(x) = x^2 ("a fast-growing function for sparse
    # matrices"; SPEC default p = 2), constant for dense
    wk = C.WEIGHT_POWER if sparse else C.WEIGHT_CONST
    ccfg = CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed, residual_samples=samples, weight_kind=wk)
    pipe = CabsPipeline(A, cfg.m, cfg.n, ccfg, rank, world, comm=comm, plan=plan)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MiB > 126 MB L2

    args.warmup = max(args.warmup, 3)  # timing rule: at least 3 warm-up steps
    for _ in range(args.warmup):
        pipe.run()
    torch.cuda.synchronize()

    # per-step breakdown: eager steps with an event between entry points
    per_step = {s: [] for s in STEPS}
    stream = torch.cuda.current_stream()
    for _ in range(min(args.steps, 3)):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        pipe.run(timed=True)
        for s, v in pipe.step_ms().items():
            per_step[s].append(v)
    # the timed steps: one pass of the hot path as ONE CUDA-graph launch on a single GPU (the
    # capture holds every library launch, the side-stream fork/join and the memsets); eager
    # stream-ordered launches with the collectives on N > 1
    graph, graph_launches = (None, 0)
    if world == 1 and not args.eager:
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            pipe.run()  # warm the capture stream
            graph, graph_launches = pipe.capture(stream=cap)
        stream.wait_stream(cap)
        torch.cuda.synchronize()
    step_ms = []
    launches0 = C.cabs_launch_count()
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.fill_(1.0)
            barrier(world)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            if graph is not None:
                graph.replay()
            else:
                pipe.run()
            e1.record(stream)
            torch.cuda.synchronize()
            barrier(world)
            step_ms.append(e0.elapsed_time(e1))
    launches = graph_launches if graph is not None else (C.cabs_launch_count() - launches0) // max(args.steps, 1)
    total_ms = allreduce_max(sum(step_ms), world)
    ms = total_ms / args.steps
    step_mean = {s: allreduce_max(statistics.mean(v), world) for s, v in per_step.items()}
    res = pipe.results()

    # ---- end to end: host-resident A, copied in every step; the sketch and metric read back
    e2e = None
    A_host = None
    if not args.no_e2e:
        if rbf:  # the inputs are the points x, y
            ins = [(A.x, xh.pin_memory()), (A.y, yh.pin_memory())]
        elif sparse:  # the CSR and CSC arrays
            ins = [(t, t.cpu().pin_memory()) for t in sp_arrays]
        else:
            A_host = A.cpu().pin_memory()
            ins = [(A, A_host)]
        outs = [pipe.U, pipe.s2, pipe.V, pipe.Ib, pipe.Jb, pipe.out]
        host_outs = [torch.empty_like(t, device="cpu").pin_memory() for t in outs]
        d2h = sum(t.numel() * t.element_size() for t in outs)
        h2d = sum(h.numel() * h.element_size() for _, h in ins)
        e2e_ms = []
        for _ in range(max(2, min(args.steps, 5))):
            flush.fill_(1.0)
            barrier(world)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for dst, h in ins:
                dst.copy_(h, non_blocking=True)
            if graph is not None:
                graph.replay()
            else:
                pipe.run()
            for h, t in zip(host_outs, outs):
                h.copy_(t, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier(world)
            e2e_ms.append(e0.elapsed_time(e1))
        e2e_t = allreduce_max(statistics.mean(e2e_ms), world)
        e2e = {"value": (cfg.m + cfg.n) / (e2e_t / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": e2e_t}

    # ---- linear access end to end ("never knowing the remaining entries"): A never leaves pinned
    # host memory (cabs_source.host_resident); S1-S9 read only the sampled rows and columns through the mapped
    # address, the error is the sampled estimate (Z17) on LIN_SAMPLES seeded pairs; the sketch and the metric
    # are read back as in `e2e`.  Not the contract's `e2e` (which copies all of A): an extra line.
    e2e_lin = None
    At = None  # A^T on the device (block-wise transpose: no second full-size temporary), when it fits
    if (world == 1 and isinstance(A, torch.Tensor) and not (args.no_variants and A_host is None)
            and 2.4 * A.numel() * 4 < torch.cuda.get_device_properties(dev).total_memory):
        At = torch.empty((cfg.n, cfg.m), dtype=torch.float32, device=dev)
        for r0 in range(0, cfg.m, 8192):
            At[:, r0:r0 + 8192] = A[r0:r0 + 8192, :cfg.n].t()
    if A_host is not None and world == 1:
        from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
        lcfg = CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed, residual_samples=LIN_SAMPLES)
        At_host = None  # both layouts in host memory (cabs_source.at)
        if At is not None:
            At_host = torch.empty(At.shape, dtype=torch.float32, pin_memory=True)
            At_host.copy_(At)
        hp = CabsPipeline(C.HostDense(A_host, dev, At=At_host), cfg.m, cfg.n, lcfg, plan=plan)
        for _ in range(2):
            hp.run()
        torch.cuda.synchronize()
        outs_h = [hp.U, hp.s2, hp.V, hp.Ib, hp.Jb, hp.out]
        host_h = [torch.empty_like(t, device="cpu").pin_memory() for t in outs_h]
        lin_ms = []
        for _ in range(max(2, min(args.steps, 5))):
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hp.run()
            for h, t in zip(host_h, outs_h):
                h.copy_(t, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            lin_ms.append(e0.elapsed_time(e1))
        lt = statistics.mean(lin_ms)
        hp.run(timed=True)
        lin_steps = hp.step_ms()
        same = bool(torch.equal(hp.Ib, pipe.Ib) and torch.equal(hp.Jb, pipe.Jb) and torch.equal(hp.U, pipe.U)
                    and torch.equal(hp.V, pipe.V) and torch.equal(hp.s2, pipe.s2))
        kk = cfg.k1 + cfg.k2
        e2e_lin = {"value": (cfg.m + cfg.n) / (lt / 1e3), "unit": UNIT, "ms_per_step": lt,
                   "what": "S1-S9 + sampled error with A resident in pinned HOST memory (zero-copy gathers of the "
                           "sampled rows / columns only; nothing else of A crosses the interconnect)",
                   "residual_samples": LIN_SAMPLES, "breakdown_ms": lin_steps,
                   "interconnect_bytes_per_step": {"useful": 4 * kk * (cfg.m + cfg.n) + 4 * LIN_SAMPLES,
                                                   "as_32B_sectors": kk * (32 * cfg.m + 4 * cfg.n) + 32 * LIN_SAMPLES},
                   "d2h_bytes_per_step": sum(t.numel() * t.element_size() for t in outs_h),
                   "factors_identical_to_device_resident_run": same,
                   "rel_err_sampled": math.sqrt(max(float(hp.out[0]), 0.0) / float(hp.out[1]))}
        e2e_lin["layouts"] = "row-major + column-major copies in host memory (cabs_source.at)" if At_host is not None \
            else "row-major only"
        if At_host is not None:  # the single-layout figure beside it: column gathers as one 32-byte sector per element
            hp1 = CabsPipeline(C.HostDense(A_host, dev), cfg.m, cfg.n, lcfg, plan=plan)
            hp1.run()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            hp1.run()
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_lin["row_major_only_ms_per_step"] = e0.elapsed_time(e1)
            e2e_lin["interconnect_bytes_per_step"]["as_32B_sectors_row_major_only"] = \
                e2e_lin["interconnect_bytes_per_step"].pop("as_32B_sectors")
            del hp1
        del hp, At_host

    # ---- the paper's follow-up variant (f) (hard threshold) on the same
    # matrix: S6-S8 replaced by cabs_hard_select_pair; timed the same way (graph on one GPU)
    variants = {}
    for fu_name, fu, fu_desc in (("hard_threshold", "hard", "P:312 variant (f): top-k2 weighting coefficients "
                                  "(cabs_hard_select_pair)"),
                                 ("leverage", "leverage", "P:312 variant (e): Supp. 3 orthogonalization + leverage-"
                                  "score sampling (cabs_orthogonalize, cabs_leverage_select_pair)")):
        if args.no_variants:
            break
        variants[fu_name] = time_variant(args, cfg, A, plan, rank, world, comm, flush, stream, fu, fu_desc)
    if not args.no_variants and At is not None:
        # the same CABS with the block held column-major (cabs_source.transposed): contiguous column
        # gathers, k (n + m/8) gather sectors instead of k (m + n/8); results identical (tests/test_gpu_transposed.py)
        variants["colmajor_layout"] = time_variant(args, cfg, C.TransposedDense(At), plan, rank, world, comm, flush,
                                                   stream, "kmeans", "Algorithm 2 unchanged; A held column-major "
                                                   "(cabs_source.transposed = 1)")
        # and with both layouts resident (cabs_source.at): every gather a contiguous copy
        variants["dual_layout"] = time_variant(args, cfg, C.DualDense(A, At), plan, rank, world, comm, flush, stream,
                                               "kmeans", "Algorithm 2 unchanged; A held row-major and column-major "
                                               "(cabs_source.at)")
    del At
    torch.cuda.empty_cache()
    if not args.no_variants and world == 1:
        variants["sketch_cur"] = time_sketch_cur(args, cfg, A, flush, samples)
        variants["rank_sweep"] = time_rank_sweep(pipe)

    if rank != 0:
        return 0
    peaks, peak_src = load_peaks()
    traffic = load_traffic()
    # ---- rooflines, algorithmic work per SURVEY.md section 8(d):
    #   k-means (S6-S7): 2 r k2 flop per point per Lloyd pass, c passes over m + n points;
    #   residual (S10): A once (4 m n bytes) plus the factors F (4 m k2) and G (4 n k2).
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    ffma_tf = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    tf32_tf = 0.5 * float(peaks.get("bf16_tflops", 1627.4))
    d_emb = int(pipe.r1.item())  # embedding dimension r <= k1 the k-means runs on
    km_path = C.cabs_kmeans_path(cfg.k2, d_emb)
    km_flops = 2.0 * cfg.iters * (m_loc_rows(plan) + n_loc_cols(plan)) * cfg.k2 * d_emb
    km_ms = step_mean["kmeans"]
    if km_path == "prune":
        km_peak, km_bound = ffma_tf, "alu"
        km_src = (f"derived: FFMA peak 148 SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz = {ffma_tf:.1f} TFLOP/s; "
                  f"achieved counts the method's 2 r k2 flop per point and pass (SURVEY 8(d)); the pruned kernel "
                  f"evaluates only the candidates the triangle-inequality bounds leave")
        km_kernel = ("lloyd_prune_kernel (cabs_kmeans_pair: exact Hamerly/Elkan bounds + FP32 direct differences, "
                     "both sides, all iterations, one launch)")
    elif km_path == "tc":
        km_peak, km_bound = tf32_tf / 3.0, "tensor"
        km_src = (f"MEASURED_PEAKS bf16_tflops {peaks.get('bf16_tflops')} x 0.5 (nominal TF32:BF16) / 3 "
                  f"(3xTF32: three MMAs per algorithmic flop)")
        km_kernel = "lloyd_tc_kernel (cabs_kmeans_pair: tcgen05 3xTF32 cross-term + FP32 direct-difference refine)"
    else:
        km_peak, km_bound = ffma_tf, "alu"
        km_src = f"derived: FFMA peak 148 SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz = {ffma_tf:.1f} TFLOP/s"
        km_kernel = "lloyd_persistent_kernel (cabs_kmeans_pair: both sides, all iterations, one launch; FFMA)"
    kmeans = {"kernel": km_kernel, "bound": km_bound, "achieved": km_flops / (km_ms / 1e3) / 1e12, "peak": km_peak,
              "unit": "TFLOP/s", "traffic": traffic_of(traffic, f"{cfg.name}_lloyd"), "peak_source": km_src,
              "algorithmic_flops_per_launch": km_flops, "launch_ms": km_ms,
              "timing": "CUDA events around cabs_kmeans_pair (eager runs): the persistent kernel plus its "
                        "weight / Floyd / init launches"}
    kmeans["frac"] = kmeans["achieved"] / kmeans["peak"]
    m_loc = plan.row_end - plan.row_begin
    r2n = int(pipe.r2.item())
    if rbf:  # sampled: two random factor rows per owned pair; entries generated
        res_bytes = 4.0 * 2 * r2n * samples * (m_loc / cfg.m)
        res_kernel = "residual_sampled_kernel (Philox pairs, generated entries, warp dot of random factor rows)"
    elif sparse:  # the nonzeros once (value + column index), the row pointers, F and G once
        res_bytes = 8.0 * A.nnz + 8.0 * (m_loc + 1) + 4.0 * r2n * (m_loc + 2 * cfg.n)
        res_kernel = ("sparse_res_nnz_kernel + orth_gram (cabs_residual on a CSR source: nonzeros + the r x r "
                      "Gram products, A - F S G^T never formed)")
    else:
        res_bytes = 4.0 * (m_loc * cfg.n + m_loc * cfg.k2 + cfg.n * cfg.k2)
        res_tc = C.cabs_residual_path(r2n) == "tc"
        res_kernel = (("residual_tc_kernel (tcgen05 3xTF32, TMA)" if res_tc else "residual_ffma_kernel") +
                      " (cabs_residual: fused F diag(s) G^T - A, squared-sum)")
    res_ms = step_mean["residual"]
    achieved = res_bytes / (res_ms / 1e3) / 1e9
    peak = float(peaks["hbm_gbs"])
    residual = {"kernel": res_kernel, "bound": "hbm",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic_of(traffic, f"{cfg.name}_residual"),
                "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json, copy bandwidth)",
                "algorithmic_bytes_per_launch": res_bytes, "launch_ms": res_ms,
                "timing": "CUDA events around cabs_residual (eager runs): G split + the fused kernel + final reduce"}
    dominant = kmeans if km_ms >= res_ms else residual
    kmeans_pts = cfg.iters * (cfg.m + cfg.n) / (step_mean["kmeans"] / 1e3)
    sketch_ms = sum(step_mean[s] for s in STEPS if s != "residual")
    a_gb = cfg.m * cfg.n * 4 / 1e9
    l2_note = (f"flushed (256 MiB write) before every timed step; implicit A, {samples:.0e} sampled entries read "
               f"{4.0 * 2 * r2n * samples / 1e12:.1f} TB of random factor rows (> L2)" if rbf else
               f"flushed (256 MiB write) before every timed step; sparse A, {A.nnz} nonzeros "
               f"({A.nnz / (cfg.m * cfg.n):.4%}), CSR + CSC {16.0 * A.nnz / 1e9:.2f} GB" if sparse else
               f"flushed (256 MiB write) before every timed step; A ({a_gb:.1f} GB) > L2")
    line = {
        "metric": METRIC, "value": (cfg.m + cfg.n) / (ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(cfg),
                   "m": cfg.m, "n": cfg.n, "weights": "power 2" if sparse else "const",
                   "k1": cfg.k1, "k2": cfg.k2, "iters": cfg.iters, "mode": "stabilized", "parallelism": f"rows{world}",
                   "l2": l2_note, "residual_samples": samples or "exact",
                   "timing": "per-step CUDA events on the launching stream, barrier+sync both sides, max over ranks",
                   "launch": "one CUDA graph per step (captured S1-S10)" if graph is not None else "stream-ordered"},
        "breakdown_ms": step_mean,
        "sketch_ms": sketch_ms,
        "sketch_rows_cols_per_s": (cfg.m + cfg.n) / (sketch_ms / 1e3),
        "kmeans_pts_per_s": kmeans_pts,
        "roofline": dominant,
        "rooflines": {"kmeans": kmeans, "residual": residual},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "quality": {"rel_err_followup": math.sqrt(max(res["resid_sq"], 0) / res["a_sq"]),
                    "near_ties_rows": int(res["tie_r"].sum()), "near_ties_cols": int(res["tie_c"].sum())},
    }
    line["variants"] = variants
    if e2e_lin is not None:
        line["e2e_linear_access"] = e2e_lin
    if e2e:
        line["e2e"] = e2e
    if world == 1 and not (args.no_cpu_baseline and args.no_parity):
        if rbf:
            A_np = None
            if not args.no_parity:
                line["parity"] = parity_block_rbf(cfg, xh, yh, sigma, pipe, res, plan, dev)
        elif sparse:
            A_np = None
            if not args.no_parity:
                line["parity"] = parity_block_sparse(cfg, sp_full, pipe, res)
        else:
            A_np = A_host.numpy() if A_host is not None else A.cpu().numpy()
            if not args.no_parity:
                line["parity"] = parity_block(cfg, A_np, pipe, res, plan, dev)
        if not args.no_cpu_baseline:
            line["cpu_baseline"] = oracle_cpu_baseline(cfg, A_np)
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
