#!/usr/bin/env python
"""Benchmark of the CABS hot path (S1-S10) on B200 -- prints ONE JSON line.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

A step is one pass of the whole hot path -- pilot sampling + gathers, pilot
sketch + embeddings, weighted Lloyd k-means on both sides, snap, follow-up
gathers + sketch, and the fused residual -- over the synthetic matrix of
BASELINE.json configs[1] (c2, 20000 x 10000, k1 = k2 = 50, 20 Lloyd iterations)
held in HBM.  Timing: W untimed warm-ups, then K steps, each bracketed by a
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

import torch  # noqa: E402

from workloads import CHUNK, CONFIGS, Generator  # noqa: E402

METRIC = "CABS sketch wall time & k-means pts/s at 1/2/4/8 GPU; HBM GB/s vs peak"
UNIT = "rows+cols/s"
BASE_CFG = {1: "c2"}  # BASELINE.json configs[1]


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
def run_reference(args, cfg):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    from oracle import cabs as O
    from workloads import make_A
    cores = len(os.sched_getaffinity(0))
    A = make_A(cfg, device="cpu").numpy()
    budget = 240.0
    times = []
    t_start = time.time()
    for i in range(args.warmup + args.steps):
        if i < args.warmup:  # warm-up: a small sample (page-in, BLAS init)
            O.cabs_run(A[:2000], min(cfg.k1, 20), min(cfg.k2, 20), 2, seed=cfg.seed)
            continue
        t0 = time.perf_counter()
        O.cabs_run(A, cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed)
        times.append(time.perf_counter() - t0)
        if time.time() - t_start > budget:
            break
    t = statistics.mean(times)
    v = (cfg.m + cfg.n) / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{cfg.name}: {cfg.note}", "m": cfg.m, "n": cfg.n, "k1": cfg.k1, "k2": cfg.k2,
                       "iters": cfg.iters},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"full {cfg.name} step S1-S10 (FP64 NumPy oracle), {len(times)} step(s)"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def oracle_cpu_baseline(cfg, A_cpu):
    """The oracle as it stands, on the host cores, on a bounded sample (one full step)."""
    from oracle import cabs as O
    cores = len(os.sched_getaffinity(0))
    t0 = time.perf_counter()
    O.cabs_run(A_cpu, cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed)
    t = time.perf_counter() - t0
    return {"value": (cfg.m + cfg.n) / t, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"one full {cfg.name} step S1-S10 of the FP64 NumPy oracle ({t:.1f} s)"}


# ---------------------------------------------------------------------- our arm
def time_variant(args, cfg, A, plan, rank, world, comm, flush, stream, followup, desc):
    """One of the paper's follow-up variants on the same matrix, timed like the main step."""
    from paper_1607_07395_b200.pipeline import CabsConfig, CabsPipeline
    vp = CabsPipeline(A, cfg.m, cfg.n, CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed, followup=followup),
                      rank, world, comm=comm, plan=plan)
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
    ap.add_argument("--no-variants", action="store_true", help="skip the variant (f) timing")
    ap.add_argument("--eager", action="store_true", help="time stream-ordered launches instead of the CUDA graph")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
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
    gen = Generator(cfg, device=dev)
    A = gen.rows(plan.row_begin, plan.row_end)
    del gen
    torch.cuda.empty_cache()
    comm = TorchComm(dev) if world > 1 else None
    ccfg = CabsConfig(cfg.k1, cfg.k2, cfg.iters, seed=cfg.seed)
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
    if not args.no_e2e:
        A_host = A.cpu().pin_memory()
        outs = [pipe.U, pipe.s2, pipe.V, pipe.Ib, pipe.Jb, pipe.out]
        host_outs = [torch.empty_like(t, device="cpu").pin_memory() for t in outs]
        d2h = sum(t.numel() * t.element_size() for t in outs)
        h2d = A_host.numel() * A_host.element_size()
        e2e_ms = []
        for _ in range(max(2, min(args.steps, 5))):
            flush.fill_(1.0)
            barrier(world)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            pipe.A.copy_(A_host, non_blocking=True)
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

    if rank != 0:
        return 0
    peaks, peak_src = load_peaks()
    traffic = load_traffic()
    # ---- rooflines.  The dominant kernel of the step is the persistent
    # Lloyd kernel (S6-S7, both sides in one launch): FP32 ALU-bound -- per (point, centre,
    # dimension) one FADD + one FFMA (direct differences) = 3 flops in 2 FP32 lane-ops, so the
    # attainable peak is 3/4 of the FFMA peak 148 SM x 128 lanes x 2 flops x max SM clock.
    # Timed as the k-means phase (the launch plus the small weight / init kernels before it).
    sm_mhz = float(peaks.get("sm_max_mhz", 1965.0))
    ffma_tf = 148 * 128 * 2 * sm_mhz * 1e6 / 1e12
    lloyd_peak = 0.75 * ffma_tf
    d_emb = int(pipe.r1.item())  # embedding dimension r <= k1 the k-means runs on
    lloyd_flops = 3.0 * cfg.iters * (m_loc_rows(plan) + n_loc_cols(plan)) * cfg.k2 * d_emb
    km_ms = step_mean["kmeans"]
    lloyd = {"kernel": "lloyd_persistent_kernel (cabs_kmeans_pair: both sides, all iterations, one launch)",
             "bound": "alu", "achieved": lloyd_flops / (km_ms / 1e3) / 1e12, "peak": lloyd_peak, "unit": "TFLOP/s",
             "traffic": traffic_of(traffic, "lloyd"),
             "peak_source": f"derived: 0.75 x FFMA peak (148 SM x 128 FP32 lanes x 2 x {sm_mhz:.0f} MHz = "
                            f"{ffma_tf:.1f} TFLOP/s); direct-difference op mix FADD+FFMA",
             "algorithmic_flops_per_launch": lloyd_flops, "launch_ms": km_ms}
    lloyd["frac"] = lloyd["achieved"] / lloyd["peak"]
    # the fused residual (S10), HBM-bound: it must stream A once (m*n*4 bytes) plus the factors
    # F (m*k2*4) and G (n*k2*4).
    m_loc = plan.row_end - plan.row_begin
    res_bytes = 4.0 * (m_loc * cfg.n + m_loc * cfg.k2 + cfg.n * cfg.k2)
    res_ms = step_mean["residual"]
    achieved = res_bytes / (res_ms / 1e3) / 1e9
    peak = float(peaks["hbm_gbs"])
    residual = {"kernel": "residual_tc_kernel (cabs_residual: fused F diag(s) G^T - A, squared-sum)", "bound": "hbm",
                "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": traffic_of(traffic, "residual"),
                "peak_source": f"{peak_src} hbm_gbs (MEASURED_PEAKS.json)",
                "algorithmic_bytes_per_launch": res_bytes, "launch_ms": res_ms}
    kmeans_pts = cfg.iters * (cfg.m + cfg.n) / (step_mean["kmeans"] / 1e3)
    sketch_ms = sum(step_mean[s] for s in STEPS if s != "residual")
    line = {
        "metric": METRIC, "value": (cfg.m + cfg.n) / (ms / 1e3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{cfg.name} = BASELINE.json configs[1]: {cfg.note}", "m": cfg.m, "n": cfg.n,
                   "k1": cfg.k1, "k2": cfg.k2, "iters": cfg.iters, "mode": "stabilized", "parallelism": f"rows{world}",
                   "l2": "flushed (256 MiB write) before every timed step; A (800 MB) > L2",
                   "timing": "per-step CUDA events on the launching stream, barrier+sync both sides, max over ranks",
                   "launch": "one CUDA graph per step (captured S1-S10)" if graph is not None else "stream-ordered"},
        "breakdown_ms": step_mean,
        "sketch_ms": sketch_ms,
        "sketch_rows_cols_per_s": (cfg.m + cfg.n) / (sketch_ms / 1e3),
        "kmeans_pts_per_s": kmeans_pts,
        "roofline": lloyd,
        "rooflines": {"lloyd": lloyd, "residual": residual},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "quality": {"rel_err_followup": math.sqrt(max(res["resid_sq"], 0) / res["a_sq"]),
                    "near_ties_rows": int(res["tie_r"].sum()), "near_ties_cols": int(res["tie_c"].sum())},
    }
    line["variants"] = variants
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = oracle_cpu_baseline(cfg, A.cpu().numpy())
    print(json.dumps(line))
    return 0


if __name__ == "__main__":
    sys.exit(main())
