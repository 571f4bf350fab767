#!/usr/bin/env python3
"""Headline benchmark: config 4 of BASELINE.json — the Gauss-Newton-Laplace
posterior (mean + marginal variances) of the 1M-unknown space-time Burgers
GMRF (P1, 1000 nodes × 1000 implicit-Euler slices), 10 GN steps + Laplace +
selected-inversion variances.

A step is one full posterior from the IC data: prior assembly on the device,
IC conditioning (factor + solve), 10 GN iterations (residual, Jacobian,
H = q_eff + JᵀΛJ into the factor storage, numeric factorization, solve, Armijo
line search), the Laplace precision, its factorization and the variances.
Host symbolic analysis (nested dissection, supernodes, plans) is one-off per
problem shape and reported separately as ``host_setup_s``.

  value : device-timed seconds per posterior (CUDA events on the library's
          stream; results stay in HBM), max over ranks.
  e2e   : the same posterior through the C-ABI with host buffers (IC values in,
          mean + variances out; copies inside the timed region).
  --impl reference : the unmodified reference (oracle/_ref, compiled from
          /root/reference) on a bounded sample of the same workload,
          extrapolated to full size with the reference's own measured per-stage
          rates.

Multi-GPU (torchrun, N>1): batch sharding — each rank solves its own
independent posterior (BASELINE config 5's "independent problems one per GPU"
mode); no data-path collective; scaling "weak". With --partition: ONE
posterior whose factorization, solves and selected inversion are partitioned
along the top nested-dissection separators across the ranks (Schur
complements and solve vectors over NCCL, paper_2503_08343_b200/partition.py);
scaling "strong".
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gauss-Newton-Laplace posterior time (s) & Cholesky FP64 TFLOP/s, % roofline"
UNIT = "s"
# Reference AMD symbolic of the full config-4 matrix, computed with oracle/_ref
# (the unmodified reference amd_order + symbolic_analyze) in the build
# container; equals SURVEY §6's measurement.
C4_FULL_AMD_FLOPS = 266698072912.0
C4_FULL_AMD_NNZL = 223320550.0
C4_FULL_N = 1_000_000
SAMPLE = (149, 150)  # reference CPU sample: 150 nodes × 150 slices (~18 s single-core)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except OSError:
        return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline
# ---------------------------------------------------------------------------
def reference_sample(n_el=SAMPLE[0], n_t=SAMPLE[1]):
    """Times the unmodified reference (run_burgers chain: spatiotemporal_prior →
    condition_on → gauss_newton(10) → laplace_posterior → variance_takahashi) on
    a bounded sample, then extrapolates each stage to the full config-4 size:
    numeric factorizations and Takahashi by the AMD flop ratio Σc², AMD +
    symbolic by the nnz(L) ratio, everything else linearly in n."""
    from oracle.pyoracle import Ref
    ref = Ref()
    p = [1, n_el, -1.0, 1.0, n_t, 1.0, 0.01 / math.pi, 0.5, 10, 1, 1, 10, 2, 1, 1.0, 1e-10, 1e8,
         0, 1e12, 10, 1, 1]
    t0 = time.perf_counter()
    b = ref.build("spatiotemporal", p)
    wall = time.perf_counter() - t0
    q = b.mat("Q_la")
    st = ref.time_stages(q.nrows, q.col_ptr, q.row_idx, q.values, 1)
    n_gn = len(b.vec("gn_objective"))
    n_fact = 1 + n_gn + 1          # conditioning, GN refactors, fresh Laplace factor
    n_sym = 3                      # AMD + symbolic: conditioning, GN (once), Laplace
    fact = n_fact * st["numeric_s"]
    taka = st["takahashi_s"]
    sym = n_sym * (st["amd_s"] + st["symbolic_s"])
    rest = max(0.0, wall - fact - taka - sym)
    sf = C4_FULL_AMD_FLOPS / st["flops"]
    sl = C4_FULL_AMD_NNZL / st["nnz_l"]
    sn = C4_FULL_N / q.nrows
    full = (fact + taka) * sf + sym * sl + rest * sn
    return {
        "value": full, "unit": UNIT, "cores": 1, "kind": "reference",
        "sample": (f"unmodified reference (oracle/_ref) run_burgers chain at {n_el + 1} nodes x "
                   f"{n_t} slices (n={q.nrows}), {n_gn} GN steps + Laplace + Takahashi: "
                   f"{wall:.2f} s measured single-threaded; extrapolated to n=1e6 by stage: "
                   f"factorizations+Takahashi x{sf:.0f} (AMD flops), AMD+symbolic x{sl:.0f} "
                   f"(nnz L), rest x{sn:.0f} (n)"),
        "measured_sample_s": wall,
        "stages_sample_s": {"numeric_x%d" % n_fact: fact, "takahashi": taka, "amd_symbolic": sym,
                            "rest": rest},
        "cpu": cpu_model(),
        **measured_full_reference(),
    }


def measured_full_reference():
    """The reference's own stage timings for the FULL config-4 workload, when the
    full-size fixture is committed (tests/golden/c4_burgers_full.npz, written by
    make_golden_full.py in the build container: single core, other jobs running
    beside it): a measured anchor for the extrapolation above, not timed on this box."""
    try:
        import numpy as np
        z = np.load(os.path.join(ROOT, "tests", "golden", "c4_burgers_full.npz"))
        t = json.loads(str(z["ref_times_json"]))
        return {"reference_full_run": {
            "stages_s": t, "wall_s": t.get("t_wall"),
            "where": "build container, 1 core (tests/golden/make_golden_full.py c4), n=1e6, "
                     "10 GN steps + Laplace + Takahashi; not this box"}}
    except Exception:  # noqa: BLE001 - fixture absent: no anchor
        return {}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} threads visible)"
    except OSError:
        pass
    return f"{os.cpu_count()} threads visible"


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def fp64_peak_tflops():
    """cuBLAS DGEMM 8192³ (torch.matmul float64), best of 5 — the measured FP64
    tensor-core denominator (MEASURED_PEAKS.json carries no FP64 entry)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    torch.cuda.empty_cache()
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


# ---------------------------------------------------------------------------
# sub-records of the default run: config 2 end to end against the reference
# measured on this host, and the config-5 shape one B200 holds
# ---------------------------------------------------------------------------
def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def run_c2(steps, warmup, with_reference=True):
    """Config 2 (2D Matérn regression, 256² nodes, 2000 points, mean + Takahashi
    variances + 16 samples) through the product's public API, e2e from host data
    (points in at setup; y, Λ in and mean, variances, samples out per step), and
    the unmodified reference (oracle/_ref) on the same seeded inputs, measured
    single-threaded on this host (no extrapolation)."""
    import torch
    from paper_2503_08343_b200.regression import RegressionPosterior, seeded_inputs
    mesh, spec, pts, y, lam, ns, seed = seeded_inputs(2)
    t0 = time.perf_counter()
    post = RegressionPosterior(mesh, spec, pts)
    setup_s = time.perf_counter() - t0
    for _ in range(max(warmup, 1)):
        post.run(y, lam, True, ns, seed)
    torch.cuda.synchronize()
    dev_ms, e2e = [], []
    for _ in range(steps):
        w0 = time.perf_counter()
        mean, var, smp = post.run(y, lam, True, ns, seed)
        e2e.append(time.perf_counter() - w0)
        dev_ms.append(post.info().run_ms)
    info = post.info()
    out = {"workload": "config 2: 2D Matern regression posterior, P1 256x256 nodes (n=65,536), "
                       "2000 seeded points, mean + Takahashi variances + 16 samples",
           "value": float(np.median(dev_ms)) * 1e-3, "unit": "s",
           "e2e": {"value": float(np.median(e2e)), "unit": "s",
                   "h2d_bytes_per_step": 16 * post.m,
                   "d2h_bytes_per_step": 8 * post.n * (2 + ns)},
           "host_setup_s": setup_s, "nnz_l": info.nnz_l, "gpu_launches": int(info.kernel_launches),
           "timing": "value: CUDA events around the device pipeline (y upload .. samples), median "
                     "of steps; e2e: wall clock of RegressionPosterior.run incl. copies"}
    if with_reference:
        try:
            from oracle.pyoracle import Ref
            w0 = time.perf_counter()
            b = Ref().build("matern2d", [255, 10.0, 2, 1.0, 2000, 1002, 400.0, 0.05, ns, 2002, 1])
            ref_s = time.perf_counter() - w0
            out["reference"] = {
                "value": ref_s, "unit": "s", "cores": 1, "kind": "reference",
                "sample": "the full config-2 chain (matern_prior, point_observation_operator, "
                          "condition_on = AMD + factor + solve, variance_takahashi, 16 "
                          "sample_direct), unmodified reference, measured (not extrapolated)",
                "stages_s": {k: b.scalar(k) for k in ("t_prior", "t_condition", "t_variance",
                                                      "t_samples")}}
            out["speedup_e2e"] = ref_s / out["e2e"]["value"]
            out["parity"] = {"mean_rel": _rel(mean, b.vec("mean_post")),
                             "var_rel": _rel(var, b.vec("var_post"))}
        except Exception as exc:  # oracle/_ref absent on this box
            out["reference"] = {"value": None, "unavailable": str(exc)}
    return out


def run_c5(n_cells, n_t, steps, warmup, peak_fp64):
    """The config-5 shape one B200 holds (Allen-Cahn, 8 GN steps + Laplace +
    variances, seed 1005): device seconds per posterior and the Cholesky's
    fraction of the FP64 peak."""
    import torch
    from paper_2503_08343_b200 import Rng
    from paper_2503_08343_b200.spacetime import (GaussNewtonConfig, SpaceTimePosterior,
                                                 SpaceTimeSpec)
    spec = SpaceTimeSpec.allen_cahn(n_cells=n_cells, n_t=n_t)
    t0 = time.perf_counter()
    post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=8))
    setup_s = time.perf_counter() - t0
    u0 = -0.1 + 0.2 * Rng(1005).uniforms(spec.n_space)
    for _ in range(max(warmup, 1)):
        post.run(u0, variances=True, copy_back=False)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        _, _, trace, _ = post.run(u0, variances=True, copy_back=False)
    e1.record()
    torch.cuda.synchronize()
    info = post.info()
    numeric_ms = _pure_numeric_ms(info)
    tf = info.flops_ref / (numeric_ms * 1e-3) / 1e12
    nn = n_cells + 1
    return {"workload": f"config-5 shape: Allen-Cahn GN-Laplace posterior, {nn}x{nn} nodes x "
                        f"{n_t} slices (n={post.n:,}), 8 GN steps + Laplace + variances, seed 1005",
            "value": e0.elapsed_time(e1) / steps * 1e-3, "unit": "s", "host_setup_s": setup_s,
            "cholesky_fp64": {"tflops": tf, "frac": tf / peak_fp64,
                              "numeric_ms_per_factorization": numeric_ms,
                              "factorizations_per_step": info.n_factorizations},
            "phases_ms": {"gauss_newton": info.gn_ms, "laplace": info.laplace_ms,
                          "variances": info.selinv_ms},
            "gn_steps": len(trace), "nnz_l": info.nnz_l,
            "factor_device_gb": info.factor_device_bytes / 1e9}


def _pure_numeric_ms(info):
    """ms per numeric factorization, from the factorizations that run alone (the
    GN / conditioning ones carry the fused forward sweep of their solve)."""
    if info.n_pure_factorizations > 0:
        return info.numeric_pure_ms / info.n_pure_factorizations
    return info.numeric_ms / max(info.n_factorizations, 1)


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--n-el", type=int, default=999)
    ap.add_argument("--n-t", type=int, default=1000)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the config-2 (with its measured reference) and config-5-shape "
                         "sub-records of the default run")
    ap.add_argument("--workload", choices=["c4", "c5"], default="c4",
                    help="c4 (default, the headline): config-4 Burgers posterior at full size; "
                         "c5: config-5 Allen-Cahn posterior at the largest shape one B200 holds "
                         "(--c5-cells x --c5-cells cells x --c5-slices), seed 1005+rank")
    ap.add_argument("--c5-cells", type=int, default=64)
    ap.add_argument("--c5-slices", type=int, default=128)
    ap.add_argument("--partition", action="store_true",
                    help="N>1: one posterior, its factorization / solves / selected inversion "
                         "partitioned along the top ND separators across the ranks (NCCL), "
                         "strong scaling; default: one independent posterior per GPU")
    ap.add_argument("--torch-exchange", action="store_true",
                    help="--partition: move the messages through the torch.distributed callback "
                         "instead of the library's own NCCL calls")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    config = {"workload": "config 4: space-time Burgers GN-Laplace posterior (mean + marginal "
                          "variances), P1 1000 nodes x 1000 implicit-Euler slices, n=1,000,000, "
                          "10 GN steps",
              "n_el": args.n_el, "n_t": args.n_t, "gn_steps": 10,
              "l2": "inputs larger than L2 (factor storage ~3 GB, Sigma panels ~1.6 GB)",
              "parallelism": f"replicas x{world} (batch sharding, one posterior per GPU)"}
    c5 = args.workload == "c5"
    if c5:
        nn = args.c5_cells + 1
        config = {"workload": f"config 5 (reduced to one B200): space-time Allen-Cahn GN-Laplace "
                              f"posterior, P1 {nn}x{nn}-node unit square x {args.c5_slices} "
                              f"implicit-Euler slices over [0, 0.5], n={nn * nn * args.c5_slices:,}, "
                              f"8 GN steps (full config 5 is 128x128x256: nnz(L) ~2.5e10, over "
                              f"one GPU's HBM)",
                  "n_cells": args.c5_cells, "n_t": args.c5_slices, "gn_steps": 8,
                  "l2": "inputs larger than L2",
                  "parallelism": f"replicas x{world} (batch of independent seeds 1005+rank, one "
                                 f"per GPU)"}
    partitioned = args.partition and world > 1
    if partitioned:
        config["parallelism"] = (f"nd-partition x{world} (one posterior; supernodal tree split "
                                 f"along its top nested-dissection separators, NCCL exchange)")

    if args.impl == "reference":
        if rank != 0:
            return
        if c5:
            print(json.dumps({"impl": "reference", "unavailable": (
                "config 5 at >= 64x64x128 overflows the reference's int32 nnz(L) "
                "(BASELINE.md §2); its CPU arm is measured on config 4")}), flush=True)
            return
        rb = reference_sample()
        line = {"impl": "reference", "metric": METRIC, "value": rb["value"], "unit": UNIT,
                "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": rb["value"] * 1e3, "higher_is_better": False, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY §8(d))",
                "config": config, "cpu_baseline": {k: rb[k] for k in
                                                   ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": rb["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0},
                "extra": {"measured_sample_s": rb["measured_sample_s"],
                          "stages_sample_s": rb["stages_sample_s"], "cpu": rb["cpu"]}}
        print(json.dumps(line), flush=True)
        return

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    from paper_2503_08343_b200.spacetime import (GaussNewtonConfig, SpaceTimePosterior,
                                                 SpaceTimeSpec)

    peak_fp64 = fp64_peak_tflops()
    peaks = load_peaks()
    if c5:
        spec = SpaceTimeSpec.allen_cahn(n_cells=args.c5_cells, n_t=args.c5_slices)
        gn_iters = 8
    else:
        spec = SpaceTimeSpec.burgers(n_el=args.n_el, n_t=args.n_t)
        gn_iters = 10
    t0 = time.perf_counter()
    if partitioned:
        from paper_2503_08343_b200.partition import NcclExchange, TorchExchange
        post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=gn_iters),
                                  partition=(world, rank, TorchExchange() if args.torch_exchange else NcclExchange()))
    else:
        post = SpaceTimePosterior(spec, GaussNewtonConfig(max_iters=gn_iters))
    host_setup_s = time.perf_counter() - t0
    if c5:  # u0_d = -0.1 + 0.2·Rng(1005+b).uniform() in DoF order
        from paper_2503_08343_b200 import Rng
        u0 = -0.1 + 0.2 * Rng(1005 + rank).uniforms(spec.n_space)
    else:
        x = spec.node_x()
        u0 = -np.sin(np.pi * x)

    for _ in range(max(args.warmup, 0)):
        post.run(u0, variances=True, copy_back=False)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-timed region: value ----
    sampler = ClockSampler(local_rank)
    barrier()
    sampler.start()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    traces = []
    e0.record()
    for _ in range(args.steps):
        _, _, trace, conv = post.run(u0, variances=True, copy_back=False)
        launches += post.info().kernel_launches
        traces.append(trace)
    e1.record()
    barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())

    # ---- e2e through the C-ABI with host buffers ----
    barrier()
    w0 = time.perf_counter()
    for _ in range(args.steps):
        mean, var, _, _ = post.run(u0, variances=True, copy_back=True)
    barrier()
    e2e_s = (time.perf_counter() - w0) / args.steps
    te = torch.tensor([e2e_s], device="cuda", dtype=torch.float64)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    n = post.n

    # ---- one profiled (untimed) run for the per-kernel roofline ----
    info = post.info()
    post.set_profile(True)
    post.run(u0, variances=True, copy_back=False)
    stats = post.kernel_stats()
    post.set_profile(False)
    pinfo = post.info()
    step_kernel_ms = sum(v["ms"] for v in stats.values())
    dom_name, dom = max(stats.items(), key=lambda kv: kv[1]["ms"])
    # DRAM traffic per launch of the dominant kernel class, from the committed ncu
    # capture (profiles/r02_ncu_traffic.json, tools/ncu_traffic.py), when present
    traffic = None
    try:
        tpath = os.path.join(ROOT, "profiles", "r02_ncu_traffic.json")
        if not os.path.exists(tpath):
            tpath = os.path.join(ROOT, "profiles", "r01_ncu_traffic.json")
        with open(tpath) as fh:
            tr = json.load(fh).get(dom_name, {})
            if tr.get("workload", "c4") == args.workload:
                traffic = tr.get("dram_bytes_per_launch")
    except (OSError, ValueError):
        traffic = None
    if dom["flops"] > 0:
        achieved = dom["flops"] / (dom["ms"] * 1e-3) / 1e12
        roof = {"kernel": dom_name, "bound": "tensor", "achieved": achieved, "peak": peak_fp64,
                "unit": "TFLOP/s", "frac": achieved / peak_fp64, "traffic": traffic,
                "peak_source": "measured in-run: cuBLAS DGEMM 8192^3 (FP64 tensor cores)",
                "share_of_step": dom["ms"] / step_kernel_ms,
                "avg_launch_ms": dom["ms"] / max(dom["launches"], 1),
                "launches_per_step": dom["launches"]}
    else:
        hbm = peaks.get("hbm_gbs", 6650.0)
        achieved = dom["bytes"] / (dom["ms"] * 1e-3) / 1e9
        roof = {"kernel": dom_name, "bound": "hbm", "achieved": achieved, "peak": hbm,
                "unit": "GB/s", "frac": achieved / hbm, "traffic": traffic,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                "share_of_step": dom["ms"] / step_kernel_ms}
    numeric_ms = _pure_numeric_ms(info)
    chol_tflops = info.flops_ref / (numeric_ms * 1e-3) / 1e12
    kernels = {k: {"ms": v["ms"], "launches": v["launches"],
                   "achieved": (v["flops"] / (v["ms"] * 1e-3) / 1e12 if v["flops"] > 0
                                else v["bytes"] / (v["ms"] * 1e-3) / 1e9),
                   "unit": "TFLOP/s" if v["flops"] > 0 else "GB/s"}
               for k, v in sorted(stats.items(), key=lambda kv: -kv[1]["ms"])}
    # north_star's per-subsystem rooflines: FP64 tensor peak for the
    # factorization, HBM for assembly, the conditioning update and the solves; the
    # selected inversion is reported against both (its GEMM part dominates)
    hbm_peak = peaks.get("hbm_gbs", 6650.0)

    def agg(prefix):
        sel = [v for k, v in stats.items() if k.startswith(prefix)]
        ms_ = sum(v["ms"] for v in sel)
        fl, by = sum(v["flops"] for v in sel), sum(v["bytes"] for v in sel)
        out = {"ms_per_step": ms_, "launches": sum(v["launches"] for v in sel)}
        if ms_ > 0:
            out["gbs"] = by / (ms_ * 1e-3) / 1e9
            out["hbm_frac"] = out["gbs"] / hbm_peak
            if fl > 0:
                out["tflops"] = fl / (ms_ * 1e-3) / 1e12
                out["fp64_frac"] = out["tflops"] / peak_fp64
        return out

    fac_row = agg("factor.")
    for k in ("gbs", "hbm_frac"):  # extend-add bytes over all factor time: not a roofline
        fac_row.pop(k, None)
    fac_row["profiled_tflops"] = fac_row.pop("tflops", None)
    fac_row["profiled_fp64_frac"] = fac_row.pop("fp64_frac", None)
    fac_row["graph_tflops"] = chol_tflops
    fac_row["graph_fp64_frac"] = chol_tflops / peak_fp64
    rows = {"1_assembly": agg("assemble."), "2_conditioning_update": agg("update."),
            "3_factorization": fac_row,
            "4_solves": agg("solve."), "5_selected_inversion": agg("selinv."),
            "residual_jacobian": agg("residual."),
            "note": "profiled (serialized) kernel time per step; bytes = algorithmic (DESIGN.md §3); "
                    "factorization: profiled_* = executed (padded) flops over the serialized "
                    "profiled kernels, graph_* = Sigma c_j^2 over the CUDA-graph numeric time "
                    "(the headline)"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    line = {
        "metric": METRIC, "value": ms / 1e3, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False,
        "scaling": "strong" if partitioned else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, SURVEY §8(d))",
        "config": config,
        "e2e": {"value": e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * len(u0),
                "d2h_bytes_per_step": 16 * n},
        "gpu_launches": int(launches),
        "clocks": clocks,
        "roofline": roof,
        "cholesky_fp64": {"tflops": chol_tflops, "frac": chol_tflops / peak_fp64,
                          "flops_per_factorization": info.flops_ref,
                          "flops_executed_padded": info.flops_sn,
                          "numeric_ms_per_factorization": numeric_ms,
                          "numeric_ms_incl_fused_forward_sweep":
                              info.numeric_ms / max(info.n_factorizations, 1),
                          "factorizations_per_step": info.n_factorizations,
                          "note": "Sigma c_j^2 over the ND symbolic / numeric time (BASELINE.md §3); "
                                  "timed on the factorizations with nothing fused (the Laplace "
                                  "precision): the others carry the forward sweep of their solve"},
        "phases_ms": {"assemble": info.assemble_ms, "condition": info.condition_ms,
                      "gauss_newton": info.gn_ms, "laplace": info.laplace_ms,
                      "variances": info.selinv_ms},
        "host_setup_s": host_setup_s,
        "kernels": kernels,
        "rooflines_by_row": rows,
        "gn_trace": [[t.objective, t.decrement, t.step_size, t.backtracks] for t in traces[-1]],
        "nnz_l": info.nnz_l, "nnz_l_padded": info.nnz_l_padded,
        "factor_device_gb": info.factor_device_bytes / 1e9,
        "peaks": {"fp64_tflops_dgemm": peak_fp64, "hbm_gbs": peaks.get("hbm_gbs")},
    }
    if c5:
        line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                "sample": "not run for config 5: the reference's int32 nnz(L) "
                                          "overflows at this shape (BASELINE.md §2)"}
    elif not args.no_cpu_baseline and world == 1:
        try:
            rb = reference_sample()
            line["cpu_baseline"] = {k: rb[k] for k in ("value", "unit", "cores", "kind", "sample")}
        except Exception as exc:  # oracle/_ref missing on this box
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"unavailable: {exc}"}
    if world == 1 and not c5 and not args.no_extras:
        del post
        torch.cuda.empty_cache()
        line["c2"] = run_c2(args.steps, args.warmup, with_reference=not args.no_cpu_baseline)
        line["c5_shape"] = run_c5(args.c5_cells, args.c5_slices, 1, 1, peak_fp64)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
