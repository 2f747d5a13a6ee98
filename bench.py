#!/usr/bin/env python3
"""bench.py — Newton-updated training views/s (one Trainer::step per view) on B200.

Workload (BASELINE.json configs[1], "c2"): 300K Gaussians, SH degree 3, 100
training views at 800x800, K=3 neighbour views at 1/4 resolution, default
TrainConfig (trainer.hpp:58-77). One "step" = Trainer::newton_step on one
training view: 4 renders of the 1+K views, 4 backward passes, 5 solve+commit
passes (trainer.hpp:299-417). Synthetic data (paper_2501_13975_b200/workload.py);
ground-truth targets are rendered on the GPU from the truth scene.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1|c2|c3]

Prints ONE JSON line (rank 0). Multi-GPU (torchrun): every rank runs the same
sequence of Newton steps; each view of a step is split into tile-row bands
across ranks, and the per-Gaussian FP64 accumulators are summed by an NCCL
all-reduce after every backward pass before the replicated solve (
strong scaling of one step, exact reference semantics).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

from paper_2501_13975_b200 import capi  # noqa: E402
from paper_2501_13975_b200.workload import CONFIGS, Config, cameras_for, make_scenes  # noqa: E402

METRIC = "Newton-updated training views/sec"
PEAKS_PATH = os.path.join(REPO, "MEASURED_PEAKS.json")
# Algorithmic FP32 work per contributing (pixel, splat) record of the position
# backward (DESIGN.md §4 "K8 position", FMA = 2): phase 1 (G, alpha, T, behind)
# ~40 flop, phase 2 in the 2-D position subspace ~250 flop (derivatives of q
# along u_x, u_y, the three-channel Gauss-Newton + curvature assembly).
POSITION_FLOPS_PER_PAIR = 290


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self, t0=None, t1=None):
        """Samples taken inside [t0, t1] (the timed region); the sampler is started
        before the warm-up so that nvidia-smi is already polling when timing starts."""
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ts, line in self.lines:
            if t0 is not None and not (t0 <= ts <= t1 + 0.1):
                continue
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    try:
        with open(PEAKS_PATH) as f:
            return json.load(f)
    except OSError:
        return {}


def l2_flush(buf):
    if buf is not None:
        buf.zero_()
        import torch
        torch.cuda.synchronize()


# ---------------------------------------------------------------------------
# CPU reference (oracle/_ref/libngs_ref.so): bounded sample of the workload
# ---------------------------------------------------------------------------

def reference_sample_config(cfg: Config, shrink: int = 16) -> tuple[Config, float]:
    """Same footprint size (px) and splat depth as `cfg` at 1/shrink of the
    Gaussians; returns (sample config, extrapolation factor = pixel ratio)."""
    n = cfg.kernels // shrink
    f = (100.0 / n) ** (1.0 / 3.0)
    lin = f / cfg.scale_factor  # kernels grow by this factor in world units
    w = max(48, int(round(cfg.width / lin)))
    h = max(48, int(round(cfg.height / lin)))
    sample = Config(cfg.name + f"/ref-sample-1:{shrink}", n, cfg.views, w, h, cfg.sh_degree, f)
    return sample, (cfg.width * cfg.height) / float(w * h)


def run_reference_sample(cfg: Config, steps: int, warmup: int, shrink: int, target_ctx=None):
    """Times the reference Trainer::step (all host threads) on a bounded sample.
    `target_ctx` (optional) renders the sample's ground-truth targets (data
    generation only, outside the timed region)."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from refimpl import ref
    sample, factor = reference_sample_config(cfg, shrink)
    truth, init = make_scenes(sample)
    cams = cameras_for(sample)
    lib = ref()
    ctx = lib.context()
    rctx = target_ctx if target_ctx is not None else ctx
    rctx.set_scene(truth)
    ropts = rctx.L.default_raster()
    ropts.threads = os.cpu_count() or 1
    targets = [rctx.render(c, ropts) for c in cams]
    ctx.set_scene(init)
    tc = lib.default_train()
    threads = os.cpu_count() or 1
    tc.threads = threads
    ctx.trainer_configure(tc, cams, targets, list(range(sample.views)))
    order = np.random.default_rng(7).permutation(sample.views)
    for i in range(warmup):
        ctx.trainer_step(int(order[i % len(order)]))
    times = []
    for i in range(steps):
        rep = ctx.trainer_step(int(order[(warmup + i) % len(order)]))
        times.append(rep.dt_ms)
    ms = float(np.mean(times))
    views_per_s = 1000.0 / (ms * factor)
    return dict(value=views_per_s, unit="views/s", cores=threads, ms_per_sample_step=ms,
                sample=(f"Trainer::step on {sample.desc} (1/{shrink} of the Gaussians, same footprint in px and "
                        f"splat depth), {steps} steps; views/s extrapolated x{factor:.2f} by pixel count"),
                kind="reference")


def reference_arm(args, cfg: Config):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    r = run_reference_sample(cfg, max(args.steps, 1), args.warmup, args.ref_shrink)
    line = {"metric": METRIC, "value": r["value"], "unit": "views/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1000.0 / r["value"], "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": cfg.name, "desc": cfg.desc, "knn": 3, "secondary_downsample": 4},
            "cpu_baseline": {"value": r["value"], "unit": "views/s", "cores": r["cores"], "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# CUDA implementation
# ---------------------------------------------------------------------------

def ours_arm(args, cfg: Config):
    import torch
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = capi.product()
    ctx = lib.context(local)
    nccl_id = None
    if world > 1:
        obj = [capi.dist_unique_id(lib) if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    truth, init = make_scenes(cfg)
    cams = cameras_for(cfg)
    ctx.set_scene(truth)
    targets = [ctx.render(c) for c in cams]
    tc = lib.default_train()
    if os.environ.get("NGS_BENCH_KNN"):  # diagnostics only (the headline uses the reference default, 3)
        tc.knn = int(os.environ["NGS_BENCH_KNN"])

    def configure(c, host_targets):
        if args.deterministic:
            c.set_deterministic(True)
        c.set_scene(init)
        tc.host_targets = 1 if host_targets else 0
        c.trainer_configure(tc, cams, targets, list(range(cfg.views)))

    configure(ctx, False)
    if world > 1:
        ctx.dist_init(nccl_id, rank, world)
    order = [int(v) for v in np.random.default_rng(7).permutation(cfg.views)]
    shard = order  # every rank steps the same views; the work of each step is sharded
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2

    def view(i):
        return shard[i % len(shard)]

    dts = []
    prof_range = os.environ.get("NGS_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    with ClockSampler(local) as clocks:
        for i in range(args.warmup):
            ctx.trainer_step(view(i))
        ctx.profile_reset()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        t_timed0 = time.time()
        for i in range(args.steps):
            l2_flush(flush)
            if prof_range:
                torch.cuda.profiler.start()
            rep = ctx.trainer_step(view(args.warmup + i))
            if prof_range:
                torch.cuda.profiler.stop()
            dts.append(rep.dt_ms)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t_timed1 = time.time()
    counters = ctx.profile_read()
    total_ms = float(sum(dts))

    # Profiled re-run of the same K steps (views serialised, every launch
    # bracketed by CUDA events on its stream) for the per-kernel roofline.
    pctx = lib.context(local)
    configure(pctx, False)
    if world > 1:
        obj = [capi.dist_unique_id(lib) if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        pctx.dist_init(obj[0], rank, world)
    for i in range(args.warmup):
        pctx.trainer_step(view(i))
    pctx.profile_reset()
    pctx.profile_enable(True)
    prof_dts = []
    for i in range(args.steps):
        l2_flush(flush)
        prof_dts.append(pctx.trainer_step(view(args.warmup + i)).dt_ms)
    prof = pctx.profile_read()
    pctx.close()

    # End to end through the C-ABI with host-resident targets (pinned H2D per step).
    ectx = lib.context(local)
    ectx.set_scene(init)
    configure(ectx, True)
    if world > 1:
        obj = [capi.dist_unique_id(lib) if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        ectx.dist_init(obj[0], rank, world)
    for i in range(args.warmup):
        ectx.trainer_step(view(i))
    e2e_ms = []
    for i in range(args.steps):
        l2_flush(flush)
        t0 = time.perf_counter()
        ectx.trainer_step(view(args.warmup + i))
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    ectx.close()

    # First-order baselines on the same workload (first_order_step, trainer.hpp:419-509):
    # device time per step, for the Newton-vs-GD cost ratio (not the headline).
    fo = {}
    if world == 1:
        for name, opt in (("gd", capi.OPT_GD),):  # Adam's cost follows its (diverging) splat sizes here
            fctx = lib.context(local)
            fctx.set_scene(init)
            tc.optimizer = opt
            fctx.trainer_configure(tc, cams, targets, list(range(cfg.views)))
            for i in range(args.warmup):
                fctx.trainer_step(view(i))
            fdt = []
            for i in range(args.steps):
                l2_flush(flush)
                fdt.append(fctx.trainer_step(view(args.warmup + i)).dt_ms)
            fctx.close()
            fo[f"{name}_ms_per_step"] = float(sum(fdt)) / args.steps
        tc.optimizer = capi.OPT_NEWTON
    ds = 4
    h2d = 3 * 8 * (cfg.width * cfg.height + 3 * (cfg.width // ds) * (cfg.height // ds))
    d2h = 8 * 5 + 8  # delta norms + error word

    if world > 1:
        t = torch.tensor([total_ms, sum(e2e_ms)], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, e2e_total = float(t[0]), float(t[1])
    else:
        e2e_total = float(sum(e2e_ms))

    if rank != 0:
        return
    views_total = args.steps  # each step is one view, done jointly by all ranks
    value = views_total / (total_ms / 1e3)
    e2e_value = views_total / (e2e_total / 1e3)

    # Roofline of the dominant kernel (position backward, FP32 CUDA-core bound).
    fp32_peak = ctx.microbench_fp32()
    fp64_peak = ctx.microbench_fp64()
    bwd_ms = prof["ms"]["bwd_position"]
    bwd_launches = max(prof["launches"]["bwd_position"], 1)
    pairs = prof["contrib_pairs"][0]
    achieved = POSITION_FLOPS_PER_PAIR * pairs / (bwd_ms * 1e-3) / 1e12 if bwd_ms > 0 else 0.0
    step_stage_ms = {k: round(v / args.steps, 4) for k, v in prof["ms"].items()}

    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # (ncu numbers are never bench values; this only sizes traffic vs algorithmic bytes).
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(REPO, "profiles", "r1_roofline_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj["dram_bytes_read"] + tj["dram_bytes_write"]
        traffic_src = f"{tj['kernel']}: {tj['source']}"
    except (OSError, KeyError, ValueError):
        pass

    # Newton-solve microbenchmark (BASELINE config 4): 10M Gaussians, random SPD blocks
    # for every attribute group, colour rank-4 (V = 4 views), HBM-roofline bound.
    solve_mb = None
    if world == 1 and not args.no_solve_microbench:
        mb_n = 10_000_000
        ms5 = ctx.microbench_solve(mb_n, sh_degree=3, views=4, reps=5)
        upd_s = mb_n / (sum(ms5) * 1e-3)
        bytes_per_update = 684  # SH3, V = 4 compact accumulators + params in/out
        hbm = float(measured_peaks().get("hbm_gbs", 6552.0))
        solve_mb = {"gaussians": mb_n, "ms_per_attr": dict(zip(("position", "rotation", "scaling", "opacity", "color"),
                                                                [round(x, 4) for x in ms5])),
                    "gaussian_updates_per_s": upd_s, "algorithmic_bytes_per_update": bytes_per_update,
                    "achieved_GBps": upd_s * bytes_per_update / 1e9,
                    "hbm_frac": upd_s * bytes_per_update / 1e9 / hbm}

    cpu = None
    if not args.no_cpu_baseline:
        cpu = run_reference_sample(cfg, 2, 0, args.ref_shrink, target_ctx=lib.context(local))
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
    line = {
        "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": cfg.name, "desc": cfg.desc, "knn": int(tc.knn), "secondary_downsample": 4,
                   "deterministic": bool(args.deterministic),
                   "parallelism": f"tile-row bands x{world} + NCCL all-reduce of accumulators", "l2": "flushed (256 MB write) between steps",
                   "targets": "GPU-rendered from the truth scene"},
        "gaussian_solves_per_s": value * cfg.kernels,
        "e2e": {"value": e2e_value, "unit": "views/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "gpu_launches": int(counters["total_launches"]),
        "roofline": {"bound": "fp32", "kernel": "backward_k<position>", "achieved": achieved,
                     "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak if fp32_peak else None,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": "measured FFMA microbenchmark (ngs_microbench_fp32)",
                     "algorithmic": f"{POSITION_FLOPS_PER_PAIR} flop x {pairs} contributing records / "
                                    f"{bwd_launches} launches"},
        "profiled_pass": {"note": "same K steps re-run with views serialised and per-launch CUDA events; "
                                  "stage times below come from it", "ms_per_step": float(sum(prof_dts)) / args.steps},
        "stage_ms_per_step": step_stage_ms,
        "group_ms_per_step_concurrent": {k: round(v / args.steps, 4) for k, v in counters["group_ms"].items()},
        "measured_fp64_tflops": fp64_peak,
        "solve_microbench": solve_mb,
        "first_order_baselines": dict(fo, newton_ms_per_step=total_ms / args.steps,
                                      newton_over_gd=(total_ms / args.steps) / fo["gd_ms_per_step"],
                                      note="GD steps (first_order_step: primary view only, one gradient traversal) "
                                           "on the same workload: the paper's Newton-vs-GD per-step cost") if fo else None,
        "contrib_pairs_per_step": [p / args.steps for p in prof["contrib_pairs"]],
        "clocks": clocks.summary(t_timed0, t_timed1),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    p.add_argument("--ref-shrink", type=int, default=64)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-solve-microbench", action="store_true")
    p.add_argument("--deterministic", action="store_true", help="exact fixed-point accumulation (bitwise reproducible)")
    args = p.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        reference_arm(args, cfg)
    else:
        ours_arm(args, cfg)


if __name__ == "__main__":
    main()
