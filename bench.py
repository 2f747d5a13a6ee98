#!/usr/bin/env python3
"""bench.py — Newton-updated training views/s (one Trainer::step per view) on B200.

Workload (BASELINE.json configs[1], "c2"): 300K Gaussians, SH degree 3, 100
training views at 800x800, K=3 neighbour views at 1/4 resolution, default
TrainConfig (trainer.hpp:58-77). One "step" = Trainer::newton_step on one
training view: 4 renders of the 1+K views, 4 backward passes, 5 solve+commit
passes (trainer.hpp:299-417). Synthetic data (paper_2501_13975_b200/workload.py);
ground-truth targets are rendered on the GPU from the truth scene.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c1|c2|c3]

Prints ONE JSON line (rank 0). Multi-GPU (torchrun, or `--gpus N` which spawns N
ranks itself): every rank runs the same sequence of Newton steps; the 1+K views
of each step are partitioned over the ranks (ngs_dist_plan: whole secondaries,
primary tile-row bands), and the per-Gaussian accumulators are summed by an
NCCL all-reduce (FP32 payload) after every backward pass before the replicated
solve (strong scaling of one step, exact reference semantics).

Side fields (world 1): `c3` (3M Gaussians, 1080p — the north-star workload) and
`c1` (10K, 256^2, with the reference CPU step measured on the SAME config,
unsliced) with device and e2e views/s; `solve_microbench` (c4, commits
included); `first_order_baselines` (GD). `--impl reference` times the
reference's own CPU Trainer::step on a 1/64 slice of the workload with the same
per-pixel and per-Gaussian work.
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

def reference_sample_config(cfg: Config, shrink: int = 8) -> tuple[Config, float]:
    """A bounded slice of `cfg` with the same per-pixel and per-Gaussian work: image sides
    / shrink, Gaussians / shrink^2, kernel sizes (and init jitter) x shrink in world units.
    Each splat then keeps its footprint in pixels and every pixel keeps its splat depth, so
    records per pixel, records per Gaussian and Gaussians per pixel all match `cfg`; the
    sample is 1/shrink^2 of one view's work (pixels, Gaussians, records alike).
    Returns (sample config, views of `cfg` per sample step = 1/shrink^2)."""
    n = max(1, cfg.kernels // (shrink * shrink))
    w = max(48, cfg.width // shrink)
    h = max(48, cfg.height // shrink)
    sample = Config(cfg.name + f"/ref-slice-1:{shrink * shrink}", n, cfg.views, w, h, cfg.sh_degree,
                    cfg.scale_factor * shrink)
    frac = (w * h) / float(cfg.width * cfg.height)
    return sample, frac


def run_reference_sample(cfg: Config, steps: int, warmup: int, shrink: int, target_ctx=None):
    """Times the reference Trainer::step (trainer.hpp:185-207, all host threads) on a bounded
    slice of `cfg` (reference_sample_config). `target_ctx` (optional) renders the slice's
    ground-truth targets (data generation only, outside the timed region)."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from refimpl import ref
    sample, frac = reference_sample_config(cfg, shrink)
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
    views_per_s = frac / (ms * 1e-3)
    return dict(value=views_per_s, unit="views/s", cores=threads, ms_per_sample_step=ms, views_per_step=frac,
                sample=(f"Trainer::step on a 1/{round(1 / frac)} slice of {cfg.name} ({sample.desc}, kernels x{shrink} "
                        f"larger in world units: same splat footprint in px, same splats per pixel, same records per "
                        f"Gaussian), {steps} steps of {ms:.0f} ms; each step is {frac:.6f} of a {cfg.name} view"),
                kind="reference")


def run_reference_full(cfg: Config, steps: int, target_ctx=None):
    """The reference Trainer::step on the FULL config (no slicing): used for c1, whose
    step the CPU finishes in seconds (BASELINE.json configs[0])."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from refimpl import ref
    truth, init = make_scenes(cfg)
    cams = cameras_for(cfg)
    lib = ref()
    ctx = lib.context()
    rctx = target_ctx if target_ctx is not None else ctx
    rctx.set_scene(truth)
    ropts = rctx.L.default_raster()
    ropts.threads = os.cpu_count() or 1
    targets = [rctx.render(c, ropts) for c in cams]
    ctx.set_scene(init)
    tc = lib.default_train()
    tc.threads = os.cpu_count() or 1
    ctx.trainer_configure(tc, cams, targets, list(range(cfg.views)))
    order = np.random.default_rng(7).permutation(cfg.views)
    ms = [ctx.trainer_step(int(order[i % len(order)])).dt_ms for i in range(steps)]
    return dict(value=1000.0 / float(np.mean(ms)), unit="views/s", cores=tc.threads, kind="reference",
                ms_per_step=float(np.mean(ms)), sample=f"{steps} full Trainer::step of {cfg.desc} (no slicing)")


def reference_arm(args, cfg: Config):
    """--impl reference: the reference's own CPU implementation (oracle/_ref: the unmodified
    reference headers compiled here) on every host thread. One step = Trainer::step on a
    bounded slice of the workload (reference_sample_config: 1/64 of a c2 view with the same
    per-pixel and per-Gaussian work); `value` is c2 views/s = slice fraction / step time."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    r = run_reference_sample(cfg, max(args.steps, 1), args.warmup, args.ref_shrink)
    line = {"metric": METRIC, "value": r["value"], "unit": "views/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": r["ms_per_sample_step"], "views_per_step": r["views_per_step"],
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": cfg.name, "desc": cfg.desc, "knn": 3, "secondary_downsample": 4,
                       "step": "Trainer::step on a 1/64 slice of one view (same per-pixel and per-Gaussian work)"},
            "cpu_baseline": {"value": r["value"], "unit": "views/s", "cores": r["cores"], "kind": "reference",
                             "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# CUDA implementation
# ---------------------------------------------------------------------------

def _setup_nccl(lib, ctx, rank, world):
    import torch
    obj = [capi.dist_unique_id(lib) if rank == 0 else None]
    torch.distributed.broadcast_object_list(obj, src=0)
    ctx.dist_init(obj[0], rank, world)


def _prepare(lib, ctx, cfg: Config):
    """Synthetic scene of `cfg` (workload.py, SynthParams semantics) and its ground-truth
    targets rendered on the GPU from the truth scene (data generation, untimed)."""
    truth, init = make_scenes(cfg)
    cams = cameras_for(cfg)
    ctx.set_scene(truth)
    targets = [ctx.render(c) for c in cams]
    return init, cams, targets


def time_steps(lib, local, rank, world, cfg, init, cams, targets, tc, steps, warmup, flush, deterministic=False,
               host_targets=False, profile=False, e2e=False, clocks=None):
    """Runs `warmup` + `steps` Trainer::step calls on a fresh context. Device time per step =
    CUDA events on the context stream around the whole step (ngs_iteration_report.dt_ms);
    e2e = host wall clock around the C-ABI call (host-resident targets: the pinned H2D copy of
    the step's 1+K target images and the report D2H are inside). L2 flushed between steps."""
    import torch
    ctx = lib.context(local)
    if deterministic:
        ctx.set_deterministic(True)
    ctx.set_scene(init)
    tc.host_targets = 1 if host_targets else 0
    ctx.trainer_configure(tc, cams, targets, list(range(cfg.views)))
    if world > 1:
        _setup_nccl(lib, ctx, rank, world)
    order = [int(v) for v in np.random.default_rng(7).permutation(cfg.views)]
    for i in range(warmup):
        ctx.trainer_step(order[i % len(order)])
    ctx.profile_reset()
    if profile:
        ctx.profile_enable(True)
    dts, walls = [], []
    prof_range = os.environ.get("NGS_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    t0 = time.time()
    for i in range(steps):
        l2_flush(flush)
        if prof_range:
            torch.cuda.profiler.start()
        w0 = time.perf_counter()
        rep = ctx.trainer_step(order[(warmup + i) % len(order)])
        walls.append((time.perf_counter() - w0) * 1e3)
        if prof_range:
            torch.cuda.profiler.stop()
        dts.append(rep.dt_ms)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    t1 = time.time()
    stats = ctx.profile_read()
    ctx.close()
    return dict(device_ms=float(sum(dts)), wall_ms=float(sum(walls)), stats=stats, t0=t0, t1=t1,
                knn=int(tc.knn))


def max_over_ranks(world, *vals):
    if world == 1:
        return vals
    import torch
    t = torch.tensor(list(vals), dtype=torch.float64, device="cuda")
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return tuple(float(x) for x in t)


def h2d_bytes(cfg: Config, knn=3, ds=4):
    return 3 * 8 * (cfg.width * cfg.height + knn * (cfg.width // ds) * (cfg.height // ds))


def side_config(lib, local, cfg: Config, steps, warmup, flush, clocks=None):
    """Device and e2e views/s of another BASELINE config on this GPU (world 1)."""
    ctx = lib.context(local)
    init, cams, targets = _prepare(lib, ctx, cfg)
    ctx.close()
    tc = lib.default_train()
    d = time_steps(lib, local, 0, 1, cfg, init, cams, targets, tc, steps, warmup, flush)
    e = time_steps(lib, local, 0, 1, cfg, init, cams, targets, tc, steps, warmup, flush, host_targets=True)
    del targets
    out = {"workload": cfg.name, "desc": cfg.desc, "steps": steps, "warmup": warmup,
           "value": steps / (d["device_ms"] / 1e3), "unit": "views/s", "ms_per_step": d["device_ms"] / steps,
           "e2e": {"value": steps / (e["wall_ms"] / 1e3), "unit": "views/s", "h2d_bytes_per_step": h2d_bytes(cfg),
                   "d2h_bytes_per_step": 48},
           "gaussian_solves_per_s": steps / (d["device_ms"] / 1e3) * cfg.kernels}
    if clocks is not None:
        out["clocks"] = clocks.summary(d["t0"], d["t1"])
    return out


def ours_arm(args, cfg: Config):
    import torch
    rank, world, local = dist_env()
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = capi.product()
    ctx = lib.context(local)
    init, cams, targets = _prepare(lib, ctx, cfg)
    tc = lib.default_train()
    if os.environ.get("NGS_BENCH_KNN"):  # diagnostics only (the headline uses the reference default, 3)
        tc.knn = int(os.environ["NGS_BENCH_KNN"])
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2

    with ClockSampler(local) as clocks:
        main = time_steps(lib, local, rank, world, cfg, init, cams, targets, tc, args.steps, args.warmup, flush,
                          deterministic=args.deterministic)
        clk = clocks.summary(main["t0"], main["t1"])
        # Profiled re-run of the same K steps (views serialised, every launch bracketed by
        # CUDA events on its stream) for the per-kernel roofline.
        prof = time_steps(lib, local, rank, world, cfg, init, cams, targets, tc, args.steps, args.warmup, flush,
                          deterministic=args.deterministic, profile=True)
        # End to end through the C-ABI with host-resident targets (pinned H2D per step).
        e2e = time_steps(lib, local, rank, world, cfg, init, cams, targets, tc, args.steps, args.warmup, flush,
                         deterministic=args.deterministic, host_targets=True)
        total_ms, e2e_total = max_over_ranks(world, main["device_ms"], e2e["wall_ms"])
        extras = {}
        if world == 1 and not args.no_extras:
            # First-order baseline on the same workload (first_order_step, trainer.hpp:419-509).
            tgd = lib.default_train()
            tgd.optimizer = capi.OPT_GD
            gd = time_steps(lib, local, 0, 1, cfg, init, cams, targets, tgd, args.steps, args.warmup, flush)
            extras["first_order_baselines"] = {
                "gd_ms_per_step": gd["device_ms"] / args.steps, "newton_ms_per_step": total_ms / args.steps,
                "newton_over_gd": total_ms / gd["device_ms"],
                "note": "GD steps (first_order_step: primary view only, one gradient traversal) on the same "
                        "workload: the paper's Newton-vs-GD per-step cost"}
            del targets
            # The other BASELINE configs on this GPU: c3 (1080p north-star workload) and c1.
            for name in ("c3", "c1"):
                if name != cfg.name:
                    extras[name] = side_config(lib, local, CONFIGS[name], min(args.steps, 10), args.warmup, flush,
                                               clocks)
    if rank != 0:
        return
    value = args.steps / (total_ms / 1e3)  # each step is one view, done jointly by all ranks
    e2e_value = args.steps / (e2e_total / 1e3)
    counters = main["stats"]
    pst = prof["stats"]

    # Roofline of the dominant kernel: the primary view's position backward launch
    # (backward_k<PositionUV, 16>), FP32 CUDA-core bound. Algorithmic work = 290 flop per
    # contributing record x the primary's records; time = that launch alone (CUDA events on
    # its stream in the profiled re-run).
    fp32_peak = ctx.microbench_fp32()
    fp64_peak = ctx.microbench_fp64()
    bwd_ms = pst["primary_bwd_ms"][0]
    bwd_launches = args.steps
    pairs = pst["primary_contrib_pairs"][0]
    achieved = POSITION_FLOPS_PER_PAIR * pairs / (bwd_ms * 1e-3) / 1e12 if bwd_ms > 0 else 0.0
    all_views = {"ms_per_step": pst["ms"]["bwd_position"] / args.steps,
                 "records_per_step": pst["contrib_pairs"][0] / args.steps,
                 "tflops": POSITION_FLOPS_PER_PAIR * pst["contrib_pairs"][0] / (pst["ms"]["bwd_position"] * 1e-3) / 1e12
                 if pst["ms"]["bwd_position"] > 0 else 0.0}
    # DRAM traffic of the dominant kernel from the committed ncu --set full capture
    # (ncu numbers are never bench values; this only sizes traffic vs algorithmic bytes).
    traffic, traffic_src = None, None
    try:
        with open(os.path.join(REPO, "profiles", "roofline_traffic.json")) as f:
            tj = json.load(f)
        traffic = tj["dram_bytes_read"] + tj["dram_bytes_write"]
        traffic_src = f"{tj['kernel']}: {tj['source']}"
    except (OSError, KeyError, ValueError):
        pass

    # Newton-solve microbenchmark (BASELINE config 4): 10M Gaussians, random SPD blocks
    # for every attribute group, colour rank-4 (V = 4 views), HBM-roofline bound; every
    # timed launch solves and commits.
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
                    "color_fast_path_frac": getattr(ctx, "last_color_fast_frac", None),
                    "achieved_GBps": upd_s * bytes_per_update / 1e9, "hbm_frac": upd_s * bytes_per_update / 1e9 / hbm,
                    "commits": "every timed launch commits all parameters (restored between launches, untimed)"}

    cpu = cpu_c1 = None
    if not args.no_cpu_baseline:
        cpu = run_reference_sample(cfg, 2, 0, args.ref_shrink, target_ctx=lib.context(local))
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if "c1" in extras:
            c1 = run_reference_full(CONFIGS["c1"], 2, target_ctx=lib.context(local))
            cpu_c1 = {k: c1[k] for k in ("value", "unit", "cores", "kind", "sample", "ms_per_step")}
            extras["c1"]["cpu_reference"] = cpu_c1
            extras["c1"]["gpu_over_cpu_e2e"] = extras["c1"]["e2e"]["value"] / cpu_c1["value"]
    line = {
        "metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": cfg.name, "desc": cfg.desc, "knn": main["knn"], "secondary_downsample": 4,
                   "deterministic": bool(args.deterministic),
                   "parallelism": (f"views of each step partitioned over {world} ranks (whole secondaries, primary "
                                   f"tile-row bands) + NCCL all-reduce of FP32 accumulators") if world > 1 else "1 GPU",
                   "l2": "flushed (256 MB write) between steps", "targets": "GPU-rendered from the truth scene"},
        "gaussian_solves_per_s": value * cfg.kernels,
        "e2e": {"value": e2e_value, "unit": "views/s", "h2d_bytes_per_step": h2d_bytes(cfg, main["knn"]),
                "d2h_bytes_per_step": 48},
        "gpu_launches": int(counters["total_launches"]),
        "allreduce_bytes_per_step": counters["allreduce_bytes"] / args.steps,
        "roofline": {"bound": "fp32", "kernel": "backward_k<PositionUV,16> (primary view, position pass)",
                     "achieved": achieved,
                     "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak if fp32_peak else None,
                     "traffic": traffic, "traffic_source": traffic_src,
                     "peak_source": "measured FFMA microbenchmark (ngs_microbench_fp32)",
                     "algorithmic": f"{POSITION_FLOPS_PER_PAIR} flop x {pairs} contributing records / "
                                    f"{bwd_launches} launches",
                     "flop_crosscheck": _flop_crosscheck(),
                     "all_views_position_backward": all_views},
        "profiled_pass": {"note": "same K steps re-run with views serialised and per-launch CUDA events; "
                                  "stage times below come from it", "ms_per_step": prof["device_ms"] / args.steps},
        "stage_ms_per_step": {k: round(v / args.steps, 4) for k, v in pst["ms"].items()},
        "group_ms_per_step_concurrent": {k: round(v / args.steps, 4) for k, v in counters["group_ms"].items()},
        "measured_fp64_tflops": fp64_peak,
        "solve_microbench": solve_mb,
        "contrib_pairs_per_step": [p / args.steps for p in pst["contrib_pairs"]],
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    line.update(extras)
    print(json.dumps(line), flush=True)


def _flop_crosscheck():
    """Executed FP32 flops of the same launch from the committed ncu instruction counts
    (2 FFMA + 4 FFMA2 + FMUL + 2 FMUL2 + FADD + 2 FADD2 per thread instruction), divided by
    its contributing records: the check of the 290 flop/record constant."""
    try:
        with open(os.path.join(REPO, "profiles", "r2_flops_backward.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def spawn_ranks(args):
    """`python bench.py --gpus N` without torchrun: re-launch as N ranks on this node."""
    import socket
    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    raise SystemExit(subprocess.call(cmd))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    p.add_argument("--ref-shrink", type=int, default=8, help="reference slice: sides / s, Gaussians / s^2")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-solve-microbench", action="store_true")
    p.add_argument("--no-extras", action="store_true", help="skip the GD baseline and the c3 / c1 side configs")
    p.add_argument("--deterministic", action="store_true", help="exact fixed-point accumulation (bitwise reproducible)")
    args = p.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "ours" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        spawn_ranks(args)
    if args.impl == "reference":
        reference_arm(args, cfg)
    else:
        ours_arm(args, cfg)


if __name__ == "__main__":
    main()
