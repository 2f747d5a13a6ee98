"""Multi-process (gloo, world_size 2) CPU test of the multi-GPU decomposition:
the CUDA library's own partition (ngs_dist_plan, a pure host function of
libngs_b200.so: whole secondary views per rank, the primary in tile-row bands)
decides which records each rank accumulates (the float64 oracle restricted to
those pixels), the per-Gaussian accumulators are all-reduced, and the sum
equals the single-process accumulation — the exchange step of the CUDA trainer
(NCCL all-reduce after every backward pass, newton.hpp:591-597)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(REPO, "oracle"))
sys.path.insert(0, os.path.join(REPO, "tests"))


def _plan(world, rank, sizes, tiles, window=11):
    from paper_2501_13975_b200 import capi
    return capi.dist_plan(capi.NgsLibrary(capi.PRODUCT_LIB), world, rank, sizes, tiles, window)


STEPS = [  # (view sizes, tile sizes) of one trainer step: primary + K secondaries at 1/4 resolution
    ([(800, 800), (200, 200), (200, 200), (200, 200)], [16, 8, 8, 8]),
    ([(1920, 1080), (480, 270), (480, 270), (480, 270)], [16, 8, 8, 8]),
    ([(256, 256), (64, 64), (64, 64), (64, 64)], [16, 8, 8, 8]),
    ([(48, 48), (32, 32), (32, 32)], [16, 16, 16]),
    ([(33, 61)], [16]),
]


@pytest.mark.parametrize("window", [3, 11, 21])
def test_dist_plan_partitions_every_view(window):
    """ngs_dist_plan (C-ABI, libngs_b200.so; pure host code): every primary tile row is owned
    by exactly one rank, every secondary by exactly one rank (whole), the rendered band is the
    owned range plus ceil((window - 1) / tile) rows, and the pixel load is balanced to within
    the largest secondary view."""
    for sizes, tiles in STEPS:
        for world in (1, 2, 3, 4, 8):
            rows_owned = [[] for _ in sizes]
            load = []
            for rank in range(world):
                plan = _plan(world, rank, sizes, tiles, window)
                px = 0
                for i, ((w, h), t, (b0, b1, o0, o1)) in enumerate(zip(sizes, tiles, plan)):
                    ty = (h + t - 1) // t
                    if o1 > o0:
                        halo = (window - 1 + t - 1) // t
                        assert (b0, b1) == (max(0, o0 - halo), min(ty, o1 + halo))
                        if i > 0 or world == 1:
                            if i > 0:
                                assert (b0, b1, o0, o1) == (0, ty, 0, ty)   # secondaries whole
                        rows_owned[i] += list(range(o0, o1))
                        px += (o1 - o0) * t * w
                    else:
                        assert (b0, b1) == (0, 0)   # projection only
                load.append(px)
            for i, ((w, h), t) in enumerate(zip(sizes, tiles)):
                assert sorted(rows_owned[i]) == list(range((h + t - 1) // t)), (sizes, world, i)
            if len(sizes) > 1 and world > 1:
                biggest_sec = max(w * h for w, h in sizes[1:])
                assert max(load) - min(load) <= biggest_sec + 2 * tiles[0] * sizes[0][0], (sizes, world, load)


def test_dist_plan_rejects_bad_arguments():
    from paper_2501_13975_b200 import capi
    for args in ((0, 0), (2, 2), (2, -1)):
        with pytest.raises(capi.InvalidInput):
            _plan(*args, [(64, 64)], [16])
    with pytest.raises(capi.InvalidInput):
        _plan(2, 0, [(64, 64)], [12])


def _band_terms(rank, world, attr, q):
    import ngs_oracle as O
    from test_oracle import cam_from, load, scene_from
    g = load("newton.npz")
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "s_"))
    ctx.build_view(0, cam_from(g, "c_"), g["target"])
    for i in range(2):
        ctx.build_view(1 + i, cam_from(g, f"sec{i}_"), g[f"sec{i}_target"])
    # this rank's share of the step (ngs_dist_plan of the CUDA library): keep only records
    # whose pixel row lies in its owned tile rows of each view
    slots = sorted(ctx.views)
    sizes = [(ctx.views[k].cam.width, ctx.views[k].cam.height) for k in slots]
    plan = _plan(world, rank, sizes, [16] * len(slots))
    for k, (_, _, o0, o1) in zip(slots, plan):
        v = ctx.views[k]
        v.records = {kk: [r for r in recs if o0 * 16 <= r["py"] < o1 * 16] for kk, recs in v.records.items()}
    gr, hs, _ = ctx.accumulate(attr, 0, [1, 2])
    return gr, hs


def _worker(rank, world, port, attr, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gr, hs = _band_terms(rank, world, attr, q)
    t = torch.from_numpy(np.concatenate([gr.ravel(), hs.ravel()]))
    dist.all_reduce(t)
    if rank == 0:
        q.put(t.numpy())
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("attr", [0, 2, 3])
def test_band_allreduce_equals_full_accumulation(attr):
    from test_oracle import load
    g = load("newton.npz")
    name = ["position", "rotation", "scaling", "opacity", "color"][attr]
    full = np.concatenate([g[f"terms_{name}_grad"].ravel(), g[f"terms_{name}_hess"].ravel()])
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, attr, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    floor = 1e-6 * np.max(np.abs(full))
    assert np.max(np.abs(out - full) / np.maximum(np.maximum(np.abs(out), np.abs(full)), floor)) < 1e-7
