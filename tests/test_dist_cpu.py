"""Multi-process (gloo, world_size 2) CPU test of the multi-GPU decomposition:
each rank accumulates the terms of its tile-row band of every view (the float64
oracle restricted to the band's pixels), the per-Gaussian accumulators are
all-reduced, and the sum equals the single-process accumulation — the exchange
step of the CUDA trainer (NCCL all-reduce after every backward pass)."""
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


def test_shard_rows_partition_covers_every_row_once():
    from paper_2501_13975_b200.capi import shard_rows
    for tiles_y in (1, 2, 3, 13, 50, 68):
        for world in (1, 2, 3, 4, 8):
            owned = []
            for r in range(world):
                b0, b1, o0, o1 = shard_rows(tiles_y, r, world)
                assert b0 <= o0 <= o1 <= b1 and b0 >= 0 and b1 <= tiles_y
                assert o0 - b0 <= 1 and b1 - o1 <= 1   # one-tile-row halo (16 px >= 10 px SSIM support)
                owned += list(range(o0, o1))
            assert owned == list(range(tiles_y))


def _band_terms(rank, world, attr, q):
    import ngs_oracle as O
    from test_oracle import cam_from, load, scene_from
    from paper_2501_13975_b200.capi import shard_rows
    g = load("newton.npz")
    ctx = O.OracleContext()
    ctx.set_scene(scene_from(g, "s_"))
    ctx.build_view(0, cam_from(g, "c_"), g["target"])
    for i in range(2):
        ctx.build_view(1 + i, cam_from(g, f"sec{i}_"), g[f"sec{i}_target"])
    # keep only records whose pixel row lies in this rank's owned tile rows
    for v in ctx.views.values():
        ty = (v.cam.height + 15) // 16
        _, _, o0, o1 = shard_rows(ty, rank, world)
        v.records = {k: [r for r in recs if o0 * 16 <= r["py"] < o1 * 16] for k, recs in v.records.items()}
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


@pytest.mark.parametrize("attr", [0, 3])
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
