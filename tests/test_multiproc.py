"""Multi-process (world_size 2, gloo on CPU) checks of the benchmark's job logic: each rank
gets its own clip (no data-path collective), and the step time reported is the max over
ranks.  The GPU path itself is single-process per GPU; this covers the host-side plumbing."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w, r, local = bench.dist_setup()
    assert (w, r, local) == (world, rank, rank)
    clip, tw, th = bench.rank_workload("C1", r, frames=3)
    digest = float(np.asarray(clip, dtype=np.float64).sum())
    times = [digest, digest]  # gather both ranks' digests through the same reduction the bench uses
    worst = bench.reduce_max(10.0 + rank, w, "cpu")
    t = torch.tensor([digest], dtype=torch.float64)
    got = [torch.zeros(1, dtype=torch.float64) for _ in range(w)]
    dist.all_gather(got, t)
    out[rank] = (worst, [float(x.item()) for x in got], tw, th, clip.shape)
    dist.destroy_process_group()


def test_two_ranks_distinct_clips_and_max_time():
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0][0] == res[1][0] == 11.0          # max over ranks
    d0, d1 = res[0][1]
    assert d0 != d1                                # each rank carves a different clip
    assert res[0][1] == res[1][1]
    assert res[0][2:] == res[1][2:]                # same config geometry on every rank


def _shard_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_1903_03180_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    runs = [(0, 5), (5, 3), (8, 4), (12, 1), (13, 6)]
    T = 19
    for mode in ("buffered", "scpl"):
        # each rank writes only the spans it owns (value = 100 + frame index), the rest is junk
        x = torch.full((T, 2, 3), -1, dtype=torch.int32)
        for s, n in sharding.owned_spans(runs, rank, world, mode, T):
            for t in range(s, s + n):
                x[t] = 100 + t
        sharding.gather_runs(x, runs, world, mode)
        res[mode] = x[:, 0, 0].tolist()
    out[rank] = res
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_clip_gather(world):
    """One clip split across ranks (sharding.py): every frame is owned by exactly
    one rank (buffered: run r on rank r % world; scpl/raw: a contiguous frame block), and after
    the per-span broadcasts every rank holds every frame."""
    from paper_1903_03180_b200 import sharding
    runs = [(0, 5), (5, 3), (8, 4), (12, 1), (13, 6)]
    for mode in ("buffered", "scpl"):
        cover = sorted(t for r in range(world) for s, n in sharding.owned_spans(runs, r, world, mode, 19)
                       for t in range(s, s + n))
        assert cover == list(range(19))
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_shard_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for r in range(world):
        for mode in ("buffered", "scpl"):
            assert res[r][mode] == [100 + t for t in range(19)]
