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
    one rank (buffered: runs dealt to the least-loaded rank as they close; scpl/raw: a contiguous
    frame block), and after the per-span broadcasts every rank holds every frame."""
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


def _scan_once_worker(rank, world, port, out):
    """scan_once mode's host plumbing: rank 0's run list reaches every rank (broadcast of host
    objects), every rank computes the same LPT owners, and the spans gather back whole."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_1903_03180_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    runs = [(0, 62), (62, 38), (100, 3)] + [(103 + 4 * k, 4) for k in range(24)] + [(199, 2), (201, 52), (253, 47)]
    got = sharding.broadcast_runs(runs if rank == 0 else None)
    owners = sharding.lpt_owners(got, world)
    T = 300
    x = torch.full((T, 2), -1, dtype=torch.int32)
    for s, n in sharding.owned_spans(got, rank, world, "buffered", T, owners):
        x[s:s + n] = torch.arange(s, s + n, dtype=torch.int32)[:, None] + 1000
    sharding.gather_runs(x, got, world, "buffered", owners=owners)
    out[rank] = (got, owners, x[:, 0].tolist())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_scan_once_lpt_gather(world):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_scan_once_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    runs0, owners0, _ = res[0]
    for r in range(world):
        runs, owners, x = res[r]
        assert runs == runs0 and owners == owners0          # identical on every rank
        assert x == [1000 + t for t in range(300)]          # every frame gathered
    # LPT balance: no rank carries more than one run's cost above the least loaded one
    load = [0.0] * world
    for run, o in zip(runs0, owners0):
        load[o] += 1000.0 + run[1]
    assert max(load) - min(load) <= 1000.0 + max(n for _, n in runs0)


def test_run_owner_assignments():
    """libscpl's online assignment (runs in scan order to the least-loaded rank) and the LPT
    deal: deterministic, every run owned once, loads balanced to within one run."""
    from paper_1903_03180_b200 import sharding
    runs = [(0, 62), (62, 38), (100, 3)] + [(103 + 4 * k, 4) for k in range(24)] + [(199, 2), (201, 52), (253, 47)]
    for world in (1, 2, 4, 8):
        for fn in (sharding.run_owners, sharding.lpt_owners):
            owners = fn(runs, world)
            assert owners == fn(runs, world) and len(owners) == len(runs)
            assert set(owners) <= set(range(world))
            load = [0.0] * world
            for run, o in zip(runs, owners):
                load[o] += 1000.0 + run[1]
            assert max(load) - min(load) <= 1000.0 + 62
    assert sharding.run_owners([(0, 5), (5, 3), (8, 4)], 2) == [0, 1, 1]  # least loaded (5 + 1000 > 3 + 1000)


def _c4_worker(rank, world, port, out):
    """BASELINE C4 across ranks: 64 clips, 64/world per rank (clip i's seed is i), no exchange
    on the data path; the bench's max-over-ranks time reduction."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    from paper_1903_03180_b200 import sharding
    from paper_1903_03180_b200.synth import C4_CLIPS, config_clip
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = sharding.shard_clips(C4_CLIPS, rank, world)
    digests = [int(config_clip("C4", frames=1, clip=i)[0][0, :8, :8].astype(np.int64).sum()) for i in mine[:2]]
    worst = bench.reduce_max(float(len(mine)) + 0.5 * rank, world, "cpu")
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    out[rank] = (mine, digests, worst, gathered)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_c4_clip_sharding(world):
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_c4_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    allc = sorted(c for r in range(world) for c in res[r][0])
    assert allc == list(range(64))                           # every clip exactly once
    assert all(len(res[r][0]) == 64 // world for r in range(world))
    assert res[0][3] == res[world - 1][3]
    assert res[0][2] == 64 // world + 0.5 * (world - 1)       # max over ranks
    d = [x for r in range(world) for x in res[r][1]]
    assert len(set(d)) == len(d)                             # different seeds, different clips


def _shared_buf_worker(rank, world, port, name, out):
    """Host gather through one shared buffer (sharding.shared_host_buffer): every rank writes its
    runs' frames (LPT owners) straight into the mapping, and after a barrier every rank reads the
    whole clip -- no collective carries frames."""
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_1903_03180_b200 import sharding
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    runs = [(0, 7), (7, 3), (10, 12), (22, 2), (24, 9)]
    owners = sharding.lpt_owners(runs, world)
    buf = sharding.shared_host_buffer(name, (33, 4, 5, 3), pin=False)
    for (s, n), o in zip(runs, owners):
        if o == rank:
            buf[s:s + n] = torch.arange(s, s + n, dtype=torch.uint8)[:, None, None, None] + 100
    dist.barrier()
    out[rank] = buf[:, 0, 0, 0].tolist()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_shared_host_buffer_gather(world):
    import uuid
    from paper_1903_03180_b200 import sharding
    name = f"scpl_test_{uuid.uuid4().hex[:8]}"
    port = _free_port()
    try:
        with mp.Manager() as mgr:
            out = mgr.dict()
            mp.spawn(_shared_buf_worker, args=(world, port, name, out), nprocs=world, join=True)
            res = dict(out)
    finally:
        try:
            os.unlink(os.path.join("/dev/shm", name))
        except FileNotFoundError:
            pass
    for r in range(world):
        assert res[r] == [100 + t for t in range(33)]
    assert sharding is not None
