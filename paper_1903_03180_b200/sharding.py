"""One clip across several GPUs ("one serial scan + independent runs"), and a
batch of clips across GPUs (BASELINE config C4).

The buffer scan (buffering.py:93-127) is serial over the clip, but once it has placed the runs
they are independent (pipeline.py:246-277 carves each from its own frames).  Two ways to split:

* every rank holds the clip, computes the energy codes and the whole scan (cheap next to the
  carves, and no rank waits on another) and carves the runs the online assignment gives it as
  they close (libscpl shard_rank / shard_count: each run goes to the least-loaded rank so far;
  every rank sees the same runs in the same order, so every rank computes the same owners);
* scan_once: rank 0 runs the scan alone, the run list goes to every rank through the host
  (a broadcast of a few integers), and the runs are dealt longest-processing-time first; each
  rank then carves exactly its runs (libscpl runs_in).

In scpl / raw modes every frame is a run: a contiguous block of frames per rank.  A run's cost
is dominated by its carve (one representative frame, ~40 DP passes: about as long as replaying
~1000 frames), so the cost model is 1000 + run length.  Outputs are gathered either with one
broadcast per run from its owner (CUDA outputs: NCCL over NVLink, or gloo on CPU) or on the
host: every rank's host-buffer call writes its runs' frames into one shared host buffer (no
collective at all).  There is no collective on the compute path.
"""

from __future__ import annotations

import os

RUN_COST0 = 1000.0  # a run's carve, in frames of replay


def _cost(run) -> float:
    return RUN_COST0 + run[1]


def run_owners(runs, world: int) -> list[int]:
    """Owner of each buffered run under libscpl's shard mode: runs in scan order, each to the
    least-loaded rank so far (lowest rank on ties) -- scpl_api.cu `mine`."""
    load = [0.0] * world
    owners = []
    for run in runs:
        best = min(range(world), key=lambda k: (load[k], k))
        load[best] += _cost(run)
        owners.append(best)
    return owners


def lpt_owners(runs, world: int) -> list[int]:
    """Longest-processing-time-first assignment of the runs (scan_once mode)."""
    load = [0.0] * world
    owners = [0] * len(runs)
    for i in sorted(range(len(runs)), key=lambda i: (-_cost(runs[i]), i)):
        best = min(range(world), key=lambda k: (load[k], k))
        load[best] += _cost(runs[i])
        owners[i] = best
    return owners


def frame_block(rank: int, world: int, T: int) -> tuple[int, int]:
    """Frames [a, b) a rank carves in scpl / raw mode (libscpl: T*rank/world .. T*(rank+1)/world)."""
    return T * rank // world, T * (rank + 1) // world


def owned_spans(runs, rank: int, world: int, mode: str, T: int, owners=None):
    """(start, length) frame spans this rank produces (owners: a run -> rank list, default the
    online assignment)."""
    if mode == "buffered":
        owners = run_owners(runs, world) if owners is None else owners
        return [tuple(r) for r, o in zip(runs, owners) if o == rank]
    a, b = frame_block(rank, world, T)
    return [(a, b - a)] if b > a else []


def gather_runs(out, runs, world: int, mode: str, group=None, owners=None):
    """Make `out` (T, ...) complete on every rank: each span is broadcast by its owner."""
    import torch.distributed as dist
    T = out.shape[0]
    for rank in range(world):
        for s, n in owned_spans(runs, rank, world, mode, T, owners):
            dist.broadcast(out[s:s + n], src=rank, group=group)
    return out


def broadcast_runs(runs, group=None, src: int = 0):
    """The scan's run list from `src` to every rank (host objects, a few integers)."""
    import torch.distributed as dist
    box = [list(map(tuple, runs)) if runs is not None else None]
    dist.broadcast_object_list(box, src=src, group=group)
    return [tuple(r) for r in box[0]]


def retarget_clip_sharded(clip, config, group=None, out=None, scan_once=False, gather=True):
    """retarget_video_tensor of one CUDA clip split across the ranks of `group`: returns the
    output (whole on every rank when gather, else this rank's runs only) and RunMetrics with
    dp_passes summed over the ranks."""
    import torch
    import torch.distributed as dist

    from .pipeline import retarget_video_tensor, scan_runs
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    owners = None
    if scan_once and config.mode == "buffered":
        runs = scan_runs(clip, config) if rank == 0 else None
        runs = broadcast_runs(runs, group) if world > 1 else runs
        owners = lpt_owners(runs, world)
        mine = [r for r, o in zip(runs, owners) if o == rank]
        res, m = retarget_video_tensor(clip, config, out=out, runs=mine)
        m.runs = runs
    else:
        res, m = retarget_video_tensor(clip, config, out=out, shard=(rank, world))
    if world > 1:
        if gather:
            gather_runs(res, m.runs, world, config.mode, group, owners)
        dp = torch.tensor([m.dp_passes], dtype=torch.int64, device=res.device)
        dist.all_reduce(dp, group=group)
        m.dp_passes = int(dp.item())
    return res, m


def shared_host_buffer(name: str, shape, pin: bool = True):
    """A host uint8 buffer every process of the node maps (/dev/shm/<name>): the ranks of a split
    clip write their runs' output frames straight into it (their D2H copies land there), so the
    outputs are gathered on the host with no collective.  Pinned (cudaHostRegister) when CUDA is
    up, so the copies run asynchronously.  The creator (rank 0) sizes it; the others attach."""
    import math
    import torch
    nbytes = int(math.prod(shape))
    path = os.path.join("/dev/shm", name)
    t = torch.from_file(path, shared=True, size=nbytes, dtype=torch.uint8).view(*shape)
    if pin and torch.cuda.is_available():
        rc = torch.cuda.cudart().cudaHostRegister(t.data_ptr(), nbytes, 0)
        if int(rc) != 0:
            raise RuntimeError(f"cudaHostRegister failed ({int(rc)}) for the shared output buffer")
    return t


def release_host_buffer(t, name: str) -> None:
    import torch
    if torch.cuda.is_available():
        torch.cuda.cudart().cudaHostUnregister(t.data_ptr())
    try:
        os.unlink(os.path.join("/dev/shm", name))
    except FileNotFoundError:
        pass


def retarget_clip_sharded_host(clip, config, out, group=None):
    """One HOST clip split across the ranks of `group`, outputs gathered on the host: rank 0 scans
    (scan_runs), the run list goes to every rank, runs are dealt longest-processing-time first,
    and every rank's host-buffer call (chunked H2D, per-run D2H) writes its runs' frames into
    `out` -- a shared_host_buffer all ranks map.  After the barrier every rank sees the whole
    output.  Returns RunMetrics with dp_passes summed over the ranks."""
    import torch
    import torch.distributed as dist

    from .pipeline import RunMetrics, _run_device, _targets, scan_runs
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    tw, th = _targets(clip, config)
    if config.mode == "buffered":
        runs = scan_runs(clip, config) if rank == 0 else None
        runs = broadcast_runs(runs, group) if world > 1 else runs
        owners = lpt_owners(runs, world)
        mine = [r for r, o in zip(runs, owners) if o == rank]
        _, dp, _, _ = _run_device(clip.contiguous(), config, tw, th, out=out, runs_in=mine)
    else:  # scpl / raw: a contiguous block of frames per rank
        _, dp, runs, _ = _run_device(clip.contiguous(), config, tw, th, out=out, shard=(rank, world))
    if world > 1:
        t = torch.tensor([dp], dtype=torch.int64)
        dist.all_reduce(t, group=group)
        dp = int(t.item())
        dist.barrier(group=group)
    return out, RunMetrics(dp_passes=dp, frames_out=clip.shape[0], runs=runs)


def shard_clips(n_clips: int, rank: int, world: int) -> list[int]:
    """Clips of a batch a rank retargets (BASELINE C4: 64 clips, 64/G per GPU): a contiguous
    block, sizes differing by at most one."""
    return list(range(n_clips * rank // world, n_clips * (rank + 1) // world))
