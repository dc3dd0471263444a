"""One clip across several GPUs ("one serial scan + independent runs").

The buffer scan (buffering.py:93-127) is serial over the clip, but once it has placed the runs
they are independent (pipeline.py:246-277 carves each from its own frames).  Every rank holds
the clip, computes the energy codes and the whole scan -- cheap next to the carves, and no
rank waits on another -- then carves and replays only its own runs: run r belongs to rank
r % world (scpl / raw modes, where every frame is a run: a contiguous block of frames per
rank).  The output frames are then exchanged with one broadcast per run from its owner (NCCL
over NVLink, or gloo on CPU), so every rank ends with the whole retargeted clip.  There is no
collective on the compute path.
"""

from __future__ import annotations


def run_owner(r: int, world: int) -> int:
    """Rank that carves buffered run r (libscpl: r % shard_count == shard_rank)."""
    return r % world


def frame_block(rank: int, world: int, T: int) -> tuple[int, int]:
    """Frames [a, b) a rank carves in scpl / raw mode (libscpl: T*rank/world .. T*(rank+1)/world)."""
    return T * rank // world, T * (rank + 1) // world


def owned_spans(runs, rank: int, world: int, mode: str, T: int):
    """(start, length) frame spans this rank produces."""
    if mode == "buffered":
        return [tuple(r) for i, r in enumerate(runs) if run_owner(i, world) == rank]
    a, b = frame_block(rank, world, T)
    return [(a, b - a)] if b > a else []


def gather_runs(out, runs, world: int, mode: str, group=None):
    """Make `out` (T, ...) complete on every rank: each span is broadcast by its owner."""
    import torch.distributed as dist
    T = out.shape[0]
    for rank in range(world):
        for s, n in owned_spans(runs, rank, world, mode, T):
            dist.broadcast(out[s:s + n], src=rank, group=group)
    return out


def retarget_clip_sharded(clip, config, group=None, out=None):
    """retarget_video_tensor of one CUDA clip split across the ranks of `group`: returns the
    whole output on every rank and RunMetrics with dp_passes summed over the ranks."""
    import torch
    import torch.distributed as dist

    from .pipeline import retarget_video_tensor
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    res, m = retarget_video_tensor(clip, config, out=out, shard=(rank, world))
    if world > 1:
        gather_runs(res, m.runs, world, config.mode, group)
        dp = torch.tensor([m.dp_passes], dtype=torch.int64, device=res.device)
        dist.all_reduce(dp, group=group)
        m.dp_passes = int(dp.item())
    return res, m
