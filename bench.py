#!/usr/bin/env python
"""Benchmark: buffered SCPL video retargeting on B200 (BASELINE.json metric).

One step = one pass of the hot path over one synthetic clip: retarget_video(mode="buffered")
on config C2 (300 x 1080x1920 RGB, width 1920 -> 1440), the BASELINE metric's 1080p
width -25% workload.  Prints ONE JSON line on rank 0.

  value     frames/s with the clip resident in HBM (device-timed, CUDA events, max over ranks)
  e2e       frames/s through the public API with pinned HOST buffers: H2D of the clip, the
            carve, D2H of the output, every step
  roofline  the dominant kernel (carve_pass_kernel): algorithmic bytes per launch / mean launch
            duration, against the measured copy bandwidth (see pass_roofline)
  step_roofline  the whole step: algorithmic HBM bytes per frame B = 6*H*W + 3*H'*W' (SURVEY.md
            §8d: the input is read by the energy/statistics pass and by the replay, the output
            written once) times frames per step / step time
  cpu_baseline  the CPU oracle port (numpy restatement of the reference) on a bounded sample

Multi-GPU (torchrun): each rank retargets its own clip (C2 recipe, seed = rank) -- clips are
independent, there is no collective on the data path ("scaling": "weak").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

if "reference" in sys.argv:  # one BLAS thread per worker process: the workers use every core
    for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ.setdefault(_v, "1")

import numpy as np

os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")  # before CUDA initialises (see package)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1903_03180_b200.synth import CONFIGS, config_clip  # noqa: E402

METRIC = "retargeted frames/sec (1080p, width -25%)"
UNIT = "frames/s"


PRIME_CALLS = 3  # untimed calls before the warm-up steps (graph-pool initialisation)


def metric_for(name: str) -> str:
    """BASELINE.json's metric on its own workload (C2); the other configs name theirs."""
    if name == "C2":
        return METRIC
    spec, tw, th = CONFIGS[name]
    what = f"width {spec.width}->{tw}" if tw else f"height {spec.height}->{th}"
    n = "64 clips x " if name == "C4" else ""
    return f"retargeted frames/sec ({name}: {n}{spec.frames}x{spec.height}x{spec.width}, {what})"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def alg_bytes_per_frame(h, w, th, tw, c=3):
    return 2 * c * h * w + c * th * tw


def pass_roofline(ph, H, W, tw, peak, peak_src):
    """Roofline of the dominant kernel, carve_pass_kernel (DP + select + trace of every run of a
    group, one cluster per run; ~70% of kernel time in the committed launch list).

    Per run and pass the algorithmic bytes are the gradient plane read once (rows x width B) and
    the 32-row choice words + landing deltas written and read back (2 x (8 + 1) B per column per
    32 rows); a launch carries dp_passes / launches runs.  The launch duration is the slowest
    cluster's SM-clock cycles (clock64 in the kernel) -- the passes run inside conditional
    graphs on the library's own streams, where events cannot bracket a single kernel.
    traffic: DRAM bytes per launch from the committed ncu --set full capture, scaled to the
    same runs per launch."""
    launches = ph.get("pass_launches") or 0
    launch_ms = ph.get("pass_launch_ms") or 0.0
    if not launches or not launch_ms:
        return None
    runs_per_launch = ph["dp_passes"] / launches
    cols = 0.5 * (W + tw)  # mean width over the passes
    per_run = H * cols * (1.0 + 2 * 9 / 32)
    alg = per_run * runs_per_launch
    achieved = alg / (launch_ms / 1e3) / 1e9
    traffic = None
    try:
        k = json.load(open(os.path.join(ROOT, "profiles", "kernel_shares.json")))
        d = k.get("_carve_pass_dram_bytes_per_launch") or {}
        if d.get("read") is not None:
            traffic = (d["read"] + d.get("write", 0)) / d["runs_per_launch"] * runs_per_launch
        share = k.get("carve_pass_kernel")
    except Exception:
        share = None
    return {"kernel": "carve_pass_kernel", "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
            "alg_bytes_per_launch": alg, "runs_per_launch": runs_per_launch, "avg_launch_us": launch_ms * 1e3,
            "launches_per_step": launches, "share_of_kernel_time": share,
            "timing": "in-kernel SM clock (clock64), slowest cluster per launch, over the timed steps",
            "limit": "latency: one dependent DP row after another (min-plus recurrence), not HBM"}


class ClockSampler:
    """SM clocks and throttle reasons sampled every 10 ms during the timed region (NVML; the
    nvidia-smi CLI polled at 100 ms as a fallback)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.sm, self.mx, self.reasons = gpu, [], [], set()
        self.proc, self.stop, self.thread, self.nv = None, threading.Event(), None, None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()

        try:  # the NVML device behind this CUDA ordinal (CUDA_VISIBLE_DEVICES may reorder)
            import torch
            p = torch.cuda.get_device_properties(self.gpu)
            want = (int(p.pci_domain_id), int(p.pci_bus_id), int(p.pci_device_id))
            for k in range(pynvml.nvmlDeviceGetCount()):
                h = pynvml.nvmlDeviceGetHandleByIndex(k)
                q = pynvml.nvmlDeviceGetPciInfo(h)
                if (int(q.domain), int(q.bus), int(q.device)) == want:
                    return pynvml, h
        except Exception:
            pass
        return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.gpu)

    def __enter__(self):
        try:
            if os.environ.get("SCPL_BENCH_CLOCKS") == "off":
                return self
            if os.environ.get("SCPL_BENCH_CLOCKS") == "smi":
                raise RuntimeError("nvidia-smi sampler requested")
            self.nv, h = self._handle()
            self.mx.append(float(self.nv.nvmlDeviceGetMaxClockInfo(h, self.nv.NVML_CLOCK_SM)))
            self.thread = threading.Thread(target=self._poll_nvml, args=(h,), daemon=True)
            self.thread.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read_smi, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _poll_nvml(self, h):
        nv = self.nv
        while not self.stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, const in self.REASONS:
                    if r & getattr(nv, const):
                        self.reasons.add(name)
            except Exception:
                pass
            self.stop.wait(0.01)

    def _read_smi(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                if parts[1].replace(".", "").isdigit():
                    self.sm.append(float(parts[1]))
                if parts[2].replace(".", "").isdigit():
                    self.mx.append(float(parts[2]))
                for (name, _), v in zip(self.REASONS, parts[4:8]):
                    if v.lower() == "active":
                        self.reasons.add(name)

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait()
        if self.thread:
            self.thread.join(timeout=2)

    def summary(self):
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": max(self.mx) if self.mx else None, "reasons": sorted(self.reasons),
                    "samples": 0}
        top = max(self.mx) if self.mx else max(self.sm)
        loaded = [s for s in self.sm if s > 0.5 * top] or self.sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": top, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml" if self.nv else "nvidia-smi"}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def reduce_max(x: float, world: int, device: str) -> float:
    """Max of a per-rank time over the job (the slowest rank bounds the step)."""
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def rank_workload(name: str, rank: int, frames=None):
    """Each rank retargets its own clip of the config's recipe (seed = rank): clips are
    independent, so the data path has no collective (weak scaling)."""
    if rank == 0 or name == "C4":
        return config_clip(name, frames=frames, clip=rank)
    from dataclasses import replace
    from paper_1903_03180_b200.synth import generate_clip
    spec, tw, th = CONFIGS[name]
    return generate_clip(replace(spec, seed=spec.seed + 1000 * rank), frames=frames), tw, th


# ------------------------------------------------------------------ CPU legs (oracle port)
def workload(name: str) -> str:
    """The config's workload name, identical on both arms."""
    spec, tw, th = CONFIGS[name]
    return (f"{name}: {spec.frames}x{spec.height}x{spec.width}x3 -> {th or spec.height}x{tw or spec.width}, "
            f"buffered SCPL, alpha 0.2, max_len 64, wm/wg 0.6/0.4")


def _golden_runs(name: str):
    """The config clip's real run list (tests/golden, produced by the reference itself)."""
    path = os.path.join(ROOT, "tests", "golden", f"{name}{'_clip0' if name == 'C4' else ''}.json")
    with open(path) as f:
        g = json.load(f)
    return [tuple(r) for r in g["runs"]], int(g["dp_passes"]), float(g.get("reference_wall_s") or 0.0)


def _oracle_run(args):
    """One real run of the config clip through the oracle port (worker process): the energy and
    buffer pushes of its first k_e frames, the carve of its representative frame (batch_carve on
    the run's mean energy) and the literal replay of one frame (remove_batch per batch,
    pipeline.py:140-154).  Returns (run length, its single-core time: per-frame costs x length +
    the carve)."""
    name, start, n, k_e = args
    sys.path.insert(0, ROOT)
    from oracle import scpl_oracle as O
    from paper_1903_03180_b200.synth import generate_clip
    spec, tw, th = CONFIGS[name]
    lo = max(0, start - 1)
    k_e = min(n, k_e)
    fr = generate_clip(spec, frames=k_e + (start - lo), threads=1, start=lo)
    prev = fr[0] if start > 0 else None
    fr = fr[start - lo:]
    t0 = time.perf_counter()
    maps = [O.motion_energy(fr[0], prev)] + [O.motion_energy(f, p) for p, f in zip(fr[:k_e - 1], fr[1:k_e])]
    O.buffer_scan(maps, O.BufferPolicy())  # (the pushes of these frames)
    u = maps[0] if k_e == 1 else O.uniform_energy(maps)
    t1 = time.perf_counter()
    if tw is not None and tw < fr[0].shape[1]:
        work, target, pe = fr[0], tw, u
    else:  # height carve: the reference transposes frames and energy (pipeline.py:263-265)
        work, target, pe = O._transpose(fr[0]), th, O._transpose(u)
    _, batches = O.batch_carve(work, target, energy=pe)
    t2 = time.perf_counter()
    O.replay_batches([work], batches)
    t3 = time.perf_counter()
    return n, (t1 - t0) / k_e * n + (t2 - t1) + (t3 - t2) * n


def run_reference(a, world, rank):
    """--impl reference: the oracle port (numpy restatement of vidcarve's path) on the host
    cores, rank 0 only.  Each step, every core takes one REAL run of the config clip (the
    reference's own run list, cycled so the run-length mix is the clip's) and times its energy +
    pushes, its carve and the literal replay of its frames (measured on its first frames,
    extrapolated to the run's length: the per-frame costs are per-frame work); the step's value is
    the runs' frames over their summed single-core time divided by the cores."""
    if rank != 0:
        return
    from concurrent.futures import ProcessPoolExecutor
    spec, tw, th = CONFIGS[a.config]
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    workers = max(1, cores)  # every host thread: one oracle run per core, one BLAS thread each
    runs, dp, ref_wall = _golden_runs(a.config)
    k_e = 2
    nxt = 0

    def step(pool):
        nonlocal nxt
        jobs = [(a.config, runs[(nxt + w) % len(runs)][0], runs[(nxt + w) % len(runs)][1], k_e)
                for w in range(workers)]
        nxt += workers
        res = list(pool.map(_oracle_run, jobs))
        frames = sum(n for n, _ in res)
        core_s = sum(t for _, t in res)
        return frames, core_s

    with ProcessPoolExecutor(max_workers=workers) as pool:
        for _ in range(min(a.warmup, 1)):  # (CPU code: one warm-up step loads the modules)
            step(pool)
        samples = [step(pool) for _ in range(a.steps)]
    frames = sum(f for f, _ in samples)
    core_s = sum(t for _, t in samples)
    per_frame_core = core_s / frames            # single-core seconds per output frame
    value = workers / per_frame_core            # frames/s on `workers` cores
    clip_frames = sum(n for _, n in runs)
    per_step = clip_frames * per_frame_core / workers
    sample = (f"per step {workers} real runs of {a.config} (the reference's run list, cycled: mix "
              f"{clip_frames} frames / {len(runs)} runs), each through the oracle port: energy + pushes of its "
              f"first {k_e} frames, the carve of its representative frame, the literal replay (remove_batch "
              f"per batch) of a frame; per-frame costs x run length; {workers} cores; the reference itself "
              f"took {ref_wall:.0f} s for the clip on one core of the build host "
              f"({clip_frames / ref_wall if ref_wall else 0:.3f} frames/s)")
    line = {
        "metric": metric_for(a.config), "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
        "warmup": a.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8/f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": workload(a.config), "frames_per_step": clip_frames,
                   "sample": f"{workers} real runs per step, per-frame costs extrapolated to the run lengths",
                   "single_core_s_per_frame": per_frame_core},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU leg
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--frames", type=int, default=None, help="truncate the clip (debug only)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--clips", type=int, default=None, help="C4: clips per step (default 64)")
    ap.add_argument("--scan-once", action="store_true",
                    help="with --split-runs: rank 0 scans, runs dealt longest-first (sharding.py)")
    ap.add_argument("--no-list-e2e", action="store_true")
    ap.add_argument("--split-runs", action="store_true",
                    help="one clip across the GPUs (sharding.py: every rank scans, carves its runs, "
                         "outputs exchanged by NCCL broadcasts); strong scaling")
    a = ap.parse_args()
    world, rank, local = dist_setup()
    if a.impl == "reference":
        return run_reference(a, world, rank)

    import torch
    import torch.distributed as dist

    import paper_1903_03180_b200 as P
    from paper_1903_03180_b200 import _lib, pipeline

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    name = a.config
    split = a.split_runs and world > 1
    batch = name == "C4"  # BASELINE configs[3]: 64 clips per step, 64/N per rank, one batch call
    from paper_1903_03180_b200 import sharding
    from paper_1903_03180_b200.synth import C4_CLIPS
    if batch:
        mine = sharding.shard_clips(a.clips or C4_CLIPS, rank, world)
        host_clips = []
        for i in mine:
            c, tw, th = config_clip("C4", frames=a.frames, clip=i)
            host_clips.append(torch.from_numpy(c).pin_memory())
            del c
    else:
        clip, tw, th = rank_workload(name, 0 if split else rank, a.frames)
        host_clips = [torch.from_numpy(clip).pin_memory()]
        del clip
    T, H, W, C = host_clips[0].shape
    tw = tw or W
    th = th or H
    cfg = P.RetargetConfig(target_width=tw, target_height=th, mode="buffered")
    devs = [h.cuda() for h in host_clips]
    host_in = host_clips[0]
    dev = devs[0]
    frames_per_rank = T * len(devs)
    lib = _lib.load()

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        return reduce_max(x, world, "cuda")

    def step(clips_dev):
        if batch:
            res = P.retarget_videos(clips_dev, cfg)
            return res[0][0], res
        if split:
            return sharding.retarget_clip_sharded(clips_dev[0], cfg, scan_once=a.scan_once)
        return P.retarget_video_tensor(clips_dev[0], cfg)

    def total_dp(m):
        return sum(x[1].dp_passes for x in m) if batch else m.dp_passes

    def all_runs(m):
        return sum(len(x[1].runs) for x in m) if batch else len(m.runs)

    # initialisation: the library instantiates its pooled CUDA graphs (one per group shape in
    # flight) on first use; a few untimed calls fill the pool before the W warm-up steps
    for _ in range(PRIME_CALLS):
        step(devs)
    for _ in range(a.warmup):
        out, m = step(devs)
    torch.cuda.synchronize()

    # ---- device-resident timed region
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    phases = []
    with ClockSampler(local) as clocks:
        launches0 = lib.scpl_kernel_launches()
        barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(a.steps):
            out, m = step(devs)
            phases.append(dict(pipeline.last_phase_ms))
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        launches = (lib.scpl_kernel_launches() - launches0) / a.steps
    ms = max_over_ranks(e0.elapsed_time(e1) / a.steps)
    frames_job = T if split else frames_per_rank * world
    value = frames_job / (ms / 1e3)

    # ---- end to end through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        host_outs = [torch.empty((T, th, tw, C), dtype=torch.uint8, pin_memory=True) for _ in host_clips]

        def e2e_step():
            if batch:
                return P.retarget_videos(host_clips, cfg, outs=host_outs)
            if not split:
                return P.retarget_video(host_in, cfg, out=host_outs[0])
            # one clip across the ranks: every rank copies it in, carves its runs; after the
            # exchange rank 0 copies the whole output back
            dev.copy_(host_in, non_blocking=True)
            res, m_ = sharding.retarget_clip_sharded(dev, cfg, scan_once=a.scan_once)
            if rank == 0:
                host_outs[0].copy_(res, non_blocking=True)
            return host_outs[0], m_

        for _ in range(max(1, min(a.warmup, 3))):
            e2e_step()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            e2e_step()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / a.steps)
        barrier()
        e2e = {"value": frames_job / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": int(sum(h.numel() for h in host_clips)),
               "d2h_bytes_per_step": int(sum(o.numel() for o in host_outs)) if (rank == 0 or not split) else 0,
               "api": "retarget_videos(pinned host clips)" if batch else "retarget_video(pinned host tensor)"}
        if not batch and not split and not a.no_list_e2e:
            # the reference's own call shape: a list of numpy frames in, a list out (the API
            # stacks the list into pinned memory and copies the output frames back)
            frames_list = list(host_in.numpy())
            P.retarget_video(frames_list, cfg)
            t0 = time.perf_counter()
            for _ in range(max(1, a.steps // 4)):
                P.retarget_video(frames_list, cfg)
            lst_ms = (time.perf_counter() - t0) * 1e3 / max(1, a.steps // 4)
            e2e["list_api"] = {"value": T / (lst_ms / 1e3), "unit": UNIT, "ms_per_step": lst_ms,
                               "api": "retarget_video(list of numpy frames) -> list of numpy frames"}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    peak, peak_src = peaks()
    bpf = alg_bytes_per_frame(H, W, th, tw, C)
    achieved = bpf * frames_per_rank / (ms / 1e3) / 1e9  # per GPU
    ph = {k: statistics.mean(p[k] for p in phases) for k in phases[0]} if phases else {}
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(name)
        except Exception:
            traffic = None

    cpu = None
    if not a.no_cpu_baseline and world == 1:
        # one core, the clip's real runs in order (the reference's run list) until ~20 s of work
        runs, _, ref_wall = _golden_runs(name)
        fr_done, core_s, k, t_start = 0, 0.0, 0, time.perf_counter()
        while time.perf_counter() - t_start < 20.0 and k < len(runs):
            n_, t_ = _oracle_run((name, runs[k][0], runs[k][1], 2))
            fr_done += n_
            core_s += t_
            k += 1
        cpu = {"value": fr_done / core_s, "unit": UNIT, "cores": 1, "kind": "port",
               "sample": f"the first {k} real runs of {name} ({fr_done} frames) through the oracle port on one "
                         f"core: energy + pushes, carve, literal replay (per-frame costs x run length); the "
                         f"reference itself: {ref_wall:.0f} s for the {sum(n for _, n in runs)}-frame clip on one "
                         f"build-host core"}

    line = {
        "metric": metric_for(name), "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong" if split else "weak", "vs_baseline": None,
        "dtype": "u8/f64", "data": "synthetic",
        "config": {"workload": workload(name) if a.frames is None else f"{name} (first {T} frames)",
                   "frames_per_step": frames_job, "clips_per_step": len(devs) * (1 if split else world),
                   "runs": all_runs(m), "dp_passes": total_dp(m),
                   "l2": f"inputs ({sum(h.numel() for h in host_clips) / 1e9:.2f} GB per rank) larger than L2",
                   "init": f"{PRIME_CALLS} untimed calls before the warm-up steps (pooled CUDA graphs instantiated)",
                   "parallelism": (f"one clip, runs split over {world} GPUs ("
                                   + ("rank 0 scans, runs dealt LPT-first" if a.scan_once else "every rank scans")
                                   + "; outputs exchanged by NCCL broadcasts)") if split else
                                  (f"{len(devs)} clips per GPU in one batch call x{world} GPUs" if batch
                                   else f"clip-per-GPU x{world}")},
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": pass_roofline(dict(ph, dp_passes=total_dp(m)), H, W, tw, peak, peak_src),
        "step_roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                          "frac": achieved / peak, "traffic": traffic,
                          "scope": "whole step (all kernels), per GPU; B = 6HW + 3H'W' bytes per frame",
                          "peak_source": peak_src},
        "phases_ms": ph,
        "clocks": clocks.summary(),
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
