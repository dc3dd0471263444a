"""`vidcarve` command line on the GPU path (the reference's cli.py:1-232 flags, defaults,
exit codes 0 success / 1 usage / 2 I/O or format, one-line diagnostics on stderr).

`video` streams PNM input straight into pinned memory and through the GPU pipeline
(media.read_clip_pinned -> retarget_video -> media.write_clip); `image` and `bench` use the
same API as the reference. `--figures` (matplotlib plots) is not provided.

    python -m paper_1903_03180_b200.cli video in.ppm out.ppm --scale 0.75
"""

from __future__ import annotations

import argparse
import sys

import numpy as np

from .buffering import BufferPolicy
from .media import MediaFormatError, read_clip_pinned, read_frames, write_clip, write_frames
from .pipeline import MODES, RetargetConfig, retarget_image, retarget_video
from .quality import SYNTHETIC_KINDS, SyntheticSpec, compare, format_metrics, generate, jitter


class _UsageError(Exception):
    pass


class _Parser(argparse.ArgumentParser):
    def error(self, message):
        raise _UsageError(message)


def _sizing(sp):
    sp.add_argument("--width", type=int, help="target width in pixels")
    sp.add_argument("--scale", type=float, help="target width as a fraction of source width")
    sp.add_argument("--height", type=int, help="target height in pixels")


def _tuning(sp, mode):
    sp.add_argument("--mode", choices=MODES, default=mode)
    sp.add_argument("--alpha", type=float, default=0.2, help="buffer threshold fraction")
    sp.add_argument("--motion-weight", type=float, default=0.6, help="weight of the frame difference term")
    sp.add_argument("--max-buffer", type=int, default=64, help="hard cap on buffer length")
    sp.add_argument("--metrics", metavar="PATH", help="write a key=value metrics report")
    sp.add_argument("--reaverage-energy", action="store_true",
                    help="recompute run energy from every carved frame, not the representative")
    sp.add_argument("--height-first", action="store_true", help="carve height before width")


def build_parser() -> _Parser:
    p = _Parser(prog="vidcarve", description="Content-aware image and video retargeting by seam carving (GPU).")
    sub = p.add_subparsers(dest="command", required=True, parser_class=_Parser)
    im = sub.add_parser("image", help="retarget a single image")
    im.add_argument("input", help="image file (.ppm, .pgm, .png) or '-' for stdin")
    im.add_argument("output", help="image file or '-' for stdout")
    _sizing(im)
    _tuning(im, "scpl")
    vd = sub.add_parser("video", help="retarget a frame stream")
    vd.add_argument("input", help="frame directory, concatenated .ppm, or '-' for stdin")
    vd.add_argument("output", help="frame directory, .ppm, or '-' for stdout")
    _sizing(vd)
    _tuning(vd, "buffered")
    bn = sub.add_parser("bench", help="compare modes over a corpus and report metrics")
    bn.add_argument("input", help=f"frame source, or a synthetic kind: {', '.join(SYNTHETIC_KINDS)}")
    _sizing(bn)
    _tuning(bn, "buffered")
    bn.add_argument("--modes", default=",".join(MODES), help="comma-separated modes to compare (default: all)")
    bn.add_argument("--frames", type=int, default=32, help="synthetic corpus length")
    bn.add_argument("--size", default="320x240", help="synthetic frame size, WxH")
    bn.add_argument("--seed", type=int, default=0, help="synthetic corpus seed")
    bn.add_argument("--figures", metavar="DIR", help="render report figures into DIR (not provided here)")
    return p


def _check_sizing(a):
    if a.width is not None and a.scale is not None:
        raise _UsageError("--width and --scale are mutually exclusive")
    if a.width is None and a.scale is None:
        raise _UsageError("one of --width or --scale is required")
    if a.scale is not None and not 0.0 < a.scale <= 1.0:
        raise _UsageError(f"--scale must be in (0, 1], got {a.scale}")


def _policy(a) -> BufferPolicy:
    if a.max_buffer < 1:
        raise _UsageError(f"--max-buffer must be >= 1, got {a.max_buffer}")
    if a.alpha <= 0:
        raise _UsageError(f"--alpha must be positive, got {a.alpha}")
    return BufferPolicy(alpha=a.alpha, max_len=a.max_buffer)


def _config(a, mode, source_width) -> RetargetConfig:
    tw = a.width if a.width is not None else max(1, round(source_width * a.scale))
    if not 0.0 <= a.motion_weight <= 1.0:
        raise _UsageError(f"--motion-weight must be in [0, 1], got {a.motion_weight}")
    return RetargetConfig(target_width=tw, target_height=a.height, mode=mode, policy=_policy(a),
                          w_motion=a.motion_weight, w_grad=1.0 - a.motion_weight,
                          reaverage_energy=a.reaverage_energy, height_first=a.height_first)


def _report(path, text):
    with open(path, "w", encoding="ascii") as fh:
        fh.write(text)


def _image(a) -> int:
    _check_sizing(a)
    frame = next(read_frames(a.input), None)
    if frame is None:
        raise MediaFormatError(f"no frames in {a.input}")
    out, metrics = retarget_image(frame, _config(a, a.mode, frame.shape[1]))
    write_frames(a.output, [out])
    if a.metrics:
        _report(a.metrics, format_metrics(metrics))
    return 0


def _video(a) -> int:
    _check_sizing(a)
    clip = read_clip_pinned(a.input)  # validated like read_frames, decoded into pinned memory
    if clip.numel() == 0:
        raise MediaFormatError(f"no frames in {a.input}")
    out, metrics = retarget_video(clip, _config(a, a.mode, clip.shape[2]))
    if out.shape[0] >= 2:
        metrics.jitter = jitter(out).value
    write_clip(a.output, out)
    if a.metrics:
        _report(a.metrics, format_metrics(metrics))
    return 0


def _bench(a) -> int:
    _check_sizing(a)
    if a.input in SYNTHETIC_KINDS:
        try:
            w, h = (int(v) for v in a.size.lower().split("x"))
        except ValueError:
            raise _UsageError(f"--size must look like 320x240, got {a.size!r}") from None
        frames = generate(SyntheticSpec(kind=a.input, width=w, height=h, frames=a.frames, seed=a.seed))
    else:
        frames = list(read_frames(a.input))
        if not frames:
            raise MediaFormatError(f"no frames in {a.input}")
    modes = [m.strip() for m in a.modes.split(",") if m.strip()]
    if not modes or any(m not in MODES for m in modes):
        raise _UsageError(f"--modes must name modes from {MODES}, got {a.modes!r}")
    if a.figures:
        raise _UsageError("--figures is not provided by this build")
    results = compare(frames, {m: _config(a, m, frames[0].shape[1]) for m in modes})
    text = format_metrics(results)
    print(text, end="")
    if a.metrics:
        _report(a.metrics, text)
    return 0


def cli_main(argv=None) -> int:
    parser = build_parser()
    try:
        a = parser.parse_args(argv)
        return {"image": _image, "video": _video}.get(a.command, _bench)(a)
    except _UsageError as e:
        parser.print_usage(sys.stderr)
        print(f"vidcarve: error: {e}", file=sys.stderr)
        return 1
    except SystemExit as e:  # --help
        return 0 if e.code in (None, 0) else int(e.code)
    except (MediaFormatError, OSError) as e:
        print(f"vidcarve: error: {e}", file=sys.stderr)
        return 2
    except ValueError as e:
        print(f"vidcarve: error: {e}", file=sys.stderr)
        return 1


def main() -> None:
    sys.exit(cli_main())


if __name__ == "__main__":
    main()
