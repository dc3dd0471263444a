"""Frame ingestion and emission, feeding the GPU path from pinned memory.

Same sources, sinks and byte grammar as the reference's `vidcarve.media`
(pkg/src/vidcarve/media.py:1-252): single PPM (P6) / PGM (P5) / PNG files, directories of
numbered image files, and concatenated binary PNM streams (`"-"` = stdin/stdout, or any
binary file object). Header tokens are whitespace separated, `#` comments run to the end
of the line, maxval must be 255, one whitespace byte precedes the payload. Errors raise
MediaFormatError with the reference's messages and frame indices.

GPU additions: `read_clip_pinned` decodes a whole stream straight into one
pinned host tensor (payloads are read in place with `readinto`, no per-frame copies), which
`retarget_video` then streams to the device in chunks overlapped with the energy pass and
the scan; `write_clip` emits P6/P5 records from a (pinned) output tensor without copies;
`retarget_stream` is the `vidcarve video - -` pipe on the GPU.
"""

from __future__ import annotations

import re
import sys
from pathlib import Path
from typing import BinaryIO, Iterable, Iterator

import numpy as np

IMAGE_SUFFIXES = (".ppm", ".pgm", ".png")
_SPACE = frozenset(b" \t\r\n\x0b\x0c")


class MediaFormatError(Exception):
    """Malformed or unsupported media data."""


# ------------------------------------------------------------------ PNM records
class _PnmReader:
    """Tokenises PNM headers from a binary stream, one byte at a time (the payload that follows
    a header must start exactly after the single delimiter byte, so no read-ahead)."""

    def __init__(self, stream: BinaryIO, label: str):
        self.stream, self.label = stream, label

    def _fail(self, idx: int, what: str) -> MediaFormatError:
        return MediaFormatError(f"{self.label}, frame {idx}: {what}")

    def token(self, idx: int, at_start: bool = False) -> bytes | None:
        out = bytearray()
        read = self.stream.read
        while True:
            c = read(1)
            if not c:
                if out:
                    return bytes(out)
                if at_start:
                    return None
                raise self._fail(idx, "malformed header, unexpected end of data")
            b = c[0]
            if b in _SPACE:
                if out:
                    return bytes(out)
            elif b == 0x23 and not out:  # '#': comment to end of line
                while c and c != b"\n":
                    c = read(1)
            else:
                out += c

    def integer(self, idx: int, what: str) -> int:
        tok = self.token(idx)
        try:
            return int(tok)
        except ValueError:
            raise self._fail(idx, f"malformed header, bad {what} {tok!r}") from None

    def header(self, idx: int):
        """(height, width, channels) of the next record, or None at a clean end of data."""
        magic = self.token(idx, at_start=True)
        if magic is None:
            return None
        if magic not in (b"P6", b"P5"):
            raise self._fail(idx, f"bad magic {magic!r}, expected P6 or P5")
        width = self.integer(idx, "width")
        height = self.integer(idx, "height")
        maxval = self.integer(idx, "maxval")
        if width < 1 or height < 1:
            raise self._fail(idx, f"bad dimensions {width}x{height}")
        if maxval != 255:
            raise self._fail(idx, f"unsupported maxval {maxval}, need 255")
        return height, width, (3 if magic == b"P6" else 1)

    def payload_into(self, idx: int, view: memoryview) -> None:
        """Fill `view` from the stream (short reads retried); truncation is an error."""
        need, got = len(view), 0
        readinto = getattr(self.stream, "readinto", None)
        while got < need:
            if readinto is not None:
                n = readinto(view[got:])
            else:
                chunk = self.stream.read(need - got)
                n = len(chunk)
                view[got:got + n] = chunk
            if not n:
                break
            got += n
        if got < need:
            raise self._fail(idx, f"truncated payload, need {need} bytes, got {got}")


def _pnm_frames(stream: BinaryIO, label: str = "stream") -> Iterator[np.ndarray]:
    rd = _PnmReader(stream, label)
    idx = 0
    while (hdr := rd.header(idx)) is not None:
        h, w, c = hdr
        arr = np.empty((h, w, c) if c == 3 else (h, w), dtype=np.uint8)
        rd.payload_into(idx, memoryview(arr).cast("B"))
        yield arr
        idx += 1


def _pnm_bytes_header(h: int, w: int, rgb: bool) -> bytes:
    return (b"P6" if rgb else b"P5") + f"\n{w} {h}\n255\n".encode("ascii")


def _pnm_record(frame: np.ndarray, force_rgb: bool = False) -> bytes:
    a = np.ascontiguousarray(np.asarray(frame, dtype=np.uint8))
    if a.ndim == 2 and force_rgb:
        a = np.repeat(a[:, :, None], 3, axis=2)
    if a.ndim == 3 and a.shape[2] != 3:
        raise MediaFormatError(f"cannot encode frame with {a.shape[2]} channels")
    if a.ndim not in (2, 3):
        raise MediaFormatError(f"cannot encode array of shape {a.shape}")
    return _pnm_bytes_header(a.shape[0], a.shape[1], a.ndim == 3) + a.tobytes()


# ------------------------------------------------------------------ sources / sinks
def _sort_key(path: Path):
    """Numbered files in number order (last number of the stem), unnumbered ones after."""
    m = re.findall(r"\d+", path.stem)
    return (0, int(m[-1]), path.name) if m else (1, 0, path.name)


def _png_frame(path: Path) -> np.ndarray:
    try:
        from PIL import Image
    except ImportError as e:  # pragma: no cover
        raise MediaFormatError(f"PNG support needs Pillow: {path}") from e
    with Image.open(path) as img:
        return np.asarray(img if img.mode == "L" else img.convert("RGB"), dtype=np.uint8)


def _file_frames(path: Path) -> Iterator[np.ndarray]:
    ext = path.suffix.lower()
    if ext == ".png":
        yield _png_frame(path)
    elif ext in (".ppm", ".pgm"):
        with open(path, "rb") as fh:
            yield from _pnm_frames(fh, label=str(path))
    else:
        raise MediaFormatError(f"unsupported image format: {path}")


def _source_frames(source) -> Iterator[np.ndarray]:
    if source == "-":
        yield from _pnm_frames(sys.stdin.buffer)
    elif hasattr(source, "read"):
        yield from _pnm_frames(source)
    else:
        path = Path(source)
        if path.is_dir():
            for f in sorted((p for p in path.iterdir() if p.suffix.lower() in IMAGE_SUFFIXES), key=_sort_key):
                yield from _file_frames(f)
        elif not path.exists():
            raise FileNotFoundError(f"no such file or directory: {path}")
        else:
            yield from _file_frames(path)


def read_frames(source: str | Path | BinaryIO) -> Iterator[np.ndarray]:
    """Frames of a file, directory or stream in index order (media.py:33-44)."""
    shape = None
    for idx, f in enumerate(_source_frames(source)):
        if shape is None:
            shape = f.shape[:2]
        elif f.shape[:2] != shape:
            raise MediaFormatError(f"frame {idx}: dimension change mid-stream, "
                                   f"expected {shape[1]}x{shape[0]}, got {f.shape[1]}x{f.shape[0]}")
        yield f


def _stream_out(stream: BinaryIO, frames: Iterable[np.ndarray]) -> None:
    for f in frames:
        stream.write(_pnm_record(f, force_rgb=True))
        stream.flush()


def write_frames(sink: str | Path | BinaryIO, frames: Iterable[np.ndarray]) -> None:
    """Frames to a stream (P6 records, gray promoted), a .ppm/.pgm file (concatenated
    records), a .png file (exactly one frame) or a directory of numbered files (media.py:47-79)."""
    if sink == "-":
        return _stream_out(sys.stdout.buffer, frames)
    if hasattr(sink, "write"):
        return _stream_out(sink, frames)
    path = Path(sink)
    ext = path.suffix.lower()
    if ext == ".png":
        frames = list(frames)
        if len(frames) != 1:
            raise MediaFormatError(f"PNG sink {path} holds exactly one frame, got {len(frames)}")
        a = np.ascontiguousarray(np.asarray(frames[0], dtype=np.uint8))
        if a.ndim not in (2, 3) or (a.ndim == 3 and a.shape[2] != 3):
            raise MediaFormatError(f"cannot encode array of shape {a.shape}")
        from PIL import Image
        Image.fromarray(a).save(path, format="PNG")
    elif ext in (".ppm", ".pgm"):
        with open(path, "wb") as fh:
            for f in frames:
                fh.write(_pnm_record(f, force_rgb=ext == ".ppm"))
    else:
        path.mkdir(parents=True, exist_ok=True)
        for idx, f in enumerate(frames):
            a = np.asarray(f)
            with open(path / (f"frame_{idx:05d}" + (".ppm" if a.ndim == 3 else ".pgm")), "wb") as fh:
                fh.write(_pnm_record(a))


# ------------------------------------------------------------------ pinned GPU feed
def read_clip_pinned(source: str | Path | BinaryIO, capacity: int = 64):
    """A PNM stream / file decoded straight into one pinned host tensor (T, H, W[, 3]).

    Payloads land in pinned memory via readinto (no intermediate copies); the tensor grows
    by doubling. Validation and messages are read_frames'. Non-PNM sources fall back to
    read_frames and one copy per frame.
    """
    import torch
    if (source != "-" and not hasattr(source, "read")
            and (Path(source).is_dir() or Path(source).suffix.lower() not in (".ppm", ".pgm")
                 or not Path(source).exists())):
        frames = list(read_frames(source))  # directories, PNG, missing paths: read_frames' behaviour
        if not frames:
            return torch.empty((0,), dtype=torch.uint8)
        return torch.from_numpy(np.stack(frames)).pin_memory()
    own = None
    if source == "-":
        stream, label = sys.stdin.buffer, "stream"
    elif hasattr(source, "read"):
        stream, label = source, "stream"
    else:
        stream = own = open(source, "rb")
        label = str(source)
    try:
        rd = _PnmReader(stream, label)
        buf, shape, t = None, None, 0
        while (hdr := rd.header(t)) is not None:
            h, w, c = hdr
            fshape = (h, w, 3) if c == 3 else (h, w)
            if shape is None:
                shape = fshape
                buf = torch.empty((capacity,) + fshape, dtype=torch.uint8, pin_memory=True)
            elif fshape[:2] != shape[:2]:
                raise MediaFormatError(f"frame {t}: dimension change mid-stream, "
                                       f"expected {shape[1]}x{shape[0]}, got {w}x{h}")
            elif fshape != shape:
                raise MediaFormatError(f"frame {t}: channel count change mid-stream")
            if t == buf.shape[0]:
                grown = torch.empty((2 * t,) + shape, dtype=torch.uint8, pin_memory=True)
                grown[:t].copy_(buf)
                buf = grown
            rd.payload_into(t, memoryview(buf[t].numpy()).cast("B"))
            t += 1
        if buf is None:
            return torch.empty((0,), dtype=torch.uint8)
        return buf[:t]
    finally:
        if own is not None:
            own.close()


def write_clip(sink: str | Path | BinaryIO, clip) -> None:
    """P6 (or P5 for gray files) records of a (T, H, W[, 3]) host tensor / array, written
    from its memory without copies (gray frames are promoted to RGB on streams, as write_frames)."""
    arr = clip.numpy() if hasattr(clip, "numpy") else np.asarray(clip)
    is_stream = sink == "-" or hasattr(sink, "write")
    if not is_stream and Path(sink).suffix.lower() != ".ppm":
        return write_frames(sink, list(arr))
    if arr.ndim == 3 and is_stream:  # gray stream: P6 has no gray form
        return write_frames(sink, list(arr))
    own = None
    stream = sys.stdout.buffer if sink == "-" else (sink if is_stream else None)
    if stream is None:
        stream = own = open(sink, "wb")
    try:
        for f in arr:
            stream.write(_pnm_bytes_header(f.shape[0], f.shape[1], f.ndim == 3))
            stream.write(memoryview(np.ascontiguousarray(f)).cast("B"))
            if is_stream:
                stream.flush()
    finally:
        if own is not None:
            own.close()


def retarget_stream(source, sink, config):
    """`vidcarve video SRC DST` on the GPU: decode into pinned memory, retarget (chunked H2D
    overlapped with the energy pass and scan, per-run D2H), write the records."""
    from .pipeline import retarget_video
    clip = read_clip_pinned(source)
    if clip.numel() == 0:
        return [], None
    out, metrics = retarget_video(clip, config)
    write_clip(sink, out)
    return out, metrics


__all__ = ["IMAGE_SUFFIXES", "MediaFormatError", "read_frames", "write_frames", "read_clip_pinned", "write_clip",
           "retarget_stream"]
