"""PNM ingestion/emission (media.py) against the reference's own outcomes (tests/golden/small.json
"media": frames or the exact MediaFormatError message, and the bytes write_frames emits)."""
import io
import json
import os

import numpy as np
import pytest

import cases
from paper_1903_03180_b200 import media

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "small.json")


sha = cases.sha


@pytest.fixture(scope="module")
def gold():
    return json.load(open(GOLD))["media"]


@pytest.mark.parametrize("name,data", cases.media_streams(), ids=[n for n, _ in cases.media_streams()])
def test_read_write_frames_match_reference(gold, name, data):
    g = gold[name]
    if "error" in g:
        with pytest.raises(media.MediaFormatError) as ei:
            list(media.read_frames(io.BytesIO(data)))
        assert str(ei.value) == g["message"]
        return
    fr = list(media.read_frames(io.BytesIO(data)))
    assert [sha(f) for f in fr] == g["frames"]
    assert [list(f.shape) for f in fr] == g["shapes"]
    buf = io.BytesIO()
    media.write_frames(buf, fr)
    got = sha(np.frombuffer(buf.getvalue(), np.uint8)) if fr else None
    assert got == g["written"]


def test_files_and_directories(tmp_path):
    rng = np.random.default_rng(3)
    frames = [rng.integers(0, 256, (6, 9, 3), dtype=np.uint8) for _ in range(3)]
    media.write_frames(tmp_path / "clip.ppm", frames)
    assert all(np.array_equal(a, b) for a, b in zip(media.read_frames(tmp_path / "clip.ppm"), frames))
    media.write_frames(tmp_path / "dir", frames)
    names = sorted(p.name for p in (tmp_path / "dir").iterdir())
    assert names == ["frame_00000.ppm", "frame_00001.ppm", "frame_00002.ppm"]
    assert all(np.array_equal(a, b) for a, b in zip(media.read_frames(tmp_path / "dir"), frames))
    with pytest.raises(FileNotFoundError):
        list(media.read_frames(tmp_path / "missing.ppm"))
    with pytest.raises(media.MediaFormatError):
        list(media.read_frames(tmp_path / "x.txt")) if (tmp_path / "x.txt").write_bytes(b"x") else None
