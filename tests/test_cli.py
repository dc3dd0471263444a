"""`vidcarve` CLI drop-in (cli.py:1-232): usage errors and exit codes on CPU; the GPU commands
against the reference's outputs (small.json: clip frames, cli_bench metrics)."""
import io
import json
import os

import numpy as np
import pytest

import cases
from paper_1903_03180_b200.cli import cli_main

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "small.json")


@pytest.mark.parametrize("argv,msg", [
    (["video", "a", "b"], "one of --width or --scale is required"),
    (["video", "a", "b", "--width", "3", "--scale", "0.5"], "--width and --scale are mutually exclusive"),
    (["video", "a", "b", "--scale", "1.5"], "--scale must be in (0, 1], got 1.5"),
    (["image", "a", "b", "--width", "3", "--mode", "nope"], "invalid choice"),
    (["bench", "static", "--width", "3", "--size", "3by3"], "--size must look like 320x240"),
])
def test_usage_errors_exit_1(argv, msg, capsys):
    assert cli_main(argv) == 1
    assert msg in capsys.readouterr().err


def test_missing_input_exit_2(tmp_path, capsys):
    assert cli_main(["video", str(tmp_path / "none.ppm"), str(tmp_path / "o.ppm"), "--scale", "0.5"]) == 2
    assert "no such file or directory" in capsys.readouterr().err
    bad = tmp_path / "bad.ppm"
    bad.write_bytes(b"P3 1 1 255\n0")
    assert cli_main(["video", str(bad), str(tmp_path / "o.ppm"), "--scale", "0.5"]) == 2
    assert "bad magic" in capsys.readouterr().err


@pytest.mark.gpu
def test_video_and_image_commands(tmp_path):
    from paper_1903_03180_b200 import media
    small = json.load(open(GOLD))
    ck, cfg = cases.CLIP_CASES["buf_w"]
    frames = cases.small_clip(**ck)
    src, dst, rep = tmp_path / "in.ppm", tmp_path / "out.ppm", tmp_path / "m.txt"
    media.write_frames(src, frames)
    assert cli_main(["video", str(src), str(dst), "--width", str(cfg["target_width"]), "--metrics", str(rep)]) == 0
    out = list(media.read_frames(dst))
    assert [cases.sha(f) for f in out] == small["clips"]["buf_w"]["frames"]
    kv = dict(line.split("=") for line in rep.read_text().split())
    assert int(kv["dp_passes"]) == small["clips"]["buf_w"]["dp_passes"] and "jitter" in kv
    img = tmp_path / "one.ppm"
    media.write_frames(img, frames[:1])
    assert cli_main(["image", str(img), str(tmp_path / "o1.ppm"), "--scale", "0.75"]) == 0


@pytest.mark.gpu
def test_bench_command_matches_reference(capsys):
    small = json.load(open(GOLD))
    for kind, per_mode in small["cli_bench"].items():
        assert cli_main(["bench", kind, "--width", "30", "--size", "40x30", "--frames", "9", "--seed", "2"]) == 0
        kv = dict(line.split("=") for line in capsys.readouterr().out.split())
        for mode, g in per_mode.items():
            assert int(kv[f"{mode}.dp_passes"]) == g["dp_passes"], (kind, mode)
            assert int(kv[f"{mode}.frames_out"]) == g["frames_out"]
            assert kv[f"{mode}.jitter"] == g["jitter"], (kind, mode)
