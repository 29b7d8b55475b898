"""The sequence harness (paper_2003_13493_b200/cli/fastlk_cli.cpp, SURVEY §8(f)
f4): PGM ingest -> detect / track CSV through the C ABI.

The same harness source is also linked against the reference build
(oracle/_ref/fastlk_cli_ref, `make -C oracle cli`): on a GPU box both binaries
must write byte-identical CSVs for the same frames and options. On CPU the
argument handling and exit codes are checked, and the product binary must
refuse to run without a GPU (no CPU fallback).
"""
import os
import subprocess

import numpy as np
import pytest

import sessions
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OURS = os.path.join(ROOT, "paper_2003_13493_b200", "fastlk_b200")
REF = os.path.join(ROOT, "oracle", "_ref", "fastlk_cli_ref")


def write_pgm(path, img):
    h, w = img.shape
    with open(path, "wb") as fh:
        fh.write(b"P5\n%d %d\n255\n" % (w, h) + np.ascontiguousarray(img).tobytes())


@pytest.fixture(scope="module")
def seq_dir(tmp_path_factory):
    d = tmp_path_factory.mktemp("seq")
    for i, f in enumerate(sessions.sliding_sequence(6, 320, 240, step=3)):
        write_pgm(d / f"frame_{i:04d}.pgm", f)
    # not a frame: ignored by the harness
    (d / "notes.txt").write_text("x")
    return d


def run(binary, *args, cwd=None):
    return subprocess.run([binary, *map(str, args)], capture_output=True, text=True, cwd=cwd,
                          timeout=300)


def need(binary):
    if not os.path.exists(binary):
        pytest.skip(f"{binary} not built")


def test_argument_errors(tmp_path):
    need(OURS)
    assert run(OURS).returncode == 1
    assert run(OURS, "--help").returncode == 0
    assert run(OURS, "frobnicate", tmp_path).returncode == 1
    r = run(OURS, "detect", tmp_path / "missing")
    assert r.returncode == 1 and "not a directory" in r.stderr
    r = run(OURS, "detect", tmp_path)
    assert r.returncode == 1 and "no .pgm frames" in r.stderr
    r = run(OURS, "detect", tmp_path, "--bogus")
    assert r.returncode == 1 and "unknown option" in r.stderr
    r = run(OURS, "detect", tmp_path, "--levels", "x")
    assert r.returncode == 1


def test_reference_harness_writes_the_csv(seq_dir, tmp_path):
    need(REF)
    out = tmp_path / "ref.csv"
    r = run(REF, "detect", seq_dir, "--out", out, "--levels", "2", "--oracle", "--strict")
    assert r.returncode == 0, r.stderr
    lines = out.read_text().splitlines()
    assert lines[0] == "frame,x,y,score,level,cell_x,cell_y"
    assert len(lines) > 6 and lines[1].startswith("0,")
    assert "false_positives: 0" in (tmp_path / "ref.csv.report.txt").read_text()


def test_no_cpu_fallback(seq_dir, tmp_path):
    import torch
    need(OURS)
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    r = run(OURS, "detect", seq_dir, "--out", tmp_path / "o.csv")
    assert r.returncode == 1 and "no CPU fallback" in r.stderr


CASES = [
    ("detect", ["--levels", "3"]),
    ("detect", ["--levels", "2", "--oracle", "--strict"]),
    ("detect", ["--config", "CFG"]),
    ("track", ["--levels", "2"]),  # target 100 > 40 cells: both fail the same way
    ("track", ["--config", "CFG", "--oracle"]),
    ("track", ["--levels", "2", "--sweep", "10,30"]),
]


@pytest.mark.gpu
@pytest.mark.parametrize("cmd,opts", CASES, ids=[f"{c}-{i}" for i, (c, _) in enumerate(CASES)])
def test_csv_identical_to_the_reference_library(seq_dir, tmp_path, cmd, opts):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    need(OURS)
    need(REF)
    cfg = tmp_path / "run.cfg"
    cfg.write_text("epsilon = 12\nN = 10\nscore_kind = mt\nl = 3\nh = 8\ntarget_count = 40\n"
                   "redetect_ratio = 0.6\nparam_mode = translation_gain\n")
    opts = [str(cfg) if o == "CFG" else o for o in opts]
    outs, codes = [], []
    for name, binary in (("ours", OURS), ("ref", REF)):
        out = tmp_path / f"{name}.csv"
        r = run(binary, cmd, seq_dir, "--out", out, *opts)
        codes.append((r.returncode, r.stderr.split(":")[-2].split("(")[0].strip()
                      if r.returncode else ""))
        if r.returncode:
            outs.append(None)
            continue
        if "--sweep" in opts:
            outs.append([(tmp_path / f"{name}.target{t}.csv").read_bytes() for t in (10, 30)])
        else:
            outs.append(out.read_bytes())
    assert codes[0] == codes[1]
    assert outs[0] == outs[1]
