"""A plain C program against the drop-in ABI (examples/detect_pgm.c): builds
with the C compiler against include/fastlk.h and libfastlk_b200.so; on a GPU
box its output is the oracle's feature list, on CPU it fails with
FLK_E_INTERNAL (no CPU fallback)."""
import os
import subprocess

import numpy as np
import pytest

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2003_13493_b200")


@pytest.fixture(scope="module")
def binary(tmp_path_factory):
    if not os.path.exists(os.path.join(LIBDIR, "libfastlk_b200.so")):
        pytest.skip("library not built")
    out = str(tmp_path_factory.mktemp("cex") / "detect_pgm")
    subprocess.run(["cc", "-std=c11", "-Wall", "-Wextra", "-Werror", f"-I{ROOT}/include",
                    f"{ROOT}/examples/detect_pgm.c", f"-L{LIBDIR}", "-lfastlk_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    return out


def frame_pgm(tmp_path):
    img = synth.texture(21, 320, 240)
    p = tmp_path / "f.pgm"
    p.write_bytes(b"P5\n320 240\n255\n" + img.tobytes())
    return img, p


def test_c_example_without_gpu(binary, tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    _, p = frame_pgm(tmp_path)
    r = subprocess.run([binary, str(p), "l=2", "h=16"], capture_output=True, text=True)
    assert r.returncode == 5 and "no CPU fallback" in r.stderr  # FLK_E_INTERNAL
    r = subprocess.run([binary, str(p), "N=20"], capture_output=True, text=True)
    assert r.returncode == 1  # FLK_E_INVALID_ARG at create, before any device work
    r = subprocess.run([binary, str(p), "bogus=1"], capture_output=True, text=True)
    assert r.returncode == 4  # FLK_E_CONFIG


@pytest.mark.gpu
def test_c_example_matches_oracle(binary, tmp_path, orc):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    img, p = frame_pgm(tmp_path)
    r = subprocess.run([binary, str(p), "l=2", "h=16", "N=10", "score_kind=mt"],
                       capture_output=True, text=True, check=True)
    rows = [list(map(int, l.split())) for l in r.stdout.splitlines() if not l.startswith("#")]
    ref, st = orc.detect(img, oracle.make_params(N=10, score_kind="mt", l=2, h=16))
    got = np.array(rows)
    assert len(got) == len(ref)
    for k, name in enumerate(("x", "y", "score", "level", "cell_x", "cell_y")):
        assert (got[:, k] == ref[name].astype(np.int64)).all()
    assert f"candidates={st.candidates} comparisons={st.comparisons}" in r.stdout
