"""bench.py keeps the driver's contract: one JSON line with the required keys
(the reference arm on CPU here; our arm on a GPU box, at a small batch)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libfastlk_ref.so")


def run_bench(*args, timeout=600, torchrun=0):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), *args]
    if torchrun:
        import socket
        so = socket.socket()
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
        so.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={torchrun}", "--master-addr", "127.0.0.1",
               "--master-port", str(port), os.path.join(ROOT, "bench.py"), *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def common_keys(d):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e"):
        assert k in d, k
    assert d["unit"] == "frames/s" and d["higher_is_better"] is True
    assert d["config"]["workload"].startswith("C4")
    assert d["value"] > 0 and d["e2e"]["value"] > 0
    for k in ("unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"]


def test_reference_arm_line():
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built")
    d = run_bench("--impl", "reference", "--steps", "1", "--warmup", "1")
    common_keys(d)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0


@pytest.mark.gpu
def test_our_arm_line():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = run_bench("--steps", "3", "--warmup", "3", "--global-batch", "1024", "--e2e-steps", "2",
                  "--no-extras", "--no-cpu-baseline")
    common_keys(d)
    assert d["scaling"] == "strong" and d["config"]["global_batch"] == 1024
    assert d["parity"]["frames"] == 1024 and d["parity"]["mismatches"] == 0
    assert d["e2e"]["results_equal_device_path"] is True
    assert d["e2e_handles"]["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s"
    assert 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["traffic"] is None or r["traffic"] > 0
    assert d["gpu_launches"] >= 3 * 3  # steps x (k_detect launches + compaction)
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert 0 < d["pyramid_roofline"]["frac"] < 1.05
    assert d["dtype"] == "u8" and d["n_gpus"] == 1


def test_both_arms_share_the_config():
    """The driver compares the two arms' `config`: same keys, same values."""
    import bench
    import argparse
    a = argparse.Namespace(batch=0, global_batch=4096)
    assert bench.bench_config(a, 1) == bench.bench_config(a, 8)
    assert set(bench.bench_config(a, 1)) == {"workload", "global_batch"}


@pytest.mark.gpu
def test_torchrun_two_ranks_match_one_rank():
    """C4's N>1 path on a one-GPU box: two ranks under torchrun,
    both on cuda:0 (--same-device), each detecting its contiguous shard of a
    512-frame global batch; the gathered per-frame results are bit-identical
    to the one-rank run and to the reference build on every frame."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    args = ("--steps", "2", "--warmup", "3", "--global-batch", "512", "--e2e-steps", "1",
            "--no-extras", "--no-cpu-baseline")
    one = run_bench(*args)
    two = run_bench("--gpus", "2", "--same-device", *args, torchrun=2)
    assert two["n_gpus"] == 2 and two["frames_per_rank"] == [256, 256]
    assert len(two["frames_per_s_per_rank"]) == 2 and min(two["frames_per_s_per_rank"]) > 0
    assert one["parity"]["mismatches"] == 0 and two["parity"]["mismatches"] == 0
    assert two["parity"]["frames"] == 512
    assert two["parity"]["digest_sha256"] == one["parity"]["digest_sha256"]
    assert two["config"] == one["config"]
    # weak scaling: 128 frames per rank
    w = run_bench("--gpus", "2", "--same-device", "--batch", "128", *args[:6],
                  "--no-extras", "--no-cpu-baseline", torchrun=2)
    assert w["scaling"] == "weak" and w["parity"]["frames"] == 256
    assert w["parity"]["mismatches"] == 0
