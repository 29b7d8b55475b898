"""Multi-GPU host logic on CPU: frame shards and the rank-0 feature gather
with the gloo backend at world size 2 (the data path has no collective)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2003_13493_b200.shard import FEATURE_WORDS, gather_features, shard_range


@pytest.mark.parametrize("total", [0, 1, 7, 4096, 4097])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shards_cover_every_frame_once(total, world):
    seen = []
    for r in range(world):
        start, n = shard_range(total, r, world)
        seen.extend(range(start, start + n))
    assert seen == list(range(total))
    sizes = [shard_range(total, r, world)[1] for r in range(world)]
    assert max(sizes) - min(sizes) <= 1


def fake_frame(g: int, cap: int):
    """Deterministic per-frame 'detector output' keyed by the global index."""
    n = (g * 7) % (cap + 1)
    f = np.zeros((cap, FEATURE_WORDS), np.int32)
    f[:n] = np.arange(n * FEATURE_WORDS, dtype=np.int32).reshape(n, FEATURE_WORDS) + 1000 * g
    return n, f.reshape(-1)


def _worker(rank, world, port, total, cap, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, n = shard_range(total, rank, world)
    counts = np.zeros(n, np.int32)
    feats = np.zeros((n, cap * FEATURE_WORDS), np.int32)
    for i in range(n):
        counts[i], feats[i] = fake_frame(start + i, cap)
    res = gather_features(counts, feats.view(np.int32).reshape(n, -1).view(
        [("w", np.int32, FEATURE_WORDS)]).reshape(n, cap), total)
    if rank == 0:
        q.put((res[0].tolist(), res[1].tobytes()))
    dist.barrier()
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("total", [9, 64])
def test_gloo_world2_gather(total):
    cap = 12
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, total, cap, q)) for r in range(2)]
    for p in procs:
        p.start()
    counts, raw = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    feats = np.frombuffer(raw, np.int32).reshape(total, cap * FEATURE_WORDS)
    for g in range(total):
        n, f = fake_frame(g, cap)
        assert counts[g] == n
        assert (feats[g] == f).all()


def _detect_worker(rank, world, port, total, q):
    """One rank of the N>1 path with the reference build standing in for the
    GPU (no device here): detect this rank's contiguous shard, then gather."""
    import sys
    import torch.distributed as dist
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import oracle
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    start, n = shard_range(total, rank, world)
    orc, ref = oracle.load_oracle(), oracle.load_reference()
    p = oracle.make_params(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=2, n=1)
    frames = np.stack([orc.synth(1, start + i, 256, 192) for i in range(n)])
    counts, feats = ref.detect_batch(frames, p, workers=1)
    res = gather_features(counts, feats, total)
    if rank == 0:
        q.put((res[0].tolist(), res[1].tobytes()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [5, 12])
def test_gloo_world2_detect_and_gather(total):
    """World size 2 over gloo: each rank detects its shard of S2 frames
    (global frame indices) and rank 0 gathers; the result equals one
    process detecting every frame (bench.py's N>1 parity path)."""
    import oracle
    if oracle.load_reference() is None:
        pytest.skip("reference build unavailable")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_detect_worker, args=(r, 2, port, total, q)) for r in range(2)]
    for p in procs:
        p.start()
    counts, raw = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc, ref = oracle.load_oracle(), oracle.load_reference()
    p = oracle.make_params(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=2, n=1)
    frames = np.stack([orc.synth(1, i, 256, 192) for i in range(total)])
    want_c, want_f = ref.detect_batch(frames, p)
    assert counts == want_c.tolist()
    got = np.frombuffer(raw, np.int32).reshape(total, -1)
    assert (got == np.ascontiguousarray(want_f).view(np.int32).reshape(total, -1)).all()
    assert sum(counts) > 0
