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
