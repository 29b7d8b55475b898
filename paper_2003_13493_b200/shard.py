"""Host-side frame sharding across GPUs (SURVEY §8 e).

Frames are independent: no cell reduction crosses frames, so a batch splits
into contiguous frame ranges, one per rank, with no collective on the data
path. This module holds the two host pieces of that scheme:

* :func:`shard_range` -- rank r of W detects frames [start, start + count);
* :func:`gather_features` -- rank 0 collects every rank's per-frame counts
  and feature lists into one array ordered by global frame index (disjoint
  slots; used after detection, outside any timed region).

Works with any torch.distributed backend (gloo on CPU tensors, NCCL on CUDA
tensors).
"""
from __future__ import annotations

import numpy as np

FEATURE_WORDS = 6  # flk_feature = 6 x 32-bit


def shard_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced split: the first total % world ranks get one extra."""
    if world < 1 or not 0 <= rank < world or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, base + (1 if rank < extra else 0)


def gather_features(counts: np.ndarray, feats: np.ndarray, total: int, device=None):
    """All ranks call; rank 0 returns (counts[total], feats[total, cap]) in
    global frame order, other ranks return None.

    counts: int32[n_local]; feats: structured FEATURE_DTYPE or int32 array of
    shape [n_local, cap] (cap = grid cells per frame, equal on all ranks).
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size()
    rank = dist.get_rank()
    n_local = counts.shape[0]
    cap = feats.shape[1] if feats.ndim == 2 else 0
    raw = np.ascontiguousarray(feats).view(np.int32).reshape(n_local, cap * FEATURE_WORDS)
    max_local = shard_range(total, 0, world)[1]
    dev = device if device is not None else torch.device("cpu")
    c = torch.zeros(max_local, dtype=torch.int32, device=dev)
    f = torch.zeros((max_local, cap * FEATURE_WORDS), dtype=torch.int32, device=dev)
    c[:n_local] = torch.from_numpy(np.ascontiguousarray(counts, dtype=np.int32)).to(dev)
    f[:n_local] = torch.from_numpy(raw).to(dev)
    cs = [torch.empty_like(c) for _ in range(world)]
    fs = [torch.empty_like(f) for _ in range(world)]
    dist.all_gather(cs, c)
    dist.all_gather(fs, f)
    if rank != 0:
        return None
    out_c = np.zeros(total, np.int32)
    out_f = np.zeros((total, cap * FEATURE_WORDS), np.int32)
    for r in range(world):
        start, n = shard_range(total, r, world)
        out_c[start:start + n] = cs[r][:n].cpu().numpy()
        out_f[start:start + n] = fs[r][:n].cpu().numpy()
    return out_c, out_f
