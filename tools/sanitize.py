#!/usr/bin/env python
"""Small representative runs for compute-sanitizer (memcheck / racecheck /
synccheck / initcheck): the fused detector (both pyramid plans, radius 1-3,
every score kind, unaligned pitch, multi-round corner lists, a chunked device
batch), the staged kernels, the conformance kernels and a short tracking
session. Checks parity
with the oracle on each so a sanitizer run is also a correctness run.

    compute-sanitizer --tool racecheck python tools/sanitize.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import numpy as np  # noqa: E402

import oracle  # noqa: E402
import paper_2003_13493_b200 as fl  # noqa: E402
import sessions  # noqa: E402
import synth  # noqa: E402


def main():
    orc = oracle.load_oracle()
    cases = [
        (synth.texture(1, 256, 160), dict(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=8, n=1), "1"),
        (synth.noise(2, 200, 120), dict(epsilon=10, N=12, score_kind="mt", l=2, w=1, h=16, n=2), "0"),
        (synth.texture(3, 193, 97), dict(epsilon=5, N=10, score_kind="sad_a", l=2, w=2, h=4, n=3), "1"),
        (synth.noise(4, 160, 96), dict(epsilon=0, N=9, score_kind="sad_b", l=1, w=1, h=32, n=1), "0"),
    ]
    for img, cfg, fuse in cases:
        det = fl.Detector(fl.Config(**cfg), plan={"fuse_pyramid": int(fuse)})
        feats, extra = det.run(img, stats=True, conformance=True)
        ref, st = orc.detect(img, oracle.make_params(**cfg))
        assert (feats == ref).all() and extra["stats"]["nms_comparisons"] == st.comparisons
        assert (det.run(img) == ref).all()
        maps = det.responses(img, cfg["l"])
        fmaps = det.responses(img, cfg["l"], fused=True)  # the fused kernel's own score tiles
        for a, b, c in zip(maps, fmaps, orc.responses(img, oracle.make_params(**cfg))):
            assert (a == c).all() and (b == c).all()
    img = synth.noise(5, 200, 120)  # multi-round corner lists
    cfg = dict(epsilon=0, N=9, score_kind="sad_b", l=2, w=1, h=16, n=1)
    feats = fl.Detector(fl.Config(**cfg), plan={"list_cap": 256}).run(img)
    assert (feats == orc.detect(img, oracle.make_params(**cfg))[0]).all()
    # a device batch in the chunked two-launch plan (side-stream level 1-2
    # launches) and its GPU conformance tally
    import torch
    W, H, n = 256, 160, 8
    cfg = dict(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=8, n=1)
    batch = fl.DeviceBatch(fl.Detector(fl.Config(**cfg), plan={"fuse_pyramid": 1,
                                                               "pyramid_chunk": 3}), W, H, n)
    d = torch.empty((n, H, W), dtype=torch.uint8, device="cuda")
    fl.synth_frames_device(d.data_ptr(), 1, 40, n, W, H, W, W * H)
    batch.run_device(d.data_ptr(), W * H, W, n)
    torch.cuda.synchronize()
    res = batch.results(n)
    for f in (0, n - 1):
        assert (res[f] == orc.detect(synth.texture(40 + f, W, H), oracle.make_params(**cfg))[0]).all()
    total, _ = batch.conformance(d.data_ptr(), W * H, W, 0, n)
    assert total["false_positives"] == 0 and total["matched"] == sum(len(r) for r in res)
    # host batches through the multi-device entry point (device 0 twice)
    hb = [synth.texture(60 + f, 256, 160) for f in range(5)]
    # initcheck does not follow cudaMemcpyBatchAsync (tools/probes/batchcopy_initcheck.cu):
    # under it (SANITIZE_TOOL=initcheck) the host batches copy frame by frame
    per_frame = os.environ.get("SANITIZE_TOOL") == "initcheck"
    d2 = fl.Detector(fl.Config(**cfg), plan={"batch_copies": 0} if per_frame else None)
    d1 = fl.Detector(fl.Config(**cfg), plan={"batch_copies": 0} if per_frame else None)
    for a, b in zip(d2.run_batch_multi(hb, [0, 0]), d1.run_batch(hb)):
        assert (a == b).all()
    frames = sessions.drifting_sequence(3, 192, 128)
    scfg = dict(epsilon=10, N=9, score_kind="sad_b", l=2, w=1, h=16, n=1, target_count=12,
                redetect_ratio=0.5, param_mode="full", max_iterations=30, convergence_epsilon=0.01)
    sessions.run_capi_session(fl.load_library(), scfg, frames)
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
