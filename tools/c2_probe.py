"""C2 single-frame latency breakdown: the device timeline of flk_detector_run
(H2D, kernels, D2H) from the CUDA activity trace (torch.profiler / CUPTI),
beside the host wall time per call.

    python tools/c2_probe.py            (on a GPU box)
"""
import ctypes
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def session_timeline():
    """Same trace for the tracking session (flk_session_process per frame)."""
    from torch.profiler import ProfilerActivity, profile

    import bench
    import paper_2003_13493_b200 as fl
    frames = bench.session_frames(0)
    lib = fl.load_library()
    imgs = [fl.Image.from_array(f) for f in frames]
    th = ctypes.c_void_p()
    s = fl.Session(fl.Config(**bench.SESSION_CFG))
    ts = []
    for im in imgs[:8]:
        assert lib.flk_session_process(s.handle, im.handle, ctypes.byref(th), None, None) == 0
        lib.flk_tracks_destroy(th)
    for im in imgs[8:]:
        t0 = time.perf_counter()
        assert lib.flk_session_process(s.handle, im.handle, ctypes.byref(th), None, None) == 0
        ts.append(time.perf_counter() - t0)
        lib.flk_tracks_destroy(th)
    print("session host wall per frame: median %.1f us" % (np.median(ts) * 1e6))
    s = fl.Session(fl.Config(**bench.SESSION_CFG))
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for im in imgs[:12]:
            assert lib.flk_session_process(s.handle, im.handle, ctypes.byref(th), None, None) == 0
            lib.flk_tracks_destroy(th)
    dump(prof, 4)


def dump(prof, last):
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    evs.sort(key=lambda e: e.time_range.start)
    calls, cur, last_end = [], [], None
    for e in evs:
        if last_end is not None and e.time_range.start - last_end > 15:
            calls.append(cur)
            cur = []
        cur.append(e)
        last_end = max(last_end or 0, e.time_range.end)
    calls.append(cur)
    for c in calls[-last:]:
        t0 = c[0].time_range.start
        print("--- call: device span %.1f us" % (max(e.time_range.end for e in c) - t0))
        for e in c:
            print("  %7.1f +%6.1f us  %s" % (e.time_range.start - t0, e.time_range.end - e.time_range.start,
                                            e.name[:70]))


def main():
    if "--session" in sys.argv:
        return session_timeline()
    import torch
    from torch.profiler import ProfilerActivity, profile

    import bench
    import paper_2003_13493_b200 as fl

    det = fl.Detector(fl.Config(**bench.CFG), device=0)
    img = fl.Image.from_array(np.ascontiguousarray(
        torch.empty((bench.H, bench.W), dtype=torch.uint8).random_(0, 256).numpy()))
    lib = fl.load_library()
    fh = ctypes.c_void_p()

    def call():
        assert lib.flk_detector_run(det.handle, img.handle, ctypes.byref(fh), None, None) == 0
        lib.flk_features_destroy(fh)

    for _ in range(50):
        call()
    ts = []
    for _ in range(300):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    print("host wall per call: median %.1f us, p5 %.1f, p95 %.1f" %
          tuple(np.percentile(np.array(ts) * 1e6, [50, 5, 95])))

    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        for _ in range(20):
            call()
    dump(prof, 3)


if __name__ == "__main__":
    main()
