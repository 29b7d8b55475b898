"""flkb_detector_run_batch throughput on host images (flk_image handles):
the raw C-ABI call (results freed unread) and the Python mirror (results as
arrays)."""
import ctypes
import sys
import time
sys.path[:0] = [".", "tests"]
import synth  # noqa: E402
import paper_2003_13493_b200 as fl  # noqa: E402
import bench  # noqa: E402

frames = [synth.texture(i, 752, 480) for i in range(1024)]
imgs = [fl.Image.from_array(f) for f in frames]
det = fl.Detector(fl.Config(**bench.CFG))
lib = fl.load_library()
det.run_batch(imgs[:64])
for n in (64, 1024):
    arr = (ctypes.c_void_p * n)(*[i.handle.value for i in imgs[:n]])
    outs = (ctypes.c_void_p * n)()
    t0 = time.perf_counter()
    for _ in range(3):
        assert lib.flkb_detector_run_batch(det.handle, arr, n, outs, None) == 0
        for i in range(n):
            lib.flk_features_destroy(ctypes.c_void_p(outs[i]))
    dt = (time.perf_counter() - t0) / 3
    t0 = time.perf_counter()
    det.run_batch(imgs[:n])
    dp = time.perf_counter() - t0
    print(f"run_batch n={n}: C ABI {n / dt:.0f} frames/s, Python mirror {n / dp:.0f} frames/s")
