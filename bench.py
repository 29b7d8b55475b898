#!/usr/bin/env python
"""FAST + grid-NMS throughput on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...

Workload (BASELINE configs[3] "C4"): 4096 frames of 752x480 per step over all
ranks, 3-level pyramid, FAST-9 SAD-B, eps=10, 32x32 cells (w=1, h=8), n=1.
Rank r of N detects the contiguous shard shard_range(4096, r, N) (strong
scaling, `--global-batch`); `--batch B` gives B frames per GPU instead (weak
scaling). Frames are independent: no collective on the data path; gloo on CPU
tensors carries the barrier, the max over ranks and the post-run gather of
results. Frames are S2 synthetic texture with global frame indices, generated
on the device; 4096 frames are 1.48 GB, so inputs exceed the 126 MB L2 and
every step streams them from HBM.

value     frames/s over all ranks, inputs resident in HBM, CUDA-event timed,
          max over ranks.
e2e       the same metric through flkb_batch_detect_host from pinned host
          memory: H2D of every frame and D2H of every count and feature list
          inside the timed region (overlapped with the kernels).
e2e_handles  flkb_detector_run_batch over flk_image handles (drop-in-adjacent).
roofline  algorithmic bytes (sum_k w_k*h_k + 16*F per frame) per
          step / device time of the detection kernels, against the measured
          HBM copy bandwidth in MEASURED_PEAKS.json; L2 GB/s from the ncu L2
          bytes per frame.
parity    every frame of the timed batch against the reference build
          (oracle/_ref) run frame-parallel on the same frames, bit-exact.
cpu_baseline  that reference run (frame-parallel over the whole workload) plus
          the as-shipped mode (one threads=0 detector, frames in sequence) on a
          bounded sample; per-stage split from flk_frame_stats; lscpu.
other_configs  C1, C2 (single-frame latency), C3, C5 (on every rank) with their
          roofline fractions and CPU baselines; the tracking session (F12).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

W, H, LEVELS = 752, 480, 3
PITCH = 768
CFG = dict(epsilon=10, N=9, score_kind="sad_b", l=3, w=1, h=8, n=1)
METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
WORKLOAD = ("C4: 752x480, l=3, FAST-9 sad_b eps=10, 32x32 cells (w=1,h=8), n=1; "
            "BASELINE configs[3]")


def level_pixels():
    w, h, s = W, H, 0
    for _ in range(LEVELS):
        s += w * h
        w //= 2
        h //= 2
    return s


def hbm_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        try:
            return float(json.load(open(p))["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (measured)"
        except Exception:
            pass
    return 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"


def profiled_instructions():
    """Warp instructions per frame of the two k_detect launches (committed ncu
    capture, profiles/traffic.json) for the issue roofline."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        return d["warp_instr_per_frame"], d["instr_source"]
    except Exception:
        return None, None


def profiled_lts():
    """L2 (lts__t_bytes) bytes per frame of the k_detect launches from the
    committed ncu capture (profiles/traffic.json)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        d = json.load(open(p))
        return d["lts_bytes_per_frame"], d.get("lts_source", d["source"])
    except Exception:
        return None, None


def profiled_traffic(frames: int):
    """DRAM bytes of the fused kernel from the committed ncu capture
    (profiles/traffic.json: per-frame dram__bytes_read + dram__bytes_write),
    scaled to this launch's frame count."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None, None
    try:
        d = json.load(open(p))
        return d["dram_bytes_per_frame"] * frames, d["source"]
    except Exception:
        return None, None


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._ready = threading.Event()  # the first sample is in (or sampling failed)
        self._t = None
        self._nvml = None

    def _sample(self):
        if self._nvml is not None:
            nv, hnd, mx, bits = self._nvml
            sm = nv.nvmlDeviceGetClockInfo(hnd, nv.NVML_CLOCK_SM)
            r = nv.nvmlDeviceGetCurrentClocksEventReasons(hnd)
            self.samples.append([str(sm), str(mx)] +
                                ["Active" if r & b else "Not Active" for b in bits])
            return
        out = subprocess.run(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True,
                             text=True, timeout=5).stdout.strip()
        if out:
            self.samples.append([x.strip() for x in out.split(",")])

    def _run(self):
        try:  # NVML directly: ~1 ms per sample instead of a process per sample
            import pynvml as nv
            nv.nvmlInit()
            hnd = nv.nvmlDeviceGetHandleByIndex(self.device)
            mx = nv.nvmlDeviceGetMaxClockInfo(hnd, nv.NVML_CLOCK_SM)
            bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                    nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
            self._nvml = (nv, hnd, mx, bits)
        except Exception:
            self._nvml = None
        period = 0.05 if self._nvml is not None else 0.2
        while not self._stop.is_set():
            try:
                self._sample()
            except Exception:
                self._ready.set()
                return
            self._ready.set()
            self._stop.wait(period)
        self._ready.set()

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        self._ready.wait(timeout=15)  # sampling is live when the timed region starts
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        if len(self.samples) < 2:  # a short region: one more sample right at its end
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def host_cpu():
    """nproc plus lscpu's model / sockets of this host (the CPU baselines' cores)."""
    info = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k = k.strip()
            if k in ("Model name", "Socket(s)", "Thread(s) per core", "Core(s) per socket", "CPU(s)"):
                info[k] = v.strip()
    except Exception:
        pass
    return info


def ref_cfg(cfg: dict) -> dict:
    """The reference's config keys (config.cpp:70-131) for flk_config_set."""
    return {k: cfg[k] for k in ("epsilon", "N", "score_kind", "l", "w", "h", "n")}


def synth_host_frames(kind: int, first: int, count: int, w: int, h: int, device: int):
    """S1/S2 frames first..first+count-1 on the host: generated on the device
    (bit-identical to the host generator, tests/test_gpu_parity.py) and copied."""
    import torch
    import paper_2003_13493_b200 as fl
    buf = torch.empty((count, h, w), dtype=torch.uint8, device=f"cuda:{device}")
    fl.synth_frames_device(buf.data_ptr(), kind, first, count, w, h, w, w * h,
                           torch.cuda.current_stream().cuda_stream)
    return buf.cpu().numpy()


def cpu_reference(cfg: dict, w: int, h: int, frames_n: int, mode: int, device: int,
                  first: int = 10_000, collect: bool = False):
    """The reference build (oracle/_ref) through its public flk_detector_run on
    host cores: mode 0 = as shipped (one detector, threads=0, frames in
    sequence, as `fastlk detect`); mode 1 = best effort (nproc threads, one
    threads=1 detector each, frame-parallel). Per-stage split from
    flk_frame_stats (frontend.cpp:38-57)."""
    import oracle
    ref = oracle.load_reference()
    if ref is None:
        return None
    workers = os.cpu_count() or 1
    frames = synth_host_frames(1, first, frames_n, w, h, device)
    res = ref.bench(frames, ref_cfg(cfg), mode=mode, workers=workers, collect=collect, stages=True)
    secs, nfeat, st = res[0], res[1], res[-1]
    cores = workers
    out = {"value": frames_n / secs, "unit": "frames/s", "cores": cores, "kind": "reference",
           "mode": "as-shipped (one detector, threads=0 = all cores inside each frame, frames in "
                   "sequence; fastlk_cli.cpp:199-232)" if mode == 0 else
                   f"frame-parallel ({workers} threads, one threads=1 detector each)",
           "sample": f"{frames_n} S2 frames {w}x{h} (indices {first}..{first + frames_n - 1}), "
                     f"{secs:.2f} s wall",
           "mpix_per_s": frames_n / secs * w * h / 1e6,
           "stage_us_per_frame": {"pyramid": st[0] / frames_n, "crf": st[1] / frames_n,
                                  "nms": st[2] / frames_n},
           "features_per_frame": nfeat / frames_n}
    if collect:
        return out, res[2]
    return out


def level_pixels_of(w: int, h: int, levels: int) -> int:
    s = 0
    for _ in range(levels):
        s += w * h
        w //= 2
        h //= 2
    return s


def side_config(name: str, spec: dict, device: int, peak: float, steps: int = 10,
                cpu: bool = True):
    """One BASELINE side configuration on this GPU: device-resident batch
    throughput, the fused kernel's roofline fraction, and the reference on
    the host's cores beside it."""
    import torch
    import paper_2003_13493_b200 as fl
    cfg, w, h, n = spec["cfg"], spec["W"], spec["H"], spec["frames"]
    c = fl.Config(**cfg)
    if spec.get("cell"):
        c.set_cell_size_px(*spec["cell"])
    b = fl.DeviceBatch(fl.Detector(c, device=device), w, h, n)
    pitch = (w + 15) // 16 * 16
    buf = torch.empty((n, h, pitch), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    fl.synth_frames_device(buf.data_ptr(), 1, 0, n, w, h, pitch, pitch * h, st)
    for _ in range(3):
        b.run_device(buf.data_ptr(), pitch * h, pitch, n, st)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        b.run_device(buf.data_ptr(), pitch * h, pitch, n, st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    fps = n / (ms / 1e3)
    counts = np.zeros(n, np.int32)
    b.download(0, n, counts.ctypes.data, None, st)
    t = [0.0, 0.0, 0.0]
    for _ in range(3):
        t = [x + y / 3 for x, y in zip(t, b.run_device_timed(buf.data_ptr(), pitch * h, pitch, n, st))]
    torch.cuda.synchronize()
    bpf = level_pixels_of(w, h, cfg["l"]) + 16 * float(counts.mean())
    kern = bpf * n / (t[1] / 1e6) / 1e9
    out = {"workload": spec["desc"], "frames_per_s": fps, "mpix_per_s": fps * w * h / 1e6,
           "ms_per_step": ms, "frames_per_step": n,
           "roofline": {"bound": "hbm", "bytes_per_frame": bpf, "peak": peak,
                        "step_gbs": bpf * fps / 1e9, "step_frac": bpf * fps / 1e9 / peak,
                        "kernel_gbs": kern, "kernel_frac": kern / peak,
                        "kernel_us_per_step": t[1],
                        "note": "algorithmic bytes (sum_k w_k h_k + 16 F) per frame x frames / "
                                "time; kernel_* over the fused k_detect launches' CUDA-event time"}}
    del buf
    if cpu and spec.get("cpu_frames"):
        rc = dict(cfg)
        if spec.get("cpu_cfg"):
            rc.update(spec["cpu_cfg"])
        cb = cpu_reference(rc, w, h, spec["cpu_frames"], 1, device, first=0)
        if cb is not None:
            if spec.get("cpu_note"):
                cb["note"] = spec["cpu_note"]
            out["cpu_baseline"] = cb
    return out


SIDE_CONFIGS = {
    "C1": {"cfg": dict(epsilon=10, N=9, score_kind="mt", l=1, w=1, h=32, n=1), "W": 752, "H": 480,
           "frames": 4096, "cpu_frames": 384,
           "desc": "752x480 l=1 FAST-9 mt (threshold score), 32x32 cells, batch 4096, S2 frames "
                   "on device (BASELINE configs[0])"},
    "C3": {"cfg": dict(epsilon=10, N=12, score_kind="sad_b", l=4, w=1, h=2, n=1), "W": 1920,
           "H": 1080, "frames": 256, "cell": (16, 16), "cpu_frames": 64,
           "cpu_note": "the reference API cannot express 16x16 cells: its 32x16 twin (w=1, h=2) "
                       "through flk_detector_run",
           "desc": "1920x1080 l=4 FAST-12 sad_b, 16x16 cells (extension), batch 256, S2 frames "
                   "on device (BASELINE configs[2])"},
    "C5": {"cfg": dict(epsilon=10, N=10, score_kind="sad_b", l=5, w=1, h=2, n=1), "W": 3840,
           "H": 2160, "frames": 64, "cpu_frames": 32,
           "desc": "3840x2160 l=5 FAST-10 sad_b, 32x32 cells (w=1,h=2), batch 64 per GPU, S2 "
                   "frames on device (BASELINE configs[4])"},
}


def c2_latency(device: int):
    """C2: one S2 752x480 frame per flk_detector_run (H2D, then a
    CUDA-graph replay of pyramid + fused + compaction kernels that leaves the
    feature list in mapped page-locked memory), host wall time per call over
    1000 calls; and separately device-only (CUDA events around one frame's
    kernels on a device-resident frame)."""
    import ctypes
    import torch
    import paper_2003_13493_b200 as fl
    det = fl.Detector(fl.Config(**CFG), device=device)
    dframe = torch.empty((H, PITCH), dtype=torch.uint8, device="cuda")
    fl.synth_frames_device(dframe.data_ptr(), 1, 0, 1, W, H, PITCH, PITCH * H,
                           torch.cuda.current_stream().cuda_stream)
    img = fl.Image.from_array(np.ascontiguousarray(dframe[:, :W].cpu().numpy()))
    lib = fl.load_library()
    fh = ctypes.c_void_p()

    def call():  # the raw C-ABI call a C caller makes, then free the result
        assert lib.flk_detector_run(det.handle, img.handle, ctypes.byref(fh), None, None) == 0
        lib.flk_features_destroy(fh)

    for _ in range(50):
        call()
    ts = []
    for _ in range(1000):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    ts = np.array(ts) * 1e6
    one = fl.DeviceBatch(fl.Detector(fl.Config(**CFG), device=device), W, H, 1)
    st = torch.cuda.current_stream()
    dev = []
    for i in range(1050):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        one.run_device(dframe.data_ptr(), PITCH * H, PITCH, 1, st.cuda_stream)
        b.record(st)
        b.synchronize()
        if i >= 50:
            dev.append(a.elapsed_time(b) * 1e3)
    return {"workload": "752x480 S2 frame, l=3 FAST-9 sad_b, 1 frame via flk_detector_run "
                        "(BASELINE configs[1])",
            "e2e_us_median": float(np.median(ts)), "e2e_us_p95": float(np.percentile(ts, 95)),
            "calls": len(ts), "device_us_median": float(np.median(dev)),
            "includes": "H2D of the frame from its page-locked pixels, pyramid + fused + "
                        "compaction kernels (graph replay), feature list written to mapped "
                        "page-locked memory, list copied into the returned handle",
            "device_only": "CUDA events around one run_device of a device-resident frame "
                           "(pyramid + fused + compaction launches), median of 1000"}


SESSION_CFG = dict(CFG, target_count=200, redetect_ratio=0.3, param_mode="full",
                   max_iterations=30, convergence_epsilon=0.01)
SESSION_FRAMES, SESSION_STEP = 60, 2


def session_frames(device: int):
    """A 752x480 sequence moving SESSION_STEP px left per frame: crops of one
    wide S2 texture generated on the device (host copies for the host API)."""
    import torch
    import paper_2003_13493_b200 as fl
    wide = W + SESSION_STEP * SESSION_FRAMES + 8
    buf = torch.empty((H, wide), dtype=torch.uint8, device=f"cuda:{device}")
    fl.synth_frames_device(buf.data_ptr(), 1, 77, 1, wide, H, wide, wide * H,
                           torch.cuda.current_stream().cuda_stream)
    master = buf.cpu().numpy()
    return [np.ascontiguousarray(master[:, SESSION_STEP * f:SESSION_STEP * f + W])
            for f in range(SESSION_FRAMES)]


def session_line(device: int):
    """SURVEY 8(f) f1+f2: the detect-track session (flk_session_process, host
    frames in, track list out) per-frame latency on this GPU."""
    import paper_2003_13493_b200 as fl
    import ctypes
    frames = session_frames(device)
    lib = fl.load_library()
    imgs = [fl.Image.from_array(f) for f in frames]
    th = ctypes.c_void_p()

    def run_sequence():  # raw C-ABI calls, as a C caller makes them
        s = fl.Session(fl.Config(**SESSION_CFG))
        ts = []
        for im in imgs:
            t0 = time.perf_counter()
            assert lib.flk_session_process(s.handle, im.handle, ctypes.byref(th), None, None) == 0
            ts.append(time.perf_counter() - t0)
            live = lib.flk_tracks_count(th)
            lib.flk_tracks_destroy(th)
        return np.array(ts) * 1e6, live

    run_sequence()  # warm-up (allocations, module load)
    ts, live = run_sequence()

    def run_many(k):  # k sessions advanced together (flkb_sessions_process)
        ss = [fl.Session(fl.Config(**SESSION_CFG)) for _ in range(k)]
        sh = (ctypes.c_void_p * k)(*[x.handle.value for x in ss])
        outs = (ctypes.c_void_p * k)()
        arrs = [(ctypes.c_void_p * k)(*([im.handle.value] * k)) for im in imgs]
        t0 = 0.0
        for j, ih in enumerate(arrs):
            if j == 1:  # frame 0 is the cold start (detection + templates)
                t0 = time.perf_counter()
            assert lib.flkb_sessions_process(sh, ih, k, outs, None) == 0
            for i in range(k):
                lib.flk_tracks_destroy(ctypes.c_void_p(outs[i]))
        return k * (len(arrs) - 1) / (time.perf_counter() - t0)

    many = {}
    for k in (1, 4, 8, 16):
        many[k] = max(run_many(k) for _ in range(3))
    cold, ts = ts[0] / 1e6, ts[1:]
    parts = []
    s3 = fl.Session(fl.Config(**SESSION_CFG))
    for f in frames:
        _, ex = s3.process(f, stats=True)
        parts.append((ex["stats"]["pyramid_us"], ex["stats"]["track_us"],
                      ex["stats"]["tracks_entering"], ex["stats"]["track_iterations"]))
    parts = np.array(parts[1:])
    return {"workload": f"752x480 l=3 FAST-9 sad_b session, target 200 tracks, full LK "
                        f"(translation+gain+offset), sequence moving {SESSION_STEP} px/frame, "
                        f"{SESSION_FRAMES} frames",
            "us_per_frame_median": float(np.median(ts)), "us_per_frame_p95": float(np.percentile(ts, 95)),
            "frames_per_s": float(1e6 / np.median(ts)), "cold_start_us": cold * 1e6,
            "live_tracks_last_frame": live,
            "stage_us_median": {"pyramid": float(np.median(parts[:, 0])),
                                "track": float(np.median(parts[:, 1]))},
            "lk_iterations_per_track": float(parts[:, 3].sum() / max(1, parts[:, 2].sum())),
            "concurrent_sessions_frames_per_s": {str(k): v for k, v in many.items()},
            "includes": "H2D of the frame, pyramid, LK kernel over every live track, D2H of "
                        "warps, host lifecycle; re-detection + template kernels when fired"}


def session_reference(device: int):
    """The reference's own flk_session_process (oracle/_ref) on the host on the
    same sequence: median per-frame latency (one session, threads=0 = all cores)."""
    import oracle
    ref = oracle.load_reference()
    if ref is None:
        return None
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import sessions
    import ctypes
    frames = session_frames(device)
    s = sessions.CapiSession(ref.lib, SESSION_CFG)  # sets the ctypes signatures
    lib = ref.lib
    imgs = []
    for f in frames:
        h = ctypes.c_void_p()
        assert lib.flk_image_create(W, H, f.ctypes.data, ctypes.byref(h)) == 0
        imgs.append(h)
    th = ctypes.c_void_p()
    ts = []
    for im in imgs:  # raw C-ABI calls, as for the GPU line
        t0 = time.perf_counter()
        assert lib.flk_session_process(s.h, im, ctypes.byref(th), None, None) == 0
        ts.append(time.perf_counter() - t0)
        lib.flk_tracks_destroy(th)
    s.close()
    for im in imgs:
        lib.flk_image_destroy(im)
    ts = np.array(ts[1:]) * 1e6
    return {"us_per_frame_median": float(np.median(ts)), "frames_per_s": float(1e6 / np.median(ts)),
            "cores": os.cpu_count(), "kind": "reference",
            "sample": f"{SESSION_FRAMES} frames of the same sequence, one session, threads=0"}


def run_reference_arm(args, rank: int, world: int):
    """bench.py --impl reference: the reference's own CPU implementation
    (oracle/_ref, compiled from /root/reference) through its public
    flk_detector_run on this host's cores, frame-parallel, each step a bounded
    sample of the same C4 workload. Rank 0 alone runs (the others exit)."""
    if rank != 0:
        return
    workers = os.cpu_count() or 1
    per_step = max(16, 4 * workers)
    import oracle
    ref = oracle.load_reference()
    if ref is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref not built and "
                          "/root/reference absent"}))
        return
    orc = oracle.load_oracle()
    frames = np.stack([orc.synth(1, i, W, H) for i in range(per_step)])
    cfg = ref_cfg(CFG)
    for _ in range(args.warmup):
        ref.bench(frames, cfg, mode=1, workers=workers)
    total, nf = 0.0, 0
    for _ in range(args.steps):
        secs, _ = ref.bench(frames, cfg, mode=1, workers=workers)
        total += secs
        nf += per_step
    fps = nf / total
    line = {"metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
            "higher_is_better": True, "scaling": "strong" if not args.batch else "weak",
            "vs_baseline": None, "dtype": "u8", "data": "synthetic (S2 texture)",
            "impl": "reference", "mpix_per_s": fps * W * H / 1e6,
            "config": bench_config(args, world),
            "parallelism": f"{workers} host threads, one threads=1 reference detector each",
            "host_cpu": host_cpu(),
            "cpu_baseline": {"value": fps, "unit": "frames/s", "cores": workers,
                             "kind": "reference",
                             "sample": f"{per_step} frames (indices 0..{per_step - 1}) per step x "
                                       f"{args.steps} steps, frame-parallel"},
            "e2e": {"value": fps, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def bench_config(args, world: int) -> dict:
    """The `config` object, identical in both arms (same workload, same global batch)."""
    g = args.batch * world if args.batch else args.global_batch
    return {"workload": WORKLOAD, "global_batch": g}


def parity_check(counts: np.ndarray, feats: np.ndarray, device: int, workers: int):
    """Every frame of the timed batch (global frame indices 0..n-1) against the
    reference build run frame-parallel on the same frames through its public
    flk_detector_run (capi.cpp:232-274); that run doubles as the frame-parallel
    CPU baseline over the whole workload."""
    import hashlib
    import oracle
    n = counts.shape[0]
    cap = feats.shape[1]
    digest = hashlib.sha256()
    for i in range(n):
        digest.update(feats[i, :counts[i]].tobytes())
    out = {"frames": n, "digest_sha256": digest.hexdigest()}
    if oracle.load_reference() is None:
        out.update(mismatches=None, against="unavailable (oracle/_ref not built)")
        return out, None
    bad, secs, nfeat, stages, step = [], 0.0, 0, [0.0, 0.0, 0.0], 512
    for c0 in range(0, n, step):
        m = min(step, n - c0)
        fr = synth_host_frames(1, c0, m, W, H, device)
        res = oracle.load_reference().bench(fr, ref_cfg(CFG), mode=1, workers=workers,
                                            collect=True, stages=True)
        secs += res[0]
        nfeat += res[1]
        rc, rf = res[2]
        stages = [a + b for a, b in zip(stages, res[3])]
        assert rf.shape[1] == cap
        for j in range(m):
            i = c0 + j
            if counts[i] != rc[j] or (feats[i, :counts[i]].view(np.int32) !=
                                      rf[j, :rc[j]].view(np.int32)).any():
                bad.append(i)
    out.update(mismatches=len(bad), first_mismatches=bad[:8],
               against="oracle/_ref (the unmodified reference build) flk_detector_run, "
                       "frame-parallel on host cores, bit-exact per frame (x, y, score, level, "
                       "cell_x, cell_y)")
    cb = {"value": n / secs, "unit": "frames/s", "cores": workers, "kind": "reference",
          "mode": f"frame-parallel ({workers} threads, one threads=1 detector each)",
          "sample": f"the whole timed workload: {n} S2 frames 752x480 (the parity pass), "
                    f"{secs:.2f} s wall",
          "mpix_per_s": n / secs * W * H / 1e6,
          "stage_us_per_frame": {"pyramid": stages[0] / n, "crf": stages[1] / n,
                                 "nms": stages[2] / n},
          "features_per_frame": nfeat / n}
    return out, cb


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--global-batch", type=int, default=4096,
                    help="frames per step over all ranks (strong scaling: rank r detects "
                         "shard_range(G, r, world); BASELINE configs[3])")
    ap.add_argument("--batch", type=int, default=0,
                    help="frames per GPU per step instead (weak scaling)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the C1/C2/C3/C5/session lines")
    ap.add_argument("--plan", default="", help="launch-plan overrides key=value,... (tuning)")
    ap.add_argument("--same-device", action="store_true",
                    help="every rank on cuda:0 (exercises the N>1 path on a one-GPU box)")
    args = ap.parse_args()

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.same_device:
        local = 0

    if args.impl == "reference":
        return run_reference_arm(args, rank, world)

    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    if world > 1:
        # the data path has no collective (frames are independent): gloo on
        # CPU tensors carries only the timing barrier, the max over ranks and
        # the post-run gather of results for the parity check
        dist.init_process_group("gloo")

    import paper_2003_13493_b200 as fl
    from paper_2003_13493_b200.shard import gather_features, shard_range
    if args.batch:
        start, B = rank * args.batch, args.batch
        scaling = "weak"
    else:
        start, B = shard_range(args.global_batch, rank, world)
        scaling = "strong"
    G = args.batch * world if args.batch else args.global_batch
    plan = {}
    for kv in filter(None, args.plan.split(",")):
        k, v = kv.split("=")
        plan[k] = int(v)
    det = fl.Detector(fl.Config(**CFG), device=local, plan=plan)
    batch = fl.DeviceBatch(det, W, H, max(B, 1))
    frames = torch.empty((max(B, 1), H, PITCH), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    if B:
        # global frame index start + i: every N sees the same 4096 frames
        fl.synth_frames_device(frames.data_ptr(), 1, start, B, W, H, PITCH, PITCH * H, stream)
    torch.cuda.synchronize()

    def step():
        if B:
            batch.run_device(frames.data_ptr(), PITCH * H, PITCH, B, stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> list:
        t = torch.tensor([v], dtype=torch.float64)
        if world == 1:
            return [v]
        out = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(out, t)
        return [float(x.item()) for x in out]

    warm = max(args.warmup, 3)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()

    start_ev, end_ev = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    launches0 = fl.kernel_launch_count()
    with ClockSampler(local) as clocks:
        start_ev.record()
        for _ in range(args.steps):
            step()
        end_ev.record()
        torch.cuda.synchronize()
    launches = fl.kernel_launch_count() - launches0
    barrier()
    ms_ranks = max_over_ranks(start_ev.elapsed_time(end_ev))
    ms_max = max(ms_ranks)
    ms_step = ms_max / args.steps
    fps = G * args.steps / (ms_max / 1e3)
    shards = [shard_range(G, r, world)[1] if not args.batch else args.batch for r in range(world)]
    per_rank = [shards[r] * args.steps / (ms_ranks[r] / 1e3) if ms_ranks[r] > 0 else 0.0
                for r in range(world)]

    # results of the timed workload (the last step's lists), for parity
    cap = batch.frame_capacity
    counts = np.zeros(max(B, 1), np.int32)
    feats = np.zeros((max(B, 1), cap), fl.FEATURE_DTYPE)
    if B:
        batch.download(0, B, counts.ctypes.data, feats.ctypes.data, stream)
    torch.cuda.synchronize()
    counts, feats = counts[:B], feats[:B]

    # end to end through the public API from pinned host memory: one
    # flkb_batch_detect_host call per step = H2D of every frame, the kernels,
    # D2H of every count and feature list, copies overlapped with the kernels
    host = frames[:max(B, 1), :, :W].contiguous().cpu().pin_memory()
    hcounts = torch.empty(max(B, 1), dtype=torch.int32).pin_memory()
    hfeats = torch.empty(max(B, 1) * cap * 6, dtype=torch.int32).pin_memory()

    def e2e_step():
        if B:
            batch.detect_host(host.data_ptr(), W * H, W, B, hcounts.data_ptr(), hfeats.data_ptr(),
                              stream)

    e2e_step()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.e2e_steps):
        e2e_step()
    e1.record()
    torch.cuda.synchronize()
    te = max(max_over_ranks(e0.elapsed_time(e1)))
    e2e_fps = G * args.e2e_steps / (te / 1e3)
    e2e_same = bool(B == 0 or ((hcounts.numpy()[:B] == counts).all() and
                               (hfeats.numpy().view(fl.FEATURE_DTYPE).reshape(B, cap) == feats).all()))
    h2d = B * W * H
    d2h = 4 * B + 24 * cap * B
    # the e2e line's own roof: one pinned H2D copy of the same step's frames
    # (the PCIe link; CUDA events, best of 3)
    h2d_gbs = None
    if B:
        dcopy = torch.empty_like(host, device="cuda")
        best = None
        for _ in range(3):
            c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            c0.record()
            dcopy.copy_(host, non_blocking=True)
            c1.record()
            torch.cuda.synchronize()
            ms = c0.elapsed_time(c1)
            best = ms if best is None else min(best, ms)
        h2d_gbs = host.numel() / (best / 1e3) / 1e9
        del dcopy

    # the drop-in-adjacent path: flk_image handles through flkb_detector_run_batch
    # (two-slot pipeline, one flk_features handle per frame), synchronous calls
    hn = min(B, 1024)
    handle_fps = mirror_fps = None
    if hn:
        imgs = [fl.Image.from_array(host[i].numpy()) for i in range(hn)]
        det_h = fl.Detector(fl.Config(**CFG), device=local, plan=plan)
        det_h.run_batch(imgs)
        lib = fl.load_library()
        arr = (ctypes.c_void_p * hn)(*[i.handle.value for i in imgs])
        outs = (ctypes.c_void_p * hn)()
        barrier()
        # the raw C-ABI call, as a C/C++ consumer of the drop-in makes it: the
        # call's wall time (H2D from the images' page-locked pixels, kernels,
        # one flk_features handle per frame); the handles are freed between
        # calls, outside the timed calls
        hsteps, th = 5, 0.0
        for _ in range(hsteps):
            t0 = time.perf_counter()
            assert lib.flkb_detector_run_batch(det_h.handle, arr, hn, outs, None) == 0
            th += time.perf_counter() - t0
            for i in range(hn):
                lib.flk_features_destroy(ctypes.c_void_p(outs[i]))
        th = max(max_over_ranks(th))
        handle_fps = world * hn * hsteps / th
        # the Python mirror (Detector.run_batch: results copied into numpy arrays)
        t0 = time.perf_counter()
        det_h.run_batch(imgs)
        mirror_fps = world * hn / max(max_over_ranks(time.perf_counter() - t0))
        del imgs

    # dominant-kernel time for the roofline: CUDA events around each launch of
    # one step, on the launching stream, averaged over a few synchronized steps
    reps = 5
    acc = [0.0, 0.0, 0.0]
    if B:
        for _ in range(reps):
            t3 = batch.run_device_timed(frames.data_ptr(), PITCH * H, PITCH, B, stream)
            acc = [a + b for a, b in zip(acc, t3)]
    pyr_us, fused_us, comp_us = (a / reps for a in acc)
    # the standalone pyramid kernel, reported on its own: the
    # one-launch plan builds levels 1-2 from level 0 in one k_pyramid_down2
    # launch (the plan small batches and the tracking session use)
    pyr_alone_us = 0.0
    if B:
        batch.set_plan(fuse_pyramid=0)
        pyr_alone_us = sum(batch.run_device_timed(frames.data_ptr(), PITCH * H, PITCH, B, stream)[0]
                           for _ in range(reps)) / reps
        batch.set_plan(fuse_pyramid=plan.get("fuse_pyramid", -1))
    fused_rank = max_over_ranks(fused_us)

    # every rank's results to rank 0 in global frame order (disjoint slots)
    if world > 1:  # (weak scaling: equal shards, shard_range(G, r, N) = [r*B, (r+1)*B))
        got = gather_features(counts, feats, G)
    else:
        got = (counts, feats.view(np.int32).reshape(B, -1))
    extras = {}
    if rank == 0:
        gc, gf = got
        gf = np.ascontiguousarray(gf).view(fl.FEATURE_DTYPE).reshape(G, cap)
        workers = os.cpu_count() or 1
        parity, cb_par = (None, None)
        if not args.no_parity:
            parity, cb_par = parity_check(gc, gf, local, workers)
        peak, peak_src = hbm_peak()
        feats_mean = float(gc.mean()) if G else 0.0
        # every pyramid pixel crosses HBM once + 16 B per feature
        bytes_frame = level_pixels() + 16 * feats_mean
        step_achieved = bytes_frame * G / (ms_step / 1e3) / 1e9
        fmax = max(fused_rank)
        achieved = bytes_frame * B / (fused_us / 1e6) / 1e9 if fused_us else 0.0
        traffic, traffic_src = profiled_traffic(B)
        lts_pf, lts_src = profiled_lts()
        line = {
            "metric": METRIC, "value": fps, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": warm, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (S2 counter-hash texture generated on device, SURVEY 8d)",
            "mpix_per_s": fps * W * H / 1e6,
            "config": bench_config(args, world),
            "parallelism": f"contiguous frame shards x{world} (shard_range), no collective on "
                           "the data path; gloo for the barrier / max over ranks / result gather",
            "frames_per_rank": shards, "frames_per_s_per_rank": per_rank,
            "l2": f"inputs {B * W * H / 1e9:.2f} GB/GPU > 126 MB L2 (no flush needed)",
            "e2e": {"value": e2e_fps, "unit": "frames/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": args.e2e_steps,
                    "api": "flkb_batch_detect_host (pinned host frames in, pinned counts + "
                           "feature lists out; chunked over two streams, H2D and D2H "
                           "overlapped with the kernels)",
                    "results_equal_device_path": e2e_same,
                    "roofline": {"bound": "pcie_h2d", "unit": "GB/s",
                                 "achieved": (h2d / 1e9) * e2e_fps / max(G, 1) if G else None,
                                 "peak": h2d_gbs,
                                 "frac": ((h2d / 1e9) * e2e_fps / max(G, 1) / h2d_gbs)
                                 if G and h2d_gbs else None,
                                 "peak_source": "one pinned host-to-device copy of the step's "
                                                "frames (torch copy_, CUDA events, best of 3)"}},
            "e2e_handles": {"value": handle_fps, "unit": "frames/s",
                            "frames_per_call": hn, "calls": 5,
                            "api": "flkb_detector_run_batch over flk_image handles (page-locked "
                                   "pixels), one flk_features handle per frame, host wall time "
                                   "of the raw C-ABI calls",
                            "python_mirror": mirror_fps},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic,
                         "kernel": "flkb::fused::k_detect (FAST + score + NMS + cell keys) over "
                                   f"a {B}-frame shard, in chunks of frames whose pyramid levels "
                                   "1-2 fit in a quarter of L2: per chunk a level-0 launch that "
                                   "also writes levels 1-2 from its staged rows, then a level 1-2 "
                                   "launch (side stream, overlapping the next chunk's level-0 "
                                   "launch) that reads them back from L2; achieved = the shard's "
                                   "algorithmic bytes / the CUDA-event time from the first to the "
                                   "last of these launches (rank 0)",
                         "kernel_launches_per_step": int(launches) // max(args.steps, 1) - 1,
                         "kernel_us_per_step": fused_us, "kernel_us_per_step_ranks": fused_rank,
                         "kernel_share_of_step": fused_us / max(fused_us + pyr_us + comp_us, 1e-9),
                         "other_kernels_us": {"pyramid": pyr_us, "compact": comp_us},
                         "bytes_per_frame": bytes_frame, "bytes_per_step": bytes_frame * G,
                         "traffic_over_algorithmic": (traffic / (bytes_frame * B)) if traffic else None,
                         "l2_gbs": (lts_pf * B / (fused_us / 1e6) / 1e9) if lts_pf and fused_us else None,
                         "l2_bytes_per_frame": lts_pf, "l2_source": lts_src,
                         "step_achieved_gbs": step_achieved, "step_frac": step_achieved / peak,
                         "peak_source": peak_src, "traffic_source": traffic_src},
            "gpu_launches": int(launches),
            "clocks": clocks.summary(),
            "host_cpu": host_cpu(),
        }
        if parity is not None:
            line["parity"] = parity
        pyr_bytes = level_pixels()  # level 0 read once, levels >= 1 written once
        if pyr_alone_us:
            pyr_gbs = pyr_bytes * B / (pyr_alone_us / 1e6) / 1e9
            line["pyramid_roofline"] = {
                "bound": "hbm", "achieved": pyr_gbs, "peak": peak, "unit": "GB/s",
                "frac": pyr_gbs / peak, "kernel_us": pyr_alone_us, "bytes_per_frame": pyr_bytes,
                "kernel": f"flkb::k_pyramid_down2 alone over the {B}-frame shard (levels 1-2 "
                          "from level 0, one 16x4-block per thread; the one-launch plan's "
                          "pyramid), CUDA events on its stream"}
        # The path is instruction-issue bound: the same kernels
        # against the SM issue rate (148 SMs x 4 schedulers x 1 warp-instr/clk
        # at the live SM clock), from the committed ncu instruction count.
        wipf, wsrc = profiled_instructions()
        mhz = line["clocks"].get("sm_mhz") or 1965.0
        if wipf and fused_us:
            peak_i = 148 * 4 * mhz * 1e6 / 1e9
            kern_i = B * wipf / (fused_us / 1e6) / 1e9
            line["issue_roofline"] = {
                "bound": "issue", "unit": "G warp-instr/s", "achieved": kern_i, "peak": peak_i,
                "frac": kern_i / peak_i, "warp_instr_per_frame": wipf,
                "note": "k_detect warp instructions per frame (ncu) x frames per step / the "
                        "step's k_detect CUDA-event time, against 148 SMs x 4 issue slots x SM clock",
                "source": wsrc}
        if not args.no_cpu_baseline:
            cbs = {}
            if cb_par is not None:
                cbs["frame_parallel"] = cb_par
            else:
                cbs["frame_parallel"] = cpu_reference(CFG, W, H, min(2048, 128 * workers), 1, local)
            cbs["as_shipped"] = cpu_reference(CFG, W, H, 96, 0, local)
            if cbs["frame_parallel"] is not None:
                line["cpu_baseline"] = dict(cbs["frame_parallel"])
                line["cpu_baseline"]["as_shipped"] = cbs["as_shipped"]
        extras["line"] = line

    # side configurations: C5 on every rank (the 8-GPU batch line of BASELINE
    # configs[4], weak: 64 frames per GPU), the others on one GPU
    if not args.no_extras:
        import torch as _t
        spec = SIDE_CONFIGS["C5"]
        barrier()
        c5 = side_config("C5", spec, local, hbm_peak()[0], cpu=False)
        fr = max_over_ranks(c5["ms_per_step"])
        if rank == 0:
            c5["frames_per_s_all_gpus"] = world * spec["frames"] / (max(fr) / 1e3)
            c5["n_gpus"] = world
            c5["note"] = ("per-GPU batch of 64 frames on each of n_gpus GPUs; frames_per_s_all_gpus "
                          "= n_gpus x 64 / max over ranks of the step time")
            extras["C5"] = c5
        _t.cuda.synchronize()
    if rank == 0:
        line = extras["line"]
        if not args.no_extras:
            oc = {}
            oc["C2_latency"] = c2_latency(local) if world == 1 else None
            for name in ("C1", "C3"):
                if world == 1:
                    oc[name] = side_config(name, SIDE_CONFIGS[name], local, hbm_peak()[0],
                                           cpu=not args.no_cpu_baseline)
            c5 = extras["C5"]
            if not args.no_cpu_baseline:
                cb = cpu_reference(SIDE_CONFIGS["C5"]["cfg"], 3840, 2160,
                                   SIDE_CONFIGS["C5"]["cpu_frames"], 1, local, first=0)
                if cb is not None:
                    c5["cpu_baseline"] = cb
            oc["C5"] = c5
            if world == 1:
                if not args.no_cpu_baseline and oc["C2_latency"] is not None:
                    cb = cpu_reference(CFG, W, H, 48, 0, local)
                    if cb is not None:
                        cb["us_per_frame"] = 1e6 / cb["value"]
                        oc["C2_latency"]["cpu_baseline"] = cb
                oc["F12_session"] = session_line(local)
                if not args.no_cpu_baseline:
                    oc["F12_session"]["cpu_baseline"] = session_reference(local)
            line["other_configs"] = {k: v for k, v in oc.items() if v is not None}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
