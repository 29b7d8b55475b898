"""One C4 detection step (4096 frames, after two warm-up steps) inside a
cudaProfilerStart/Stop window, for one-pass ncu counters of every kernel of
the step under a given launch plan:

    ncu --profile-from-start off --cache-control none --clock-control none \
        --metrics gpu__time_duration.sum,dram__bytes_read.sum,... --csv --log-file X.csv \
        python tools/counters.py [--plan staged=1] [--batch 4096]

tools/counters_summary.py turns the CSV into per-kernel totals per frame.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", default="")
    ap.add_argument("--batch", type=int, default=4096)
    a = ap.parse_args()
    import torch

    import bench
    import paper_2003_13493_b200 as fl
    plan = {k: int(v) for k, v in (kv.split("=") for kv in filter(None, a.plan.split(",")))}
    B, W, H, P = a.batch, bench.W, bench.H, bench.PITCH
    det = fl.Detector(fl.Config(**bench.CFG), plan=plan)
    batch = fl.DeviceBatch(det, W, H, B)
    frames = torch.empty((B, H, P), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    fl.synth_frames_device(frames.data_ptr(), 1, 0, B, W, H, P, P * H, st)
    for _ in range(2):
        batch.run_device(frames.data_ptr(), P * H, P, B, st)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    batch.run_device(frames.data_ptr(), P * H, P, B, st)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print("plan", plan, "launches", batch.kernels_per_run)


if __name__ == "__main__":
    main()
