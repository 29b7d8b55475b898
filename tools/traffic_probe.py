"""One C4 detection step (4096 frames) after one warm-up step, for an ncu
DRAM-traffic capture of its k_detect launches:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum --cache-control none \
        -k regex:k_detect -s <launches per step> python tools/traffic_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    import bench
    import paper_2003_13493_b200 as fl
    B, W, H, P = 4096, bench.W, bench.H, bench.PITCH
    chunk = int(os.environ.get("PYR_CHUNK", "0"))  # tool option, passed as a launch plan
    det = fl.Detector(fl.Config(**bench.CFG), plan={"pyramid_chunk": chunk} if chunk else None)
    batch = fl.DeviceBatch(det, W, H, B)
    frames = torch.empty((B, H, P), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    fl.synth_frames_device(frames.data_ptr(), 1, 0, B, W, H, P, P * H, st)
    for _ in range(2):
        batch.run_device(frames.data_ptr(), P * H, P, B, st)
    torch.cuda.synchronize()
    print("launches per step", batch.kernels_per_run)


if __name__ == "__main__":
    main()
