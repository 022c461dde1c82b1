"""Per-launch time of the headline chain: back-to-back graph replays vs isolated replays (synchronize
and idle between launches) vs direct (non-graph) launches, each device-timed with CUDA events."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    st = bench.build_stack(32, 1000, dev, "chain")
    st.capture()
    for _ in range(5):
        st.replay()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(20):
        st.replay()
    e[1].record()
    torch.cuda.synchronize()
    print(f"back-to-back graph replays: {e[0].elapsed_time(e[1]) / 20 * 1000:.1f} us per launch")
    iso = []
    for _ in range(20):
        torch.cuda.synchronize()
        time.sleep(0.002)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.replay()
        b.record()
        torch.cuda.synchronize()
        iso.append(a.elapsed_time(b) * 1000)
    iso.sort()
    print(f"isolated graph replays: median {iso[10]:.1f} min {iso[0]:.1f} max {iso[-1]:.1f} us")
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device=dev)
    iso = []
    for _ in range(20):
        flush.fill_(1)  # write 512 MB: evicts (and writes back) everything in the 126 MB L2
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        st.replay()
        b.record()
        torch.cuda.synchronize()
        iso.append(a.elapsed_time(b) * 1000)
    iso.sort()
    print(f"replays after an L2 flush: median {iso[10]:.1f} min {iso[0]:.1f} max {iso[-1]:.1f} us")
    e[0].record()
    for _ in range(20):
        st.launch_all()
    e[1].record()
    torch.cuda.synchronize()
    print(f"back-to-back direct launches: {e[0].elapsed_time(e[1]) / 20 * 1000:.1f} us per launch")


if __name__ == "__main__":
    main()
