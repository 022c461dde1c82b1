"""Host overhead of the e2e path: LinearStack.forward(host x) vs its parts (host graph replay + sync)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def wall(fn, n=50):
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        for _ in range(n):
            fn()
        best = min(best, (time.perf_counter() - t) / n * 1e6)
    return best


def main():
    dev = torch.device("cuda", 0)
    st = bench.build_stack(32, 1000, dev, "chain")
    st.capture()
    x0 = torch.from_numpy(np.random.default_rng(0).standard_normal(st.x.numel()).astype(np.float32))
    st.forward(x0)
    s = torch.cuda.current_stream(dev)
    print(f"forward(host tensor):          {wall(lambda: st.forward(x0)):7.1f} us")
    print(f"host graph replay + sync:      {wall(lambda: (st.host_graph.replay(), s.synchronize())):7.1f} us")
    print(f"device graph replay + sync:    {wall(lambda: (st.graph.replay(), s.synchronize())):7.1f} us")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        st.host_graph.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"host graph, device time:       {e0.elapsed_time(e1) / 50 * 1000:7.1f} us")


if __name__ == "__main__":
    main()
