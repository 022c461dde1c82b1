"""Fixed cost of one chain launch: ms per graph replay of tiny chains (1 / 2 / 8 stages of 256 x 256)
next to the Llama-2-7B stack, i.e. launch + prologue (descriptor cache, barriers, epoch check-in) +
final fold, which the per-token time carries whatever the weights.

    python tools/chain_overhead.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_27914_b200 as P  # noqa: E402
from paper_2603_27914_b200.stack import LinearStack  # noqa: E402


def time_stack(st, n=50):
    st.capture()
    for _ in range(5):
        st.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        st.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1000.0


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    for S in (1, 2, 8, 32, 128):
        qs = [P.quantize_tensor(torch.randn((256, 256), generator=g, device=dev) / 16) for _ in range(S)]
        print(f"{S:4d} stages of 256x256: {time_stack(LinearStack(qs, limbs=3, mode='chain')):7.2f} us per launch")


if __name__ == "__main__":
    main()
