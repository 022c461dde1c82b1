"""Single-shot MMQ call for an ncu capture: rotate + itq3_mmq at one shape (default 14336x4096, M=2048).

    ncu --set full -k regex:mmq_pair -c 1 python tools/mmq_ncu_target.py [--rows R --cols K --m M]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_27914_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=14336)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--m", type=int, default=2048)
    ap.add_argument("--calls", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    q = P.quantize_tensor(torch.randn((a.rows, a.cols), generator=g, device=dev) / a.cols ** 0.5)
    X = torch.randn((a.cols, a.m), generator=g, device=dev)
    for _ in range(a.calls):
        P.fused_matmul(q, X)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
