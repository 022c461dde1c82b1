"""End-to-end time of the public fused_matmul call (CUDA X in, CUDA Y out; includes its allocations,
the activation rotation, the fused finiteness check and the host sync the DomainError semantics need).

    python tools/api_matmul_bench.py
"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_27914_b200 as P  # noqa: E402

SHAPES = [(14336, 4096), (4096, 14336), (4096, 4096)]


def main():
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    out = []
    for rows, K in SHAPES:
        q = P.quantize_tensor(torch.randn((rows, K), generator=g, device=dev) / K ** 0.5)
        for M in (16, 64, 256, 2048):
            X = torch.randn((K, M), generator=g, device=dev)
            for _ in range(3):
                P.fused_matmul(q, X)
            torch.cuda.synchronize()
            n = 20
            t0 = time.perf_counter()
            for _ in range(n):
                P.fused_matmul(q, X)
            torch.cuda.synchronize()
            us = (time.perf_counter() - t0) / n * 1e6
            t0 = time.perf_counter()
            for _ in range(n):
                P.fused_matmul(q, X, check_finite=False)
            torch.cuda.synchronize()
            us_nc = (time.perf_counter() - t0) / n * 1e6
            r = {"rows": rows, "K": K, "M": M, "api_us": us, "tflops": 2 * rows * K * M / us / 1e6,
                 "api_us_no_check": us_nc, "tflops_no_check": 2 * rows * K * M / us_nc / 1e6}
            out.append(r)
            print(json.dumps(r), flush=True)
    return out


if __name__ == "__main__":
    main()
