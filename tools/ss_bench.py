"""Variant ss (per-32 sub-scales) and block_n 32..128 on the fast MMQ path vs block_n 256 variant s, and vs
the generic fp64 kernel those formats took before.

    python tools/ss_bench.py [--rows 4096 --cols 4096] [--out profiles/r01/ss_mmq.json]

Device time per fused_matmul call (CUDA events around 10 back-to-back calls, check_finite=False, so the
call is rotation + MMQ), and the generic fp64 kernel (itq3_matmul_generic, the path variant ss took before).
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_27914_b200 as P  # noqa: E402
from paper_2603_27914_b200 import _lib  # noqa: E402


def dev_time(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3  # us


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    w = torch.randn((a.rows, a.cols), generator=g, device=dev) / a.cols ** 0.5
    qs = {"s": P.quantize_tensor(w), "ss": P.quantize_tensor(w, P.QuantConfig(variant="ss"))}
    for n in (128, 64, 32):
        qs[f"s{n}"] = P.quantize_tensor(w, P.QuantConfig(block_n=n))
    res = []
    for m in (16, 64, 256, 2048):
        X = torch.randn((a.cols, m), generator=g, device=dev)
        row = {"rows": a.rows, "K": a.cols, "M": m}
        for v, q in qs.items():
            us = dev_time(lambda: P.fused_matmul(q, X, check_finite=False))
            row[f"{v}_us"] = us
            row[f"{v}_tflops"] = 2.0 * a.rows * a.cols * m / us / 1e6
        q = qs["ss"]
        p = q.ensure_decodable()
        Xd = X.double()
        ws = torch.empty(_lib.load().itq3_generic_ws_nbytes(a.rows, a.cols, 256, m), dtype=torch.uint8, device=dev)
        Y = torch.empty((a.rows, m), dtype=torch.float64, device=dev)
        gen = lambda: _lib.call("itq3_matmul_generic", _lib.ptr(p), a.rows, a.cols, 256, 1, _lib.ptr(Xd), m,
                                Xd.stride(0), Xd.stride(1), _lib.ptr(Y), _lib.ptr(ws), _lib.stream_ptr(dev))
        row["ss_generic_fp64_us"] = dev_time(gen, reps=3)
        res.append(row)
        print(json.dumps(row), flush=True)
    if a.out:
        json.dump({"results": res}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
