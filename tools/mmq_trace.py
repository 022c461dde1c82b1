"""Per-role cycle accounting of the K5 CTA-pair MMQ kernel (csrc/mmq.cu, g_mmq_trace).

    python tools/mmq_trace.py [--rows 14336 --cols 4096 --m 2048]
Prints the median over CTAs of: producer wait on `empty`, expander wait on `full`, expander busy
(decode + tcgen05.st + arrive), MMA-issuer wait on `ready` / `dempty` (leaders only), epilogue wait
on `dfull` and busy time, total producer cycles, and chunks per CTA.
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_27914_b200 as P  # noqa: E402
from paper_2603_27914_b200 import _lib  # noqa: E402

NAMES = ["prod_wait_empty", "exp_wait_full", "exp_busy", "mma_wait_ready", "mma_wait_dempty",
         "epi_wait_dfull", "epi_busy", "prod_total", "chunks", "mma_total", "prod_issue", "exp_wait_aempty"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=14336)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--m", type=int, default=2048)
    ap.add_argument("--flags", type=int, default=0, help="diagnostic knockouts (when compiled in)")
    ap.add_argument("--data", choices=["randn", "zeros", "ones"], default="randn", help="activation values")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    q = P.quantize_tensor(torch.randn((a.rows, a.cols), generator=g, device=dev) / a.cols ** 0.5)
    X = torch.randn((a.cols, a.m), generator=g, device=dev)
    if a.data == "zeros":
        X.zero_()
    elif a.data == "ones":
        X.fill_(1.0)
    P.fused_matmul(q, X)
    tr = torch.zeros(4096 * 16, dtype=torch.int64, device=dev)
    tr[4095 * 16] = a.flags
    _lib.call("itq3_mmq_set_trace", _lib.ptr(tr))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    P.fused_matmul(q, X)
    e1.record()
    torch.cuda.synchronize()
    _lib.call("itq3_mmq_set_trace", None)
    if P.compute.MMQ_MIN_TOKENS <= a.m <= P.compute.MMQ8_MAX_TOKENS:  # K5b: its own counter layout
        _lib.call("itq3_mmq_set_trace", None)
        t = tr.view(-1, 16).cpu().numpy()
        t = t[t[:, 10] > 0]
        names8 = ["prod_wait_empty", "mma_wait_aready", "mma_wait_full", "mma_wait_dempty", "mma_total",
                  "exp_wait_full", "exp_wait_aempty", "exp_total", "epi_wait_dfull", "epi_total", "blocks", "cta_total"]
        print(f"K5b {a.rows}x{a.cols} M={a.m}: {e0.elapsed_time(e1) * 1e3:.1f} us (rotate + mmq8), {len(t)} CTAs")
        for i, n in enumerate(names8):
            print(f"  {n:18s} median {np.median(t[:, i]):10.0f}  max {t[:, i].max():10.0f}")
        print(f"  cycles per block: {np.median(t[:, 11]) / np.median(t[:, 10]):.0f}")
        return
    # separate timings (no trace): rotation and the MMQ kernel, 10 calls each
    lib = _lib.load()
    act = torch.empty(lib.itq3_mmq_act_nbytes(a.cols, a.m), dtype=torch.uint8, device=dev)
    Y = torch.empty((a.rows, a.m), dtype=torch.float32, device=dev)
    wsn = lib.itq3_mmq_ws_nbytes(a.rows, a.cols, a.m)
    ws = torch.empty(max(wsn, 1), dtype=torch.uint8, device=dev)
    s = _lib.stream_ptr(dev)
    rot = lambda: _lib.call("itq3_rotate_act_f16", _lib.ptr(X), 0, a.cols, a.m, X.stride(0), X.stride(1),
                            _lib.ptr(act), None, s)
    mmq = lambda: _lib.call("itq3_mmq", _lib.ptr(q.mmq_layout()), a.rows, a.cols, 0, _lib.ptr(act), a.m,
                            _lib.ptr(Y), 0, Y.stride(0), Y.stride(1), _lib.ptr(ws) if wsn else None, s)
    for name, fn in (("rotate_act_f16", rot), ("mmq", mmq)):
        fn()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 100
        extra = f"  {2 * a.rows * a.cols * a.m / us / 1e6:.0f} TFLOP/s" if name == "mmq" else ""
        print(f"  {name}: {us:.1f} us{extra}")
    t = tr.view(-1, 16).cpu().numpy()
    used = t[:, 8] > 0
    t = t[used]
    print(f"{a.rows}x{a.cols} M={a.m}: {e0.elapsed_time(e1) * 1e3:.1f} us (rotate + mmq), {used.sum()} CTAs")
    for i, n in enumerate(NAMES):
        col = t[:, i]
        if i in (3, 4, 9):
            col = col[::2]
        print(f"  {n:18s} median {np.median(col):12.0f}  max {col.max():12.0f}")
    ch = np.median(t[:, 8])
    print(f"  cycles per chunk (prod_total / chunks): {np.median(t[:, 7]) / ch:.0f}")


if __name__ == "__main__":
    main()
