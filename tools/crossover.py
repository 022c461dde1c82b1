"""Where does the tensor-core MMQ (K5) overtake the mma.sync GEMV (K3+K4) as the token count M grows?

    python tools/crossover.py
Times both device paths (rotate + multiply, CUDA events, 20 reps, >= 160 MB of distinct weight copies
rotated so the weights stream from HBM) at Llama-3-8B shapes, M = 1..128.
"""
import json
import os
import sys

import torch


def graph_time(fn, reps):
    """GPU time per call of fn(i): the reps calls are captured in one CUDA graph and replayed, so host
    launch overhead (ctypes + driver, ~5-7 us per launch) is off the measured path."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for i in range(3):
            fn(i)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_27914_b200 as P  # noqa: E402
from paper_2603_27914_b200 import _lib  # noqa: E402

SHAPES = [(4096, 4096), (14336, 4096), (4096, 14336)]
MS = [1, 2, 4, 8, 16, 24, 32, 48, 64, 96, 128]


def main():
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    out = []
    for rows, K in SHAPES:
        g = torch.Generator(device=dev)
        g.manual_seed(rows + K)
        ncopy = min(8, max(2, int(160e6 // (rows * K * 66 / 256)) + 1))
        qs = [P.quantize_tensor(torch.randn((rows, K), generator=g, device=dev) / K ** 0.5) for _ in range(ncopy)]
        tiled = [q.tiled() for q in qs]
        mmq = [q.mmq_layout() for q in qs]
        mmq8 = [q.mmq8_layout() for q in qs]
        for M in MS:
            X = torch.randn((K, M), generator=g, device=dev)
            Y = torch.empty((rows, M), dtype=torch.float32, device=dev)
            limbs = 3 if M == 1 else 2
            act = torch.empty(lib.itq3_act_nbytes(K, M, limbs), dtype=torch.uint8, device=dev)
            actf = torch.empty(lib.itq3_mmq_act_nbytes(K, M), dtype=torch.uint8, device=dev)
            wsn = lib.itq3_mmq_ws_nbytes(rows, K, M)
            ws = torch.empty(max(wsn, 1), dtype=torch.uint8, device=dev)

            def gemv(i):
                s = _lib.stream_ptr(dev)
                _lib.call("itq3_rotate_act", _lib.ptr(X), _lib.F32, K, M, X.stride(0), X.stride(1), limbs,
                          _lib.ptr(act), s)
                _lib.call("itq3_gemv", _lib.ptr(tiled[i % ncopy]), rows, K, 0, _lib.ptr(act), M, limbs, _lib.ptr(Y),
                          _lib.F32, Y.stride(0), Y.stride(1), s)

            def mmqf(i):
                s = _lib.stream_ptr(dev)
                _lib.call("itq3_rotate_act_f16", _lib.ptr(X), _lib.F32, K, M, X.stride(0), X.stride(1),
                          _lib.ptr(actf), None, s)
                _lib.call("itq3_mmq", _lib.ptr(mmq[i % ncopy]), rows, K, 0, _lib.ptr(actf), M, _lib.ptr(Y), _lib.F32,
                          Y.stride(0), Y.stride(1), _lib.ptr(ws) if wsn else None, s)

            act8 = torch.empty(lib.itq3_mmq8_act_nbytes(K, M), dtype=torch.uint8, device=dev) if M <= 64 else None
            ws8n = lib.itq3_mmq8_ws_nbytes(rows, K, M) if M <= 64 else 0
            ws8 = torch.empty(max(ws8n, 1), dtype=torch.uint8, device=dev)

            def mmq8f(i):
                s = _lib.stream_ptr(dev)
                _lib.call("itq3_rotate_act_i8", _lib.ptr(X), _lib.F32, K, M, X.stride(0), X.stride(1), _lib.ptr(act8), None, s)
                _lib.call("itq3_mmq8", _lib.ptr(mmq8[i % ncopy]), rows, K, _lib.ptr(act8), M, _lib.ptr(Y), _lib.F32,
                          Y.stride(0), Y.stride(1), _lib.ptr(ws8) if ws8n else None, s)

            row = {"rows": rows, "K": K, "M": M}
            for name, fn in (("gemv_us", gemv), ("mmq_us", mmqf), ("mmq8_us", mmq8f)):
                if name == "mmq_us" and M < 8:
                    continue
                if name == "mmq8_us" and M > 64:
                    continue
                row[name] = graph_time(fn, 20) * 1000
            row["weight_gbps_gemv"] = rows * K * 66 / 256 / (row["gemv_us"] * 1e-6) / 1e9
            if "mmq8_us" in row:
                row["weight_gbps_mmq8"] = rows * K * 67 / 256 / (row["mmq8_us"] * 1e-6) / 1e9
            print(json.dumps(row), flush=True)
            out.append(row)
    return out


if __name__ == "__main__":
    main()
