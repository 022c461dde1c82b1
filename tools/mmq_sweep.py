"""C3 sweep: batched MMQ (tcgen05, csrc/mmq.cu) at Llama-3-8B shapes x M = 16..2048.

    python tools/mmq_sweep.py [--out profiles/r01/mmq_sweep.json]
Times itq3_rotate_act_f16 + itq3_mmq with CUDA events over a CUDA graph of 20 calls (host launch
overhead excluded; weights of
>= 2 distinct copies rotated to defeat L2 at small M), reports TFLOPS = 2*rows*K*M / t and the
fraction of the measured dense bf16/f16 peak (MEASURED_PEAKS.json).
"""
import argparse
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

SHAPES = [(4096, 4096), (1024, 4096), (14336, 4096), (4096, 14336)]
MS = [16, 32, 64, 128, 256, 512, 1024, 2048]


def M_SMALL(m):
    return P.compute.MMQ_MIN_TOKENS <= m <= P.compute.MMQ8_MAX_TOKENS


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    except (OSError, KeyError, ValueError):
        peak = 1590.0  # B200_PROFILING.md's fallback dense bf16 figure
    lib = _lib.load()
    res = []
    for rows, K in SHAPES:
        g = torch.Generator(device=dev)
        g.manual_seed(rows + K)
        copies = []
        ncopy = max(2, int(160e6 // (rows * K * 66 / 256)) + 1)
        for c in range(min(ncopy, 8)):
            q = P.quantize_tensor(torch.randn((rows, K), generator=g, device=dev) / K ** 0.5)
            copies.append((q.mmq_layout(), q.mmq8_layout()))
        for M in MS:
            X = torch.randn((K, M), generator=g, device=dev)
            kinds = (["i8"] if M_SMALL(M) else []) + (["f16"] if M >= 32 else [])
            for kind in kinds:
                small = kind == "i8"
                act = torch.empty(lib.itq3_mmq8_act_nbytes(K, M) if small else lib.itq3_mmq_act_nbytes(K, M),
                                  dtype=torch.uint8, device=dev)
                Y = torch.empty((rows, M), dtype=torch.float32, device=dev)
                wsn = lib.itq3_mmq8_ws_nbytes(rows, K, M) if small else lib.itq3_mmq_ws_nbytes(rows, K, M)
                ws = torch.empty(max(wsn, 1), dtype=torch.uint8, device=dev)

                def rot(i):
                    s = _lib.stream_ptr(dev)
                    if small:
                        _lib.call("itq3_rotate_act_i8", _lib.ptr(X), _lib.F32, K, M, X.stride(0), X.stride(1),
                                  _lib.ptr(act), None, s)
                    else:
                        _lib.call("itq3_rotate_act_f16", _lib.ptr(X), _lib.F32, K, M, X.stride(0), X.stride(1),
                                  _lib.ptr(act), None, s)

                def mm(i):
                    s = _lib.stream_ptr(dev)
                    if small:  # K5b, kind::i8
                        _lib.call("itq3_mmq8", _lib.ptr(copies[i % len(copies)][1]), rows, K, _lib.ptr(act), M,
                                  _lib.ptr(Y), _lib.F32, Y.stride(0), Y.stride(1), _lib.ptr(ws) if wsn else None, s)
                    else:  # K5, kind::f16 CTA pairs
                        _lib.call("itq3_mmq", _lib.ptr(copies[i % len(copies)][0]), rows, K, 0, _lib.ptr(act), M,
                                  _lib.ptr(Y), _lib.F32, Y.stride(0), Y.stride(1), _lib.ptr(ws) if wsn else None, s)

                def run(i):
                    rot(i)
                    mm(i)

                ms = graph_time(run, args.reps)
                ms_k = graph_time(mm, args.reps)
                tf = 2.0 * rows * K * M / (ms * 1e-3) / 1e12
                tf_k = 2.0 * rows * K * M / (ms_k * 1e-3) / 1e12
                wbytes = rows * K * 66 / 256
                r = {"rows": rows, "K": K, "M": M, "kernel": "K5b kind::i8" if small else "K5 kind::f16 pair",
                     "us": ms * 1e3, "tflops": tf, "frac_of_bf16_peak": tf / peak, "kernel_us": ms_k * 1e3,
                     "kernel_tflops": tf_k, "kernel_frac_of_bf16_peak": tf_k / peak,
                     "weight_gbps": wbytes / (ms * 1e-3) / 1e9}
                res.append(r)
                print(json.dumps(r), flush=True)
    if args.out:
        json.dump({"peak_bf16_tflops": peak, "results": res}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
