"""Config C2: one batch-1 fused GEMV (Llama-2-7B shapes 4096x4096, 4096x11008) through the public API.

    python tools/gemv_c2.py [--out profiles/r01/gemv_c2.json]
Device time: fused_matvec(q, x) on a CUDA x (one-stage chain kernel: in-kernel rotation + TMA weight
stream), 50 calls captured in a CUDA graph, over enough distinct weight copies (>= 200 MB) that
every call streams its weights from HBM.  Also the previous two-kernel path (K3 rotate + K4 GEMV)
for comparison, and the end-to-end call from a host numpy vector (H2D + kernel + D2H, fp64 parity
mode) as a user of the reference would make it.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_27914_b200 as P  # noqa: E402
from paper_2603_27914_b200 import _lib  # noqa: E402
from paper_2603_27914_b200.compute import _matvec_chain  # noqa: E402


def graph_time(fn, reps):
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    import bench  # noqa: E402  (the bench's peak: MEASURED_PEAKS.json, else the profiling guide's fallback)

    peak, peak_source = bench.measured_peak()
    res = []
    for rows, K in [(4096, 4096), (4096, 11008)]:
        g = torch.Generator(device=dev)
        g.manual_seed(rows + K)
        wbytes = rows * K * 66 // 256
        ncopy = int(200e6 // wbytes) + 1
        qs = [P.quantize_tensor(torch.randn((rows, K), generator=g, device=dev) / K ** 0.5) for _ in range(ncopy)]
        for q in qs:
            q.tiled()
        x = torch.randn(K, generator=g, device=dev)
        lib = _lib.load()
        act = torch.empty(lib.itq3_act_nbytes(K, 1, 3), dtype=torch.uint8, device=dev)
        y = torch.empty(rows, dtype=torch.float32, device=dev)

        def chain(i):
            _matvec_chain(qs[i % ncopy], x[:, None])

        def two_kernels(i):
            s = _lib.stream_ptr(dev)
            _lib.call("itq3_rotate_act", _lib.ptr(x), _lib.F32, K, 1, 1, K, 3, _lib.ptr(act), s)
            _lib.call("itq3_gemv", _lib.ptr(qs[i % ncopy].tiled()), rows, K, 0, _lib.ptr(act), 1, 3, _lib.ptr(y),
                      _lib.F32, 1, 1, s)

        for i in range(ncopy):  # build each tensor's chain context outside graph capture
            chain(i)
        t_chain = graph_time(chain, 50)
        t_two = graph_time(two_kernels, 50)
        xh = np.random.default_rng(0).standard_normal(K)
        P.fused_matvec(qs[0], xh)
        t0 = time.perf_counter()
        for _ in range(20):
            P.fused_matvec(qs[0], xh)
        e2e = (time.perf_counter() - t0) / 20
        r = {"rows": rows, "K": K, "packed_bytes": wbytes, "copies": ncopy,
             "chain_us": t_chain * 1e3, "chain_gbps": wbytes / (t_chain * 1e-3) / 1e9,
             "chain_frac_hbm": wbytes / (t_chain * 1e-3) / 1e9 / peak,
             "two_kernel_us": t_two * 1e3, "two_kernel_gbps": wbytes / (t_two * 1e-3) / 1e9,
             "e2e_parity_host_us": e2e * 1e6}
        print(json.dumps(r), flush=True)
        res.append(r)
    if args.out:
        json.dump({"hbm_peak_gbs": peak, "peak_source": peak_source, "results": res}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
