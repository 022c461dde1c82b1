"""Cost of the fused all-gather epilogue (itq3_mmq_peers) against the plain K5 MMQ on one GPU.

    python tools/tp_mmq_bench.py [--out profiles/r01/tp_mmq.json]

Per shape and M (workspace splits allowed in both): itq3_mmq (bulk row stores to one Y), itq3_mmq_peers with one
peer (the rank itself) and with 2 / 4 peers (extra copies on the same GPU stand in for NVLink peers:
HBM write traffic grows like the NVLink traffic would).  CUDA-graph timing of 20 calls, rotation excluded.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_27914_b200 as P  # noqa: E402
from paper_2603_27914_b200 import _lib  # noqa: E402
from mmq_sweep import graph_time  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    lib = _lib.load()
    res = []
    for rows, K in ((14336, 4096), (4096, 14336)):
        g = torch.Generator(device=dev)
        g.manual_seed(rows)
        q = P.quantize_tensor(torch.randn((rows, K), generator=g, device=dev) / K ** 0.5)
        mmq = q.mmq_layout()
        for M in (256, 2048):
            X = torch.randn((K, M), generator=g, device=dev)
            act = torch.empty(lib.itq3_mmq_act_nbytes(K, M), dtype=torch.uint8, device=dev)
            _lib.call("itq3_rotate_act_f16", _lib.ptr(X), _lib.F32, K, M, M, 1, _lib.ptr(act), None,
                      _lib.stream_ptr(dev))
            ys = [torch.empty((rows, M), dtype=torch.float32, device=dev) for _ in range(4)]
            wsn = lib.itq3_mmq_ws_nbytes(rows, K, M)
            ws = torch.empty(max(wsn, 1), dtype=torch.uint8, device=dev)
            row = {"rows": rows, "K": K, "M": M}
            plain = lambda i: _lib.call("itq3_mmq", _lib.ptr(mmq), rows, K, 0, _lib.ptr(act), M, _lib.ptr(ys[0]),
                                        _lib.F32, M, 1, _lib.ptr(ws) if wsn else None, _lib.stream_ptr(dev))
            row["mmq_us"] = graph_time(plain, 20) * 1000
            for npeer in (1, 2, 4):
                peers = torch.tensor([y.data_ptr() for y in ys[:npeer]], dtype=torch.int64, device=dev)
                fn = lambda i: _lib.call("itq3_mmq_peers", _lib.ptr(mmq), rows, K, 0, _lib.ptr(act), M,
                                         _lib.ptr(peers), npeer, 0, _lib.F32, M, 1, _lib.ptr(ws) if wsn else None,
                                         _lib.stream_ptr(dev))
                row[f"peers{npeer}_us"] = graph_time(fn, 20) * 1000
                if npeer > 1:
                    torch.testing.assert_close(ys[npeer - 1], ys[0], rtol=0, atol=0)
            row["tflops_mmq"] = 2.0 * rows * K * M / row["mmq_us"] / 1e6
            row["tflops_peers1"] = 2.0 * rows * K * M / row["peers1_us"] / 1e6
            print(json.dumps(row), flush=True)
            res.append(row)
    if a.out:
        json.dump({"results": res}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
