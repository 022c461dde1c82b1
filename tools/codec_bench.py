"""C1 codec throughput: K1 encode, K7 validate, K2 dequant (float32 / float64) on B200 vs the CPU oracle.

    python tools/codec_bench.py [--rows 4096 --cols 4096] [--big 16384] [--out profiles/r01/codec_bench.json]

Device times are CUDA events around graph-free back-to-back launches (after warm-up), on inputs of
the stated size; `--big` repeats the device legs on a big x big matrix (> 126 MB L2 in both directions).
Algorithmic bytes: encode = 4 B in (fp32) + 100/256 B out per weight; dequant =
100/256 B in + 4 (fp32) or 8 (fp64) B out per weight; validate = 100/256 B in per weight.  The CPU leg is
the oracle's vectorised encoder/decoder (numpy, 1 host thread) on the C1 matrix, checked byte-equal.
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
from oracle import itq3_oracle as O  # noqa: E402  (checker / CPU baseline only)


def dev_time(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3  # seconds


def legs(rows, cols, dev, peak):
    n = rows * cols
    nb = n // 256
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    w = torch.randn((rows, cols), generator=g, device=dev, dtype=torch.float32)
    payload = torch.empty((nb, 100), dtype=torch.uint8, device=dev)
    s = _lib.stream_ptr(dev)
    enc = lambda: _lib.call("itq3_encode", _lib.ptr(w), _lib.F32, n, 256, 0, 0, P.ScalePolicy().coefficient(), 1,
                            _lib.ptr(payload), s)
    word = _lib.first_bad_word(dev)
    mask = _lib.CHECK_PLANES | _lib.CHECK_SCALE_NAN | _lib.CHECK_ZP | _lib.CHECK_SUB_NAN
    val = lambda: _lib.call("itq3_validate", _lib.ptr(payload), nb, 256, 0, mask, _lib.ptr(word), s)
    out32 = torch.empty(n, dtype=torch.float32, device=dev)
    out64 = torch.empty(n, dtype=torch.float64, device=dev)
    dq32 = lambda: _lib.call("itq3_dequant", _lib.ptr(payload), nb, 256, 0, n, _lib.ptr(out32), _lib.F32, s)
    dq64 = lambda: _lib.call("itq3_dequant", _lib.ptr(payload), nb, 256, 0, n, _lib.ptr(out64), _lib.F64, s)
    res = {}
    for name, fn, bpw in (("encode_f32", enc, 4 + 100 / 256), ("validate", val, 100 / 256),
                          ("dequant_f32", dq32, 100 / 256 + 4), ("dequant_f64", dq64, 100 / 256 + 8)):
        t = dev_time(fn)
        gbs = n * bpw / t / 1e9
        res[name] = {"us": t * 1e6, "gweights_per_s": n / t / 1e9, "algorithmic_gbps": gbs,
                     "hbm_frac": gbs / peak, "blocks_per_s": nb / t}
    assert _lib.read_first_bad(word) is None
    return w, payload, res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows", type=int, default=4096)
    ap.add_argument("--cols", type=int, default=4096)
    ap.add_argument("--big", type=int, default=16384)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    w, payload, c1 = legs(a.rows, a.cols, dev, peak)
    # CPU oracle (1 thread, vectorised numpy) on the same C1 matrix; byte-equal check
    wc = w.cpu().numpy()
    t0 = time.perf_counter()
    ref_pay, _ = O.quantize_payload(wc)
    t_enc = time.perf_counter() - t0
    assert np.array_equal(ref_pay, payload.cpu().numpy()), "encoder bytes differ from the oracle"
    t0 = time.perf_counter()
    deq = O.dequantize(ref_pay, a.rows, a.cols, 256, False)
    t_dec = time.perf_counter() - t0
    out = {"c1": {"rows": a.rows, "cols": a.cols, "device": c1,
                  "cpu_oracle": {"encode_s": t_enc, "dequant_f64_s": t_dec, "cores": 1,
                                 "kind": "port (vectorised numpy restatement)",
                                 "speedup_encode": t_enc / (c1["encode_f32"]["us"] * 1e-6),
                                 "speedup_dequant_f64": t_dec / (c1["dequant_f64"]["us"] * 1e-6)},
                  "eps_q_frob_rel": float(np.linalg.norm(deq - wc) / np.linalg.norm(wc))},
           "peak_hbm_gbs": peak}
    if a.big:
        del w, payload
        torch.cuda.empty_cache()
        _, _, big = legs(a.big, a.big, dev, peak)
        out["big"] = {"rows": a.big, "cols": a.big, "device": big}
    print(json.dumps(out, indent=1))
    if a.out:
        json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
