"""Generate the golden fixtures from the REAL reference package (run in the build container).

    python tests/golden/make_golden.py [--full]

Imports ``itq3`` from /root/reference/pkg/src (read-only, never copied) and writes
  * tests/golden/small_cases.npz   -- container bytes / dequant / matvec / matmul outputs
                                      for ~100 small seeded tensors over every block size,
                                      variant, zero-point mode and scale policy;
  * tests/golden/full_digests.json -- (--full) SHA-256 of the reference container bytes
                                      and dequantised tensor at config C1 (4096x4096) plus
                                      the eval_error eps_q fields;
  * tests/golden/gemv_c2_*.npy      -- (--full) reference fused_matvec outputs at the C2
                                      shapes, and a fused_matmul output at a C3 row sample.
Inputs are regenerated on the GPU box from seeds with numpy (same image), and the
input digests are stored so a drift in numpy's generators is caught, not silent.
"""

from __future__ import annotations

import argparse
import hashlib
import io
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from cases import case_inputs, case_list  # noqa: E402


def sha(b) -> str:
    if isinstance(b, np.ndarray):
        b = np.ascontiguousarray(b).tobytes()
    return hashlib.sha256(b).hexdigest()


def container(itq3, q) -> bytes:
    buf = io.BytesIO()
    itq3.write_container(q, buf)
    return buf.getvalue()


def small_cases(itq3):
    from itq3.codec import QuantConfig
    from itq3.quantizer import ScalePolicy

    out = {}
    meta = []
    for i, c in enumerate(case_list()):
        w, x, X = case_inputs(i, tuple(c["shape"]), c["dist"])
        cfg = QuantConfig(block_n=c["block_n"], variant=c["variant"], symmetric=c["symmetric"],
                          policy=ScalePolicy(kind=c["policy"]))
        q = itq3.quantize_tensor(w, cfg)
        key = c["key"]
        deq = itq3.dequantize_tensor(q)
        out[key + "_container"] = np.frombuffer(container(itq3, q), np.uint8)
        out[key + "_y"] = itq3.fused_matvec(q, x)
        out[key + "_Y"] = itq3.fused_matmul(q, X)
        c = dict(c, w_sha256=sha(w), deq_sha256=sha(deq), deq_signbit_sha256=sha(np.signbit(deq)))
        meta.append(c)
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **out)
    with open(os.path.join(HERE, "small_cases.json"), "w") as f:
        json.dump(meta, f, indent=1)
    print(f"small cases: {len(meta)}")


def full(itq3):
    from itq3.codec import QuantConfig
    from itq3.compute import generate_weights

    digests = {"inputs": {}, "c1": [], "c2": [], "c3": []}
    for dist in ("gaussian", "outlier"):
        w = generate_weights(dist, 4096, 4096, seed=0).astype(np.float32)
        digests["inputs"][f"{dist}_4096x4096_seed0_f32"] = sha(w)
        combos = [("s", True), ("ss", True)] + ([("s", False)] if dist == "gaussian" else [])
        for variant, sym in combos:
            t = time.time()
            cfg = QuantConfig(variant=variant, symmetric=sym)
            q = itq3.quantize_tensor(w, cfg)
            data = container(itq3, q)
            deq = itq3.dequantize_tensor(q)
            r = itq3.eval_error(w, cfg)
            digests["c1"].append(dict(dist=dist, rows=4096, cols=4096, variant=variant, symmetric=sym,
                                      container_sha256=sha(data), container_len=len(data),
                                      dequant_f64_sha256=sha(deq),
                                      dequant_f32_sha256=sha(deq.astype(np.float32)),
                                      mse=r.mse, frobenius_rel=r.frobenius_rel,
                                      zero_fraction=r.zero_fraction, clamp_fraction=r.clamp_fraction))
            print(dist, variant, sym, f"{time.time() - t:.1f}s")
    # C2 GEMV at Llama-2-7B shapes (rows x cols, K = cols)
    for rows, cols in ((4096, 4096), (4096, 11008)):
        t = time.time()
        w = generate_weights("gaussian", rows, cols, seed=0).astype(np.float32)
        x = np.random.default_rng(1).standard_normal(cols).astype(np.float32)
        q = itq3.quantize_tensor(w, QuantConfig())
        data = container(itq3, q)
        y = itq3.fused_matvec(q, x)
        name = f"gemv_c2_{rows}x{cols}.npy"
        np.save(os.path.join(HERE, name), y)
        digests["c2"].append(dict(rows=rows, cols=cols, input_sha256=sha(w), x_sha256=sha(x),
                                  container_sha256=sha(data), y_file=name))
        print("gemv", rows, cols, f"{time.time() - t:.1f}s")
    # C3 MMQ sample: 256 rows of a Llama-3-8B (14336 x 4096) layer at M = 16
    t = time.time()
    w = generate_weights("gaussian", 256, 4096, seed=3).astype(np.float32)
    X = np.random.default_rng(2).standard_normal((4096, 16)).astype(np.float32)
    q = itq3.quantize_tensor(w, QuantConfig())
    Y = itq3.fused_matmul(q, X)
    np.save(os.path.join(HERE, "mmq_c3_256x4096_m16.npy"), Y)
    digests["c3"].append(dict(rows=256, cols=4096, m=16, input_sha256=sha(w), x_sha256=sha(X),
                              container_sha256=sha(container(itq3, q)), y_file="mmq_c3_256x4096_m16.npy"))
    print("mmq sample", f"{time.time() - t:.1f}s")
    with open(os.path.join(HERE, "full_digests.json"), "w") as f:
        json.dump(digests, f, indent=1)


# Extra C3 row samples (rows x K, M, weight seed): embedded by tests/test_gpu_c3_shapes.py into the
# LAST rows of a full Llama-3-8B-shaped layer, so the reference's outputs pin the kernels at the
# shapes the sweep times (K5 for M = 128 / 1024 / 2048, K5b for M = 64).
C3_EXTRA = [(256, 4096, 128, 4), (128, 4096, 2048, 5), (128, 14336, 64, 6), (128, 14336, 1024, 7)]


def c3_extra(itq3):
    from itq3.codec import QuantConfig
    from itq3.compute import generate_weights

    path = os.path.join(HERE, "full_digests.json")
    with open(path) as f:
        digests = json.load(f)
    digests["c3"] = digests["c3"][:1]
    for rows, cols, m, seed in C3_EXTRA:
        t = time.time()
        w = generate_weights("gaussian", rows, cols, seed=seed).astype(np.float32)
        X = np.random.default_rng(seed + 100).standard_normal((cols, m)).astype(np.float32)
        q = itq3.quantize_tensor(w, QuantConfig())
        Y = itq3.fused_matmul(q, X)
        name = f"mmq_c3_{rows}x{cols}_m{m}.npy"
        np.save(os.path.join(HERE, name), Y)
        digests["c3"].append(dict(rows=rows, cols=cols, m=m, seed=seed, x_seed=seed + 100, input_sha256=sha(w),
                                  x_sha256=sha(X), container_sha256=sha(container(itq3, q)), y_file=name))
        print("mmq sample", rows, cols, m, f"{time.time() - t:.1f}s")
    with open(path, "w") as f:
        json.dump(digests, f, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--full-only", action="store_true")
    ap.add_argument("--c3-extra", action="store_true", help="only (re)generate the extra C3 row samples")
    args = ap.parse_args()
    sys.path.insert(0, REF)
    import itq3  # noqa: E402  (the reference, read-only)

    if args.c3_extra:
        c3_extra(itq3)
        return
    if not args.full_only:
        small_cases(itq3)
    if args.full or args.full_only:
        full(itq3)
        c3_extra(itq3)


if __name__ == "__main__":
    main()
