"""eps_q evaluation throughput at config C1 (4096x4096 fp32): K8 (itq3_eval) vs the CPU oracle.

    python tools/eval_bench.py

Device timing with CUDA events (inputs resident), end-to-end timing from a host numpy array,
and the oracle's error_report (the reference's vectorised numpy harness restated) on one core.
"""

import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_27914_b200 as P  # noqa: E402
from paper_2603_27914_b200.evaluate import _EvalRun  # noqa: E402
from oracle import itq3_oracle as O  # noqa: E402


def main():
    rows = cols = 4096
    w = O.generate_weights("gaussian", rows, cols, seed=0).astype(np.float32)
    t = torch.from_numpy(w).cuda()
    cfg = P.QuantConfig()
    for _ in range(3):
        _EvalRun(t, 256, False, cfg.policy, True, None)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        _EvalRun(t, 256, False, cfg.policy, True, None)
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / reps
    t0 = time.perf_counter()
    r = P.eval_error(w, cfg)
    e2e_ms = (time.perf_counter() - t0) * 1e3
    t0 = time.perf_counter()
    ref = O.error_report(w)
    cpu_s = time.perf_counter() - t0
    assert r.mse == ref["mse"]
    nb = rows * cols // 256
    print(json.dumps({"workload": "eval_error C1 4096x4096 fp32, block 256 / s / constant",
                      "device_ms": dev_ms, "e2e_ms_from_host_numpy": e2e_ms, "cpu_oracle_s": cpu_s,
                      "cpu_cores": 1, "speedup_device_vs_cpu": cpu_s * 1e3 / dev_ms,
                      "blocks_per_s_device": nb / (dev_ms / 1e3),
                      "algorithmic_bytes_per_block": 1024 + 3 * 2048 + 3 * 2048,
                      "achieved_GBps": nb * (1024 + 12288) / (dev_ms / 1e3) / 1e9}))


if __name__ == "__main__":
    main()
