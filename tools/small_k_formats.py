"""fused_matmul at k = 1 / 4 for variant ss and block_n 64 (4096 x 4096): the zero-padded K5 path (CUDA fp32
X) next to the exact fp64 generic kernel these formats used before (CUDA fp64 X takes it), device-timed."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_27914_b200 as P  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1000


def main():
    rng = np.random.default_rng(0)
    w = torch.from_numpy(rng.standard_normal((4096, 4096)).astype(np.float32) * 0.02).cuda()
    for fmt in (dict(variant="ss"), dict(block_n=64)):
        q = P.quantize_tensor(w, P.QuantConfig(**fmt))
        for k in (1, 4):
            X = torch.randn((4096, k), device="cuda")
            fast = timed(lambda: P.fused_matmul(q, X, check_finite=False))
            exact = timed(lambda: P.fused_matmul(q, X.double(), check_finite=False), reps=3)
            print(f"{fmt} k={k}: K5 (padded to 8) {fast:8.1f} us   exact fp64 generic {exact:9.1f} us")


if __name__ == "__main__":
    main()
