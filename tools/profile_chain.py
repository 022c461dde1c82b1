"""Run the chain kernel a few times for ncu (optionally in independent-stage mode)."""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2603_27914_b200.stack import LinearStack  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--independent", action="store_true")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
dev = torch.device("cuda", 0)
st = bench.build_stack(a.layers, 1000, dev, "chain")
if a.independent:
    st = LinearStack(st.qs, limbs=3, mode="chain", independent=True)
x = np.random.default_rng(0).standard_normal(st.x.numel()).astype(np.float32)
for _ in range(a.reps):
    st.x.copy_(torch.from_numpy(x))
    st.launch_all()
torch.cuda.synchronize()
print("done")
