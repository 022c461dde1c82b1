"""GPU (world size 1): the tensor-parallel decode stack (parallel.TPStack) with its graph-captured
kernels equals the single-GPU per-stage chain (stack.LinearStack, mode="kernels") bit for bit.
The multi-rank sharding/gather logic is covered on CPU by tests/test_parallel_gloo.py."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")
from paper_2603_27914_b200.parallel import TPStack  # noqa: E402
from paper_2603_27914_b200.stack import LinearStack  # noqa: E402


def test_tp_world1_matches_linear_stack():
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    shapes = [(768, 512), (512, 512), (1300, 512), (512, 1280)]
    qs = [P.quantize_tensor(torch.randn((r, c), generator=g, device="cuda") / c ** 0.5) for r, c in shapes]
    tp = TPStack(qs, [r for r, _ in shapes], [c for _, c in shapes])
    ref = LinearStack(qs, mode="kernels")
    x = np.random.default_rng(0).standard_normal(512).astype(np.float32)
    tp.x.copy_(torch.from_numpy(x))
    tp.replay()
    y_tp = tp.output().cpu().numpy()
    y_ref = ref.forward(x)
    np.testing.assert_array_equal(y_tp, y_ref)
