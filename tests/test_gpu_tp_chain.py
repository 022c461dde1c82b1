"""GPU: the fused tensor-parallel chain (parallel.TPChainStack; the all-gather is the reducers'
peer stores, csrc/chain.cu) is bit-exact with the single-GPU chain.  World 1 runs in-process; world 2
and 4 are simulated on the one GPU by tools/tp_chain_sim.py (co-resident cooperative kernels, one per
virtual rank, exchanging stage outputs through the peer-store path), in a subprocess with a watchdog."""

import os
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")
from paper_2603_27914_b200.parallel import TPChainStack  # noqa: E402
from paper_2603_27914_b200.stack import LinearStack  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_tp_chain_world1_matches_chain():
    g = torch.Generator(device="cuda")
    g.manual_seed(11)
    shapes = [(768, 512), (512, 768), (5120, 512), (512, 5120)]
    qs = [P.quantize_tensor(torch.randn((r, c), generator=g, device="cuda") / c ** 0.5) for r, c in shapes]
    rows, cols = [r for r, _ in shapes], [c for _, c in shapes]
    tp = TPChainStack(qs, rows, cols)
    ref = LinearStack(qs, mode="chain", lo=False)
    rng = np.random.default_rng(2)
    for _ in range(3):  # graph replays alternate the epoch-parity halves of y
        x = rng.standard_normal(512).astype(np.float32)
        tp.x.copy_(torch.from_numpy(x))
        tp.replay()
        np.testing.assert_array_equal(tp.output().cpu().numpy(), ref.forward(x))


@pytest.mark.parametrize("args", [["--ranks", "2"], ["--ranks", "4", "--asym"]])
def test_tp_chain_simulated_ranks(args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tp_chain_sim.py"), "--timeout", "60", *args],
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "bit-exact" in r.stdout
