"""K5b: small-batch MMQ on tcgen05.mma kind::i8 (csrc/mmq.cu) against the CPU oracle.

Each token column must lie within test_gpu_stack.chain_bound at L = 2 (the same integer rotation
with |q| <= 2^14, fp32 accumulation) of the exact fp64 product of the oracle-decoded weights.
Covers every block_n of the token tile (16 / 32 / 64), padding rows and tokens, split-K,
asymmetric zero-points, strided / bf16 inputs and bf16 outputs.
"""

import numpy as np
import pytest
import torch

from oracle import itq3_oracle as O
from test_gpu_stack import chain_bound

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")
from paper_2603_27914_b200 import _lib  # noqa: E402


def run_mmq8(q, X, out_dtype=torch.float32):
    lib = _lib.load()
    rows, cols = q.rows, q.cols
    M = X.shape[1]
    dev = X.device
    act = torch.empty(lib.itq3_mmq8_act_nbytes(cols, M), dtype=torch.uint8, device=dev)
    s = _lib.stream_ptr(dev)
    _lib.call("itq3_rotate_act_i8", _lib.ptr(X), _lib.TORCH_DTYPE_CODE[X.dtype], cols, M, X.stride(0), X.stride(1),
              _lib.ptr(act), None, s)
    Y = torch.empty((rows, M), dtype=out_dtype, device=dev)
    wsn = lib.itq3_mmq8_ws_nbytes(rows, cols, M)
    ws = torch.empty(max(wsn, 1), dtype=torch.uint8, device=dev)
    _lib.call("itq3_mmq8", _lib.ptr(q.mmq8_layout()), rows, cols, _lib.ptr(act), M, _lib.ptr(Y),
              _lib.TORCH_DTYPE_CODE[out_dtype], Y.stride(0), Y.stride(1), _lib.ptr(ws) if wsn else None, s)
    return Y


@pytest.mark.parametrize("rows,cols,M,asym", [
    (256, 512, 16, False), (300, 1024, 5, False), (128, 4096, 32, True), (1000, 768, 64, False),
    (4096, 4096, 24, False), (513, 2048, 63, True), (14336, 256, 2, False),
])
def test_mmq8_matches_oracle(rows, cols, M, asym):
    g = torch.Generator(device="cuda")
    g.manual_seed(rows * 7 + cols + M)
    w = torch.randn((rows, cols), generator=g, device="cuda") / cols ** 0.5
    q = P.quantize_tensor(w, P.QuantConfig(symmetric=not asym))
    X = torch.randn((cols, M), generator=g, device="cuda")
    Y = run_mmq8(q, X).cpu().numpy().astype(np.float64)
    pay = q.payload().cpu().numpy()
    Xn = X.cpu().numpy().astype(np.float64)
    for m in range(M):
        exact, bound = chain_bound(pay, rows, cols, Xn[:, m], limbs=2)
        err = np.abs(Y[:, m] - exact)
        assert np.all(err <= bound), (m, float(np.max(err / bound)))


def test_mmq8_strided_bf16_and_determinism():
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    q = P.quantize_tensor(torch.randn((640, 1536), generator=g, device="cuda") / 40)
    Xt = torch.randn((40, 1536), generator=g, device="cuda")
    X = Xt.t()  # strided (cols x M) view
    Y1 = run_mmq8(q, X)
    Y2 = run_mmq8(q, X.contiguous())
    assert torch.equal(Y1, Y2)
    assert torch.equal(run_mmq8(q, X), Y1)  # deterministic
    Yb = run_mmq8(q, X.to(torch.bfloat16), out_dtype=torch.bfloat16).float()
    exact = torch.from_numpy(O.dequantize(q.payload().cpu().numpy(), 640, 1536, 256, False)).cuda().float() @ \
        X.to(torch.bfloat16).float()
    assert torch.allclose(Yb, exact, rtol=2e-2, atol=2e-2 * exact.abs().max().item())
