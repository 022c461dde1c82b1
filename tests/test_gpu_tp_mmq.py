"""GPU: row-sharded MMQ with the all-gather fused into the K5 epilogue (parallel.TPMatmul,
itq3_mmq_peers).  World 1 (the rank's own buffer as its only peer) must equal the plain K5 call bit for
bit (same shape, same split plan); worlds 2 and 3 are simulated on the one GPU with one buffer per
virtual rank: every rank's copy of Y is identical, complete, and within the K5 bound of the oracle
(a shard's K-split plan can differ from the full matrix's, so not bitwise equal to it)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")
from paper_2603_27914_b200 import _lib  # noqa: E402
from paper_2603_27914_b200.parallel import TPMatmul, shard_quantized  # noqa: E402
from test_gpu_mmq import mmq_bound  # noqa: E402


def unsharded(q, X):
    """The plain K5 call (itq3_mmq with its workspace) on the full matrix, rows x k fp32."""
    k = X.shape[1]
    act = torch.empty(_lib.load().itq3_mmq_act_nbytes(q.cols, k), dtype=torch.uint8, device=X.device)
    _lib.call("itq3_rotate_act_f16_n", _lib.ptr(X), _lib.F32, q.cols, k, X.stride(0), X.stride(1), q.block_n,
              _lib.ptr(act), None, _lib.stream_ptr(X.device))
    Y = torch.empty((q.rows, k), dtype=torch.float32, device=X.device)
    wsn = _lib.load().itq3_mmq_ws_nbytes(q.rows, q.cols, k)
    ws = torch.empty(wsn, dtype=torch.uint8, device=X.device) if wsn else None
    _lib.call("itq3_mmq", _lib.ptr(q.mmq_layout()), q.rows, q.cols, q.mmq_flags(), _lib.ptr(act), k, _lib.ptr(Y),
              _lib.F32, Y.stride(0), Y.stride(1), _lib.ptr(ws) if ws is not None else None, _lib.stream_ptr(X.device))
    return Y


@pytest.mark.parametrize("m", [16, 100, 300])
@pytest.mark.parametrize("world", [1, 2, 3])
def test_tp_mmq_peer_stores(world, m):
    rows, cols = 1000, 1024
    rng = np.random.default_rng(world * 100 + m)
    q = P.quantize_tensor(rng.standard_normal((rows, cols)) * 0.05)
    X = torch.from_numpy(rng.standard_normal((cols, m)).astype(np.float32)).cuda()
    ref = unsharded(q, X)
    if world == 1:
        tp = TPMatmul(q, rows, 512)
        Y = tp(X)
        torch.cuda.synchronize()
        torch.testing.assert_close(Y, ref, rtol=0, atol=0)
        exact, bound = mmq_bound(q.payload().cpu().numpy(), rows, cols, X.cpu().numpy())
        assert np.all(np.abs(Y.cpu().numpy() - exact) <= bound)
        # double-buffered by call parity: the next call writes the other half, Y stays intact
        Y2 = tp(2 * X)
        torch.cuda.synchronize()
        assert Y2.data_ptr() != Y.data_ptr()
        torch.testing.assert_close(Y, ref, rtol=0, atol=0)
        assert tp(X).data_ptr() == Y.data_ptr()
        return
    bufs = [torch.full((2 * rows * 512,), float("nan"), dtype=torch.float32, device="cuda") for _ in range(world)]
    bases = [b.data_ptr() for b in bufs]
    tps = [TPMatmul(shard_quantized(q, world, r), rows, 512, world=world, rank=r, ybuf=bufs[r], peer_bases=bases)
           for r in range(world)]
    for tp in tps:
        tp.launch(X)
    torch.cuda.synchronize()
    y0 = bufs[0][: rows * m].view(rows, m)
    for r in range(1, world):
        torch.testing.assert_close(bufs[r][: rows * m].view(rows, m), y0, rtol=0, atol=0)
    exact, bound = mmq_bound(q.payload().cpu().numpy(), rows, cols, X.cpu().numpy())
    assert np.all(np.abs(y0.cpu().numpy() - exact) <= bound)  # also: no NaN left from the fill


@pytest.mark.parametrize("m", [40, 300])
def test_tp_mmq_peer_stores_bf16(m):
    """bf16 outputs through the peer-store epilogue (two simulated ranks, each computing half the rows
    and writing both buffers): every copy equals the plain K5 call's bf16 output of the same rows."""
    rows, cols, world = 768, 1024, 2
    rng = np.random.default_rng(m)
    q = P.quantize_tensor(rng.standard_normal((rows, cols)) * 0.05)
    X = torch.from_numpy(rng.standard_normal((cols, m)).astype(np.float32)).cuda()
    lib = _lib.load()
    act = torch.empty(lib.itq3_mmq_act_nbytes(cols, m), dtype=torch.uint8, device="cuda")
    _lib.call("itq3_rotate_act_f16", _lib.ptr(X), _lib.F32, cols, m, X.stride(0), X.stride(1), _lib.ptr(act), None,
              _lib.stream_ptr(X.device))
    bufs = [torch.full((rows, m), float("nan"), dtype=torch.bfloat16, device="cuda") for _ in range(world)]
    peers = torch.tensor([b.data_ptr() for b in bufs], dtype=torch.int64, device="cuda")
    for r in range(world):
        shard = shard_quantized(q, world, r)
        r0 = r * (rows // world)
        _lib.call("itq3_mmq_peers", _lib.ptr(shard.mmq_layout()), shard.rows, cols, 0, _lib.ptr(act), m,
                  _lib.ptr(peers), world, r0, _lib.BF16, m, 1, None, _lib.stream_ptr(X.device))
    ref = torch.empty((rows, m), dtype=torch.bfloat16, device="cuda")
    _lib.call("itq3_mmq", _lib.ptr(q.mmq_layout()), rows, cols, 0, _lib.ptr(act), m, _lib.ptr(ref), _lib.BF16, m, 1,
              None, _lib.stream_ptr(X.device))
    torch.cuda.synchronize()
    for b in bufs:
        torch.testing.assert_close(b, ref, rtol=0, atol=0)
