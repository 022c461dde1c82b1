"""Multi-process (world_size 2, gloo, CPU) tests of the row-sharded path (parallel.py).

The sharding, payload slicing, padding and all-gather logic run for real across 2 processes; the
local product is the CPU oracle injected as `local_fn` (the CUDA kernel is the single-GPU path
tested in tests/test_gpu_*.py).  Checks: the gathered output equals the unsharded product (to BLAS blocking, 1e-12),
the chain composes, and per-rank encoding concatenates to the bit-exact full container.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import itq3_oracle as O


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class FakeQ:
    """Duck-typed QuantizedTensor for CPU: payload as a torch uint8 tensor."""

    def __init__(self, payload, rows, cols):
        self._payload = torch.from_numpy(np.ascontiguousarray(payload))
        self._validated = True
        self.rows, self.cols, self.block_n, self.variant, self.symmetric = rows, cols, 256, "s", True

    def payload(self):
        return self._payload


def oracle_local(shard, X):
    p = shard.payload().numpy()
    return torch.from_numpy(O.fused_matmul(p, shard.rows, shard.cols, 256, False, X.numpy()))


def _worker(rank, world, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2603_27914_b200.parallel as par

    # monkeypatch QuantizedTensor construction inside shard_quantized with the CPU duck type
    def shard_cpu(q, world_, rank_):
        r0, r1 = par.shard_bounds(q.rows, world_, rank_)
        nbr = q.cols // 256
        return FakeQ(q.payload().numpy()[r0 * nbr:r1 * nbr], r1 - r0, q.cols)

    par.shard_quantized = shard_cpu
    rng = np.random.default_rng(0)
    shapes = [(300, 512), (512, 256), (130, 512)]
    qs, ws = [], []
    for r, c in shapes:
        w = rng.standard_normal((r, c))
        pay, _ = O.quantize_payload(w)
        qs.append(FakeQ(pay, r, c))
        ws.append(w)
    x = torch.from_numpy(rng.standard_normal(512))
    # single linear
    lin = par.ShardedLinear(qs[0], local_fn=oracle_local)
    y = lin(x)
    full = O.fused_matmul(qs[0].payload().numpy(), 300, 512, 256, False, x.numpy()[:, None])[:, 0]
    ok1 = bool(np.allclose(y.numpy(), full, rtol=1e-12, atol=1e-12))  # BLAS blocking differs by shape
    # chain
    chain = par.ShardedChain(qs, local_fn=oracle_local)
    yc = chain(x).numpy()
    ref = x.numpy()
    for q in qs:
        ref = O.fused_matmul(q.payload().numpy(), q.rows, q.cols, 256, False, ref[: q.cols, None])[:, 0]
    ok2 = bool(np.allclose(yc, ref, rtol=1e-10, atol=1e-12))
    # per-rank encoding of the row shard concatenates to the full container bytes
    r0, r1 = par.shard_bounds(300, world, rank)
    mine, _ = O.quantize_payload(ws[0][r0:r1])
    gathered = [None] * world
    dist.all_gather_object(gathered, mine.tobytes())
    ok3 = b"".join(gathered) == qs[0].payload().numpy().tobytes()
    results[rank] = (ok1, ok2, ok3)
    dist.destroy_process_group()


def test_row_sharded_gather_world2():
    world = 2
    mgr = mp.Manager()
    results = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), results), nprocs=world, join=True)
    assert len(results) == world
    for r in range(world):
        assert results[r] == (True, True, True), (r, results[r])


@pytest.mark.parametrize("rows,world", [(300, 2), (4096, 8), (7, 4), (28672, 8)])
def test_shard_bounds_cover_rows(rows, world):
    from paper_2603_27914_b200.parallel import shard_bounds

    spans = [shard_bounds(rows, world, r) for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == rows
    for (a0, a1), (b0, b1) in zip(spans, spans[1:]):
        assert a1 == b0 and a0 <= a1


def test_tp_chain_layout_and_descriptors():
    """Host side of the fused tensor-parallel chain: the symmetric y layout (2 parity halves x
    K-chunks x full rows per stage, same offsets on every rank) and the descriptor checks of
    itq3_chain_write_desc_tp (no GPU needed)."""
    import ctypes

    from paper_2603_27914_b200 import _lib
    from paper_2603_27914_b200.parallel import shard_bounds, tp_chain_layout

    rows, cols = [12288, 4096, 11008, 4096], [4096, 4096, 4096, 11008]
    offs, total = tp_chain_layout(rows, cols)
    assert offs == [0, 2 * 12288, 2 * 12288 + 2 * 4096, 2 * 12288 + 2 * 4096 + 2 * 11008]
    assert total == offs[-1] + 2 * 3 * 4096  # cols 11008 -> 3 K-chunks of 4096
    lib = _lib.load()
    nd = lib.itq3_chain_desc_nbytes()
    host = ctypes.create_string_buffer(nd * 4)
    peers = 0x1000  # device address of the peer table: only stored, never dereferenced here
    for world in (2, 8):
        for rank in range(world):
            for i in range(4):
                r0, r1 = shard_bounds(rows[i], world, rank)
                assert lib.itq3_chain_write_desc_tp(host, i, None, 0x2000, r1 - r0, cols[i], 0, r0, rows[i],
                                                    peers, world) == 0
    # a shard running past the stage's rows, a missing peer table and too many peers are refused
    assert lib.itq3_chain_write_desc_tp(host, 0, None, 0x2000, 4096, 4096, 0, 10000, 12288, peers, 2) != 0
    assert lib.itq3_chain_write_desc_tp(host, 0, None, 0x2000, 4096, 4096, 0, 0, 12288, None, 2) != 0
    assert lib.itq3_chain_write_desc_tp(host, 0, None, 0x2000, 4096, 4096, 0, 0, 12288, peers, 9) != 0
    assert lib.itq3_chain_write_desc_tp(host, 0, None, 0x2000, 4096, 4000, 0, 0, 12288, peers, 2) != 0
