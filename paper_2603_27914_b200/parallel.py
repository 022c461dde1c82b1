"""Row-sharded (column-parallel) ITQ3_S linears across GPUs with an output all-gather.

SURVEY.md §8(e): output rows are independent -- y_r needs only row r's blocks and the full x -- so
with cols % block_n == 0 every row is a run of whole blocks and GPU g owns the contiguous payload
slice of rows [r0_g, r1_g).  Encoding shards the same way (concatenating the ranks' containers in
rank order is bit-exact with encoding the full matrix).  x is replicated; the only collective is the
all-gather of y (NCCL over NVLink via torch.distributed, one process per GPU).

The local product is the single-GPU fused kernel (K4 GEMV / K5 MMQ).  `local_fn` can be injected so
the sharding/gather logic is testable with the gloo backend on CPU (tests/test_parallel_gloo.py).
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from .codec import QuantizedTensor, block_nbytes
from .errors import ShapeError


def shard_bounds(rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous row range of `rank`: ceil-divided so all ranks but the last hold equal shards."""
    per = -(-rows // world)
    r0 = min(rows, rank * per)
    return r0, min(rows, r0 + per)


def shard_quantized(q: QuantizedTensor, world: int, rank: int) -> QuantizedTensor:
    """The rows [r0, r1) of q as a standalone QuantizedTensor (payload slice, no re-encoding)."""
    if q.cols % q.block_n:
        raise ShapeError("shard_quantized: rows must be whole blocks (cols % block_n == 0)")
    r0, r1 = shard_bounds(q.rows, world, rank)
    nbr = q.cols // q.block_n
    p = q.payload() if q._payload is None or q._payload.is_cuda else q._payload
    return QuantizedTensor(r1 - r0, q.cols, q.block_n, q.variant, q.symmetric, 0, payload=p[r0 * nbr:r1 * nbr],
                           validated=q._validated)


def assemble_payload(shards: list[torch.Tensor], n: int, ss: bool) -> torch.Tensor:
    """Concatenate rank payloads in rank order (bit-exact with the unsharded payload)."""
    bs = block_nbytes(n, ss)
    for s in shards:
        if s.shape[-1] != bs:
            raise ShapeError("assemble_payload: block size mismatch")
    return torch.cat(shards, dim=0)


class ShardedLinear:
    """One row-sharded linear: y = all_gather(local rows of w_hat @ x)."""

    def __init__(self, q: QuantizedTensor, group=None, local_fn=None):
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.rows, self.cols = q.rows, q.cols
        self.r0, self.r1 = shard_bounds(q.rows, self.world, self.rank)
        self.per = -(-q.rows // self.world)
        self.shard = shard_quantized(q, self.world, self.rank) if self.world > 1 else q
        if local_fn is None:
            from .compute import fused_matmul

            local_fn = fused_matmul
        self.local_fn = local_fn

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        """x: (cols,) or (cols, k) on this rank's device; returns the full (rows[, k]) output."""
        vec = x.ndim == 1
        X = x[:, None] if vec else x
        y = self.local_fn(self.shard, X)  # (r1 - r0, k)
        if self.world == 1:
            return y[:, 0] if vec else y
        k = y.shape[1]
        buf = torch.zeros((self.per, k), dtype=y.dtype, device=y.device)
        buf[: y.shape[0]] = y
        out = torch.empty((self.per * self.world, k), dtype=y.dtype, device=y.device)
        dist.all_gather_into_tensor(out, buf, group=self.group)
        out = out[: self.rows]
        return out[:, 0] if vec else out


class ShardedChain:
    """A dependent chain of row-sharded linears (tensor-parallel decode step)."""

    def __init__(self, qs: list[QuantizedTensor], group=None, local_fn=None):
        for a, b in zip(qs, qs[1:]):
            if b.cols > a.rows:
                raise ShapeError("ShardedChain: stage input longer than the previous output")
        self.stages = [ShardedLinear(q, group, local_fn) for q in qs]

    def __call__(self, x: torch.Tensor) -> torch.Tensor:
        for st in self.stages:
            x = st(x[: st.cols])
        return x
