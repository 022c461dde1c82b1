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


class TPStack:
    """Tensor-parallel decode chain on CUDA: every stage is row-sharded over the process group,
    computed with the K3 rotate + K4 GEMV kernels on the local rows, and all-gathered with NCCL
    (all_gather_into_tensor over NVLink) into the replicated input of the next stage.  The whole
    step -- 2 kernels + 1 collective per stage -- is captured in one CUDA graph.

    `local_qs[i]` is this rank's QuantizedTensor of rows shard_bounds(rows_i, world, rank) of stage i
    (quantized locally: row shards encode bit-exactly like the full matrix, tests/test_parallel_gloo.py);
    `rows[i]`/`cols[i]` are the full stage shapes.
    """

    def __init__(self, local_qs, rows, cols, group=None, limbs: int = 3):
        from . import _lib

        self._lib = _lib
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.qs, self.rows, self.cols, self.limbs = local_qs, list(rows), list(cols), limbs
        for i in range(1, len(rows)):
            if cols[i] > rows[i - 1]:
                raise ShapeError("TPStack: stage input longer than the previous output")
        self.dev = _lib.device()
        lib = _lib.load()
        self.per = [-(-r // self.world) for r in rows]
        self.tiled = [q.tiled() for q in local_qs]
        self.x = torch.zeros(cols[0], dtype=torch.float32, device=self.dev)
        self.acts = [torch.empty(lib.itq3_act_nbytes(c, 1, limbs), dtype=torch.uint8, device=self.dev) for c in cols]
        self.ylocal = [torch.zeros(p, dtype=torch.float32, device=self.dev) for p in self.per]
        self.yfull = [torch.zeros(p * self.world, dtype=torch.float32, device=self.dev) for p in self.per]
        self.graph = None

    def launch_all(self):
        lib = self._lib
        s = lib.stream_ptr(self.dev)
        for i, q in enumerate(self.qs):
            xin = self.x if i == 0 else self.yfull[i - 1]
            lib.call("itq3_rotate_act", lib.ptr(xin), lib.F32, self.cols[i], 1, 1, self.cols[i], self.limbs,
                     lib.ptr(self.acts[i]), s)
            if q.rows > 0:
                lib.call("itq3_gemv", lib.ptr(self.tiled[i]), q.rows, q.cols, int(not q.symmetric), lib.ptr(self.acts[i]),
                         1, self.limbs, lib.ptr(self.ylocal[i]), lib.F32, 1, 1, s)
            if self.world > 1:
                dist.all_gather_into_tensor(self.yfull[i], self.ylocal[i], group=self.group)
            else:
                self.yfull[i].copy_(self.ylocal[i])

    def capture(self):
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            self.launch_all()
        torch.cuda.current_stream(self.dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch_all()
        self.graph = g

    def replay(self):
        if self.graph is None:
            self.capture()
        self.graph.replay()

    def output(self) -> torch.Tensor:
        return self.yfull[-1][: self.rows[-1]]


def tp_chain_layout(rows: list[int], cols: list[int]) -> tuple[list[int], int]:
    """Word offsets of each stage's tagged-output buffer inside one symmetric allocation, and the total.

    Stage i holds 2 (epoch parity) x nch_i (K-chunks of 4096) x rows_i u64 words -- the layout
    itq3_chain_write_desc_tp expects -- at the same offset on every rank, so rank p's copy of stage i
    is peer_base[p] + 8 * offset_i."""
    offs, total = [], 0
    for r, c in zip(rows, cols):
        offs.append(total)
        total += 2 * (-(-c // 4096)) * r
    return offs, total


class TPChainStack:
    """Tensor-parallel decode chain in ONE persistent kernel per rank, with the all-gather fused in.

    Every rank runs the cooperative chain kernel (csrc/chain.cu) over its row shards; the reducer of
    each stage stores its tagged output words directly into every rank's copy of the stage output
    (NVLink peer stores through torch symmetric-memory peer pointers), and the next stage's consumers
    on every rank spin on those tags exactly as in the single-GPU chain.  There is no NCCL call, no
    per-stage launch and no separate gather pass: the transfer of stage i overlaps stage i's math
    unit by unit (TPStack is the unfused NCCL baseline: 2 kernels + 1 all_gather per stage).

    `local_qs[i]`: this rank's rows shard_bounds(rows[i], world, rank) of stage i.  `peer_bases`
    (optional, testing): the per-rank base addresses of `ybuf` to use instead of a symmetric-memory
    rendezvous -- with world 1 the only peer is the rank itself.
    """

    def __init__(self, local_qs, rows, cols, group=None, limbs: int = 3, world: int | None = None,
                 rank: int | None = None, ybuf: torch.Tensor | None = None, peer_bases: list[int] | None = None,
                 grid: int = 0):
        import ctypes

        from . import _lib

        self._lib = _lib
        self.group = group
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world, self.rank = world, rank
        self.qs, self.rows, self.cols, self.limbs, self.grid = local_qs, list(rows), list(cols), limbs, grid
        if not local_qs:
            raise ShapeError("TPChainStack: no stages")
        for i in range(1, len(rows)):
            if cols[i] > rows[i - 1]:
                raise ShapeError("TPChainStack: stage input longer than the previous output")
        for i, q in enumerate(local_qs):
            r0, r1 = shard_bounds(rows[i], world, rank)
            if q.rows != r1 - r0 or q.cols != cols[i]:
                raise ShapeError(f"TPChainStack: stage {i} shard is {q.rows}x{q.cols}, expected {r1 - r0}x{cols[i]}")
            if not q.fast_layout():
                raise ShapeError("TPChainStack: stages need the tiled layout (block_n 256, variant s, cols % 256 == 0)")
        self.dev = _lib.device()
        lib = _lib.load()
        self.tiled = [q.tiled() for q in local_qs]
        self.offs, total = tp_chain_layout(self.rows, self.cols)
        if ybuf is None:
            if world > 1:
                from torch.distributed import _symmetric_memory as symm

                ybuf = symm.empty(total, dtype=torch.int64, device=self.dev)
                ybuf.zero_()
                hdl = symm.rendezvous(ybuf, group if group is not None else dist.group.WORLD)
                delta = ybuf.data_ptr() - hdl.buffer_ptrs[rank]  # tensor offset inside the symmetric block
                peer_bases = [b + delta for b in hdl.buffer_ptrs]
                torch.cuda.synchronize(self.dev)
                dist.barrier(group)  # every copy zeroed before any peer stores into it
            else:
                ybuf = torch.zeros(total, dtype=torch.int64, device=self.dev)
        if peer_bases is None:
            peer_bases = [ybuf.data_ptr()]
        if len(peer_bases) != world or peer_bases[rank] != ybuf.data_ptr():
            raise ShapeError("TPChainStack: peer_bases must list every rank's buffer, this rank's at index rank")
        self.ybuf = ybuf
        S = len(local_qs)
        self.peers = torch.tensor([[b + 8 * o for b in peer_bases] for o in self.offs], dtype=torch.int64,
                                  device=self.dev)
        host = ctypes.create_string_buffer(lib.itq3_chain_desc_nbytes() * S)
        for i, q in enumerate(local_qs):
            r0, _ = shard_bounds(rows[i], world, rank)
            _lib.check(lib.itq3_chain_write_desc_tp(host, i, _lib.ptr(self.tiled[i]),
                                                    ybuf.data_ptr() + 8 * self.offs[i], q.rows, q.cols,
                                                    int(not q.symmetric), r0, rows[i],
                                                    self.peers.data_ptr() + 8 * world * i, world))
        self.desc = torch.frombuffer(bytearray(host.raw), dtype=torch.uint8).to(self.dev)
        self.epoch = torch.zeros(2, dtype=torch.int32, device=self.dev)
        self.x = torch.zeros(cols[0], dtype=torch.float32, device=self.dev)
        self.out = torch.empty(rows[-1], dtype=torch.float32, device=self.dev)
        self.graph = None

    def launch_all(self, stream: int | None = None) -> None:
        lib = self._lib
        s = stream if stream is not None else lib.stream_ptr(self.dev)
        # symmetric weights: the instantiation without the zero-point tile loop (with the peer-store paths)
        sym = 2 if all(q.symmetric for q in self.qs) else 0
        lib.call("itq3_chain_run_ex", lib.ptr(self.desc), len(self.qs), lib.ptr(self.x), self.limbs,
                 lib.ptr(self.epoch), lib.ptr(self.out), self.grid, None, s, sym)

    def capture(self) -> None:
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            self.launch_all()
        torch.cuda.current_stream(self.dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch_all()
        self.graph = g

    def replay(self) -> None:
        if self.graph is None:
            self.capture()
        self.graph.replay()

    def output(self) -> torch.Tensor:
        """The full last-stage output (all ranks' rows), identical on every rank."""
        return self.out

    def forward(self, x) -> "np.ndarray":
        """Host in -> host out on this rank: H2D of x (pinned), the graphed chain step, D2H of the
        gathered last-stage output.  Every rank must call it for the same step (the chain's peer
        stores pair the ranks' launches)."""
        import numpy as np

        if getattr(self, "host_in", None) is None:
            self.host_in = torch.empty(self.x.numel(), dtype=torch.float32).pin_memory()
            self.host_out = torch.empty(self.out.numel(), dtype=torch.float32).pin_memory()
        self.host_in.copy_(torch.as_tensor(np.asarray(x, dtype=np.float32)).reshape(-1))
        self.x.copy_(self.host_in, non_blocking=True)
        self.replay()
        self.host_out.copy_(self.out, non_blocking=True)
        torch.cuda.current_stream(self.dev).synchronize()
        return self.host_out.numpy()

    def nvlink_bytes_per_step(self) -> int:
        """Bytes this rank stores into its peers' copies per step: every tagged output word (8 B per
        row and K-chunk partial) of its row shards, once per remote rank."""
        tot = 0
        for q in self.qs:
            tot += q.rows * -(-q.cols // 4096) * 8 * (self.world - 1)
        return tot


class TPMatmul:
    """Row-sharded batched product (fused_matmul, k >= 16) with the all-gather fused into the K5 MMQ
    epilogue: every finished output row goes straight to all ranks' copies of Y through NVLink peer
    pointers (torch symmetric memory), then one symmetric-memory barrier orders the reads.  The
    unfused equivalent is ShardedLinear (local fused_matmul + NCCL all_gather_into_tensor).

    `local_q`: this rank's rows shard_bounds(rows, world, rank); Y is rows x max_tokens (fp32) on every
    rank.  `peer_bases` / `ybuf` (testing): explicit per-rank output buffers (2 * rows * max_tokens
    floats each) instead of a rendezvous.

    Y is double-buffered by call parity: call t writes half t % 2 of every rank's buffer, so a fast
    rank's call t + 1 never overwrites the words a slower rank is still reading from call t (it
    cannot start call t + 2 before every rank has passed call t + 1's barrier, which is stream-ordered
    behind that rank's reads of call t's Y).  The returned Y is a view of that half: valid until the
    second-next call on this object (clone it to keep it longer).
    """

    def __init__(self, local_q: QuantizedTensor, rows: int, max_tokens: int, group=None, world: int | None = None,
                 rank: int | None = None, ybuf: torch.Tensor | None = None, peer_bases: list[int] | None = None):
        from . import _lib

        self._lib = _lib
        self.group = group
        if world is None:
            world = dist.get_world_size(group) if dist.is_initialized() else 1
        if rank is None:
            rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world, self.rank, self.rows, self.cols, self.max_tokens = world, rank, rows, local_q.cols, max_tokens
        self.r0, r1 = shard_bounds(rows, world, rank)
        if local_q.rows != r1 - self.r0:
            raise ShapeError(f"TPMatmul: shard has {local_q.rows} rows, expected {r1 - self.r0}")
        if not (local_q.mmq_ok() and local_q.k5_range_ok()):
            raise ShapeError("TPMatmul: the shard's format is not on the K5 path (cols % 256, whole blocks)")
        self.q = local_q
        self.dev = _lib.device()
        self.hdl = None
        if ybuf is None:
            if world > 1:
                from torch.distributed import _symmetric_memory as symm

                ybuf = symm.empty(2 * rows * max_tokens, dtype=torch.float32, device=self.dev)
                self.hdl = symm.rendezvous(ybuf, group if group is not None else dist.group.WORLD)
                delta = ybuf.data_ptr() - self.hdl.buffer_ptrs[rank]
                peer_bases = [b + delta for b in self.hdl.buffer_ptrs]
            else:
                ybuf = torch.empty(2 * rows * max_tokens, dtype=torch.float32, device=self.dev)
        if peer_bases is None:
            peer_bases = [ybuf.data_ptr()]
        if len(peer_bases) != world or peer_bases[rank] != ybuf.data_ptr():
            raise ShapeError("TPMatmul: peer_bases must list every rank's buffer, this rank's at index rank")
        if ybuf.numel() < 2 * rows * max_tokens:
            raise ShapeError("TPMatmul: ybuf must hold 2 * rows * max_tokens floats (double-buffered Y)")
        self.ybuf = ybuf
        half = 4 * rows * max_tokens  # bytes per parity half
        self.peers = torch.tensor([[b + p * half for b in peer_bases] for p in (0, 1)], dtype=torch.int64,
                                  device=self.dev)
        self.calls = 0

    def launch(self, X: torch.Tensor, stream: int | None = None) -> None:
        """Rotate X (cols x k, this rank's device) and run the peer-store MMQ; no synchronisation."""
        lib, k = self._lib, X.shape[1]
        if X.shape[0] != self.cols or not 1 <= k <= self.max_tokens:
            raise ShapeError(f"TPMatmul: X must be {self.cols} x (1..{self.max_tokens}), got {tuple(X.shape)}")
        s = stream if stream is not None else lib.stream_ptr(self.dev)
        self._act = torch.empty(lib.load().itq3_mmq_act_nbytes(self.cols, k), dtype=torch.uint8, device=self.dev)
        lib.call("itq3_rotate_act_f16_n", lib.ptr(X), lib.TORCH_DTYPE_CODE[X.dtype], self.cols, k, X.stride(0),
                 X.stride(1), self.q.block_n, lib.ptr(self._act), None, s)
        wsn = lib.load().itq3_mmq_ws_nbytes(self.q.rows, self.cols, k)
        self._ws = torch.empty(wsn, dtype=torch.uint8, device=self.dev) if wsn else None
        self.parity = self.calls & 1
        self.calls += 1
        lib.call("itq3_mmq_peers", lib.ptr(self.q.mmq_layout()), self.q.rows, self.cols, self.q.mmq_flags(),
                 lib.ptr(self._act), k, lib.ptr(self.peers[self.parity]), self.world, self.r0, lib.F32, k, 1,
                 lib.ptr(self._ws) if self._ws is not None else None, s)

    def __call__(self, X: torch.Tensor) -> torch.Tensor:
        """Y = w_hat @ X for the full `rows`, identical on every rank (a view of the symmetric buffer)."""
        self.launch(X)
        if self.hdl is not None:
            self.hdl.barrier()  # every rank's peer stores have landed before anyone reads Y
        k = X.shape[1]
        base = self.parity * self.rows * self.max_tokens
        return self.ybuf[base: base + self.rows * k].view(self.rows, k)
