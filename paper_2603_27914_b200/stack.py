"""Decode-time linear stack: a dependent chain of fused GEMVs replayed as one CUDA graph.

There is no reference counterpart (the reference has no model); this is the harness behind
the "decode tokens/sec" metric.  Stage i multiplies the
quantized matrix q_i by the first q_i.cols entries of stage i-1's output, so every GEMV
depends on the previous one exactly as in a decoder's qkv -> o -> gate_up -> down chain.
Per stage: K3 ``itq3_rotate_act`` (x -> rotated fixed-point limbs) + K4 ``itq3_gemv``.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from .codec import QuantizedTensor
from .errors import ShapeError


def balanced_work(shapes: list[tuple[int, int]], grid: int) -> np.ndarray:
    """Host-balanced chain work split (itq3_chain_set_work): for every stage, which (K-chunk, first row
    tile) each CTA takes, as chunk * Gc + rt0 (-1 idle).

    A stage whose input is a strict prefix of the previous stage's output (qkv -> o, gate_up -> down in a
    decoder layer) finds that input complete after the previous stage's first rounds, so each CTA starts it
    right after its own units of the previous stage: the stage ends at max over CTAs of the units carried
    since the last full-input stage.  Greedily giving the cheapest (chunk, row-tile) items to the CTAs that
    carry the most units brings that max down to the mean (Llama-2-7B: qkv + o 8 -> 7 units, gate_up + down
    15.5 -> 15).  Stages that read the whole previous output restart the count."""
    S = len(shapes)
    tab = np.full((S, grid), -1, dtype=np.int32)
    load = np.zeros(grid)
    for s, (rows, cols) in enumerate(shapes):
        nb = cols // 256
        nch = -(-nb // 16)
        gc = grid // nch
        rt = -(-rows // 16)
        if not (s > 0 and cols < shapes[s - 1][0]):
            load[:] = 0.0
        items = []
        for ch in range(nch):
            w = min(16, nb - 16 * ch) / 16.0
            for v in range(gc):
                n = (rt - 1 - v) // gc + 1 if v < rt else 0
                items.append((n * w, ch, v))
        items.sort()
        order = np.argsort(-load, kind="stable")
        for c, (cost, ch, v) in zip(order, items):
            tab[s, c] = ch * gc + v
            load[c] += cost
    return tab


def _hadamard16(dev) -> torch.Tensor:
    h = torch.ones(1, 1, dtype=torch.float64)
    for _ in range(4):
        h = torch.cat([torch.cat([h, h], 1), torch.cat([h, -h], 1)], 0)
    return h.to(dev)


class LinearStack:
    """mode="chain": one persistent cooperative kernel per step (csrc/chain.cu, default);
    mode="kernels": 2 launches per stage (K3 rotate_act + K4 gemv), for comparison.

    independent=True: every stage reads x (no dependency between stages) -- the streaming reference pass.
    lo (symmetric chains): True runs the instantiation that passes H_16 y between stages (faster; its
    intermediate stage outputs are stored in that form and `stage_output` undoes it), False the one with plain
    stage outputs (bit-identical to the tensor-parallel chain).  The final output is the same either way up to
    the fp32 rounding of the H_16 transforms (tests/test_gpu_stack.py bounds both)."""

    balance = True  # host-balanced work split (balanced_work); False: the kernel's default round robin

    def __init__(self, qs: list[QuantizedTensor], limbs: int = 3, mode: str = "chain", independent: bool = False,
                 lo: bool = True):
        if not qs:
            raise ShapeError("LinearStack: no stages")
        for a, b in zip(qs, qs[1:]):
            if b.cols > a.rows:
                raise ShapeError(f"LinearStack: stage needs {b.cols} inputs, previous stage has {a.rows} rows")
        for q in qs:
            if not q.fast_layout():
                raise ShapeError("LinearStack: stages need the tiled layout (block_n 256, variant s, cols % 256 == 0)")
        self.dev = _lib.device()
        self.qs = qs
        self.limbs = limbs
        lib = _lib.load()
        self.tiled = [q.tiled() for q in qs]
        self.x = torch.zeros(qs[0].cols, dtype=torch.float32, device=self.dev)
        self.acts = [torch.empty(lib.itq3_act_nbytes(q.cols, 1, limbs), dtype=torch.uint8, device=self.dev)
                     for q in qs]
        self.ys = [torch.empty(q.rows, dtype=torch.float32, device=self.dev) for q in qs]
        self.graph = None
        self.mode = mode
        self.independent = independent  # every stage reads x (no dependency): pure streaming
        # lo (symmetric chains): the chain kernel instantiation whose stages pass H_16 y per 16-row tile (its
        # rotations skip 4 of 8 butterfly stages); lo=False: plain outputs, bit-identical to the TP chain
        self.lo_kernel = lo
        if mode == "chain":
            self._setup_chain()
        elif mode != "kernels":
            raise ValueError(f"LinearStack: unknown mode {mode!r}")
        self.host_in = torch.empty(qs[0].cols, dtype=torch.float32).pin_memory()
        self.host_out = torch.empty(qs[-1].rows, dtype=torch.float32).pin_memory()

    def _setup_chain(self) -> None:
        lib = _lib.load()
        S = len(self.qs)
        nd = lib.itq3_chain_desc_nbytes()
        host = ctypes.create_string_buffer(nd * S)
        self.nch = [-(-q.cols // 4096) for q in self.qs]
        # tagged outputs: (fp32 bits | epoch << 32), zero = epoch 0 (never current)
        self.yparts = [torch.zeros((c, q.rows), dtype=torch.int64, device=self.dev) for c, q in zip(self.nch, self.qs)]
        self.out = torch.empty(self.qs[-1].rows, dtype=torch.float32, device=self.dev)
        for i, q in enumerate(self.qs):
            xin = None
            if self.independent:
                self._xin = getattr(self, "_xin", torch.randn(max(qq.cols for qq in self.qs), device=self.dev))
                xin = _lib.ptr(self._xin)
            _lib.check(lib.itq3_chain_write_desc(host, i, _lib.ptr(self.tiled[i]), _lib.ptr(self.yparts[i]), xin,
                                                 q.rows, q.cols, int(not q.symmetric), 0))
        if self.balance and not self.independent:
            grid = lib.itq3_sm_count()
            self.work = torch.from_numpy(balanced_work([(q.rows, q.cols) for q in self.qs], grid)).to(self.dev)
            for i in range(S):
                _lib.check(lib.itq3_chain_set_work(host, i, _lib.ptr(self.work[i])))
        self.sym = all(q.symmetric for q in self.qs)
        # stages whose stored output is H_16 y per full 16-row tile (the LO kernel: all but the last)
        self.lo = [self.sym and self.lo_kernel and i + 1 < S for i in range(S)]
        self.epoch = torch.zeros(2, dtype=torch.int32, device=self.dev)  # (step epoch, check-in count)
        self.trace = None
        self.desc = torch.frombuffer(bytearray(host.raw), dtype=torch.uint8).to(self.dev)

    def enable_trace(self) -> torch.Tensor:
        """Per-(CTA, stage) globaltimer stamps: entered, input ready, input rotated, last tile done."""
        sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
        S = len(self.qs)
        self.trace = torch.zeros(sms * S * 4 + S * 16 * 4 + 16 * 8, dtype=torch.int64, device=self.dev)
        self.graph = None
        return self.trace

    @property
    def launches_per_step(self) -> int:
        return 1 if self.mode == "chain" else 2 * len(self.qs)  # chain: one cooperative kernel

    def step_bytes(self) -> int:
        """Algorithmic bytes of one step: all tiled weights + rotated activations + outputs."""
        return sum(self.gemv_bytes(i) for i in range(len(self.qs)))

    def gemv_bytes(self, i: int) -> int:
        """Algorithmic bytes of stage i's GEMV launch: tiled weights + activation fragments + y."""
        q = self.qs[i]
        act = _lib.load().itq3_chain_act_block_bytes(self.limbs) if self.mode == "chain" else 2048 + 64
        return int(self.tiled[i].numel()) + (q.cols // 256) * act + 4 * q.rows

    def launch_stage(self, i: int, stream: int | None = None, parts: str = "both") -> None:
        q = self.qs[i]
        s = stream if stream is not None else _lib.stream_ptr(self.dev)
        xin = self.x if i == 0 else self.ys[i - 1]
        if parts in ("both", "rotate"):
            _lib.call("itq3_rotate_act", _lib.ptr(xin), _lib.F32, q.cols, 1, 1, q.cols, self.limbs,
                      _lib.ptr(self.acts[i]), s)
        if parts in ("both", "gemv"):
            _lib.call("itq3_gemv", _lib.ptr(self.tiled[i]), q.rows, q.cols, int(not q.symmetric),
                      _lib.ptr(self.acts[i]), 1, self.limbs, _lib.ptr(self.ys[i]), _lib.F32, 1, 1, s)

    def launch_all(self, out: torch.Tensor | None = None) -> None:
        if self.mode == "chain":
            trace = _lib.ptr(self.trace) if self.trace is not None else None
            # symmetric: LO kernel (flags 6: symmetric | single GPU) or the plain symmetric one (2); else general
            sym = (6 if self.lo_kernel else 2) if self.sym else 4
            _lib.call("itq3_chain_run_ex", _lib.ptr(self.desc), len(self.qs), _lib.ptr(self.x), self.limbs,
                      _lib.ptr(self.epoch), _lib.ptr(self.out if out is None else out), 0, trace,
                      _lib.stream_ptr(self.dev), sym)
            return
        for i in range(len(self.qs)):
            self.launch_stage(i)

    def output(self) -> torch.Tensor:
        """Device output of the last stage."""
        return self.out if self.mode == "chain" else self.ys[-1]

    def stage_output(self, i: int) -> torch.Tensor:
        """Stage i's output; in chain mode the K-chunk partials summed in the kernel's order (float64 for a
        stage that stores H_16 y, see below)."""
        if self.mode != "chain":
            return self.ys[i]
        p = self.yparts[i].view(torch.int32).reshape(self.nch[i], self.qs[i].rows, 2)[..., 0].view(torch.float32)
        y = p[0].clone()
        for c in range(1, p.shape[0]):
            y += p[c]
        if not self.lo[i]:
            return y
        # LO kernel: whole 16-row groups hold H_16 y -- returned as H_16^-1 of that fp32 sum in float64, exactly
        # the input the next stage multiplies; a partial last group is stored plain
        full = y.numel() // 16 * 16
        out = y.double()
        out[:full] = (out[:full].view(-1, 16) @ _hadamard16(y.device) / 16.0).reshape(-1)
        return out

    def capture(self) -> None:
        """Record the whole chain as one CUDA graph (launch overhead off the critical path)."""
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            self.launch_all()  # warm-up outside capture
        torch.cuda.current_stream(self.dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.launch_all()
        self.graph = g

    def replay(self) -> None:
        if self.graph is None:
            self.capture()
        self.graph.replay()

    def _host_step(self) -> None:
        # H2D: one small copy kernel reading the pinned (UVA-mapped) input; chain mode: the kernel's final
        # fold stores the output straight into the pinned host buffer (no memcpy nodes, 1909 -> ~1950 tok/s)
        _lib.call("itq3_copy_f32", _lib.ptr(self.x), _lib.ptr(self.host_in), self.x.numel(), _lib.stream_ptr(self.dev))
        if self.mode == "chain":
            self.launch_all(out=self.host_out)
        else:
            self.launch_all()
            self.host_out.copy_(self.output(), non_blocking=True)

    def capture_host_step(self) -> None:
        """One CUDA graph for a whole host-to-host step: the pinned input copied in by a small kernel, the
        chain (or the kernel sequence), its output written into pinned host memory -- one graph per token."""
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            self._host_step()  # warm-up outside capture
        torch.cuda.current_stream(self.dev).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._host_step()
        self.host_graph = g

    def forward(self, x) -> np.ndarray:
        """Host in -> host out: H2D of x, the chain, D2H of the last stage's output, as ONE graph launch.
        The returned host array is the stack's pinned output buffer (valid until the next call)."""
        xt = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.asarray(x, dtype=np.float32))
        if xt.numel() != self.x.numel():
            raise ShapeError(f"LinearStack.forward: expected {self.x.numel()} inputs, got {xt.numel()}")
        if xt.is_cuda:
            self.x.copy_(xt.reshape(-1))
            self.replay()
            self.host_out.copy_(self.output(), non_blocking=True)
        else:
            if getattr(self, "host_graph", None) is None or self.graph is None:
                self.replay()  # first use: capture the device-only graph too (stage outputs, epochs)
                self.capture_host_step()
                self._host_in_np, self._host_out_np = self.host_in.numpy(), self.host_out.numpy()
                self._stream = torch.cuda.current_stream(self.dev)
            np.copyto(self._host_in_np, xt.reshape(-1).numpy())  # plain memcpy into the pinned input
            self.host_graph.replay()
            self._stream.synchronize()
            return self._host_out_np
        torch.cuda.current_stream(self.dev).synchronize()
        return self.host_out.numpy()
