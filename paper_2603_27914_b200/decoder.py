"""Decoder-stack harness (BASELINE configs[3]): a Llama-style decoder
whose every linear is an ITQ3_S tensor multiplied by the fused kernels of this package, for the
batch-1 decode tokens/s metric.  None of it exists in the reference; it only frames the hot path.

Per layer and token: [residual +] RMSNorm -> qkv GEMV -> RoPE + KV-cache append + grouped-query
attention over the cache -> o GEMV -> residual + RMSNorm -> gate_up GEMV -> SiLU(gate) * up -> down
GEMV.  qkv and o are one-stage chain launches (csrc/chain.cu, one cooperative kernel each); gate_up,
the SiLU gating and down are ONE two-stage chain launch (the down stage applies the gating while
loading its input); the rest of the glue is two small kernels (csrc/decoder_glue.cu), so a layer
is 6 launches.  A whole token step is ONE CUDA
graph: the position lives in a device tensor that the graph itself advances, the attention reads
the full cache under a position mask, so replays need no host work.
"""

from __future__ import annotations

import math

import torch

from .codec import QuantizedTensor, quantize_tensor
from .compute import fused_matvec

LLAMA3_8B = dict(hidden=4096, inter=14336, n_heads=32, n_kv=8, head_dim=128, rope_theta=500000.0)


class _GatedPair:
    """gate_up -> SiLU(gate) * up -> down as ONE two-stage chain launch (csrc/chain.cu, gated stage
    flag): the down projection's consumers read both halves of the gate_up output and apply the
    gating while loading, so neither the intermediate activation nor a second launch exists."""

    def __init__(self, q_gu: QuantizedTensor, q_down: QuantizedTensor, dev):
        import ctypes

        from . import _lib

        self._lib = _lib
        lib = _lib.load()
        host = ctypes.create_string_buffer(lib.itq3_chain_desc_nbytes() * 2)
        self.y = []
        for i, (q, flag) in enumerate(((q_gu, 0), (q_down, 2))):
            nch = -(-q.cols // 4096)
            y = torch.zeros((nch, q.rows), dtype=torch.int64, device=dev)  # tagged outputs, epoch 0
            self.y.append(y)
            _lib.check(lib.itq3_chain_write_desc(host, i, _lib.ptr(q.tiled()), _lib.ptr(y), None, q.rows, q.cols,
                                                 int(not q.symmetric) | flag, 0))
        self.desc = torch.frombuffer(bytearray(host.raw), dtype=torch.uint8).to(dev)
        self.epoch = torch.zeros(2, dtype=torch.int32, device=dev)
        self.out = torch.zeros(q_down.rows, dtype=torch.float32, device=dev)

    def __call__(self, x: torch.Tensor, stream: int) -> torch.Tensor:
        lib = self._lib
        lib.call("itq3_chain_run_gated", lib.ptr(self.desc), 2, lib.ptr(x), 3, lib.ptr(self.epoch), lib.ptr(self.out),
                 0, None, stream)
        return self.out


class DecoderStack:
    """`layers` x (qkv, o, gate_up, down) ITQ3_S linears with random N(0, 0.02^2) weights (quantised
    on the GPU by K1), RMSNorm gains near 1, a KV cache of `max_ctx` positions (fp32)."""

    def __init__(self, layers: int = 32, max_ctx: int = 1024, seed: int = 0, dev=None, shapes: dict | None = None,
                 eps: float = 1e-5, serving: bool = True):
        cfg = dict(LLAMA3_8B, **(shapes or {}))
        self.dev = dev or torch.device("cuda", torch.cuda.current_device())
        self.layers, self.max_ctx, self.eps = layers, max_ctx, eps
        self.h, self.inter = cfg["hidden"], cfg["inter"]
        self.nh, self.nkv, self.hd = cfg["n_heads"], cfg["n_kv"], cfg["head_dim"]
        g = torch.Generator(device=self.dev)
        g.manual_seed(seed)
        kv = self.nkv * self.hd
        shapes_l = [(self.h + 2 * kv, self.h), (self.h, self.h), (2 * self.inter, self.h), (self.h, self.inter)]
        self.q: list[list[QuantizedTensor]] = []
        for _ in range(layers):
            row = []
            for r, c in shapes_l:
                w = torch.randn((r, c), generator=g, device=self.dev).mul_(0.02)
                q = quantize_tensor(w)
                q.tiled()
                if serving:
                    q.drop_payload()  # only the tiled GEMV copy stays on the device
                row.append(q)
                del w
            self.q.append(row)
        self.gain = [(1.0 + 0.1 * torch.randn((2, self.h), generator=g, device=self.dev)) for _ in range(layers)]
        inv = 1.0 / (cfg["rope_theta"] ** (torch.arange(0, self.hd, 2, device=self.dev, dtype=torch.float64) / self.hd))
        ang = torch.arange(max_ctx, device=self.dev, dtype=torch.float64)[:, None] * inv[None, :]
        self.cos, self.sin = ang.cos().float(), ang.sin().float()
        self.k_cache = torch.zeros((layers, 1, self.nkv, max_ctx, self.hd), device=self.dev)
        self.v_cache = torch.zeros_like(self.k_cache)
        self.pos = torch.zeros(1, dtype=torch.long, device=self.dev)
        self.x = torch.zeros(self.h, device=self.dev)
        self.out = torch.zeros(self.h, device=self.dev)
        self.kpos = torch.arange(max_ctx, device=self.dev)
        self.xs = torch.zeros(self.h, device=self.dev)          # residual stream
        self.hbuf = torch.zeros(self.h, device=self.dev)        # normalised input of a projection
        self.att = torch.zeros(self.h, device=self.dev)         # attention output (nh * hd)
        from . import _lib

        self.attn_ws = torch.zeros(_lib.load().itq3_glue_attention_ws_nbytes(self.nh), dtype=torch.uint8,
                                   device=self.dev)  # split partials + per-head counters
        if self.hd != 128 or max_ctx > 1024 or self.nh * self.hd != self.h:
            raise ValueError("DecoderStack: the glue kernels need head_dim 128, max_ctx <= 1024, nh * hd = hidden")
        self.pairs = [_GatedPair(row[2], row[3], self.dev) for row in self.q]
        self.graph = None

    def _rms(self, x, gain):
        return torch.nn.functional.rms_norm(x, (self.h,), weight=gain, eps=self.eps)

    def _rope(self, t, cos, sin):  # t: (heads, hd), rotate-half convention
        a, b = t[:, : self.hd // 2], t[:, self.hd // 2:]
        return torch.cat((a * cos - b * sin, a * sin + b * cos), dim=1)

    def _step(self) -> None:
        """One token: 3 chain launches (qkv, o, gated gate_up+down) + 3 glue launches per layer."""
        from . import _lib

        st = _lib.stream_ptr(self.dev)
        xs, h = self.xs, self.hbuf
        xs.copy_(self.x)
        prev = None
        for li in range(self.layers):
            qkv_w, o_w = self.q[li][0], self.q[li][1]
            _lib.call("itq3_glue_residual_rmsnorm", _lib.ptr(xs), _lib.ptr(prev) if prev is not None else None,
                      _lib.ptr(self.gain[li][0]), _lib.ptr(h), self.h, self.eps, st)
            qkv = fused_matvec(qkv_w, h, check_finite=False)
            _lib.call("itq3_glue_rope_attention", _lib.ptr(qkv), _lib.ptr(self.cos), _lib.ptr(self.sin),
                      _lib.ptr(self.pos), _lib.ptr(self.k_cache[li, 0]), _lib.ptr(self.v_cache[li, 0]),
                      _lib.ptr(self.att), self.nh, self.nkv, self.hd, self.max_ctx, _lib.ptr(self.attn_ws), st)
            o = fused_matvec(o_w, self.att, check_finite=False)
            _lib.call("itq3_glue_residual_rmsnorm", _lib.ptr(xs), _lib.ptr(o), _lib.ptr(self.gain[li][1]),
                      _lib.ptr(h), self.h, self.eps, st)
            prev = self.pairs[li](h, st)  # gate_up + SiLU gating + down: one chain launch
        _lib.call("itq3_glue_residual_rmsnorm", _lib.ptr(xs), _lib.ptr(prev), None, _lib.ptr(self.out), self.h,
                  self.eps, st)
        self.pos.add_(1)

    def capture(self) -> None:
        """Record one token step (all layers, position advance included) as a CUDA graph."""
        side = torch.cuda.Stream(self.dev)
        side.wait_stream(torch.cuda.current_stream(self.dev))
        with torch.cuda.stream(side):
            self._step()  # warm-up: builds the per-tensor chain contexts outside capture
        torch.cuda.current_stream(self.dev).wait_stream(side)
        self.reset()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step()
        self.graph = g

    def reset(self, pos: int = 0) -> None:
        self.pos.fill_(pos)
        self.k_cache.zero_()
        self.v_cache.zero_()

    def step(self, x: torch.Tensor | None = None) -> torch.Tensor:
        """Decode one token: hidden state in (device, len hidden), hidden state out; advances the position."""
        if x is not None:
            self.x.copy_(x)
        if self.graph is None:
            self.capture()
        self.graph.replay()
        return self.out

    def reference_step(self, x: torch.Tensor, pos: int, k_hist: list, v_hist: list) -> torch.Tensor:  # noqa: C901
        """The same token step in plain torch fp32 with dequantised weights (numerics test only)."""
        from .codec import dequantize_tensor

        h = x.clone()
        cos, sin = self.cos[pos:pos + 1], self.sin[pos:pos + 1]
        kvd = self.nkv * self.hd
        for li in range(self.layers):
            if not hasattr(self, "_ref_w"):
                self._ref_w = {}
            if li not in self._ref_w:
                self._ref_w[li] = [torch.as_tensor(dequantize_tensor(q), device=self.dev).float() for q in self.q[li]]
            W = self._ref_w[li]
            g1, g2 = self.gain[li][0], self.gain[li][1]
            qkv = W[0] @ self._rms(h, g1)
            q = self._rope(qkv[: self.h].view(self.nh, self.hd), cos, sin)
            k = self._rope(qkv[self.h: self.h + kvd].view(self.nkv, self.hd), cos, sin)
            v = qkv[self.h + kvd:].view(self.nkv, self.hd)
            k_hist[li].append(k)
            v_hist[li].append(v)
            K = torch.stack(k_hist[li], dim=1).repeat_interleave(self.nh // self.nkv, 0)  # (nh, t, hd)
            V = torch.stack(v_hist[li], dim=1).repeat_interleave(self.nh // self.nkv, 0)
            s = (K @ q[:, :, None])[:, :, 0] / math.sqrt(self.hd)
            att = (torch.softmax(s, dim=1)[:, None, :] @ V)[:, 0, :]
            h = h + W[1] @ att.reshape(self.h)
            gu = W[2] @ self._rms(h, g2)
            h = h + W[3] @ (torch.nn.functional.silu(gu[: self.inter]) * gu[self.inter:])
        return h
