"""Decoder-stack harness (BASELINE configs[3]): a Llama-style decoder
whose every linear is an ITQ3_S tensor multiplied by the fused kernels of this package, for the
batch-1 decode tokens/s metric.  None of it exists in the reference; it only frames the hot path.

Per layer and token: [residual +] RMSNorm -> qkv GEMV -> RoPE + KV-cache append + grouped-query
attention over the cache -> o GEMV -> residual + RMSNorm -> gate_up GEMV -> SiLU(gate) * up -> down
GEMV.  Everything but the attention runs inside chain launches (csrc/chain.cu, decoder flags): the
RMSNorm in the loads of the qkv / gate_up stages (every CTA of a 4096-column stage holds the whole
input), the SiLU gating in the loads of the down stage, the residual adds in the final folds; the
attention (RoPE + KV append + split decode attention) is one glue kernel (csrc/decoder_glue.cu).
A layer is 2 launches: attention, then ONE chain [o -> RMSNorm(x + o) -> gate_up -> SiLU gating -> down
-> RMSNorm((x + o) + down) -> next layer's qkv] whose last stage also writes the new residual stream
(ping-pong buffers); the last layer's chain ends in the lm_head.  Plus one [RMSNorm -> qkv] launch for
layer 0: 2 x layers + 1 launches per token.  A whole token step is ONE CUDA
graph: the position lives in a device tensor that the graph itself advances, the attention reads
the full cache under a position mask, so replays need no host work.
"""

from __future__ import annotations

import math

import torch

from .codec import QuantizedTensor, quantize_tensor

LLAMA3_8B = dict(hidden=4096, inter=14336, n_heads=32, n_kv=8, head_dim=128, rope_theta=500000.0, vocab=128256)


class _Chain:
    """A short chain of ITQ3_S stages run as ONE cooperative launch (csrc/chain.cu, decoder flags):
    stages = [(QuantizedTensor, flags, xin)], flags bit 1 = gated input (SiLU(gate) * up of the
    previous stage), bit 2 = RMSNorm input with gain `xin`, bit 3 = the fold adds into `out` (the
    residual stream) instead of overwriting it, bit 4 = the RMSNorm input is x0 + the previous
    stage's output (residual after an o projection in the same launch), bit 5 = the fold adds stage
    0's output first, bit 6 = the RMSNorm input is (x0 + stage 0's output) + the previous stage's
    output (the residual after a whole layer), bit 7 = that stage also writes the residual it formed
    to `xout`.  A stage-0 `xin` without flag 2 is that stage's input vector."""

    def __init__(self, stages, out: torch.Tensor, dev, xout: torch.Tensor | None = None):
        import ctypes

        from . import _lib

        self._lib = _lib
        lib = _lib.load()
        host = ctypes.create_string_buffer(lib.itq3_chain_desc_nbytes() * len(stages))
        self.y, self.keep = [], []
        for i, (q, flags, gain) in enumerate(stages):
            y = torch.zeros((-(-q.cols // 4096), q.rows), dtype=torch.int64, device=dev)  # tagged outputs
            self.y.append(y)
            self.keep.append(gain)
            _lib.check(lib.itq3_chain_write_desc(host, i, _lib.ptr(q.tiled()), _lib.ptr(y),
                                                 _lib.ptr(gain) if gain is not None else None, q.rows, q.cols,
                                                 int(not q.symmetric) | flags, 0))
            if flags & XOUT:
                _lib.check(lib.itq3_chain_set_xout(host, i, _lib.ptr(xout)))
                self.keep.append(xout)
        self.n = len(stages)
        self.desc = torch.frombuffer(bytearray(host.raw), dtype=torch.uint8).to(dev)
        self.epoch = torch.zeros(2, dtype=torch.int32, device=dev)
        self.out = out

    def __call__(self, x: torch.Tensor, stream: int) -> torch.Tensor:
        lib = self._lib
        lib.call("itq3_chain_run_gated", lib.ptr(self.desc), self.n, lib.ptr(x), 3, lib.ptr(self.epoch),
                 lib.ptr(self.out), 0, None, stream)
        return self.out


GATED, NORM_IN, ADD_OUT, RESID_IN, ADD_OUT0, RESID2_IN, XOUT = 2, 4, 8, 16, 32, 64, 128


class DecoderStack:
    """`layers` x (qkv, o, gate_up, down) ITQ3_S linears with random N(0, 0.02^2) weights (quantised
    on the GPU by K1), RMSNorm gains near 1, a KV cache of `max_ctx` positions (fp32)."""

    def __init__(self, layers: int = 32, max_ctx: int = 1024, seed: int = 0, dev=None, shapes: dict | None = None,
                 eps: float = 1e-5, serving: bool = True, lm_head: bool = True):
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
        # final RMSNorm + ITQ3_S lm_head (vocab x hidden): logits of the token, one more chain launch
        self.vocab = cfg["vocab"]
        self.lm_head = None
        if lm_head:
            w = torch.randn((self.vocab, self.h), generator=g, device=self.dev).mul_(0.02)
            self.lm_head = quantize_tensor(w)
            self.lm_head.tiled()
            if serving:
                self.lm_head.drop_payload()
            del w
            self.final_gain = 1.0 + 0.1 * torch.randn(self.h, generator=g, device=self.dev)
            self.logits = torch.zeros(self.vocab, device=self.dev)
        inv = 1.0 / (cfg["rope_theta"] ** (torch.arange(0, self.hd, 2, device=self.dev, dtype=torch.float64) / self.hd))
        ang = torch.arange(max_ctx, device=self.dev, dtype=torch.float64)[:, None] * inv[None, :]
        self.cos, self.sin = ang.cos().float(), ang.sin().float()
        self.k_cache = torch.zeros((layers, 1, self.nkv, max_ctx, self.hd), device=self.dev)
        self.v_cache = torch.zeros_like(self.k_cache)
        self.pos = torch.zeros(1, dtype=torch.long, device=self.dev)
        self.host_pos = 0
        self.x = torch.zeros(self.h, device=self.dev)
        self.out = torch.zeros(self.h, device=self.dev)
        self.kpos = torch.arange(max_ctx, device=self.dev)
        self.att = torch.zeros(self.h, device=self.dev)         # attention output (nh * hd)
        from . import _lib

        self.attn_ws = torch.zeros(_lib.load().itq3_glue_attention_ws_nbytes(self.nh), dtype=torch.uint8,
                                   device=self.dev)  # split partials + per-head counters
        if self.hd != 128 or max_ctx > 1024 or self.nh * self.hd != self.h:
            raise ValueError("DecoderStack: the glue kernels need head_dim 128, max_ctx <= 1024, nh * hd = hidden")
        # launch 0: [RMSNorm -> qkv_0]; layer L: attention, then [o -> RMSNorm(x + o) -> gate_up -> SiLU gating
        # -> down -> RMSNorm(x + o + down) -> qkv_{L+1} (or the lm_head)], the residual ping-ponging between
        # self.xs2[L % 2] (read) and self.xs2[(L + 1) % 2] (written by the last stage)
        self.qkv_out = torch.zeros(self.h + 2 * kv, device=self.dev)
        self.xs2 = [torch.zeros(self.h, device=self.dev), torch.zeros(self.h, device=self.dev)]
        self.first = _Chain([(self.q[0][0], NORM_IN, self.gain[0][0])], self.qkv_out, self.dev)
        self.chains = []
        for li, (_, o_w, gu_w, down_w) in enumerate(self.q):
            mlp = [(o_w, 0, self.att), (gu_w, NORM_IN | RESID_IN, self.gain[li][1])]
            if li + 1 < layers:
                nxt, out = (self.q[li + 1][0], NORM_IN | RESID2_IN | XOUT, self.gain[li + 1][0]), self.qkv_out
            elif self.lm_head is not None:
                nxt, out = (self.lm_head, NORM_IN | RESID2_IN | XOUT, self.final_gain), self.logits
            else:
                nxt, out = None, self.xs2[li % 2]
            if nxt is None:  # last layer without a head: fold x += o + down in place
                stages = mlp + [(down_w, GATED | ADD_OUT | ADD_OUT0, None)]
            else:
                stages = mlp + [(down_w, GATED, None), nxt]
            self.chains.append(_Chain(stages, out, self.dev, xout=self.xs2[(li + 1) % 2]))
        self.final_xs = self.xs2[layers % 2] if self.lm_head is not None else self.xs2[(layers - 1) % 2]
        self.graph = None

    def weight_bytes(self) -> int:
        """Packed (tiled) ITQ3_S weight bytes one token streams: every layer's linears + the lm_head."""
        n = sum(int(t.numel()) for row in self.q for q in row for t in q._tiled.values())
        if self.lm_head is not None:
            n += sum(int(t.numel()) for t in self.lm_head._tiled.values())
        return n

    def launches_per_step(self) -> int:
        return 2 * self.layers + 1

    def _rms(self, x, gain):
        return torch.nn.functional.rms_norm(x, (self.h,), weight=gain, eps=self.eps)

    def _rope(self, t, cos, sin):  # t: (heads, hd), rotate-half convention
        a, b = t[:, : self.hd // 2], t[:, self.hd // 2:]
        return torch.cat((a * cos - b * sin, a * sin + b * cos), dim=1)

    def _step(self) -> None:
        """One token: the layer-0 [RMSNorm -> qkv] chain, then per layer one glue launch (RoPE + KV append +
        split attention) and one chain [o -> ... -> down -> next qkv / lm_head]."""
        from . import _lib

        st = _lib.stream_ptr(self.dev)
        self.xs2[0].copy_(self.x)
        self.first(self.xs2[0], st)  # qkv_0 = W_qkv RMSNorm(x)
        for li in range(self.layers):
            _lib.call("itq3_glue_rope_attention", _lib.ptr(self.qkv_out), _lib.ptr(self.cos), _lib.ptr(self.sin),
                      _lib.ptr(self.pos), _lib.ptr(self.k_cache[li, 0]), _lib.ptr(self.v_cache[li, 0]),
                      _lib.ptr(self.att), self.nh, self.nkv, self.hd, self.max_ctx, _lib.ptr(self.attn_ws), st)
            # h = x + W_o att; x' = h + W_down (SiLU(gate) * up)(RMSNorm(h)); qkv_{L+1} = W_qkv RMSNorm(x')
            # (the last layer: logits = W_head RMSNorm(x'))
            self.chains[li](self.xs2[li % 2], st)
        self.out.copy_(self.final_xs)
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
        if not 0 <= pos < self.max_ctx:
            raise ValueError(f"DecoderStack: position {pos} outside the KV cache (max_ctx {self.max_ctx})")
        self.pos.fill_(pos)
        self.host_pos = pos
        self.k_cache.zero_()
        self.v_cache.zero_()

    def replay(self) -> None:
        """One graphed token step (bench loop); the host-side position guards the KV cache bound."""
        if self.host_pos >= self.max_ctx:
            raise ValueError(f"DecoderStack: KV cache full ({self.max_ctx} positions); reset() first")
        self.graph.replay()
        self.host_pos += 1

    def step(self, x: torch.Tensor | None = None) -> torch.Tensor:
        """Decode one token: hidden state in (device, len hidden), hidden state out; advances the position.
        Raises once the KV cache is full (the glue kernel also refuses positions >= max_ctx on the
        device and writes no cache entry: its error word, attn_ws's last u32, is set)."""
        if x is not None:
            self.x.copy_(x)
        if self.graph is None:
            self.capture()
        self.replay()
        return self.out

    def device_error(self) -> int:
        """The glue kernel's out-of-cache flag (non-zero after a replay at a position >= max_ctx)."""
        return int(self.attn_ws.view(torch.int32)[-1].item())

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
        if self.lm_head is not None:
            if not hasattr(self, "_ref_head"):
                self._ref_head = torch.as_tensor(dequantize_tensor(self.lm_head), device=self.dev).float()
            self.ref_logits = self._ref_head @ self._rms(h, self.final_gain)
        return h
