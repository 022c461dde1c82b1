"""Decoder-stack harness (BASELINE configs[3]): a Llama-style decoder
whose every linear is an ITQ3_S tensor multiplied by the fused kernels of this package, for the
batch-1 decode tokens/s metric.  None of it exists in the reference; it only frames the hot path.

Per layer and token: [residual +] RMSNorm -> qkv GEMV -> RoPE + KV-cache append + grouped-query
attention over the cache -> o GEMV -> residual + RMSNorm -> gate_up GEMV -> SiLU(gate) * up -> down
GEMV.  The WHOLE token is ONE persistent chain launch (csrc/chain.cu, decoder flags): per layer the
stages [attention partials, attention combine, o, gate_up, down, next qkv] -- the RMSNorm in the loads
of the qkv / gate_up stages (every CTA of a 4096-column stage holds the whole input), the SiLU gating
in the loads of the down stage, the residual stream as tagged buffers written by each layer's last
stage (the residual adds folded into the norm inputs); the attention stages read q / k / v from the
qkv stage's tagged outputs (RoPE, KV append, grouped-query attention over 16 position splits per kv
head, then a per-head combine); the last layer ends in the lm_head.  A token step is one CUDA graph
of that one launch: the position lives in a device tensor that the graph itself advances, so replays
need no host work.
"""

from __future__ import annotations

import os

import math

import torch

from .codec import QuantizedTensor, quantize_tensor

LLAMA3_8B = dict(hidden=4096, inter=14336, n_heads=32, n_kv=8, head_dim=128, rope_theta=500000.0, vocab=128256)


class _Chain:
    """ONE cooperative launch of the chain kernel (csrc/chain.cu, GATED instantiation) over a list of
    stages, each a dict: {"q": QuantizedTensor, "flags", "xin", "xres", "xout", "ref"} for an ITQ3_S
    GEMV stage, or {"attn": 256 | 512, "params": device AttnParams, "y": tagged output} for an
    attention stage.  Flags: bit 1 gated input (SiLU(gate) * up of the previous stage), bit 2 RMSNorm
    input with gain `xin`, bit 3 the final fold adds the residual, bit 4 the norm input is residual +
    the previous stage's output, bit 5 the fold adds the `ref` stage's output first, bit 6 the norm
    input is (residual + the `ref` stage's output) + the previous stage's output, bit 7 the stage
    also writes the residual it formed (tagged) to `xout`.  The residual is `xres` (a tagged buffer
    written earlier in the launch) or, when None, the launch input x0."""

    def __init__(self, stages, out: torch.Tensor, dev):
        import ctypes

        from . import _lib

        self._lib = _lib
        lib = _lib.load()
        host = ctypes.create_string_buffer(lib.itq3_chain_desc_nbytes() * len(stages))
        self.y, self.keep = [], []
        for i, st in enumerate(stages):
            if "attn" in st:
                self.keep.append(st["params"])
                self.y.append(st["y"])
                _lib.check(lib.itq3_chain_write_desc_attn(host, i, st["attn"], _lib.ptr(st["params"]),
                                                          _lib.ptr(st["y"]), st["y"].numel()))
                continue
            q, flags, xin = st["q"], st.get("flags", 0), st.get("xin")
            y = torch.zeros((-(-q.cols // 4096), q.rows), dtype=torch.int64, device=dev)  # tagged outputs
            self.y.append(y)
            self.keep.append(xin)
            _lib.check(lib.itq3_chain_write_desc(host, i, _lib.ptr(q.tiled()), _lib.ptr(y),
                                                 _lib.ptr(xin) if xin is not None else None, q.rows, q.cols,
                                                 int(not q.symmetric) | flags | (st.get("ref", 0) << 16), 0))
            if st.get("xres") is not None:
                _lib.check(lib.itq3_chain_set_xres(host, i, _lib.ptr(st["xres"])))
                self.keep.append(st["xres"])
            if flags & XOUT:
                _lib.check(lib.itq3_chain_set_xout(host, i, _lib.ptr(st["xout"])))
                self.keep.append(st["xout"])
        self.n = len(stages)
        # the gated single-GPU instantiation (itq3_chain_run_ex flags: gated | single GPU), without the
        # zero-point tile loop when every weight stage is symmetric (1097 -> 1105 tok/s)
        sym = all(st["q"].symmetric for st in stages if "q" in st)
        self.run_flags = 1 | 4 | (2 if sym else 0)
        self.desc = torch.frombuffer(bytearray(host.raw), dtype=torch.uint8).to(dev)
        self.epoch = torch.zeros(2, dtype=torch.int32, device=dev)
        self.out = out

    def __call__(self, x: torch.Tensor, stream: int) -> torch.Tensor:
        lib = self._lib
        lib.call("itq3_chain_run_ex", lib.ptr(self.desc), self.n, lib.ptr(x), 3, lib.ptr(self.epoch),
                 lib.ptr(self.out), 0, None, stream, self.run_flags)
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

        if self.hd != 128 or max_ctx > 1024 or self.nh * self.hd != self.h:
            raise ValueError("DecoderStack: the attention stages need head_dim 128, max_ctx <= 1024, nh * hd = hidden")
        # ONE launch per token: qkv_0, then per layer [attention partials, attention combine, o, gate_up,
        # down, next qkv / lm_head]; the residual after layer L lives in the tagged buffer res[L + 1]
        import os
        import struct

        G = self.nh // self.nkv
        if G != 4:
            raise ValueError("DecoderStack: the in-chain attention needs 4 query heads per kv head")
        sms = torch.cuda.get_device_properties(self.dev).multi_processor_count
        # attention items (kv head, split), at most one per SM: the combine fetches 8 splits per L2 round trip,
        # so the split count is rounded down to a multiple of 8 (B200, 8 kv heads: 16 splits, 1000 tok/s, vs
        # 18: 984 and 24 (two items on some SMs): 861).  ITQ3_ATTN_SPLITS overrides; ceil(max_ctx / splits) <= 64.
        per_sm = min(32, sms // self.nkv)
        self.splits = int(os.environ.get("ITQ3_ATTN_SPLITS", "0")) or max(1, per_sm - per_sm % 8 if per_sm >= 8 else per_sm)
        if -(-max_ctx // self.splits) > 64:  # positions per split (the chain's score scratch)
            raise ValueError("DecoderStack: ceil(max_ctx / attention splits) must be <= 64")
        if self.splits > 32:  # the combine reads split statistics one per lane
            raise ValueError("DecoderStack: at most 32 attention splits per kv head")
        self.res = [None] + [torch.zeros(self.h, dtype=torch.int64, device=self.dev) for _ in range(layers)]
        # residual + o of layer L (tagged), published by its gate_up stage: the next qkv stage's norm input is
        # then res_mid + down (two producers, one poll loop) instead of res + o + down
        self.res_mid = [torch.zeros(self.h, dtype=torch.int64, device=self.dev) for _ in range(layers)]
        self.att_y = [torch.zeros(self.h, dtype=torch.int64, device=self.dev) for _ in range(layers)]
        self.part_y = [torch.zeros(self.nkv * self.splits * 4 * 130, dtype=torch.int64, device=self.dev)
                       for _ in range(layers)]
        self.attn_params = []
        self.attn_err = torch.zeros(1, dtype=torch.int32, device=self.dev)
        for li in range(layers):
            raw = struct.pack("<QQQQQQiiii", self.k_cache[li, 0].data_ptr(), self.v_cache[li, 0].data_ptr(),
                              self.cos.data_ptr(), self.sin.data_ptr(), self.pos.data_ptr(),
                              self.attn_err.data_ptr(), self.nh, self.nkv, max_ctx, self.splits)
            assert len(raw) == _lib.load().itq3_chain_attn_params_nbytes()
            self.attn_params.append(torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(self.dev))
        stages = [dict(q=self.q[0][0], flags=NORM_IN, xin=self.gain[0][0])]
        for li, (_, o_w, gu_w, down_w) in enumerate(self.q):
            stages.append(dict(attn=256, params=self.attn_params[li], y=self.part_y[li]))
            stages.append(dict(attn=512, params=self.attn_params[li], y=self.att_y[li]))
            o_idx = len(stages)
            stages.append(dict(q=o_w))
            stages.append(dict(q=gu_w, flags=NORM_IN | RESID_IN | XOUT, xin=self.gain[li][1], xres=self.res[li],
                               xout=self.res_mid[li]))
            if li + 1 < layers:
                nxt = dict(q=self.q[li + 1][0], xin=self.gain[li + 1][0])
            elif self.lm_head is not None:
                nxt = dict(q=self.lm_head, xin=self.final_gain)
            else:
                nxt = None
            if nxt is None:  # the last layer without a head folds x + o + down into `out`
                stages.append(dict(q=down_w, flags=GATED | ADD_OUT | ADD_OUT0, ref=o_idx, xres=self.res[li]))
            else:
                stages.append(dict(q=down_w, flags=GATED))
                nxt.update(flags=NORM_IN | RESID_IN | XOUT, xres=self.res_mid[li], xout=self.res[li + 1])
                stages.append(nxt)
        self.n_stages = len(stages)
        self.token_chain = _Chain(stages, self.logits if self.lm_head is not None else self.out, self.dev)
        self.graph = None

    def weight_bytes(self) -> int:
        """Packed (tiled) ITQ3_S weight bytes one token streams: every layer's linears + the lm_head."""
        n = sum(int(t.numel()) for row in self.q for q in row for t in q._tiled.values())
        if self.lm_head is not None:
            n += sum(int(t.numel()) for t in self.lm_head._tiled.values())
        return n

    def launches_per_step(self) -> int:
        return 1

    def _rms(self, x, gain):
        return torch.nn.functional.rms_norm(x, (self.h,), weight=gain, eps=self.eps)

    def _rope(self, t, cos, sin):  # t: (heads, hd), rotate-half convention
        a, b = t[:, : self.hd // 2], t[:, self.hd // 2:]
        return torch.cat((a * cos - b * sin, a * sin + b * cos), dim=1)

    def _step(self) -> None:
        """One token: ONE chain launch over all layers (attention stages included), then the position
        advance (a device op, so the graphed step needs no host work)."""
        from . import _lib

        self.token_chain(self.x, _lib.stream_ptr(self.dev))
        if self.lm_head is not None:  # the final residual stream: low halves of the tagged words
            self.out.copy_(self.res[self.layers].view(torch.int32)[0::2].view(torch.float32))

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
        device and writes no cache entry: its error word, `device_error()`, is set)."""
        if x is not None:
            self.x.copy_(x)
        if self.graph is None:
            self.capture()
        self.replay()
        return self.out

    def device_error(self) -> int:
        """The attention stages' out-of-cache flag (non-zero after a replay at a position >= max_ctx)."""
        return int(self.attn_err.item())

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
