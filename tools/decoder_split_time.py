"""Where a decoder token's time goes: the full graphed step vs graphs of only its chain launches and
only its attention launches (same buffers, same order)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_27914_b200 import _lib  # noqa: E402
from paper_2603_27914_b200.decoder import DecoderStack  # noqa: E402


def timed(fn, reps=20):
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


dev = torch.device("cuda", 0)
st = DecoderStack(layers=32, max_ctx=1024, seed=3000, dev=dev)
st.capture()
st.reset(512)


def chains():
    s = _lib.stream_ptr(dev)
    st.first(st.xs2[0], s)
    for li in range(st.layers):
        st.chains[li](st.xs2[li % 2], s)


def attn():
    s = _lib.stream_ptr(dev)
    for li in range(st.layers):
        _lib.call("itq3_glue_rope_attention", _lib.ptr(st.qkv_out), _lib.ptr(st.cos), _lib.ptr(st.sin),
                  _lib.ptr(st.pos), _lib.ptr(st.k_cache[li, 0]), _lib.ptr(st.v_cache[li, 0]), _lib.ptr(st.att),
                  st.nh, st.nkv, st.hd, st.max_ctx, _lib.ptr(st.attn_ws), s)


full = timed(lambda: st._step_no_pos() if hasattr(st, "_step_no_pos") else st._step())
st.reset(512)
print(f"full step {full:.3f} ms; chains only {timed(chains):.3f} ms; attention only {timed(attn):.3f} ms "
      f"({st.layers} layers, position ~512)")
