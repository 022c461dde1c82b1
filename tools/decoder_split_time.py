"""Where a decoder token's time goes: the one-launch token chain vs the same chain without its attention
stages (the o projection then reads the qkv outputs directly), both graphed and device-timed."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_27914_b200 import _lib  # noqa: E402
from paper_2603_27914_b200 import decoder as D  # noqa: E402


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
st = D.DecoderStack(layers=32, max_ctx=1024, seed=3000, dev=dev)
st.reset(512)
full = timed(lambda: st.token_chain(st.x, _lib.stream_ptr(dev)))
# the same stages without attention: rebuild the stage list from the token chain's inputs
stages = [dict(q=st.q[0][0], flags=D.NORM_IN, xin=st.gain[0][0])]
for li, (_, o_w, gu_w, down_w) in enumerate(st.q):
    o_idx = len(stages)
    stages.append(dict(q=o_w))
    stages.append(dict(q=gu_w, flags=D.NORM_IN | D.RESID_IN, xin=st.gain[li][1], xres=st.res[li]))
    stages.append(dict(q=down_w, flags=D.GATED))
    nxt = dict(q=st.q[li + 1][0], xin=st.gain[li + 1][0]) if li + 1 < st.layers else dict(q=st.lm_head, xin=st.final_gain)
    nxt.update(flags=D.NORM_IN | D.RESID2_IN | D.XOUT, ref=o_idx, xres=st.res[li], xout=st.res[li + 1])
    stages.append(nxt)
no_attn = D._Chain(stages, st.logits, dev)
gemv_only = timed(lambda: no_attn(st.x, _lib.stream_ptr(dev)))
print(f"token chain {full:.3f} ms ({st.n_stages} stages, 1 launch); without the {2 * st.layers} attention stages "
      f"{gemv_only:.3f} ms; attention stages {full - gemv_only:.3f} ms = {(full - gemv_only) / st.layers * 1000:.1f} us/layer")
