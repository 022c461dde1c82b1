"""Timeline of one decoder token (the gated chain launch), per stage kind: needs an experiment build with
-DCHAIN_GATED_TRACE (tools/ab_build_src.sh trace paper_2603_27914_b200/csrc/chain.cu chain -DCHAIN_GATED_TRACE;
ITQ3_LIB=exp_libs/libitq3_trace.so python tools/trace_decoder.py).

Per stage kind (attention partials, combine, o, gate_up, down, qkv) the median over layers of: the stage's
critical path (max over CTAs of its end stamp minus the previous stage's), the median CTA's wait (entered ->
input ready), rotation and compute, and how late the earliest CTA saw its input after the previous stage's
last CTA finished (store -> L2 -> poll).
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2603_27914_b200 import _lib  # noqa: E402
from paper_2603_27914_b200.decoder import DecoderStack  # noqa: E402


def main():
    dev = torch.device("cuda", 0)
    d = DecoderStack(layers=32, max_ctx=1024, dev=dev)
    ch = d.token_chain
    S = ch.n
    G = torch.cuda.get_device_properties(dev).multi_processor_count
    trace = torch.zeros(G * S * 4 + S * 64 + 128, dtype=torch.int64, device=dev)
    d.reset(512)
    d.x.normal_()
    stream = _lib.stream_ptr(dev)
    for _ in range(4):
        trace.zero_()
        _lib.call("itq3_chain_run_ex", _lib.ptr(ch.desc), S, _lib.ptr(d.x), 3, _lib.ptr(ch.epoch), _lib.ptr(ch.out),
                 0, _lib.ptr(trace), stream, ch.run_flags)
        torch.cuda.synchronize()
    raw = trace.cpu().numpy().astype(np.float64)
    t = raw[: G * S * 4].reshape(G, S, 4)
    t0 = np.min(np.where(t[:, 0, 0] > 0, t[:, 0, 0], np.inf))
    t = np.where(t > 0, (t - t0) / 1000.0, np.nan)  # us, NaN = CTA idle in that stage
    end = np.nanmax(t[:, :, 3], axis=0)
    crit = np.diff(np.concatenate([[0.0], end]))
    print(f"token {np.nanmax(end):.1f} us over {S} stages")
    names = ["attn_part", "attn_comb", "o", "gate_up", "down", "qkv/head"]
    print("stage 0 (qkv_0): %.2f us" % crit[0])
    for k, n in enumerate(names):
        idx = list(range(1 + k, S, 6))
        c = np.median(crit[idx])
        active = np.median([np.sum(~np.isnan(t[:, i, 3])) for i in idx])
        w = np.nanmedian(t[:, idx, 1] - t[:, idx, 0]) if k >= 2 else float("nan")
        r = np.nanmedian(t[:, idx, 2] - t[:, idx, 1]) if k >= 2 else float("nan")
        cm = np.nanmedian(t[:, idx, 3] - t[:, idx, 2]) if k >= 2 else np.nanmedian(t[:, idx, 3] - t[:, idx, 0])
        first = np.median([np.nanmin(t[:, i, 1 if k >= 2 else 0]) - end[i - 1] for i in idx])
        skew = np.median([np.nanmax(t[:, i, 3]) - np.nanmedian(t[:, i, 3]) for i in idx])
        print(f"{n:9s} crit {c:6.2f} us  CTAs {active:4.0f}  wait {w:5.2f}  rotate {r:5.2f}  compute/med {cm:5.2f}  "
              f"first input after prev end {first:5.2f}  end skew (max-med) {skew:5.2f}")
    print("sum of medians x 32: %.1f us" % (32 * sum(np.median(crit[list(range(1 + k, S, 6))]) for k in range(6))))


if __name__ == "__main__":
    main()
