"""Timeline of one chain-kernel step (globaltimer stamps per CTA and stage).

    python tools/trace_chain.py [--layers 32]
Prints, per stage kind, the median over CTAs of: wait for the previous stage (entered ->
input ready), rotation (ready -> rotated), compute (rotated -> last tile published), and the
stage's critical path (max publish of s - max publish of s-1).
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=32)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    st = bench.build_stack(args.layers, 1000, dev, "chain")
    tr = st.enable_trace()
    x = np.random.default_rng(0).standard_normal(st.x.numel()).astype(np.float32)
    ap2 = os.environ.get("TRACE_INDEPENDENT")
    if ap2:
        from paper_2603_27914_b200.stack import LinearStack
        st = LinearStack(st.qs, limbs=3, mode="chain", independent=True)
        tr = st.enable_trace()
    for _ in range(3):
        st.forward(x)
    raw = tr.cpu().numpy().astype(np.float64)
    S = len(st.qs)
    G = (raw.size - S * 64 - 128) // (S * 4)
    t = raw[: G * S * 4].reshape(G, S, 4)
    wt = raw[G * S * 4: G * S * 4 + S * 64].reshape(S, 16, 4)
    cyc = raw[G * S * 4 + S * 64:G * S * 4 + S * 64 + 64].reshape(16, 4)
    c_in = raw[G * S * 4 + S * 64 + 64:G * S * 4 + S * 64 + 80]
    tot = cyc[:, 3].mean()
    print("CTA0 compute-warp cycle split (mean over warps): wait_full %.1f%%  tiles %.1f%%  rotate+input %.1f%%  "
          "(total %.0f cycles)" % (100 * cyc[:, 0].mean() / tot, 100 * cyc[:, 1].mean() / tot,
                                   100 * cyc[:, 2].mean() / tot, tot))
    print("  of which input wait+load %.1f%%, rotation proper %.1f%%; per stage: input %.0f, rotation %.0f cycles"
          % (100 * c_in.mean() / tot, 100 * (cyc[:, 2].mean() - c_in.mean()) / tot, c_in.mean() / S,
             (cyc[:, 2].mean() - c_in.mean()) / S))
    t0 = t[:, 0, 0].min()
    t = (t - t0) / 1000.0  # us
    wt = np.where(wt > 0, (wt - t0) / 1000.0, np.nan)
    names = [n for n, _, _ in bench.LAYER_SHAPES]
    crit = np.diff(np.concatenate([[0.0], t[:, :, 3].max(axis=0)]))
    print(f"step {t[:, :, 3].max():.1f} us over {S} stages; per-stage critical path median {np.median(crit):.2f} us")
    for k, n in enumerate(names):
        idx = list(range(k, S, len(names)))
        w = np.median(t[:, idx, 1] - t[:, idx, 0])
        r = np.median(t[:, idx, 2] - t[:, idx, 1])
        c = np.median(t[:, idx, 3] - t[:, idx, 2])
        cm = np.median((t[:, idx, 3] - t[:, idx, 2]).max(axis=0))
        print(f"{n:8s} wait {w:6.2f}  rotate {r:5.2f}  compute med {c:6.2f} max {cm:6.2f}  crit {np.median(crit[idx]):6.2f} us")
    # CTA 0 per-warp detail, relative to the stage's "rotated" stamp: first full wait, tiles, publish
    for k, n in enumerate(names):
        idx = list(range(k, S, len(names)))
        base = t[0, idx, 2][:, None]
        fw = np.nanmedian(wt[idx, :, 1] - base)
        td = np.nanmedian(wt[idx, :, 2] - base)
        pb = np.nanmedian(wt[idx, :, 3] - wt[idx, :, 2])
        print(f"  cta0 {n:8s} first-full {fw:6.2f}  tiles-done {td:6.2f}  publish-fence {pb:5.2f} us (warp medians)")
    # publish skew: last-first publish time of a stage
    sk = t[:, :, 3].max(axis=0) - t[:, :, 3].min(axis=0)
    print(f"publish skew across CTAs median {np.median(sk):.2f} us")
    # dependency latency: stage s+1 input ready on a CTA minus the LAST CTA's tiles-done of stage s
    # (min over CTAs ~ store -> visible -> poll; median adds the CTAs that were still busy), and the
    # imbalance of stage s (last tiles-done minus the median one)
    last = t[:, :, 3].max(axis=0)
    lat = t[:, 1:, 1] - last[None, :-1]
    imb = last - np.median(t[:, :, 3], axis=0)
    for k, n in enumerate(names):
        idx = [i for i in range(k, S, len(names)) if i >= 1]
        lo = np.median(np.nanmin(np.where(t[:, idx, 1] > 0, lat[:, [i - 1 for i in idx]], np.nan), axis=0))
        md = np.median(np.median(lat[:, [i - 1 for i in idx]], axis=0))
        print(f"  {n:8s} input ready after the last producer: min {lo:5.2f} median {md:5.2f} us; "
              f"producer-stage imbalance {np.median(imb[[i - 1 for i in idx]]):5.2f} us")


if __name__ == "__main__":
    main()
