"""Fused tensor-parallel chain (parallel.TPChainStack) checked on ONE GPU.

    python tools/tp_chain_sim.py [--ranks 2] [--steps 4] [--timeout 60]

Two legs, each compared bit for bit with the single-GPU chain (stack.LinearStack, mode="chain") on
the full matrices:
  1. world 1: one TPChainStack whose only peer is itself (the fused-store path, .sys scope loads);
  2. world R simulated on one device: R TPChainStacks, one per virtual rank, each holding its row
     shards, its own tagged-output buffer and the peer table of all R buffers (device pointers on the
     same GPU stand in for NVLink peer pointers), each launched with grid = SMs / R on its own stream
     so the R cooperative kernels are co-resident and exchange stage outputs through the peer stores
     exactly as R GPUs would.
A host watchdog bounds the wait: if the kernels do not finish in --timeout seconds the process
exits (code 3) and the CUDA context is torn down with it.
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2603_27914_b200 as P  # noqa: E402
from paper_2603_27914_b200.parallel import TPChainStack, shard_bounds, shard_quantized, tp_chain_layout  # noqa: E402
from paper_2603_27914_b200.stack import LinearStack  # noqa: E402

SHAPES = [(1280, 512), (512, 1280), (8192, 512), (512, 8192), (1024, 512)]


def wait(ev, timeout):
    t0 = time.time()
    while not ev.query():
        if time.time() - t0 > timeout:
            print(f"TIMEOUT: tensor-parallel chain did not finish in {timeout} s", flush=True)
            os._exit(3)
        time.sleep(0.001)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", type=int, default=2)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--timeout", type=float, default=60.0)
    ap.add_argument("--asym", action="store_true")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(5)
    cfg = P.QuantConfig(symmetric=not a.asym)
    qs = [P.quantize_tensor(torch.randn((r, c), generator=g, device=dev) / c ** 0.5, cfg) for r, c in SHAPES]
    rows, cols = [r for r, _ in SHAPES], [c for _, c in SHAPES]
    ref = LinearStack(qs, mode="chain", lo=False)
    rng = np.random.default_rng(0)
    xs = [rng.standard_normal(cols[0]).astype(np.float32) for _ in range(a.steps)]
    want = [ref.forward(x).copy() for x in xs]

    # leg 1: world 1, the rank is its own only peer
    tp1 = TPChainStack(qs, rows, cols)
    for x, w in zip(xs, want):
        tp1.x.copy_(torch.from_numpy(x))
        tp1.launch_all()
        ev = torch.cuda.Event()
        ev.record()
        wait(ev, a.timeout)
        np.testing.assert_array_equal(tp1.output().cpu().numpy(), w)
    print("world 1: bit-exact with the single-GPU chain over", a.steps, "steps", flush=True)

    # leg 2: R virtual ranks on one device
    R = a.ranks
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    _, total = tp_chain_layout(rows, cols)
    bufs = [torch.zeros(total, dtype=torch.int64, device=dev) for _ in range(R)]
    bases = [b.data_ptr() for b in bufs]
    ranks = []
    for r in range(R):
        local = [shard_quantized(q, R, r) for q in qs]
        for i, q in enumerate(local):
            r0, r1 = shard_bounds(rows[i], R, r)
            assert q.rows == r1 - r0
        ranks.append(TPChainStack(local, rows, cols, world=R, rank=r, ybuf=bufs[r], peer_bases=bases, grid=sms // R))
    streams = [torch.cuda.Stream(dev) for _ in range(R)]
    torch.cuda.synchronize()
    for step, (x, w) in enumerate(zip(xs, want)):
        for r in range(R):
            ranks[r].x.copy_(torch.from_numpy(x))
        torch.cuda.synchronize()
        evs = []
        for r in range(R):
            with torch.cuda.stream(streams[r]):
                ranks[r].launch_all(stream=streams[r].cuda_stream)
                ev = torch.cuda.Event()
                ev.record(streams[r])
                evs.append(ev)
        for ev in evs:
            wait(ev, a.timeout)
        for r in range(R):
            np.testing.assert_array_equal(ranks[r].output().cpu().numpy(), w, err_msg=f"rank {r} step {step}")
    print(f"world {R} (simulated, grid {sms // R} per rank): every rank bit-exact with the single-GPU chain "
          f"over {a.steps} steps", flush=True)

    # leg 3: the ranks run back to back without host synchronisation between steps (a rank may
    # enter step t+1 while a peer is still in step t: the epoch-parity double buffer keeps them apart)
    for r in range(R):
        ranks[r].x.copy_(torch.from_numpy(xs[0]))
    torch.cuda.synchronize()
    n = 20
    evs = []
    t0 = time.time()
    for r in range(R):
        with torch.cuda.stream(streams[r]):
            for _ in range(n):
                ranks[r].launch_all(stream=streams[r].cuda_stream)
            ev = torch.cuda.Event()
            ev.record(streams[r])
            evs.append(ev)
    for ev in evs:
        wait(ev, a.timeout)
    for r in range(R):
        np.testing.assert_array_equal(ranks[r].output().cpu().numpy(), want[0], err_msg=f"rank {r} free-running")
    print(f"free-running {n} steps per rank: bit-exact ({(time.time() - t0) * 1e3 / n:.3f} ms/step wall)", flush=True)


if __name__ == "__main__":
    main()
