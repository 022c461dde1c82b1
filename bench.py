#!/usr/bin/env python
"""Benchmark: batch-1 decode through a Llama-2-7B-shaped ITQ3_S linear stack (BASELINE.json configs[1]).

Step = one decode token through 32 layers x 4 dependent fused GEMV stages
      qkv 12288x4096 -> o 4096x4096 -> gate_up 22016x4096 -> down 4096x11008
(Llama-2-7B linear shapes, q/k/v and gate/up concatenated as serving engines do), each stage's
input being the previous stage's output.  Per stage: K3 rotate_act + K4 fused IFWHT-dequant
GEMV (libitq3.so), the whole chain replayed as one CUDA graph.  Weights: random-init
N(0, 1/K), quantized on the GPU by the K1 encoder (bit-exact ITQ3_S), 1.69 GB of tiled codes
per step (> 126 MB L2, so every step streams from HBM without an explicit flush).

  value        tokens/s (device-timed with CUDA events, max over ranks; N ranks = N replicas)
  e2e          tokens/s through LinearStack.forward(host x) incl. H2D of x and D2H of y
  roofline     the GEMV kernel: algorithmic bytes / CUDA-event time of a graph of all its launches
  cpu_baseline the CPU oracle (oracle/itq3_oracle.py, numpy port of the reference) on a row
               sample, all host cores
`--impl reference` times that CPU path alone (the reference arm; reference is pure Python).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# linear shapes (rows x K) per decoder layer; q/k/v and gate/up concatenated as serving engines do
MODELS = {
    "llama2-7b": (32, [("qkv", 12288, 4096), ("o", 4096, 4096), ("gate_up", 22016, 4096), ("down", 4096, 11008)]),
    "llama3-8b": (32, [("qkv", 6144, 4096), ("o", 4096, 4096), ("gate_up", 28672, 4096), ("down", 4096, 14336)]),
    "llama3-70b": (80, [("qkv", 10240, 8192), ("o", 8192, 8192), ("gate_up", 57344, 8192), ("down", 8192, 28672)]),
}
MODEL = os.environ.get("ITQ3_BENCH_MODEL", "llama2-7b")
for _i, _a in enumerate(sys.argv):  # resolved before argparse so module constants follow --model
    if _a == "--model" and _i + 1 < len(sys.argv):
        MODEL = sys.argv[_i + 1]
    elif _a.startswith("--model="):
        MODEL = _a.split("=", 1)[1]
N_LAYERS, LAYER_SHAPES = MODELS[MODEL]
WEIGHTS_PER_TOKEN = N_LAYERS * sum(r * c for _, r, c in LAYER_SHAPES)  # llama2-7b: 6,476,005,376
METRIC = "decode tokens/sec (batch-1 fused IFWHT-dequant GEMV chain, %s linear shapes)" % MODEL
WORKLOAD = "%s linear stack decode: %d layers x (%s), batch 1" % (
    MODEL, N_LAYERS, ", ".join(f"{n} {r}x{c}" for n, r, c in LAYER_SHAPES))
FALLBACK_HBM_GBS = 6650.0


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


# ------------------------------------------------------------------------------------------------
# CPU path (oracle port of the reference) -- used for cpu_baseline and --impl reference
# ------------------------------------------------------------------------------------------------
_CPU_STATE = {}


def _cpu_init(rows_per_stage: int, seed: int):
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np

    from oracle import itq3_oracle as O

    rng = np.random.default_rng(seed)
    work = []
    for _, rows, cols in LAYER_SHAPES:
        w = (rng.standard_normal((rows_per_stage, cols)) / math.sqrt(cols)).astype(np.float32)
        pay, _ = O.quantize_payload(w)
        x = rng.standard_normal(cols).astype(np.float32)
        work.append((pay, rows_per_stage, cols, x))
    _CPU_STATE["work"] = work


def _cpu_step(_):
    """One bounded sample: the reference algorithm (decode each block exactly, fp64 dot) over
    rows_per_stage rows of each of the 4 stage shapes."""
    from oracle import itq3_oracle as O

    t = time.perf_counter()
    n = 0
    for pay, rows, cols, x in _CPU_STATE["work"]:
        O.fused_matmul(pay, rows, cols, 256, False, x[:, None])
        n += rows * cols
    return n, time.perf_counter() - t


class CpuArm:
    def __init__(self, rows_per_stage: int = 64, procs: int | None = None):
        import multiprocessing as mp

        self.procs = procs or len(os.sched_getaffinity(0))
        self.rows = rows_per_stage
        # fresh interpreters with single-threaded BLAS: one core per worker, no inherited
        # thread pools or CUDA state from the parent
        for var in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
            os.environ[var] = "1"
        ctx = mp.get_context("spawn")
        self.pool = ctx.Pool(self.procs, initializer=_cpu_init, initargs=(rows_per_stage, 1234))
        self.weights_per_step = self.procs * rows_per_stage * sum(c for _, _, c in LAYER_SHAPES)

    def step(self) -> float:
        t = time.perf_counter()
        self.pool.map(_cpu_step, range(self.procs), chunksize=1)
        return time.perf_counter() - t

    def sample_desc(self) -> str:
        return (f"{self.rows} rows of each stage shape per process x {self.procs} processes = "
                f"{self.weights_per_step} weights/step ({self.weights_per_step / WEIGHTS_PER_TOKEN:.2e} of a token), "
                "oracle fused_matmul (exact block decode + fp64 dot); tokens/s extrapolated by weight count")

    def close(self):
        self.pool.terminate()


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    arm = CpuArm(rows_per_stage=args.cpu_rows)
    for _ in range(args.warmup):
        arm.step()
    times = [arm.step() for _ in range(args.steps)]
    arm.close()
    tot = sum(times)
    tok_s = arm.weights_per_step * args.steps / tot / WEIGHTS_PER_TOKEN
    line = {
        "impl": "reference", "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: N(0,1/K) weights quantized by the oracle encoder, random fp32 x",
        "config": {"workload": WORKLOAD, "global_batch": 1, "parallelism": "cpu-processes"},
        "cpu_baseline": {"value": tok_s, "unit": "tokens/s", "cores": arm.procs, "kind": "port",
                         "sample": arm.sample_desc()},
        "e2e": {"value": tok_s, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------
# GPU arm
# ------------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([f.strip() for f in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if len(r) >= 8 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 8 for i in range(4) if r[4 + i] == "Active"})
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    """dram bytes per GEMV launch from the committed ncu --set full capture, if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_gemv_traffic.json")) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def build_stack(n_layers: int, seed: int, dev, mode: str = "chain"):
    import torch

    import paper_2603_27914_b200 as P
    from paper_2603_27914_b200.stack import LinearStack

    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    qs = []
    for _ in range(n_layers):
        for _, rows, cols in LAYER_SHAPES:
            w = torch.randn((rows, cols), generator=g, device=dev, dtype=torch.float32).mul_(1.0 / math.sqrt(cols))
            q = P.quantize_tensor(w)  # K1 encoder, bit-exact ITQ3_S container payload
            q.tiled()
            q.drop_payload()  # serving keeps only the tiled copy resident
            qs.append(q)
            del w
    return LinearStack(qs, limbs=3, mode=mode)


def run_decoder(args):
    """--decoder: BASELINE configs[3], a full Llama-3-8B-shaped decoder (RMSNorm, RoPE, grouped-query
    attention over a KV cache, SiLU gating) with every linear an ITQ3_S tensor on the fused GEMV;
    random N(0, 0.02^2) weights quantised on the GPU.  One CUDA graph per token; the timed tokens
    decode positions 512.. of a 1024-position cache.  Replicas only (no collective) for N > 1."""
    import torch

    from paper_2603_27914_b200.decoder import DecoderStack

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    st = DecoderStack(layers=args.layers, max_ctx=1024, seed=3000 + rank, dev=dev)
    st.capture()
    st.reset(512)
    g = torch.Generator(device=dev)
    g.manual_seed(rank)
    st.x.copy_(torch.randn(st.h, generator=g, device=dev))
    for _ in range(args.warmup):
        st.graph.replay()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        st.graph.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    tiled = sum(int(t.numel()) for row in st.q for q in row for t in q._tiled.values())
    if rank == 0:
        print(json.dumps({
            "metric": "decode tokens/sec (batch-1 ITQ3_S decoder: fused IFWHT-dequant GEMV chains with RMSNorm, gating and residuals folded in, + a RoPE/attention kernel)",
            "value": world * 1000.0 / ms, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "u8xs8->s32 mma + fp32",
            "data": "synthetic: random-init N(0, 0.02^2) weights quantized to ITQ3_S on the GPU, random hidden state",
            "config": {"workload": f"llama3-8b decoder decode: {args.layers} layers (hidden 4096, ffn 14336, "
                                   "32 heads / 8 kv heads, head_dim 128), positions 512+ of a 1024 KV cache",
                       "model": "llama3-8b (decoder, random init)", "global_batch": world, "seq_len": 1,
                       "parallelism": "single" if world == 1 else f"replicas{world}"},
            "packed_weight_gbps": tiled / (ms / 1000.0) / 1e9,
            "gpu_launches": 4 * args.layers * args.steps}), flush=True)  # 3 chains + 1 attention kernel per layer
    if world > 1:
        torch.distributed.destroy_process_group()


def run_tp(args):
    """--tp: ONE token stream row-sharded over the ranks (strong scaling): each rank holds
    rows shard_bounds(r, world, rank) of every stage.  --tp-impl fused (default): one persistent chain
    kernel per rank whose reducers store every output word into all ranks' copies of y over NVLink
    (symmetric-memory peer pointers) -- the all-gather is fused, no NCCL call in the step.
    --tp-impl nccl: K3+K4 kernels and an NCCL all_gather per stage, one CUDA graph per step."""
    import torch

    import paper_2603_27914_b200 as P
    from paper_2603_27914_b200.parallel import TPChainStack, TPStack, shard_bounds

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    g = torch.Generator(device=dev)
    g.manual_seed(2000 + rank)
    qs, rows, cols = [], [], []
    for _ in range(args.layers):
        for _, r, c in LAYER_SHAPES:
            r0, r1 = shard_bounds(r, world, rank)
            w = torch.randn((max(r1 - r0, 1), c), generator=g, device=dev).mul_(1.0 / math.sqrt(c))
            q = P.quantize_tensor(w)
            q.tiled()
            qs.append(q)
            rows.append(r)
            cols.append(c)
            del w
    if args.tp_impl == "fused":
        st = TPChainStack(qs, rows, cols)  # one chain kernel per rank, all-gather fused into peer stores
    else:
        st = TPStack(qs, rows, cols)  # K3 + K4 + NCCL all_gather per stage
    st.capture()
    for _ in range(args.warmup):
        st.replay()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        st.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        tiled_bytes = sum(int(t.numel()) for t in st.tiled) * world
        print(json.dumps({
            "metric": METRIC.replace("GEMV chain", "GEMV chain, tensor-parallel"), "value": 1000.0 / ms,
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8xs8->s32 mma + fp32",
            "data": "synthetic: random-init N(0,1/K) row shards quantized to ITQ3_S on each GPU",
            "config": {"workload": WORKLOAD, "model": f"{MODEL} (linear layers)", "global_batch": 1, "seq_len": 1,
                       "parallelism": f"tp{world} (row-sharded stages; " + (
                           "all-gather fused into the chain kernel's peer stores)" if args.tp_impl == "fused"
                           else "NCCL all-gather per stage)")},
            "packed_weight_gbps": tiled_bytes / (ms / 1000.0) / 1e9,
            "gpu_launches": (1 if args.tp_impl == "fused" else 2 * len(qs)) * args.steps}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_ours(args):
    import numpy as np
    import torch

    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stack = build_stack(args.layers, 1000 + rank, dev, args.mode)
    stack.capture()
    x0 = torch.from_numpy(np.random.default_rng(rank).standard_normal(stack.x.numel()).astype(np.float32))
    stack.forward(x0)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    # ---- timed region: device value -------------------------------------------------------------
    for _ in range(args.warmup):
        stack.replay()
    barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        stack.replay()
    e1.record()
    barrier()
    clk = clocks.stop()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    value = world * 1000.0 / ms

    # ---- e2e: public API with host buffers (H2D x, graphed chain, D2H y) -------------------------
    for _ in range(args.warmup):
        stack.forward(x0)
    barrier()
    t = time.perf_counter()
    for _ in range(args.steps):
        stack.forward(x0)
    e2e_ms = max_over_ranks(1000.0 * (time.perf_counter() - t) / args.steps)

    # ---- roofline: the chain kernel is the only kernel of the step (1 launch + a counter memset) ----
    peak, peak_src = measured_peak()
    traffic = ncu_traffic()
    step_bytes = stack.step_bytes()
    achieved = step_bytes / (ms / 1000.0) / 1e9
    # the same kernel with the inter-stage dependency removed (every stage reads a fixed x):
    # pure weight streaming -> the kernel's own HBM roofline, separate from dependency latency
    from paper_2603_27914_b200.stack import LinearStack as _LS

    st_ind = _LS(stack.qs, limbs=stack.limbs, mode="chain", independent=True)
    st_ind.capture()
    for _ in range(3):
        st_ind.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        st_ind.replay()
    e1.record()
    torch.cuda.synchronize()
    ind_ms = e0.elapsed_time(e1) / args.steps
    streaming = {"gbps": step_bytes / (ind_ms / 1000.0) / 1e9, "frac": step_bytes / (ind_ms / 1000.0) / 1e9 / peak,
                 "ms_per_pass": ind_ms, "desc": "chain kernel, same 128 GEMVs, inter-stage dependency removed"}
    del st_ind
    # for comparison: the same chain as 2 launches per stage (rotate_act + gemv) in one graph
    sep = None
    if not args.no_compare:
        from paper_2603_27914_b200.stack import LinearStack

        st2 = LinearStack(stack.qs, limbs=stack.limbs, mode="kernels")
        st2.capture()
        for _ in range(3):
            st2.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            st2.replay()
        e1.record()
        torch.cuda.synchronize()
        sep = 1000.0 / (e0.elapsed_time(e1) / args.steps)
        del st2

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        arm = CpuArm(rows_per_stage=args.cpu_rows)
        arm.step()
        ts = [arm.step() for _ in range(args.cpu_steps)]
        arm.close()
        cpu_tok = arm.weights_per_step * len(ts) / sum(ts) / WEIGHTS_PER_TOKEN
        cpu = {"value": cpu_tok, "unit": "tokens/s", "cores": arm.procs, "kind": "port", "sample": arm.sample_desc()}
    tiled_bytes = sum(int(t.numel()) for t in stack.tiled)
    n_st = len(stack.qs)
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8xs8->s32 mma + fp32",
        "data": "synthetic: random-init N(0,1/K) weights quantized to ITQ3_S on the GPU (K1), random fp32 x0",
        "config": {"workload": WORKLOAD, "model": f"{MODEL} (linear layers)", "global_batch": world,
                   "seq_len": 1, "parallelism": f"replicas{world}" if world > 1 else "single",
                   "stages_per_step": n_st, "activation_limbs": stack.limbs,
                   "l2": f"{tiled_bytes / 1e9:.2f} GB of tiled weights per step > 126 MB L2; no flush needed"},
        "packed_weight_gbps": tiled_bytes / (ms / 1000.0) / 1e9,
        "container_equiv_gbps": WEIGHTS_PER_TOKEN * 100 / 256 / (ms / 1000.0) / 1e9,
        "separate_kernels_tokens_per_s": sep,
        "streaming_roofline": streaming,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic.get("bytes_per_launch") if traffic else None,
                     "kernel": "itq3::chain_kernel (whole step, 1 launch)", "peak_source": peak_src,
                     "bytes_per_launch": step_bytes, "launch_us": ms * 1000.0,
                     "algorithmic_bytes": "66 B per 256 weights (64 B 2-bit codes + 2 B f16 scale) + 800 B per "
                                          "256-block of rotated activation (3 limbs) + 4 B per output row"},
        "cpu_baseline": cpu,
        "e2e": {"value": world * 1000.0 / e2e_ms, "unit": "tokens/s", "h2d_bytes_per_step": 4 * stack.x.numel(),
                "d2h_bytes_per_step": 4 * stack.ys[-1].numel(), "api": "LinearStack.forward(host np.float32)"},
        "gpu_launches": stack.launches_per_step * args.steps,
        "clocks": clk,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--cpu-rows", type=int, default=64)
    ap.add_argument("--cpu-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-compare", action="store_true")
    ap.add_argument("--mode", choices=["chain", "kernels"], default="chain")
    ap.add_argument("--model", choices=sorted(MODELS), default=MODEL)
    ap.add_argument("--tp", action="store_true", help="row-shard one token stream over the ranks (C5)")
    ap.add_argument("--decoder", action="store_true", help="configs[3]: full Llama-3-8B-shaped decoder decode step")
    ap.add_argument("--tp-impl", choices=["fused", "nccl"], default="fused",
                    help="--tp: fused chain kernel with NVLink peer stores, or per-stage kernels + NCCL all_gather")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.layers is None:
        args.layers = N_LAYERS
    if args.impl == "reference":
        run_reference(args)
    elif args.tp:
        run_tp(args)
    elif args.decoder:
        run_decoder(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
