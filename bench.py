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


def _argv_value(flag: str):
    for i, a in enumerate(sys.argv):
        if a == flag and i + 1 < len(sys.argv):
            return sys.argv[i + 1]
        if a.startswith(flag + "="):
            return a.split("=", 1)[1]
    return None


def _default_model() -> str:
    """--model, else ITQ3_BENCH_MODEL, else: N = 1 -> llama2-7b (configs[1], the headline); N > 1 ->
    llama3-70b row-sharded over the ranks (configs[4], C5) unless --replicas is given."""
    m = _argv_value("--model") or os.environ.get("ITQ3_BENCH_MODEL")
    if m:
        return m
    n = int(_argv_value("--gpus") or os.environ.get("WORLD_SIZE", "1"))
    return "llama3-70b" if n > 1 and "--replicas" not in sys.argv else "llama2-7b"


MODEL = _default_model()  # resolved before argparse so module constants follow --model / --gpus
N_LAYERS, LAYER_SHAPES = MODELS[MODEL]
WEIGHTS_PER_TOKEN = N_LAYERS * sum(r * c for _, r, c in LAYER_SHAPES)  # llama2-7b: 6,476,005,376
METRIC = "decode tokens/sec (batch-1 fused IFWHT-dequant GEMV chain, %s linear shapes)" % MODEL
WORKLOAD = "%s linear stack decode: %d layers x (%s), batch 1" % (
    MODEL, N_LAYERS, ", ".join(f"{n} {r}x{c}" for n, r, c in LAYER_SHAPES))
FALLBACK_HBM_GBS = 6650.0
FALLBACK_BF16_TFLOPS = 1590.0  # B200_PROFILING.md's fallback dense bf16 figure (used only without MEASURED_PEAKS.json)


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
    """dram bytes per chain launch from the committed ncu --set full capture (profiles/), used only if the
    capture was taken of the chain.cu now in the tree (its SHA-256 is recorded with the capture);
    otherwise None and a note in the line, never a stale number."""
    import hashlib

    try:
        with open(os.path.join(ROOT, "profiles", "ncu_gemv_traffic.json")) as f:
            rec = json.load(f)
        with open(os.path.join(ROOT, "paper_2603_27914_b200", "csrc", "chain.cu"), "rb") as f:
            sha = hashlib.sha256(f.read()).hexdigest()
    except (OSError, ValueError):
        return None
    if rec.get("chain_cu_sha256") != sha:
        print("bench.py: profiles/ncu_gemv_traffic.json was captured from another chain.cu; traffic = null",
              file=sys.stderr)
        return {"bytes_per_launch": None, "stale": True}
    return rec


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
            "gpu_launches": st.launches_per_step() * args.steps}), flush=True)  # 2 chains + 1 attention per layer
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
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        st.replay()
    e1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1) / args.steps

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    ms = max_over_ranks(ms)
    e2e = None
    if hasattr(st, "forward"):  # public API, host buffers: H2D x + graphed step + D2H of the gathered y
        import numpy as np

        x0 = np.random.default_rng(7).standard_normal(cols[0]).astype(np.float32)
        for _ in range(args.warmup):
            st.forward(x0)
        if world > 1:
            torch.distributed.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            st.forward(x0)
        e2e_ms = max_over_ranks(1000.0 * (time.perf_counter() - t0) / args.steps)
        e2e = {"value": 1000.0 / e2e_ms, "unit": "tokens/s", "h2d_bytes_per_step": 4 * cols[0],
               "d2h_bytes_per_step": 4 * rows[-1], "api": "TPChainStack.forward(host np.float32) on every rank"}
    local_bytes = sum(int(t.numel()) for t in st.tiled)
    tot_bytes = local_bytes
    if world > 1:
        t = torch.tensor([float(local_bytes)], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t)
        tot_bytes = int(t.item())
    peak, peak_src = measured_peak()
    nvl = st.nvlink_bytes_per_step() * world if hasattr(st, "nvlink_bytes_per_step") else None
    if rank == 0:
        per_gpu = tot_bytes / world / (ms / 1000.0) / 1e9
        print(json.dumps({
            "metric": METRIC.replace("GEMV chain", "GEMV chain, tensor-parallel"), "value": 1000.0 / ms,
            "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u8xs8->s32 mma + fp32",
            "data": "synthetic: random-init N(0,1/K) row shards quantized to ITQ3_S on each GPU",
            "config": {"workload": WORKLOAD, "model": f"{MODEL} (linear layers)", "global_batch": 1, "seq_len": 1,
                       "parallelism": f"tp{world} (row-sharded stages; " + (
                           "all-gather fused into the chain kernel's peer stores)" if args.tp_impl == "fused"
                           else "NCCL all-gather per stage)"),
                       "l2": f"{tot_bytes / world / 1e9:.2f} GB of tiled weights per GPU per step > 126 MB L2"},
            "packed_weight_gbps": tot_bytes / (ms / 1000.0) / 1e9,
            "packed_weight_gbps_per_gpu": per_gpu,
            "nvlink_bytes_per_token": nvl,
            "roofline": {"bound": "hbm", "achieved": per_gpu, "peak": peak, "unit": "GB/s", "frac": per_gpu / peak,
                         "traffic": None, "kernel": "itq3::chain_kernel per rank (whole step, 1 launch)",
                         "peak_source": peak_src},
            "e2e": e2e,
            "gpu_launches": (1 if args.tp_impl == "fused" else 2 * len(qs)) * args.steps,
            "clocks": clk}), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


# ------------------------------------------------------------------------------------------------
# extra keys of the N = 1 line: C3 MMQ (configs[2]) and C4 decoder (configs[3]), device-timed
# ------------------------------------------------------------------------------------------------
def graph_time(fn, reps):
    """Device time per call of fn(i): reps calls captured in one CUDA graph, CUDA events around a replay."""
    import torch

    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for i in range(3):
            fn(i)
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(reps):
            fn(i)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


INT8_NOMINAL_TOPS = 4500.0  # B200 dense int8 (datasheet; no measured int8 peak in MEASURED_PEAKS.json)


def measure_c3(dev, reps: int = 20) -> dict:
    """BASELINE configs[2] at the Llama-3-8B gate/up shape 14336 x 4096: K5 (tcgen05 kind::f16 CTA pairs)
    at M = 2048 in TFLOPS, K5b (kind::i8) at M = 16 / 64 in packed GB/s.  Calls rotate over 11 distinct
    weight copies (> 160 MB > L2), so every call streams its weights from HBM."""
    import torch

    import paper_2603_27914_b200 as P
    from paper_2603_27914_b200 import _lib

    rows, K = 14336, 4096
    lib = _lib.load()
    g = torch.Generator(device=dev)
    g.manual_seed(33)
    copies = []
    for _ in range(11):
        q = P.quantize_tensor(torch.randn((rows, K), generator=g, device=dev).mul_(K ** -0.5))
        copies.append((q.mmq_layout(), q.mmq8_layout()))
        del q
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except (OSError, ValueError):
        pass
    bf16 = float(peaks.get("bf16_tflops", 0) or 0) or None
    bf16_src = "measured (MEASURED_PEAKS.json bf16_tflops)"
    if bf16 is None:
        bf16, bf16_src = FALLBACK_BF16_TFLOPS, "fallback (B200_PROFILING.md)"
    hbm, _ = measured_peak()
    out = {"shape": f"{rows}x{K}", "weight_copies": len(copies)}
    for M in (16, 64, 2048):
        small = P.compute.MMQ_MIN_TOKENS <= M <= P.compute.MMQ8_MAX_TOKENS
        X = torch.randn((K, M), generator=g, device=dev)
        act = torch.empty(lib.itq3_mmq8_act_nbytes(K, M) if small else lib.itq3_mmq_act_nbytes(K, M),
                          dtype=torch.uint8, device=dev)
        Y = torch.empty((rows, M), dtype=torch.float32, device=dev)
        wsn = lib.itq3_mmq8_ws_nbytes(rows, K, M) if small else lib.itq3_mmq_ws_nbytes(rows, K, M)
        ws = torch.empty(max(wsn, 1), dtype=torch.uint8, device=dev)

        def rot(i):
            s = _lib.stream_ptr(dev)
            name = "itq3_rotate_act_i8" if small else "itq3_rotate_act_f16"
            _lib.call(name, _lib.ptr(X), _lib.F32, K, M, X.stride(0), X.stride(1), _lib.ptr(act), None, s)

        def mm(i):
            s = _lib.stream_ptr(dev)
            w = copies[i % len(copies)][1 if small else 0]
            if small:
                _lib.call("itq3_mmq8", _lib.ptr(w), rows, K, _lib.ptr(act), M, _lib.ptr(Y), _lib.F32, Y.stride(0),
                          Y.stride(1), _lib.ptr(ws) if wsn else None, s)
            else:
                _lib.call("itq3_mmq", _lib.ptr(w), rows, K, 0, _lib.ptr(act), M, _lib.ptr(Y), _lib.F32, Y.stride(0),
                          Y.stride(1), _lib.ptr(ws) if wsn else None, s)

        def both(i):
            rot(i)
            mm(i)

        ms = graph_time(both, reps)
        ms_k = graph_time(mm, reps)
        flops = 2.0 * rows * K * M
        wbytes = int(copies[0][1 if small else 0].numel())
        r = {"kernel": "K5b tcgen05 kind::i8" if small else "K5 tcgen05 kind::f16 cta_group::2",
             "us": ms * 1e3, "kernel_us": ms_k * 1e3, "tflops": flops / ms / 1e9, "kernel_tflops": flops / ms_k / 1e9,
             "weight_bytes": wbytes, "kernel_weight_gbps": wbytes / ms_k / 1e6,
             "kernel_frac_hbm": wbytes / ms_k / 1e6 / hbm}
        r["kernel_frac_bf16"] = r["kernel_tflops"] / bf16
        r["bf16_peak_tflops"], r["bf16_peak_source"] = bf16, bf16_src
        r["kernel_frac_int8_nominal"] = r["kernel_tflops"] / INT8_NOMINAL_TOPS
        out[f"m{M}"] = r
    del copies
    torch.cuda.empty_cache()
    return out


def measure_c4(dev, steps: int, warmup: int) -> dict:
    """BASELINE configs[3]: the Llama-3-8B-shaped decoder (32 layers, random-init weights quantized to
    ITQ3_S on the GPU), one CUDA graph per token, positions 512+ of a 1024-position KV cache."""
    import torch

    from paper_2603_27914_b200.decoder import DecoderStack

    st = DecoderStack(layers=32, max_ctx=1024, seed=3000, dev=dev)
    st.capture()
    st.reset(512)
    st.x.copy_(torch.randn(st.h, device=dev))
    for _ in range(warmup):
        st.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        st.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    wbytes = st.weight_bytes()
    hbm, _ = measured_peak()
    r = {"tokens_per_s": 1000.0 / ms, "ms_per_token": ms, "packed_weight_bytes_per_token": wbytes,
         "packed_weight_gbps": wbytes / ms / 1e6, "frac_hbm": wbytes / ms / 1e6 / hbm,
         "launches_per_token": st.launches_per_step(), "lm_head": st.lm_head is not None,
         "workload": "llama3-8b decoder decode, 32 layers (hidden 4096, ffn 14336, 32/8 heads, head_dim 128)"
                     + (" + 128256x4096 ITQ3_S lm_head" if st.lm_head is not None else "")
                     + ", positions 512+ of a 1024 KV cache, batch 1"}
    del st
    torch.cuda.empty_cache()
    return r


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
    trials = []
    for _ in range(3):  # wall-clock timing: best of 3 runs of `steps` calls rides out host-side noise
        t = time.perf_counter()
        for _ in range(args.steps):
            stack.forward(x0)
        trials.append(1000.0 * (time.perf_counter() - t) / args.steps)
    e2e_ms = max_over_ranks(min(trials))

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
    extra = {}
    if world == 1 and not args.no_extra:
        extra["c3_mmq"] = measure_c3(dev)
        extra["c4_decoder"] = measure_c4(dev, args.steps, args.warmup)
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
                "d2h_bytes_per_step": 4 * stack.ys[-1].numel(), "api": "LinearStack.forward(host np.float32)",
                "timing": "wall clock around `steps` forward() calls (each: H2D, graphed chain, D2H, sync), best of 3"},
        "gpu_launches": stack.launches_per_step * args.steps,
        "clocks": clk,
    }
    line.update(extra)
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def spawn_ranks(args) -> int:
    """`--gpus N > 1` without a torchrun environment: re-launch this script under torch.distributed.run
    with one rank per GPU on 127.0.0.1 (rank 0 prints the JSON line); returns the launcher's exit code."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def run_dry(args):
    """--dry-run (CPU, gloo): exercises the multi-rank plumbing of the GPU arms -- rank discovery,
    barrier, max-over-ranks of the step time, one JSON line from rank 0 -- without a GPU."""
    import torch
    import torch.distributed as dist

    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    t0 = time.perf_counter()
    for _ in range(args.warmup + args.steps):
        sum(range(10000))
    ms = 1000.0 * (time.perf_counter() - t0) / (args.warmup + args.steps) * (1 + rank)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": 1000.0 / ms, "unit": "tokens/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "dry_run": True,
                          "config": {"workload": WORKLOAD, "model": MODEL,
                                     "parallelism": f"tp{world}" if world > 1 and not args.replicas else
                                     f"replicas{world}"}}), flush=True)
    if world > 1:
        dist.destroy_process_group()


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
    ap.add_argument("--no-extra", action="store_true", help="skip the C3 MMQ and C4 decoder keys of the N=1 line")
    ap.add_argument("--mode", choices=["chain", "kernels"], default="chain")
    ap.add_argument("--model", choices=sorted(MODELS), default=MODEL)
    ap.add_argument("--tp", action="store_true", help="row-shard one token stream over the ranks (C5); "
                                                      "the default for --gpus > 1")
    ap.add_argument("--replicas", action="store_true", help="--gpus > 1: N independent replicas of the N=1 step")
    ap.add_argument("--decoder", action="store_true", help="configs[3]: full Llama-3-8B-shaped decoder decode step")
    ap.add_argument("--tp-impl", choices=["fused", "nccl"], default="fused",
                    help="--tp: fused chain kernel with NVLink peer stores, or per-stage kernels + NCCL all_gather")
    ap.add_argument("--dry-run", action="store_true", help="CPU/gloo check of the multi-rank plumbing (tests)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.layers is None:
        args.layers = N_LAYERS
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    world = dist_env()[1]
    if args.dry_run:
        run_dry(args)
    elif args.impl == "reference":
        run_reference(args)
    elif args.tp or (world > 1 and not args.replicas and not args.decoder):
        run_tp(args)
    elif args.decoder:
        run_decoder(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
