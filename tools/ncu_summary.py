"""Summarise one kernel of an ncu report (ncu --set full) as JSON: duration, DRAM bytes, throughputs,
issue and pipe utilisation -- the figures profiles/ and bench.py's roofline.traffic quote.

    python tools/ncu_summary.py report.ncu-rep --kernel chain_kernel [--chain-sha] > summary.json
"""
import argparse
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread", "sm__cycles_elapsed.avg.per_second"]


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit)
    return float(v.replace(",", "")) * scale if scale else None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--kernel", default="")
    ap.add_argument("--chain-sha", action="store_true", help="record the SHA-256 of csrc/chain.cu")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        if a.kernel not in name:
            continue
        out["Kernel Name"] = name
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                out[k] = f"{r[i]} {units[i]}".strip()
        rd = to_bytes(r[hdr.index("dram__bytes_read.sum")], units[hdr.index("dram__bytes_read.sum")])
        wr = to_bytes(r[hdr.index("dram__bytes_write.sum")], units[hdr.index("dram__bytes_write.sum")])
        if rd is not None and wr is not None:
            out["traffic_bytes_per_launch"] = rd + wr
        break
    if a.chain_sha:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        with open(os.path.join(root, "paper_2603_27914_b200", "csrc", "chain.cu"), "rb") as f:
            out["chain_cu_sha256"] = hashlib.sha256(f.read()).hexdigest()
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
