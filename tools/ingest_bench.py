"""Container ingest throughput: write_container -> file -> read_container (pinned staging + K7).

    python tools/ingest_bench.py [rows cols]

Reports GB/s of container bytes for a warm page cache (the file was just written), which is the
case SURVEY §8(f)1 targets (the reference's per-block deserialize loop).
"""

import os
import sys
import tempfile
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_27914_b200 as P  # noqa: E402


def main():
    rows, cols = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (28672, 8192)
    g = torch.Generator(device="cuda")
    g.manual_seed(0)
    q = P.quantize_tensor(torch.randn((rows, cols), generator=g, device="cuda"))
    path = os.path.join(tempfile.mkdtemp(), "w.itq3")
    nbytes = P.write_container(q, path)
    q2 = P.read_container(path)  # warm-up (pinned staging allocation)
    assert q2 == q if rows * cols <= 1 << 20 else True
    times = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        q2 = P.read_container(path)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
    t = min(times)
    same = bool(torch.equal(q2.payload(), q.payload()))
    with open(path, "rb") as f:
        t0 = time.perf_counter()
        data = f.read()
        t_read = time.perf_counter() - t0
    print({"rows": rows, "cols": cols, "container_bytes": nbytes, "read_container_s": t,
           "GB_per_s": nbytes / t / 1e9, "plain_file_read_GB_per_s": len(data) / t_read / 1e9,
           "payload_equal": same})


if __name__ == "__main__":
    main()
