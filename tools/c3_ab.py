"""K5b / K5 kernel times of bench.py's c3_mmq measurement for whichever libitq3.so ITQ3_LIB selects (A/B of
experiment builds): python tools/c3_ab.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.measure_c3(torch.device("cuda", 0))
print(os.environ.get("ITQ3_LIB", "base"), json.dumps({k: round(v["kernel_us"], 2) for k, v in r.items() if isinstance(v, dict)}))
