"""Chain-kernel decomposition: ms per token of the Llama-2-7B linear stack as a dependent chain and with
the dependency removed (streaming), for whichever libitq3.so is loaded (ITQ3_LIB=... points at a
knock-out build, e.g. -DCHAIN_EXP_NOROT / -DCHAIN_EXP_NOTILE).  Run from the repo root:

    python tools/chain_decomp.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.getcwd())
import bench
from paper_2603_27914_b200.stack import LinearStack
LinearStack.balance = "--no-balance" not in sys.argv
dev = torch.device("cuda", 0)
res = {}
for indep in (False, True):
    st = bench.build_stack(32, 1000, dev, "chain")
    if indep:
        st = LinearStack(st.qs, limbs=3, mode="chain", independent=True)
    st.capture()
    for _ in range(5): st.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): st.replay()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    res["streaming" if indep else "chain"] = {"ms": ms, "tok_s": 1000 / ms, "gbps": st.step_bytes() / ms / 1e6}
    del st
    torch.cuda.empty_cache()
print(os.environ.get("ITQ3_LIB", "base"), json.dumps(res))
