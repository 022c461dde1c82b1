"""Per-role cycle accounting of the tensor-core dequantiser (csrc/dequant.cu, itq3_dequant_set_trace) on a 16384^2 matrix."""
import sys, os, ctypes, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2603_27914_b200 as P
from paper_2603_27914_b200 import _lib
lib = _lib.load()
lib.itq3_dequant_set_trace.argtypes = [ctypes.c_void_p]
dev = torch.device("cuda", 0)
n = 16384 * 16384
w = torch.randn(n, device=dev)
nb = n // 256
pay = torch.empty((nb, 100), dtype=torch.uint8, device=dev)
s = _lib.stream_ptr(dev)
_lib.call("itq3_encode", _lib.ptr(w), _lib.F32, n, 256, 0, 0, P.ScalePolicy().coefficient(), 1, _lib.ptr(pay), s)
for dt, code in ((torch.float32, _lib.F32), (torch.float64, _lib.F64)):
    out = torch.empty(n, dtype=dt, device=dev)
    tr = torch.zeros(148 * 16, dtype=torch.int64, device=dev)
    _lib.call("itq3_dequant", _lib.ptr(pay), nb, 256, 0, n, _lib.ptr(out), code, s)
    lib.itq3_dequant_set_trace(tr.data_ptr())
    _lib.call("itq3_dequant", _lib.ptr(pay), nb, 256, 0, n, _lib.ptr(out), code, s)
    torch.cuda.synchronize()
    lib.itq3_dequant_set_trace(None)
    t = tr.view(148, 16).cpu().numpy()
    names = ["exp_wait_aempty", "exp_total", "exp_load", "mma_wait_aready", "mma_wait_dempty", "mma_total",
             "epi_wait_dfull", "epi_total", "epi_wait_group", "tiles"]
    print(dt)
    for i, nm in enumerate(names):
        print(f"  {nm:16s} {np.median(t[:, i]):12.0f}")
