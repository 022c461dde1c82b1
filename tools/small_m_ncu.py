"""One fused_matmul at small M on the MMQ path (for ncu captures of mmq_kernel at M = 16)."""
import sys

import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2603_27914_b200 as P  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(0)
rows, K, M = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (14336, 4096, 16)
q = P.quantize_tensor(torch.randn((rows, K), generator=g, device=dev) / K ** 0.5)
X = torch.randn((K, M), generator=g, device=dev)
for _ in range(3):
    Y = P.fused_matmul(q, X)
torch.cuda.synchronize()
