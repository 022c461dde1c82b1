"""Small invocations of every concurrent kernel, for compute-sanitizer (memcheck / racecheck / synccheck).

    compute-sanitizer --tool racecheck python tools/sanitize_run.py chain1
Cases: encode (K1), dequant (K2t tensor-core IFWHT), chain1 / chain4 (persistent chain kernel with
1 and 4 dependent stages: TMA ring + mbarriers + tagged cross-CTA spin waits), tp2 (the chain's
tensor-parallel peer-store path with 2 simulated ranks on one GPU), mmq (K5 CTA pairs, tcgen05 f16),
mmq8 (K5b tcgen05 i8), gemv (K3 + K4).  Each case checks its result against the CPU oracle so a
sanitizer run that perturbs timing still has to produce the right answer.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2603_27914_b200 as P  # noqa: E402
from oracle import itq3_oracle as O  # noqa: E402


def weights(rows, cols, seed=0):
    return (np.random.default_rng(seed).standard_normal((rows, cols)) / np.sqrt(cols)).astype(np.float32)


def case_encode():
    w = weights(64, 1024)
    q = P.quantize_tensor(torch.from_numpy(w).cuda())
    assert np.array_equal(q.payload().cpu().numpy().reshape(-1), O.quantize_payload(w)[0].reshape(-1))


def case_dequant():
    w = weights(512, 1024, 1)
    q = P.quantize_tensor(w)
    pay = q.payload().cpu().numpy()
    assert np.array_equal(P.dequantize_tensor(q), O.dequantize(pay, 512, 1024, 256, False))


def case_chain(n_stages):
    from test_gpu_stack import chain_bound, lo_flags

    from paper_2603_27914_b200.stack import LinearStack

    shapes = [(1024, 512), (512, 1024), (768, 512), (512, 768)][:n_stages]
    qs = [P.quantize_tensor(weights(r, c, i)) for i, (r, c) in enumerate(shapes)]
    st = LinearStack(qs, limbs=3, mode="chain")
    x = np.random.default_rng(3).standard_normal(shapes[0][1]).astype(np.float32)
    for _ in range(2):
        st.forward(x)
    xin = x.astype(np.float64)
    for i, q in enumerate(qs):
        y = st.stage_output(i).cpu().numpy().astype(np.float64)
        exact, bound = chain_bound(q.payload().cpu().numpy(), q.rows, q.cols, xin, 3, **lo_flags(st, i))
        assert np.all(np.abs(y - exact) <= bound), i
        if i + 1 < len(qs):
            xin = y[: qs[i + 1].cols]


def case_tp2():
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import tp_chain_sim

    sys.argv = [sys.argv[0], "--ranks", "2", "--steps", "1", "--timeout", "300"]
    tp_chain_sim.main()


def case_mmq(m):
    from test_gpu_mmq import matmul_bound

    w = weights(256, 512, 5)
    q = P.quantize_tensor(w)
    X = np.random.default_rng(m).standard_normal((512, m)).astype(np.float32)
    Y = P.fused_matmul(q, torch.from_numpy(X).cuda()).cpu().numpy()
    exact, bound = matmul_bound(q.payload().cpu().numpy(), 256, 512, X)
    assert np.all(np.abs(Y - exact) <= bound)


def case_gemv():
    w = weights(300, 1024, 7)
    q = P.quantize_tensor(w)
    x = np.random.default_rng(1).standard_normal((1024, 3)).astype(np.float32)
    Y = P.fused_matmul(q, torch.from_numpy(x).cuda()).cpu().numpy()
    ref = O.dequantize(q.payload().cpu().numpy(), 300, 1024, 256, False) @ x.astype(np.float64)
    assert np.allclose(Y, ref, rtol=1e-3, atol=1e-3 * np.abs(ref).max())


CASES = {
    "encode": case_encode, "dequant": case_dequant, "chain1": lambda: case_chain(1),
    "chain4": lambda: case_chain(4), "tp2": case_tp2, "mmq": lambda: case_mmq(200),
    "mmq8": lambda: case_mmq(32), "gemv": case_gemv,
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        torch.cuda.synchronize()
        print(f"{n}: ok", flush=True)
