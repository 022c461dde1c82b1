"""Golden fixtures for the block utilities of the reference API, produced by the REAL reference.

    python tests/golden/make_golden_util.py

Imports ``itq3`` from /root/reference/pkg/src (read-only) and writes tests/golden/util_cases.npz:
block_stats on blocks of many lengths (numpy's pairwise-sum structure changes at 8 and 128),
ternary_quantize / ternary_dequantize (exact ties included), uniform_quantize, hadamard_matrix,
hadamard_oracle, fwht_staged (every stage), fwht32_warp, ternary_mse and optimal_scale.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

LENGTHS = [1, 2, 5, 7, 8, 9, 16, 31, 100, 128, 129, 135, 256, 300, 1000, 1024, 4097]


def main():
    sys.path.insert(0, REF)
    import itq3 as R

    rng = np.random.default_rng(20261017)
    out = {}
    for n in LENGTHS:
        v = rng.standard_normal(n) * rng.uniform(0.01, 100.0)
        s = R.block_stats(v)
        out[f"bs_in_{n}"] = v
        out[f"bs_out_{n}"] = np.array([s.n, s.mean, s.sigma, s.l1, s.linf, s.excess_kurtosis])
    const = np.full(64, 0.3)
    s = R.block_stats(const)
    out["bs_in_const"] = const
    out["bs_out_const"] = np.array([s.n, s.mean, s.sigma, s.l1, s.linf, s.excess_kurtosis])
    # ternary quantise / dequantise, with exact half-way points
    x = np.concatenate([rng.standard_normal(997) * 0.7, np.array([0.25, -0.25, 0.75, -0.75, 0.5, -0.5, 0.0, -0.0])])
    for d, z in ((0.5, 0), (0.37, 1), (1.3, -1)):
        g = R.TernaryGrid(d=d, z=z)
        out[f"tq_{d}_{z}"] = R.ternary_quantize(x, g)
        out[f"td_{d}_{z}"] = R.ternary_dequantize(out[f"tq_{d}_{z}"], g)
    out["tq_in"] = x
    for bits, lo, hi in ((2, -1.0, 1.0), (3, -2.5, 1.5), (8, -0.7, 0.9)):
        out[f"uq_{bits}"] = R.uniform_quantize(x, bits, lo, hi)
    for n in (2, 4, 8, 16, 32, 64):
        out[f"hm_{n}"] = R.hadamard_matrix(n)
        a = rng.standard_normal((3, n))
        out[f"ho_in_{n}"] = a
        out[f"ho_out_{n}"] = R.hadamard_oracle(a)
    for n in (2, 8, 32, 256, 512):
        for dt in (np.float64, np.float32):
            a = rng.standard_normal(n).astype(dt)
            tr = R.fwht_staged(a)
            key = f"fs_{n}_{np.dtype(dt).name}"
            out[key + "_in"] = a
            out[key + "_stages"] = np.stack(tr.stages)
            out[key + "_final"] = tr.final
    w = rng.standard_normal(32)
    out["fw_in"] = w
    out["fw_out"] = R.fwht32_warp(w)
    mse = []
    for alpha, sigma in ((0.878, 1.0), (0.1, 1.0), (2.0, 1.0), (0.5, 0.3), (3.0, 2.0), (1e-3, 1.0)):
        mse.append((alpha, sigma, R.ternary_mse(alpha, sigma)))
    out["mse"] = np.array(mse)
    st = R.block_stats(rng.standard_normal(256))
    out["os_stats"] = np.array([st.n, st.mean, st.sigma, st.l1, st.linf, st.excess_kurtosis])
    out["os_out"] = np.array([R.optimal_scale(st, R.ScalePolicy(kind=k)) for k in ("constant", "argmin", "mean-abs")])
    np.savez_compressed(os.path.join(HERE, "util_cases.npz"), **out)
    print(f"wrote {len(out)} arrays")


if __name__ == "__main__":
    main()
