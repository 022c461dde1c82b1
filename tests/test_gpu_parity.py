"""GPU parity: the CUDA path through the drop-in API vs the reference's golden outputs
(tests/golden, produced by the real reference) and the CPU oracle.

Bars:
  * container bytes: bit-exact (SHA-256 at config C1 4096x4096, byte-equal on 204 small cases)
  * dequantised weights: bit-exact float64 (incl. the sign of zero)
  * fused products, parity mode (numpy in): the reference's own tolerance rtol 1e-5 per element
    (test_compute.py:66-103) -- in practice ~1e-12
  * fused products, perf mode (CUDA fp32/bf16 in): |err| <= sum_b d_b/16 * |t_b|_1 * s_b/2 (fixed-point
    rounding of the rotated activations, a priori) + 1e-5 * sum|w_hat||x| (fp32 accumulation)
"""

import hashlib
import io
import math

import numpy as np
import pytest
import torch

from cases import case_inputs
from oracle import itq3_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_2603_27914_b200")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg_of(c):
    return P.QuantConfig(block_n=c["block_n"], variant=c["variant"], symmetric=c["symmetric"],
                         policy=P.ScalePolicy(kind=c["policy"]))


def container(q):
    buf = io.BytesIO()
    P.write_container(q, buf)
    return buf.getvalue()


def test_small_cases_against_reference(golden):
    meta, arrays, _ = golden
    for i, c in enumerate(meta):
        w, x, X = case_inputs(i, tuple(c["shape"]), c["dist"])
        q = P.quantize_tensor(w, cfg_of(c))
        assert container(q) == arrays[c["key"] + "_container"].tobytes(), c
        deq = P.dequantize_tensor(q)
        assert sha(deq) == c["deq_sha256"], c
        assert sha(np.signbit(deq)) == c["deq_signbit_sha256"], c
        y = P.fused_matvec(q, x)
        np.testing.assert_allclose(y, arrays[c["key"] + "_y"], rtol=1e-5, atol=1e-12, err_msg=str(c))
        Y = P.fused_matmul(q, X)
        np.testing.assert_allclose(Y, arrays[c["key"] + "_Y"], rtol=1e-5, atol=1e-12, err_msg=str(c))
        # fused_matvec is exactly the k=1 column of fused_matmul (test_compute.py:80-84)
        np.testing.assert_array_equal(y, P.fused_matmul(q, x[:, None])[:, 0])


def test_container_round_trip_and_reader(golden):
    meta, arrays, _ = golden
    for c in meta[::7]:
        data = arrays[c["key"] + "_container"].tobytes()
        q = P.read_container(data)
        assert container(q) == data
        assert q == P.read_container(io.BytesIO(data))


@pytest.mark.parametrize("idx", [0, 1, 2, 3, 4])
def test_full_c1_bit_exact(golden, idx):
    _, _, full = golden
    c = full["c1"][idx]
    w = O.generate_weights(c["dist"], 4096, 4096, seed=0).astype(np.float32)
    assert sha(w) == full["inputs"][f"{c['dist']}_4096x4096_seed0_f32"]
    q = P.quantize_tensor(w, P.QuantConfig(variant=c["variant"], symmetric=c["symmetric"]))
    data = container(q)
    assert len(data) == c["container_len"]
    assert hashlib.sha256(data).hexdigest() == c["container_sha256"]
    deq = P.dequantize_tensor(q)
    assert sha(deq) == c["dequant_f64_sha256"]
    out32 = torch.empty((4096, 4096), dtype=torch.float32, device="cuda")
    P.dequantize_tensor(q, out=out32)
    assert sha(out32.cpu().numpy()) == c["dequant_f32_sha256"]
    err = (deq - w.astype(np.float64)).reshape(-1)
    assert float(np.mean(err ** 2)) == pytest.approx(c["mse"], rel=1e-12)  # eps_q identical
    assert float(np.linalg.norm(err) / np.linalg.norm(w.astype(np.float64))) == pytest.approx(c["frobenius_rel"],
                                                                                            rel=1e-12)


def perf_bound(payload, rows, cols, x, limbs):
    """A-priori bound of the perf path vs the exact product (see module docstring)."""
    n = 256
    nb = cols // n
    deq = O.dequantize(payload, rows, cols, n, False)
    quants, sb, zb, _ = O.split_payload(payload, n, False)
    codes, _ = O.unpack_planes(quants, n)
    # max(|t|_1, |c|_1): the chain kernel (k = 1) subtracts the exact sum of x' (test_gpu_stack.chain_bound)
    t1 = np.maximum(np.abs(codes.astype(np.float64) - np.trunc(O.f16_value(zb))[:, None]).sum(axis=1),
                    codes.astype(np.float64).sum(axis=1)).reshape(rows, nb)
    d = O.f16_value(sb).reshape(rows, nb)
    xb = O.butterfly(np.asarray(x, np.float64).reshape(nb, n))
    amax = np.abs(xb).max(axis=1)
    ex = np.where(amax > 0, np.floor(np.log2(np.where(amax > 0, amax, 1))) + 3 - 8 * limbs, 0)
    s = 2.0 ** ex
    bound = (d / 16.0 * t1 * s[None, :] / 2.0).sum(axis=1)
    mag = np.abs(deq) @ np.abs(np.asarray(x, np.float64))
    return deq @ np.asarray(x, np.float64), bound + 1e-5 * mag


@pytest.mark.parametrize("shape", [(4096, 4096), (4096, 11008)])
def test_gemv_c2_against_reference(golden, shape):
    _, _, full = golden
    c = [e for e in full["c2"] if (e["rows"], e["cols"]) == shape][0]
    rows, cols = shape
    w = O.generate_weights("gaussian", rows, cols, seed=0).astype(np.float32)
    x = np.random.default_rng(1).standard_normal(cols).astype(np.float32)
    assert sha(w) == c["input_sha256"] and sha(x) == c["x_sha256"]
    q = P.quantize_tensor(w)
    assert hashlib.sha256(container(q)).hexdigest() == c["container_sha256"]
    y_ref = np.load(f"tests/golden/{c['y_file']}")
    # parity mode (numpy in, float64 out)
    y = P.fused_matvec(q, x)
    np.testing.assert_allclose(y, y_ref, rtol=1e-5, atol=1e-12)
    assert np.max(np.abs(y - y_ref) / (np.abs(y_ref) + 1e-12)) < 1e-9
    # perf mode (CUDA fp32 in, fp32 out, 3 limbs)
    yp = P.fused_matvec(q, torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    exact, bound = perf_bound(q.payload().cpu().numpy(), rows, cols, x, 3)
    assert np.all(np.abs(yp - y_ref) <= bound), np.max(np.abs(yp - y_ref) / bound)


def test_mmq_sample_against_reference(golden):
    _, _, full = golden
    c = full["c3"][0]
    w = O.generate_weights("gaussian", 256, 4096, seed=3).astype(np.float32)
    X = np.random.default_rng(2).standard_normal((4096, 16)).astype(np.float32)
    q = P.quantize_tensor(w)
    Y_ref = np.load(f"tests/golden/{c['y_file']}")
    np.testing.assert_allclose(P.fused_matmul(q, X), Y_ref, rtol=1e-5, atol=1e-12)
    Yp = P.fused_matmul(q, torch.from_numpy(X).cuda()).cpu().numpy()  # M = 16 -> tcgen05 MMQ (kind::i8)
    from test_gpu_mmq import matmul_bound

    _, bound = matmul_bound(q.payload().cpu().numpy(), 256, 4096, X)
    assert np.all(np.abs(Yp - Y_ref) <= bound)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.float16])
@pytest.mark.parametrize("m", [1, 3, 8, 15])
def test_perf_mode_dtypes_and_tokens(dtype, m):
    rng = np.random.default_rng(7 + m)
    w = rng.standard_normal((300, 1024)) * 0.02
    q = P.quantize_tensor(w)
    X = torch.from_numpy(rng.standard_normal((1024, m))).to(dtype).cuda()
    Y = P.fused_matmul(q, X).cpu().numpy()
    Xd = X.double().cpu().numpy()
    pay = q.payload().cpu().numpy()
    for j in range(m):
        exact, bound = perf_bound(pay, 300, 1024, Xd[:, j], P.compute.perf_limbs(m))
        assert np.all(np.abs(Y[:, j] - exact) <= bound)
    # token-major activations (torch M x K, transposed view) give identical results
    Y2 = P.fused_matmul(q, X.t().contiguous().t()).cpu().numpy()
    np.testing.assert_array_equal(Y, Y2)


def test_asymmetric_fast_path_parity():
    rng = np.random.default_rng(11)
    h = O.hadamard(256) / 16.0
    y = rng.normal(loc=0.8, scale=0.3, size=(64, 256))
    w = (y @ h).reshape(16, 1024)  # mean-shifted transform domain -> zero-points -1
    q = P.quantize_tensor(w, P.QuantConfig(symmetric=False))
    pay = q.payload().cpu().numpy()
    assert (O.split_payload(pay, 256, False)[2] == 0xBC00).any()
    x = rng.standard_normal(1024)
    np.testing.assert_allclose(P.fused_matvec(q, x), O.fused_matmul(pay, 16, 1024, 256, False, x[:, None])[:, 0],
                               rtol=1e-9, atol=1e-12)


def test_fwht_bit_exact():
    rng = np.random.default_rng(3)
    for n in (2, 4, 8, 16, 32, 64, 128, 256, 512):
        v = rng.laplace(size=(5, n)) * 10.0 ** rng.uniform(-3, 3)
        np.testing.assert_array_equal(P.fwht_forward(v), O.fwht(v))
        v32 = v.astype(np.float32)
        out = P.fwht_inverse(v32)
        assert out.dtype == np.float32
        np.testing.assert_array_equal(out, O.fwht(v32))
    np.testing.assert_array_equal(P.fwht_forward(np.array([1.0, 2.0, 3.0, 4.0])), [5.0, -1.0, -2.0, 0.0])
    with pytest.raises(P.LengthError):
        P.fwht_forward(np.ones(24))
    with pytest.raises(P.DomainError):
        P.fwht_forward(np.array([1.0, np.nan]))


def test_packing_known_answers():
    # test_packing.py:24-64,128-131
    assert P.pack_ternary(np.zeros(256, np.int8)) == b"\xff" * 32 + b"\x00" * 64
    assert P.pack_ternary(np.array([-1, 0, 1, 1, 0, -1, 0, 0], np.int8)) == bytes([0xD2, 0x0C, 0x00])
    assert P.serialize_block(np.array([-1, 0, 1, 1, 0, -1, 0, 0]), P.TernaryGrid(d=1.0)) == \
        bytes([0xD2, 0x0C, 0x00, 0x00, 0x3C, 0x00, 0x00])
    with pytest.raises(P.CorruptionError, match="index 0"):
        P.unpack_ternary(bytes([0x01, 0x01, 0x00]), 8)
    with pytest.raises(P.CorruptionError, match="index 3"):
        P.unpack_ternary(bytes([0x00, 0x00, 0x08]), 8)
    rng = np.random.default_rng(44)
    for _ in range(20):
        qc = rng.integers(-1, 2, size=256).astype(np.int8)
        np.testing.assert_array_equal(P.unpack_ternary(P.pack_ternary(qc), 256), qc)


def test_corruption_and_container_faults():
    rng = np.random.default_rng(20)
    q = P.quantize_tensor(rng.normal(size=(3, 300)))
    data = bytearray(container(q))
    bad = bytearray(data)
    bad[32 + 100 + 64] |= 0x01  # plane-2 bit in block 1 (test_codec.py:276-282)
    with pytest.raises(P.CorruptionError, match="block 1"):
        P.read_container(bytes(bad))
    bad = bytearray(data)
    bad[32 + 100 + 96:32 + 100 + 98] = bytes([0x00, 0x7E])  # NaN scale in block 1
    with pytest.raises(P.CorruptionError, match="block 1: deserialize_block: scale is NaN"):
        P.read_container(bytes(bad))
    bad = bytearray(data)
    bad[32 + 98:32 + 100] = bytes([0x00, 0x40])  # zero-point 2.0 in block 0
    with pytest.raises(P.CorruptionError, match="zero-point 2.0"):
        P.read_container(bytes(bad))
    with pytest.raises(P.BadMagicError):
        P.read_container(b"XXXX" + bytes(data[4:]))
    with pytest.raises(P.TruncatedStreamError):
        P.read_container(bytes(data[:-10]))
    with pytest.raises(P.SizeMismatchError):
        P.read_container(bytes(data) + b"\x00\x00")
    # dequantize of a tensor built from a corrupt block list names the block
    blocks = list(q.blocks)
    b1 = blocks[1]
    blocks[1] = P.PackedBlock(n=256, quants=b1.quants[:64] + b"\x01" + b1.quants[65:], scale_bits=b1.scale_bits,
                              zp_bits=b1.zp_bits)
    qq = P.QuantizedTensor(q.rows, q.cols, 256, "s", True, q.pad, blocks)
    with pytest.raises(P.CorruptionError, match="block 1"):
        P.dequantize_tensor(qq)
    broken = P.QuantizedTensor(q.rows, q.cols, 256, "s", True, q.pad, q.blocks[:-1])
    with pytest.raises(P.ShapeError):
        P.write_container(broken, io.BytesIO())


def test_api_validation_order():
    q = P.quantize_tensor(np.random.default_rng(1).normal(size=(4, 256)))
    with pytest.raises(P.ShapeError):
        P.fused_matvec(q, np.zeros(255))
    with pytest.raises(P.ShapeError):
        P.fused_matmul(q, np.zeros((255, 2)))
    with pytest.raises(P.ShapeError):
        P.fused_matvec(q, np.zeros((256, 1)))
    with pytest.raises(P.DomainError):
        P.fused_matvec(q, np.full(256, np.nan))
    with pytest.raises(P.ShapeError):
        P.quantize_tensor(np.zeros(256))
    bad = np.zeros((2, 128))
    bad[0, 0] = np.nan
    with pytest.raises(P.DomainError):
        P.quantize_tensor(bad)
    with pytest.raises(P.LengthError):
        P.encode_block(np.zeros(128), P.QuantConfig(block_n=256))
    assert P.quantize_tensor(np.zeros((1, 300))).pad == 212
    assert P.quantize_tensor(np.ones((256, 256))).bits_per_weight == pytest.approx(3.125)
    assert P.quantize_tensor(np.ones((256, 256)), P.QuantConfig(variant="ss")).bits_per_weight == pytest.approx(3.625)


def test_block_codec_single_block():
    w = np.zeros(256)
    w[37] = 16.0
    b = P.encode_block(w, P.QuantConfig())
    assert set(np.unique(b.codes())) == {-1, 1}
    err2 = float(np.sum((P.decode_block(b) - w) ** 2))
    assert err2 <= 256 * b.scale ** 2 / 4 + 1e-6
    z = P.encode_block(np.zeros(32), P.QuantConfig(block_n=32))
    assert z.scale == 0.0
    np.testing.assert_array_equal(P.decode_block(z), np.zeros(32))
    assert math.isclose(P.argmin_scale_coeff(), 0.878, abs_tol=1e-12)


@pytest.mark.parametrize("nblocks", [1, 31, 33, 70001])
def test_validate_fast_path_first_offender(nblocks):
    """K7 fast path (block_n 256, variant s, one thread per block): same first offender and message as
    the per-block reference checks, for block counts that leave ragged warps."""
    from paper_2603_27914_b200 import codec as C

    rng = np.random.default_rng(nblocks)
    w = rng.standard_normal((nblocks, 256)).astype(np.float32)
    q = P.quantize_tensor(torch.from_numpy(w).cuda())
    pay = q.payload().clone()
    C.validate_payload(pay, 256, False, True, True)  # clean: no error
    late, early = nblocks - 1, nblocks // 2
    bad = pay.clone()
    bad[late, 64 + 5] |= 0x10      # plane 2 bit -> stored code > 2 at index 8*5+4 = 44
    with pytest.raises(P.CorruptionError, match=f"block {late}:.*index 44"):
        C.validate_payload(bad, 256, False, True, True)
    if early < late:  # an earlier offender wins
        bad[early, 96:98] = torch.tensor([0x01, 0x7E], dtype=torch.uint8)  # scale NaN (0x7E01)
        with pytest.raises(P.CorruptionError, match=f"block {early}: deserialize_block: scale is NaN"):
            C.validate_payload(bad, 256, False, True, True)


@pytest.mark.parametrize("nblocks,tail", [(1, 0), (129, 0), (300, 77), (1000, 255)])
@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_dequant_tensor_core_path_bit_exact(nblocks, tail):
    """K2t (tensor-core IFWHT, block_n 256 / variant s) plus its exact float64 pass: bit-identical
    (incl. signed zeros) to the oracle's decode, for ragged element counts and for blocks the tensor-core
    path hands to the exact pass (scale +0, negative, inf; zero-point 2.0)."""
    rng = np.random.default_rng(nblocks + tail)
    numel = nblocks * 256 - tail
    w = (rng.standard_normal(numel) * 0.1).astype(np.float32)
    ref_pay, _ = O.quantize_payload(w[None, :])
    pay = ref_pay.copy()
    nb = pay.shape[0]
    specials = {0: 0x0000, 1: 0xBC00, 2: 0x7C00}  # scale +0, -1.0, +inf
    for b, sb in specials.items():
        if b < nb:
            pay[b, 96:98] = np.frombuffer(np.uint16(sb).tobytes(), np.uint8)
    if nb > 3:
        pay[3, 98:100] = np.frombuffer(np.uint16(0x4000).tobytes(), np.uint8)  # zero-point 2.0
    want = O.dequantize(pay, 1, numel, 256, False).reshape(-1)
    dev = torch.device("cuda", 0)
    p = torch.from_numpy(pay).to(dev)
    for dt in (torch.float64, torch.float32):
        out = torch.empty(numel, dtype=dt, device=dev)
        P._lib.call("itq3_dequant", P._lib.ptr(p), nb, 256, 0, numel, P._lib.ptr(out), P._lib.TORCH_DTYPE_CODE[dt],
                    P._lib.stream_ptr(dev))
        got = out.cpu().numpy().astype(np.float64)
        exp = want.astype(np.float32).astype(np.float64) if dt == torch.float32 else want
        assert np.array_equal(got.view(np.uint64), exp.view(np.uint64)) or \
            np.array_equal(np.isnan(got), np.isnan(exp)) and np.array_equal(
                np.where(np.isnan(got), 0, got).view(np.uint64), np.where(np.isnan(exp), 0, exp).view(np.uint64)), dt


def test_release_layouts_and_rebuild():
    """Weight memory per format: layouts can be released and are rebuilt on use."""
    rng = np.random.default_rng(12)
    q = P.quantize_tensor(rng.standard_normal((512, 1024)) * 0.05)
    X = torch.from_numpy(rng.standard_normal((1024, 32)).astype(np.float32)).cuda()
    x = X[:, 0].contiguous()
    y1, Y1 = P.fused_matvec(q, x).clone(), P.fused_matmul(q, X).clone()
    base = q.device_nbytes()
    q.release("tiled", "mmq8")
    assert q.device_nbytes() < base
    torch.testing.assert_close(P.fused_matvec(q, x), y1, rtol=0, atol=0)
    torch.testing.assert_close(P.fused_matmul(q, X), Y1, rtol=0, atol=0)
    with pytest.raises(ValueError):
        q.release("bogus")
