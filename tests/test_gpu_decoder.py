"""GPU: the decoder-stack harness (decoder.DecoderStack) -- graph-replayed token steps with ITQ3_S
GEMVs -- against the same step in plain torch fp32 with the dequantised weights.  Tolerance: the
GEMV's rotated activations carry 22-bit limbs (relative error ~2^-21 per product), compounded over
the layers and the attention softmax; 1e-4 of the hidden-state norm."""

import pytest
import torch

pytestmark = pytest.mark.gpu
P = pytest.importorskip("paper_2603_27914_b200")
from paper_2603_27914_b200.decoder import DecoderStack  # noqa: E402

SMALL = dict(hidden=512, inter=1024, n_heads=4, n_kv=1, head_dim=128, rope_theta=10000.0, vocab=2000)


def test_decoder_steps_match_fp32_reference():
    dev = torch.device("cuda", 0)
    st = DecoderStack(layers=2, max_ctx=320, seed=3, dev=dev, shapes=SMALL, serving=False)
    g = torch.Generator(device=dev)
    g.manual_seed(4)
    k_hist, v_hist = [[] for _ in range(2)], [[] for _ in range(2)]
    for pos in range(300):  # long enough for the attention splits' unrolled position loops
        x = torch.randn(512, generator=g, device=dev)
        got = st.step(x).clone()
        want = st.reference_step(x, pos, k_hist, v_hist)
        err = float((got - want).norm() / want.norm())
        assert err < 1e-4, (pos, err)
        lerr = float((st.logits - st.ref_logits).norm() / st.ref_logits.norm())  # RMSNorm -> lm_head chain
        assert lerr < 1e-4, (pos, lerr)
    assert int(st.pos) == 300


def test_decoder_kv_cache_bound():
    """the graphed step advances the device position with no host work, so the host keeps
    its own counter and refuses a step once the cache is full; the glue kernel also refuses a
    position >= max_ctx on the device (no cache write, error word set)."""
    dev = torch.device("cuda", 0)
    st = DecoderStack(layers=1, max_ctx=8, seed=5, dev=dev, shapes=SMALL, serving=False)
    st.capture()
    st.reset(6)
    x = torch.randn(512, device=dev)
    st.step(x)
    st.step(x)
    with pytest.raises(ValueError, match="KV cache full"):
        st.step(x)
    assert st.device_error() == 0
    kc = st.k_cache.clone()
    st.graph.replay()  # bypass the host guard: the device position is now 8 == max_ctx
    torch.cuda.synchronize()
    assert st.device_error() == 1
    assert torch.equal(st.k_cache, kc)
    with pytest.raises(ValueError):
        st.reset(8)


def test_decoder_without_head_matches_fp32_reference():
    """lm_head=False: the last layer's chain folds x += o + down in place (flags 8 | 32)."""
    dev = torch.device("cuda", 0)
    st = DecoderStack(layers=3, max_ctx=64, seed=8, dev=dev, shapes=SMALL, serving=False, lm_head=False)
    g = torch.Generator(device=dev)
    g.manual_seed(9)
    k_hist, v_hist = [[] for _ in range(3)], [[] for _ in range(3)]
    for pos in range(20):
        x = torch.randn(512, generator=g, device=dev)
        got = st.step(x).clone()
        want = st.reference_step(x, pos, k_hist, v_hist)
        err = float((got - want).norm() / want.norm())
        assert err < 1e-4, (pos, err)
