"""extract_features for wide speculative sets (K > 64: the spec_full_vocab
ablation and the tree's full-vocabulary draft probabilities, engine.py:166-168,
predictor.py:42-52) against the oracle, bit for bit: the softmax with the
strict denominator chain and numpy's pairwise prev-sum check (now summed by
the whole CTA, leaf blocks in parallel) -- including the uniform prior at
V = 32000 / 128000 that a sequential sum would wrongly reject."""
import numpy as np
import pytest

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import numerics

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K", [65, 1000, 32000, 128000])
def test_wide_features_bit_exact(oracle, K):
    rs = np.random.default_rng(K)
    lg = (rs.standard_normal(K) * 3).astype(np.float32)
    prev = np.full(K, np.float32(1.0 / K), np.float32)            # uniform prior
    ref = oracle.extract_features(lg, prev)
    with numerics.using("strict"):
        fv = spx.extract_features(lg, prev)
    assert np.array_equal(fv.local_probs.cpu().numpy(), ref.local_probs)
    assert np.array_equal(fv.prob_variation.cpu().numpy(), ref.prob_variation)
    # a random prior summing to 1 in numpy's pairwise order
    p = rs.random(K).astype(np.float32)
    p /= p.sum(dtype=np.float32)
    if abs(float(p.sum()) - 1.0) <= 1e-5:
        ref = oracle.extract_features(lg, p)
        fv = spx.extract_features(lg, p)
        assert np.array_equal(fv.prob_variation.cpu().numpy(), ref.prob_variation)
    # off by more than the reference tolerance -> the reference's ValueError
    bad = prev.copy()
    bad[0] += np.float32(3e-5)
    with pytest.raises(ValueError, match="sum to 1"):
        oracle.extract_features(lg, bad)
    with pytest.raises(ValueError, match="sum to 1"):
        spx.extract_features(lg, bad)


@pytest.mark.parametrize("n,V,K", [(1, 1000, 4), (10, 32000, 8), (3, 128000, 64)])
def test_softmax_pick_equals_feature_probs(n, V, K):
    """spx_softmax_pick (the draft proposal's probabilities) == the feature
    kernel's softmax (softmax_device, one-hot prior) at the same ids, bit for bit."""
    import torch
    from paper_2504_08850_b200 import _native as N
    from paper_2504_08850_b200.speculation import softmax_device
    rs = np.random.default_rng(V + n)
    lg = torch.as_tensor((rs.standard_normal((n, V)) * 4).astype(np.float32), device="cuda")
    ids = torch.as_tensor(rs.integers(0, V, size=(n, K)).astype(np.int32), device="cuda")
    out = torch.empty((n, K), dtype=torch.float32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    fast = torch.empty((n, K), dtype=torch.float32, device="cuda")
    N.check(N.lib().spx_softmax_pick(N.ptr(lg), n, V, N.ptr(ids), K, N.ptr(out), N.SPX_MODE_STRICT,
                                     N.ptr(err), N.stream_ptr()), "spx_softmax_pick")
    N.check(N.lib().spx_softmax_pick(N.ptr(lg), n, V, N.ptr(ids), K, N.ptr(fast), N.SPX_MODE_FAST,
                                     N.ptr(err), N.stream_ptr()), "spx_softmax_pick")
    assert err.item() == 0
    for r in range(n):
        full = softmax_device(lg[r].contiguous())
        assert torch.equal(out[r], full[ids[r].long()])          # STRICT: bit for bit
    # FAST: parallel denominator, within the FAST probability tolerance (1e-3
    # absolute).  Relative differences reach ~2e-4 at V = 128000: that is the
    # reference's own left-to-right chain drifting (~n u), not the parallel sum
    assert (fast - out).abs().max().item() <= 1e-3
    assert torch.allclose(fast, out, rtol=1e-3, atol=0)


def test_softmax_pick_id_range_error():
    """An id outside the vocabulary is the reference's ValueError, not a read."""
    import torch
    from paper_2504_08850_b200 import _native as N
    lg = torch.zeros((1, 100), dtype=torch.float32, device="cuda")
    ids = torch.as_tensor([[3, 100]], dtype=torch.int32, device="cuda")
    out = torch.empty((1, 2), dtype=torch.float32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().spx_softmax_pick(N.ptr(lg), 1, 100, N.ptr(ids), 2, N.ptr(out), N.SPX_MODE_FAST,
                                     N.ptr(err), N.stream_ptr()), "spx_softmax_pick")
    with pytest.raises(ValueError, match="out of range"):
        N.raise_device_error(err.item())
    assert out[0, 0].item() == pytest.approx(0.01)
