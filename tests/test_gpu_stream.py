"""The STREAM predictor kernel (csrc/spx_pred_stream.cuh: K <= 8 at LLM
widths, bf16 head) against the STRICT reference-order kernel on the same
inputs: every K of its range (compile-time K=4 and the generic path), both
widths, more requests than CTAs, skipped rows (row_done / row_layer_mask),
out-of-range ids and the pdl=2 ("ids ready") launch.

Tolerances (stated here): logits 2e-5 relative to the batch's max |logit|
(canonical order vs strict chain on the same bf16 weights), probabilities
1e-3 absolute, decisions equal wherever |z2 - z_cut| > 1e-4.
"""
import numpy as np
import pytest
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import _native as N
from paper_2504_08850_b200 import numerics, rng

pytestmark = pytest.mark.gpu

LOGIT_RTOL = 2e-5
PROB_ATOL = 1e-3
_HEADS = {}


def head(d, V=4096):
    if d not in _HEADS:
        cfg = spx.ModelConfig(vocab_size=V, hidden_dim=d, num_layers=2, num_heads=32,
                              ffn_dim=4 * d, max_context=64, seed=77 + d)
        _HEADS[d] = spx.init_model(cfg, dtype="bf16", head_only=True)
    return _HEADS[d]


def inputs(d, K, B, V=4096, seed=0):
    r = np.random.default_rng(seed)
    hidden = torch.as_tensor(r.standard_normal((B, d)).astype(np.float32), device="cuda")
    hidden = hidden.to(torch.bfloat16).float()
    ids = np.stack([r.choice(V, K, replace=False) for _ in range(B)]).astype(np.int32)
    prev = np.full((B, K), np.float32(1.0 / K), np.float32)
    return hidden, torch.as_tensor(ids, device="cuda"), prev


def run(m, w, hidden, ids, prev, mode, thr=0.5, **kw):
    with numerics.using(mode):
        p = torch.as_tensor(prev, device="cuda").clone()
        out = spx.evaluate_batch(m, w, hidden, ids, p, threshold=thr, **kw)
        torch.cuda.synchronize()
    return out, p


@pytest.mark.parametrize("d", [2048, 4096, 8192])
@pytest.mark.parametrize("K", [1, 2, 3, 4, 5, 8])
def test_stream_matches_strict(d, K):
    m = head(d)
    w = spx.init_predictor(K, 512, rng.derive(5, K))
    B = 333                                    # > 2 * 148 CTAs: several requests per CTA
    hidden, ids, prev = inputs(d, K, B, seed=K)
    fs, ps = run(m, w, hidden, ids, prev, "strict")
    ff, pf = run(m, w, hidden, ids, prev, "fast")
    assert fs.err.item() == 0 and ff.err.item() == 0
    ls, lf = fs.logits.cpu().numpy(), ff.logits.cpu().numpy()
    assert np.max(np.abs(lf - ls)) <= LOGIT_RTOL * np.abs(ls).max()
    assert np.max(np.abs(ff.prob.cpu().numpy() - fs.prob.cpu().numpy())) <= PROB_ATOL
    np.testing.assert_allclose(pf.cpu().numpy(), ps.cpu().numpy(), rtol=1e-4, atol=1e-6)
    zc = spx.z_cut(0.5)
    clear = np.abs(fs.z.cpu().numpy().astype(np.float64) - zc) > 1e-4
    assert np.array_equal(ff.fired.cpu().numpy()[clear], fs.fired.cpu().numpy()[clear])


def test_stream_skips_masked_and_exited_rows():
    d, K, B, layer = 4096, 4, 300, 3
    m = head(d)
    bank = spx.PredictorBank({l: spx.init_predictor(K, 512, rng.derive(9, l)) for l in range(6)}, 6)
    hidden, ids, prev = inputs(d, K, B, seed=11)
    r = np.random.default_rng(3)
    done = torch.as_tensor((r.random(B) < 0.3).astype(np.uint8), device="cuda")
    mask = torch.as_tensor(np.where(r.random(B) < 0.3, 0, 1 << layer).astype(np.int64), device="cuda")
    full, pfull = run(m, bank, hidden, ids, prev, "fast", layer=layer)
    part, ppart = run(m, bank, hidden, ids, prev, "fast", layer=layer, row_done=done,
                      row_layer_mask=mask)
    skip = (done.cpu().numpy() != 0) | (mask.cpu().numpy() == 0)
    assert skip.any() and (~skip).any()
    assert not part.fired.cpu().numpy()[skip].any()
    assert np.array_equal(part.fired.cpu().numpy()[~skip], full.fired.cpu().numpy()[~skip])
    np.testing.assert_array_equal(ppart.cpu().numpy()[skip], prev[skip])     # prev untouched
    np.testing.assert_array_equal(ppart.cpu().numpy()[~skip], pfull.cpu().numpy()[~skip])


def test_stream_id_out_of_range_sets_error():
    d, K, B = 4096, 4, 200
    m = head(d)
    w = spx.init_predictor(K, 512, 1)
    hidden, ids, prev = inputs(d, K, B, seed=5)
    ids[17, 2] = 4096                          # == V
    out, _ = run(m, w, hidden, ids, prev, "fast")
    assert out.err.item() & N.ERR_ID_RANGE
    assert out.fired[17].item() == 0
    with pytest.raises(ValueError, match="token id out of range"):
        N.raise_device_error(out.err.item())


def test_stream_pdl_ids_ready_is_identical():
    d, K, B = 4096, 4, 512
    m = head(d)
    w = spx.init_predictor(K, 512, 2)
    hidden, ids, prev = inputs(d, K, B, seed=6)
    a, pa = run(m, w, hidden, ids, prev, "fast", pdl=False)
    b, pb = run(m, w, hidden, ids, prev, "fast", pdl=2)
    assert torch.equal(a.fired, b.fired) and torch.equal(pa, pb)
    assert torch.equal(a.logits, b.logits) and torch.equal(a.z, b.z)
