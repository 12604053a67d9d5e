"""GPU label collection and offline profiling against the
reference: ``collect_training_data`` (src/specexit/predictor.py:219-275) vs
the reference's own output on the tiny-pipeline artifacts
(tests/golden/collect_tiny.npz, made by tests/golden/make_collect_golden.py),
and the profile stage (pipeline.py:168-191 -> scheduler.py:105-121) vs the
reference pipeline's profile.spxs exit counts [120,47,18,15,7,1,1,303].

STRICT: features bit-identical, labels and counts exact.  FAST: labels,
decisions and counts exact (certified predictor decisions), features within
FEAT_RTOL_FAST relative to the largest feature of the row.
"""
import os

import numpy as np
import pytest

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import numerics

pytestmark = pytest.mark.gpu

FEAT_RTOL_FAST = 1e-5
TP = os.path.join(os.path.dirname(__file__), "golden", "tiny_pipeline")
PROFILE_COUNTS = [120, 47, 18, 15, 7, 1, 1, 303]


def _tiny():
    t = spx.load_weights(os.path.join(TP, "target.spxw"))
    d = spx.load_weights(os.path.join(TP, "draft.spxw"))
    bank = spx.load_predictors(os.path.join(TP, "predictors.spxp"))
    with open(os.path.join(TP, "fixture_corpus.txt"), "rb") as fh:
        corpus = fh.read()
    return t, d, bank, corpus


@pytest.mark.parametrize("mode", ["strict", "fast"])
@pytest.mark.parametrize("case", ["a", "b"])
def test_collect_training_data_matches_reference(golden, mode, case):
    g = golden.npz("collect_tiny.npz")
    k, n, plen, max_new, seed = (int(v) for v in g[f"{case}_args"])
    t, d, _, corpus = _tiny()
    layers = list(range(t.config.num_layers - 1))
    with numerics.using(mode):
        ex = spx.collect_training_data(t, d, corpus, layers, k=k, num_prompts=n,
                                       prompt_len=plen, max_new=max_new, seed=seed)
    assert len(ex) == len(g[f"{case}_labels"]) == n * max_new * len(layers)
    feats = np.stack([e.features for e in ex]).astype(np.float32)
    assert [e.layer for e in ex] == list(g[f"{case}_layers"])
    assert [int(e.label) for e in ex] == list(g[f"{case}_labels"])
    want = g[f"{case}_features"]
    if mode == "strict":
        assert np.array_equal(feats.view(np.uint32), want.view(np.uint32))
    else:
        scale = np.abs(want).max(axis=1, keepdims=True)
        assert np.all(np.abs(feats - want) <= FEAT_RTOL_FAST * scale)


def test_collect_training_data_shapes_like_reference_test():
    """tests/test_predictor.py:140-147 of the reference, on the device."""
    t, d, _, corpus = _tiny()
    ex = spx.collect_training_data(t, d, corpus, [0, 2], k=4, num_prompts=2, prompt_len=8,
                                   max_new=6, seed=0)
    assert len(ex) == 2 * 6 * 2
    assert {e.layer for e in ex} == {0, 2}
    assert all(e.features.shape == (12,) for e in ex)
    with pytest.raises(ValueError):
        spx.collect_training_data(t, d, b"", [0])
    with pytest.raises(ValueError):
        spx.collect_training_data(t, d, corpus[:4], [0], prompt_len=8)


def _corpus_prompts(corpus, n, plen, seed):
    data = np.frombuffer(corpus, dtype=np.uint8)
    starts = spx.rng.splitmix64(seed, n) % np.uint64(data.size - plen + 1)
    return [[int(b) for b in data[int(s):int(s) + plen]] for s in starts]


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_profile_offline_device_reproduces_reference_profile(mode):
    """pipeline.py:168-191 defaults: 16 prompts of 16 bytes (seed 505),
    max_new 32, threshold 0.7, schedule 'all' -> the reference's counts."""
    t, d, bank, corpus = _tiny()
    prompts = _corpus_prompts(corpus, 16, 16, 505)
    fp = spx.weight_fingerprint(os.path.join(TP, "target.spxw"))
    with numerics.using(mode):
        prof = spx.profile_offline_device(t, d, bank, prompts, 32, fingerprint=fp, k=4,
                                          threshold=0.7)
    ref = spx.load_profile(os.path.join(TP, "profile.spxs"))
    assert list(prof.exit_counts) == PROFILE_COUNTS == list(ref.exit_counts)
    assert prof.fingerprint == ref.fingerprint
    with pytest.raises(ValueError):
        spx.profile_offline_device(t, d, bank, [], 32)
