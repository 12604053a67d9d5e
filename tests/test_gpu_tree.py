"""GPU parity of the device TreeEngine (tree.py:133-302) against the
reference's own TreeEngine runs (tests/golden/tree_tiny.json, made by
tests/golden/make_tree_golden.py on the trained tiny pipeline artifacts).

STRICT mode must reproduce every TreeStepResult field exactly and every
predictor probability (in the reference's call order) within 1e-9 abs (the
decision itself is exact: z2 >= z_cut).  FAST mode is held to the same step
results on these streams (decisions are exact unless a probability sits
within ~1e-6 of the threshold, which the golden margins exclude).
"""
import os

import numpy as np
import pytest
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import engine as E
from paper_2504_08850_b200 import numerics
from paper_2504_08850_b200 import tree as T

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PIPE = os.path.join(GOLDEN, "tiny_pipeline")
PROB_ATOL = 1e-9
PROMPT = [84, 104, 101, 32]
_MODELS = {}


def models():
    if not _MODELS:
        _MODELS["t"] = spx.load_weights(os.path.join(PIPE, "target.spxw"))
        _MODELS["d"] = spx.load_weights(os.path.join(PIPE, "draft.spxw"))
        _MODELS["bank"] = spx.load_predictors(os.path.join(PIPE, "predictors.spxp"))
        _MODELS["prof"] = spx.load_profile(os.path.join(PIPE, "profile.spxs"))
    return _MODELS["t"], _MODELS["d"], _MODELS["bank"], _MODELS["prof"]


def engine_for(case):
    t, d, bank, prof = models()
    pol = {"never_all": E.NeverExitPolicy(), "always_all": E.AlwaysExitPolicy()}.get(
        case["case"], E.PredictorPolicy(bank))
    eng = T.TreeEngine(t, d, pol, tuple(case["branching"]),
                       E.EngineConfig(k=4, threshold=case["threshold"], schedule_mode=case["mode"]),
                       profile=prof if case["mode"] == "two-level" else None,
                       schedule_config=spx.ScheduleConfig(5, 1, 4))
    eng.record_probs = True
    return eng


def step_fields(r):
    return dict(accepted_tokens=r.accepted_tokens, correction_token=r.correction_token,
                path_exit_layers=r.path_exit_layers, accepted_path=r.accepted_path,
                predictor_evals=r.predictor_evals, num_paths=r.num_paths,
                max_path_len=r.max_path_len, scheduled_layer_count=r.scheduled_layer_count)


def _cases(golden):
    return golden.json("tree_tiny.json")["cases"]


@pytest.mark.parametrize("ci", range(15))
def test_tree_engine_strict_matches_reference(golden, ci):
    case = _cases(golden)[ci]
    eng = engine_for(case)
    with numerics.using("strict"):
        eng.start(case["prompt"])
        for s, ref in enumerate(case["steps"]):
            n0 = len(eng.prob_log)
            res = eng.step()
            exp = {k: ref[k] for k in step_fields(res)}
            assert step_fields(res) == exp, (case["case"], s)
            got = eng.prob_log[n0:]
            assert [l for l, _ in got] == [l for l, _ in ref["probs"]], (case["case"], s)
            for (_, p), (_, q) in zip(got, ref["probs"]):
                assert abs(p - q) <= PROB_ATOL, (case["case"], s, p, q)
    assert eng.context == case["context"]
    assert eng.online.queue == case["online_queue"]


@pytest.mark.parametrize("ci", [0, 4, 9])
def test_tree_engine_fast_matches_reference(golden, ci):
    case = _cases(golden)[ci]
    eng = engine_for(case)
    with numerics.using("fast"):
        eng.start(case["prompt"])
        for s, ref in enumerate(case["steps"]):
            res = eng.step()
            assert step_fields(res) == {k: ref[k] for k in step_fields(res)}, (case["case"], s)


def test_merge_paths_structure():
    """tests/test_tree.py:16-26."""
    _, d, _, _ = models()
    with numerics.using("strict"):
        tree = spx.build_token_tree(d, PROMPT, (3, 2))
        hts = T.merge_paths(tree, d, PROMPT, k=4)
    assert len(hts) == 6
    for ht in hts:
        assert len(ht.path) == 2 == len(ht.per_node_spec)
        kids = tree.children(ht.path[0])
        assert ht.per_node_spec[0].tokens == tuple(tree.nodes[c].token for c in kids)
        assert len(ht.per_node_spec[1].tokens) == 4


def test_merge_paths_needs_draft_for_leaves():
    """tests/test_tree.py:29-32."""
    _, d, _, _ = models()
    tree = spx.build_token_tree(d, PROMPT, (2,))
    with pytest.raises(ValueError):
        T.merge_paths(tree)


def test_tree_no_exit_equals_greedy():
    """tests/test_tree.py:76-80."""
    t, d, _, _ = models()
    with numerics.using("strict"):
        base, _ = E.greedy_generate(t, PROMPT, 30)
        toks, _ = T.TreeEngine(t, d, E.NeverExitPolicy(), (3, 2)).generate(PROMPT, 30)
    assert toks == base


def test_tree_self_draft_accepts():
    """tests/test_tree.py:83-89."""
    t, _, _, _ = models()
    with numerics.using("strict"):
        _, steps = T.TreeEngine(t, t, E.NeverExitPolicy(), (1,)).generate(PROMPT, 12)
    assert all(len(s.accepted_tokens) >= 1 for s in steps)


def test_tree_oracle_policy_lossless():
    """tests/test_tree.py:92-96 (host-policy path of the engine)."""
    t, d, _, _ = models()
    with numerics.using("strict"):
        base, _ = E.greedy_generate(t, PROMPT, 12)
        toks, _ = T.TreeEngine(t, d, E.OraclePolicy(t), (2, 2)).generate(PROMPT, 12)
    assert toks == base


def test_mapping_complexity_bound():
    """tests/test_tree.py:99-104."""
    t, d, _, _ = models()
    _, steps = T.TreeEngine(t, d, E.NeverExitPolicy(), (3, 2)).generate(PROMPT, 20)
    for s in steps:
        assert s.predictor_evals <= s.num_paths * s.scheduled_layer_count * s.max_path_len


def test_merged_mapping_dedups_shared_feature_ids():
    """K6 reads each unique LM-head row once: sibling nodes share most of their
    draft top-k, so the unique count is below the pair count."""
    t, d, bank, _ = models()
    eng = T.TreeEngine(t, d, E.PredictorPolicy(bank), (3, 2))
    eng.start(PROMPT)
    eng.step()
    assert eng.last_unique_ids <= eng.last_pairs


def test_tree_missing_predictor_raises_keyerror():
    t, d, bank, _ = models()
    partial = {l: w for l, w in bank.items() if l != 0}
    eng = T.TreeEngine(t, d, E.PredictorPolicy(partial), (2,))
    eng.start(PROMPT)
    with pytest.raises(KeyError):
        eng.step()


def test_two_level_needs_profile():
    t, d, _, _ = models()
    with pytest.raises(ValueError):
        T.TreeEngine(t, d, E.NeverExitPolicy(), (2,), E.EngineConfig(schedule_mode="two-level"))


def test_tree_gate_and_node_eval_kernels():
    """K7b and the node-eval kernel in isolation against numpy."""
    import torch
    from paper_2504_08850_b200 import _native as N
    paths = [[1, 3], [1, 4], [2, 5]]
    ptr = torch.tensor([0, 2, 4, 6], dtype=torch.int32, device="cuda")
    nodes = torch.tensor([1, 3, 1, 4, 2, 5], dtype=torch.int32, device="cuda")
    for fire in ([0, 0, 0], [1, 0, 0], [0, 1, 1]):
        pf = torch.tensor(fire, dtype=torch.uint8, device="cuda")
        gate = torch.full((6,), 7, dtype=torch.uint8, device="cuda")
        N.check(N.lib().spx_tree_gate(N.ptr(pf), N.ptr(ptr), N.ptr(nodes), 3, 6, N.ptr(gate),
                                      N.stream_ptr()), "spx_tree_gate")
        exp = np.zeros(6, np.uint8)
        for p, f in enumerate(fire):
            if f:
                exp[0] = 1
                exp[paths[p]] = 1
        assert gate.cpu().numpy().tolist() == exp.tolist()


@pytest.mark.parametrize("n_rows,n_ids,k", [(200, 300, 16), (64, 128, 64), (26, 40, 4), (300, 700, 8)])
def test_tree_merged_tensor_cores_match_cuda_cores(n_rows, n_ids, k):
    """K6 on tcgen05 (kind::f16, xg split exactly into three bf16 parts,
    TMEM accumulators) vs the CUDA-core CDOT kernel on the same pairs: equal
    within the f32 accumulation-order tolerance stated here (1e-5 of the
    row's largest |logit| + 1e-6)."""
    from paper_2504_08850_b200.model import head_prep, merged_logits
    cfg = spx.ModelConfig(vocab_size=32000, hidden_dim=4096, num_layers=1, num_heads=32,
                          ffn_dim=11008, max_context=64, seed=5)
    m = spx.init_model(cfg, dtype="bf16", head_only=True)
    g = torch.Generator(device="cuda").manual_seed(n_rows + n_ids)
    h = torch.randn((n_rows, 4096), device="cuda", generator=g).to(torch.bfloat16).float()
    r = np.random.default_rng(n_rows)
    pool = r.choice(32000, n_ids, replace=False)
    ids = [r.choice(pool, k, replace=False) for _ in range(n_rows)]
    with numerics.using("fast"):
        prep = head_prep(m, h)
        a = merged_logits(m, prep, ids, tensor_cores=False)
        b = merged_logits(m, prep, ids, tensor_cores=True)
    for x, y in zip(a, b):
        x, y = x.cpu().numpy(), y.cpu().numpy()
        assert np.all(np.abs(x - y) <= 1e-5 * np.abs(x).max() + 1e-6)


@pytest.mark.parametrize("branching", [(5, 2, 1), (3, 2)])
def test_tree_fast_tensor_core_drafting_matches_full_logits(branching):
    """FAST, bf16 draft: the tree is drafted from K4's tensor-core form (exact
    stable top-max(K, b) ids per node, probabilities from the tensor-core
    logits) instead of the full CUDA-core draft logits.  The trees, exits,
    accepted tokens and corrections must be identical; the draft
    probabilities agree within the FAST tolerance."""
    from paper_2504_08850_b200 import rng
    V, D = 2048, 1024
    tc = spx.ModelConfig(V, D, 4, 8, 2816, 128, 41)
    dc = spx.ModelConfig(V, D, 1, 8, 2816, 128, 42)
    t, d = spx.init_model(tc, dtype="bf16"), spx.init_model(dc, dtype="bf16")
    bank = {l: spx.init_predictor(4, 512, rng.derive(43, l)) for l in range(3)}
    prof = spx.OfflineProfile(4, np.asarray([5, 3, 2, 0], np.uint64), 0)
    out = {}
    with numerics.using("fast"):
        for tcd in (False, True):
            eng = T.TreeEngine(t, d, E.PredictorPolicy(bank), branching,
                               E.EngineConfig(k=4, threshold=0.5, schedule_mode="two-level"), prof,
                               spx.ScheduleConfig(5, 1, 2))
            eng.tc_draft = tcd
            trees = []
            orig = eng._draft_tree

            def rec(orig=orig, trees=trees):
                r = orig()
                trees.append(r[0])
                return r
            eng._draft_tree = rec
            eng.start([int(x) % V for x in rng.splitmix64(44, 12)])
            steps = []
            for _ in range(3):
                r = eng.step()
                steps.append((r.accepted_tokens, r.correction_token, r.path_exit_layers,
                              r.accepted_path, r.predictor_evals))
            out[tcd] = (steps, trees)
    assert out[False][0] == out[True][0]
    for ta, tb in zip(out[False][1], out[True][1]):
        assert [(n.token, n.parent, n.depth) for n in ta.nodes] == \
            [(n.token, n.parent, n.depth) for n in tb.nodes]
        np.testing.assert_allclose([n.prob for n in tb.nodes[1:]],
                                   [n.prob for n in ta.nodes[1:]], rtol=1e-4, atol=1e-6)
