"""Pin the oracle (CPU restatement, oracle/specexit_oracle.py) against the
reference's own outputs (tests/golden/, produced by make_golden.py and the
reference pipeline).  CPU only."""
import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN


def _case_inputs(g):
    return g["hidden"], g["ids"], g["prev"]


def _check_predictor_case(o, t, g, thrs):
    w = o.PredictorWeights(g["w1"], g["b1"], g["w2"], float(g["b2"]))
    hidden = g["hidden"]
    for i in range(g["ids"].shape[0]):
        lg = o.sliced_head_logits(t, hidden[i], g["ids"][i])
        assert np.array_equal(lg.view(np.uint32), g["logits"][i].view(np.uint32)), i
        fv = o.extract_features(lg, g["prev"][i])
        assert np.array_equal(fv.concat().view(np.uint32), g["feats"][i].view(np.uint32))
        z = o.predictor_logit(w, fv)
        assert np.float32(z).view(np.uint32) == g["z2"][i].view(np.uint32)
        p = o.predictor_forward(w, fv)
        assert p == g["prob"][i]
        for thr in thrs:
            assert o.decide_exit(p, thr) == bool(g[f"fired_{thr}"][i])
        assert int(np.argmax(o.full_head_logits(t, hidden[i]))) == int(g["argmax"][i])


def test_rng_known_answers(oracle, golden):
    kat = golden.json("rng_kat.json")
    # the reference's own KAT (tests/test_rng.py:7)
    assert [int(v) for v in oracle.splitmix64(0, 3)] == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4,
                                                         0x06C45D188009454F]
    assert [int(v) for v in oracle.splitmix64(0, 3)] == kat["splitmix64_seed0"]
    assert [int(v) for v in oracle.splitmix64(12345, 5)] == kat["splitmix64_seed12345"]
    for s, i, v in kat["derive"]:
        assert oracle.derive(s, i) == v
    assert oracle.uniform(99, 64, -0.25, 0.5).view(np.uint32).tolist() == kat["uniform_bits"]


@pytest.mark.parametrize("name,thrs", [("predictor_tiny.npz", (0.5, 0.7)),
                                       ("predictor_tiny_k20.npz", (0.5,)),
                                       ("predictor_tiny_h32.npz", (0.5,))])
def test_predictor_path_tiny(oracle, golden, name, thrs):
    g = golden.npz(name)
    t = oracle.init_model(oracle.ModelConfig(num_layers=int(g["layers"]), seed=int(g["seed"])),
                          bf16=True)
    _check_predictor_case(oracle, t, g, thrs)


def _head_7b(oracle):
    cfg = oracle.ModelConfig(vocab_size=32000, hidden_dim=4096, num_layers=32, num_heads=32,
                             ffn_dim=11008, max_context=512, seed=1234)
    return cfg, oracle.init_model(cfg, bf16=True, only={"lm_head", "final_norm.g", "final_norm.b"})


def hidden_7b(oracle, n=8, seed=21):
    r = np.random.default_rng(seed)
    return oracle.round_bf16(r.standard_normal((n, 4096)).astype(np.float32))


@pytest.mark.slow
def test_predictor_path_7b_head(oracle, golden):
    g = golden.npz("predictor_7b.npz")
    _, t = _head_7b(oracle)
    g["hidden"] = hidden_7b(oracle, g["ids"].shape[0], int(g["hidden_seed"]))
    _check_predictor_case(oracle, t, g, (0.5, 0.7))


def test_scheduler_stream(oracle, golden):
    for case in golden.json("scheduler_stream.json"):
        cfg = oracle.ScheduleConfig(case["queue_len"], case["radius"], case["top_k"])
        assert oracle.ranked_layers(case["exit_counts"], case["L"]) == case["ranked"]
        st = oracle.OnlineState(case["L"], cfg)
        for e, act, nbr in zip(case["exits"], case["active"], case["neighbor_counts"]):
            oracle.update_online(st, e)
            assert st.neighbor_counts.tolist() == nbr
            assert oracle.active_layers(case["exit_counts"], st, cfg) == act
        assert st.queue == case["queue"]


def test_scheduler_reference_known_answers(oracle):
    """The reference's own scheduler goldens (tests/test_scheduler.py:16-65)."""
    assert oracle.ranked_layers([5, 9, 9, 0, 2, 0, 0, 100], 8) == [1, 2, 0, 4, 3, 5, 6]
    st = oracle.OnlineState(8, oracle.ScheduleConfig(queue_len=5, radius=2))
    oracle.update_online(st, 0)
    assert [i for i in range(7) if st.neighbor_counts[i] > 0] == [0, 1, 2]
    oracle.update_online(st, 7)
    assert st.neighbor_counts[7] == 1
    assert [i for i in range(7) if st.neighbor_counts[i] > 0] == [0, 1, 2, 5, 6]
    cfg = oracle.ScheduleConfig(queue_len=5, radius=1, offline_top_k=2)
    st = oracle.OnlineState(8, cfg)
    counts = [10, 0, 0, 0, 0, 0, 5, 0]
    assert oracle.active_layers(counts, st, cfg) == [0, 6]
    oracle.update_online(st, 4)
    assert oracle.active_layers(counts, st, cfg) == [0, 3, 4, 5, 6]


def test_grouped_logits(oracle, golden):
    g = golden.npz("grouped_tiny.npz")
    t = oracle.init_model(oracle.ModelConfig(num_layers=4, seed=3), bf16=True)
    lists = np.split(g["ids"], np.cumsum(g["sizes"])[:-1])
    got = np.concatenate(oracle.grouped_speculative_logits(t, g["hidden"], lists))
    assert np.array_equal(got.view(np.uint32), g["logits"].view(np.uint32))


def _tiny_engine_models(oracle, eg):
    tc = oracle.ModelConfig(num_layers=6, seed=eg["target_seed"])
    dc = oracle.ModelConfig(num_layers=2, seed=eg["draft_seed"])
    return tc, oracle.init_model(tc, bf16=True), dc, oracle.init_model(dc, bf16=True)


def test_engine_traces_tiny(oracle, golden):
    eg = golden.json("engine_tiny.json")
    tc, t, dc, dm = _tiny_engine_models(oracle, eg)
    bank = {l: oracle.init_predictor(4, 512, oracle.derive(eg["bank_seed"], l)) for l in range(5)}
    for tr in eg["traces"]:
        pol = {"never": "never", "always": "always"}.get(tr["policy"], bank)
        eng = oracle.ExitEngineOracle(tc, t, dc, dm, pol, k=4, threshold=tr["threshold"],
                                      schedule_mode=tr["mode"], exit_counts=eg["exit_counts"],
                                      schedule_config=oracle.ScheduleConfig(
                                          tr["queue_len"], tr["radius"], tr["top_k"]))
        toks, trace = eng.generate(tr["prompt"], len(tr["tokens"]))
        assert toks == tr["tokens"], tr["policy"]
        for rec, ref in zip(trace, tr["records"]):
            assert (rec.token, rec.exit_layer, rec.predictor_fired, rec.verified, rec.active,
                    rec.full_head_count, rec.predictor_evals) == (
                ref["token"], ref["exit_layer"], ref["predictor_fired"], ref["verified"],
                ref["active"], ref["full_head_count"], ref["predictor_evals"])


def corpus_prompts(corpus, num_prompts, prompt_len, seed, oracle):
    """pipeline.py:262-268."""
    data = np.frombuffer(corpus, dtype=np.uint8)
    starts = oracle.splitmix64(seed, num_prompts) % np.uint64(data.size - prompt_len + 1)
    return [[int(b) for b in data[int(s):int(s) + prompt_len]] for s in starts]


def tiny_pipeline_inputs(oracle):
    d = os.path.join(GOLDEN, "tiny_pipeline")
    tc, t = oracle.load_spxw(os.path.join(d, "target.spxw"))
    dc, dm = oracle.load_spxw(os.path.join(d, "draft.spxw"))
    bank = oracle.load_spxp(os.path.join(d, "predictors.spxp"))
    L, counts = oracle.load_spxs(os.path.join(d, "profile.spxs"))
    with open(os.path.join(d, "fixture_corpus.txt"), "rb") as fh:
        corpus = fh.read()
    prompts = corpus_prompts(corpus, 16, 16, 606, oracle)     # DEFAULT_CONFIG["bench"]
    with open(os.path.join(d, "trace.jsonl")) as fh:
        golden = [json.loads(line) for line in fh if line.strip()]
    return tc, t, dc, dm, bank, counts, prompts, golden


@pytest.mark.slow
def test_tiny_pipeline_trace_end_to_end(oracle):
    """The oracle replays the reference pipeline's bench stage
    (pipeline.py:193-242: greedy stream, then generate_forced with two-level
    scheduling, thr 0.7, ScheduleConfig(5, 1, 4)) and reproduces the shipped
    golden trace.jsonl record for record."""
    tc, t, dc, dm, bank, counts, prompts, golden = tiny_pipeline_inputs(oracle)
    assert list(counts) == [120, 47, 18, 15, 7, 1, 1, 303]
    out = []
    for prompt in prompts:
        greedy = oracle.ExitEngineOracle(tc, t, dc, dm, "never")
        toks, _ = greedy.generate(prompt, 48)
        eng = oracle.ExitEngineOracle(tc, t, dc, dm, bank, k=4, threshold=0.7,
                                      schedule_mode="two-level", exit_counts=counts,
                                      schedule_config=oracle.ScheduleConfig(5, 1, 4))
        out.extend(eng.generate_forced(prompt, toks))
    assert len(out) == len(golden) == 768
    for rec, ref in zip(out, golden):
        assert (rec.token, rec.exit_layer, rec.predictor_fired, rec.verified, rec.active) == (
            ref["token"], ref["exit_layer"], ref["predictor_fired"], ref["verified"], ref["active"])


def _tree_cases(golden):
    return golden.json("tree_tiny.json")["cases"]


def run_tree_oracle(oracle, case, n_steps=None):
    tc, t, dc, dm, bank, counts, _, _ = tiny_pipeline_inputs(oracle)
    pol = {"never_all": "never", "always_all": "always"}.get(case["case"], bank)
    eng = oracle.TreeEngineOracle(tc, t, dc, dm, pol, case["branching"], k=4,
                                  threshold=case["threshold"], schedule_mode=case["mode"],
                                  exit_counts=counts, schedule_config=oracle.ScheduleConfig(5, 1, 4))
    eng.start(case["prompt"])
    return eng, [eng.step() for _ in range(n_steps or len(case["steps"]))]


def assert_tree_step_equal(res, ref, where):
    got = dict(accepted_tokens=res.accepted_tokens, correction_token=res.correction_token,
               path_exit_layers=res.path_exit_layers, accepted_path=res.accepted_path,
               predictor_evals=res.predictor_evals, num_paths=res.num_paths,
               max_path_len=res.max_path_len, scheduled_layer_count=res.scheduled_layer_count)
    exp = {k: ref[k] for k in got}
    assert got == exp, where


@pytest.mark.parametrize("ci", range(0, 15, 3))
def test_tree_engine_oracle_matches_reference(oracle, golden, ci):
    """The oracle's TreeEngine restatement (tree.py:133-302) reproduces the
    reference TreeEngine's step results and every predictor probability
    (bit-exact, in call order) on the trained tiny pipeline models."""
    case = _tree_cases(golden)[ci]
    eng, steps = run_tree_oracle(oracle, case)
    for s, (res, ref) in enumerate(zip(steps, case["steps"])):
        assert_tree_step_equal(res, ref, (case["case"], s))
        assert [[l, p] for l, p in res.probs] == ref["probs"], (case["case"], s)
