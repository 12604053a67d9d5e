"""BatchedExitEngine: B independent early-exit streams stepped together
(configs[3]) -- every stream's ExitRecords equal a single-stream reference
engine's on the same prompt (oracle ExitEngineOracle, STRICT numerics:
bit-exact), including streams that exit early and are completed lazily while
the other streams keep running."""
import numpy as np
import pytest

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import engine as E
from paper_2504_08850_b200 import numerics

pytestmark = pytest.mark.gpu

PROMPTS = [[84, 104, 101, 32], [72, 101, 108, 108], [7, 200, 31, 99], [1, 2, 3, 4], [250, 9, 9, 1]]


def _models(eg):
    tc = spx.ModelConfig(num_layers=6, seed=eg["target_seed"])
    dc = spx.ModelConfig(num_layers=2, seed=eg["draft_seed"])
    return spx.init_model(tc, dtype="bf16"), spx.init_model(dc, dtype="bf16")


def _rec(r):
    return (r.token, r.exit_layer, r.predictor_fired, r.verified, list(r.active),
            r.full_head_count, r.predictor_evals)


@pytest.mark.parametrize("policy,thr,mode", [("mlp", 0.5, "two-level"), ("mlp", 0.3, "all"),
                                             ("always", 0.5, "two-level"),
                                             ("never", 0.5, "all")])
def test_batched_engine_matches_oracle_per_stream(golden, oracle, policy, thr, mode):
    eg = golden.json("engine_tiny.json")
    t, d = _models(eg)
    bank = {l: spx.init_predictor(4, 512, oracle.derive(eg["bank_seed"], l)) for l in range(5)}
    counts = np.asarray(eg["exit_counts"])
    prof = spx.OfflineProfile(6, counts, 0)
    pol = {"mlp": E.PredictorPolicy(bank), "always": E.AlwaysExitPolicy(),
           "never": E.NeverExitPolicy()}[policy]
    n = 12
    with numerics.using("strict"):
        eng = spx.BatchedExitEngine(t, d, pol, E.EngineConfig(k=4, threshold=thr,
                                                              schedule_mode=mode),
                                    prof, spx.ScheduleConfig(5, 1, 2), batch=len(PROMPTS),
                                    context=32)
        toks, recs = eng.generate(PROMPTS, n)
    ot = oracle.init_model(oracle.ModelConfig(num_layers=6, seed=eg["target_seed"]), bf16=True)
    od = oracle.init_model(oracle.ModelConfig(num_layers=2, seed=eg["draft_seed"]), bf16=True)
    opol = {"mlp": {l: oracle.PredictorWeights(w.w1, w.b1, w.w2, w.b2) for l, w in bank.items()},
            "always": "always", "never": "never"}[policy]
    for b, prompt in enumerate(PROMPTS):
        oe = oracle.ExitEngineOracle(oracle.ModelConfig(num_layers=6, seed=eg["target_seed"]), ot,
                                     oracle.ModelConfig(num_layers=2, seed=eg["draft_seed"]), od,
                                     opol, k=4, threshold=thr, schedule_mode=mode,
                                     exit_counts=counts,
                                     schedule_config=oracle.ScheduleConfig(5, 1, 2))
        _, want = oe.generate(prompt, n)
        got = [_rec(r) for r in recs[b]]
        assert got == [(r.token, r.exit_layer, r.predictor_fired, r.verified, list(r.active),
                        r.full_head_count, r.predictor_evals) for r in want], b
        assert toks[b] == [r.token for r in want]



def test_batched_engine_validation(golden):
    eg = golden.json("engine_tiny.json")
    t, d = _models(eg)
    with pytest.raises(ValueError):
        spx.BatchedExitEngine(t, d, E.NeverExitPolicy(), E.EngineConfig(schedule_mode="bogus"))
    eng = spx.BatchedExitEngine(t, d, E.NeverExitPolicy(), batch=2, context=16)
    with pytest.raises(ValueError):
        eng.start([[1, 2], [3]])
    with pytest.raises(ValueError):
        eng.generate([[1, 2], [3, 4]], 0)


@pytest.mark.parametrize("policy", ["always", "mlp"])
def test_batched_engine_trained_models_with_exits(oracle, policy):
    """The reference pipeline's TRAINED tiny target/draft and predictors
    (tests/golden/tiny_pipeline, f32): streams exit early at different layers
    and steps, their skipped rows are completed lazily while the other
    streams run on -- every stream still equals its single-stream oracle run."""
    import os
    tp = os.path.join(os.path.dirname(__file__), "golden", "tiny_pipeline")
    t = spx.load_weights(os.path.join(tp, "target.spxw"))
    d = spx.load_weights(os.path.join(tp, "draft.spxw"))
    bank = spx.load_predictors(os.path.join(tp, "predictors.spxp"))
    prof = spx.load_profile(os.path.join(tp, "profile.spxs"))
    tcfg, tt = oracle.load_spxw(os.path.join(tp, "target.spxw"))
    dcfg, dt = oracle.load_spxw(os.path.join(tp, "draft.spxw"))
    with open(os.path.join(tp, "fixture_corpus.txt"), "rb") as fh:
        data = np.frombuffer(fh.read(), np.uint8)
    prompts = [[int(x) for x in data[s_:s_ + 12]] for s_ in (0, 300, 901, 1500)]
    n, thr = 16, 0.7
    pol = E.AlwaysExitPolicy() if policy == "always" else E.PredictorPolicy(bank)
    opol = "always" if policy == "always" else {
        l: oracle.PredictorWeights(w.w1, w.b1, w.w2, w.b2) for l, w in bank.items()}
    with numerics.using("strict"):
        eng = spx.BatchedExitEngine(t, d, pol, E.EngineConfig(k=4, threshold=thr,
                                                              schedule_mode="two-level"),
                                    prof, spx.ScheduleConfig(5, 1, 4), batch=len(prompts),
                                    context=32)
        toks, recs = eng.generate(prompts, n)
    exits = 0
    for b, prompt in enumerate(prompts):
        oe = oracle.ExitEngineOracle(tcfg, tt, dcfg, dt, opol, k=4, threshold=thr,
                                     schedule_mode="two-level",
                                     exit_counts=np.asarray(prof.exit_counts),
                                     schedule_config=oracle.ScheduleConfig(5, 1, 4))
        _, want = oe.generate(prompt, n)
        assert [_rec(r) for r in recs[b]] == [
            (r.token, r.exit_layer, r.predictor_fired, r.verified, list(r.active),
             r.full_head_count, r.predictor_evals) for r in want], b
        exits += sum(r.exit_layer < t.config.num_layers - 1 for r in want)
    assert exits > 0                              # lazily completed rows exercised
