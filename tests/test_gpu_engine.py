"""GPU parity of the device-resident early-exit engine (flag-guarded decoder
layers + the graph-captured token step) against the oracle and the
reference's golden traces.

STRICT mode (reference reduction order) must reproduce the reference's
hidden states bit-for-bit and every ExitRecord field exactly.  FAST mode is
held to hidden states within 1e-4 relative (tolerance stated here) and to
self-consistency (Never policy == greedy decoding).
"""
import json
import os

import numpy as np
import pytest
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import engine as E
from paper_2504_08850_b200 import numerics
from paper_2504_08850_b200.decode import DecodeState

pytestmark = pytest.mark.gpu

HIDDEN_RTOL_FAST = 1e-4
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
PROMPT = [84, 104, 101, 32]


def _ref_rows(oracle, seed, layers, tokens):
    cfg = oracle.ModelConfig(num_layers=layers, seed=seed)
    t = oracle.init_model(cfg, bf16=True)
    st = oracle.DecodeState(cfg, t, oracle.sinusoidal_encoding(cfg.max_context, cfg.hidden_dim))
    return cfg, t, st


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_decode_state_lazy_completion(oracle, mode):
    """Layer kernels vs the oracle DecodeState, including the lazy
    completion of rows left behind by an early exit (model.py:220-270)."""
    m = spx.init_model(spx.ModelConfig(num_layers=4, seed=3), dtype="bf16")
    cfg, t, ref = _ref_rows(oracle, 3, 4, None)
    with numerics.using(mode):
        st = DecodeState(m)
        # prompt through all layers, then token A exits after layer 1,
        # token B runs all layers (dragging A's rows 2..3 along)
        plan = [(PROMPT, 4), ([65], 2), ([66], 4), ([67], 1), ([68], 4)]
        for toks, depth in plan:
            st.begin(toks)
            ref.begin(toks)
            for l in range(depth):
                got = st.run_layer(l).cpu().numpy()
                want = ref.run_layer(l)
                if mode == "strict":
                    assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), (toks, l)
                else:
                    np.testing.assert_allclose(got, want, rtol=HIDDEN_RTOL_FAST,
                                               atol=HIDDEN_RTOL_FAST * np.abs(want).max())
        st.check()
        fr = st.frontier[:st.n].cpu().numpy()
        assert list(fr) == list(ref.frontier[:ref.n])


@pytest.mark.parametrize("dims", [(1024, 2816, 8), (4096, 11008, 32), (512, 1376, 4),
                                  (5120, 13824, 40)])
def test_fast_layers_match_strict(dims):
    """The TMA-streamed FAST layer kernels (every contraction width class:
    1..3 chunks per thread) against the STRICT reference-order kernels, with
    multi-row prefill, single-row decode and lazily completed rows."""
    d, f, nh = dims
    cfg = spx.ModelConfig(vocab_size=512, hidden_dim=d, num_layers=3, num_heads=nh, ffn_dim=f,
                          max_context=32, seed=9)
    m = spx.init_model(cfg, dtype="bf16")
    outs = {}
    for mode in ("strict", "fast"):
        with numerics.using(mode):
            st = DecodeState(m)
            res = []
            for toks, depth in [(list(range(1, 13)), 3), ([6], 1), ([7], 3), ([8], 3), ([9], 1),
                                ([10], 1), ([11], 3)]:
                st.begin(toks)
                for l in range(depth):
                    res.append(st.run_layer(l).cpu().numpy())
            st.check()
            res.append(st.pending[:st.n].cpu().numpy())
            outs[mode] = res
    for a, b in zip(outs["strict"], outs["fast"]):
        np.testing.assert_allclose(b, a, rtol=1e-3, atol=1e-3 * np.abs(a).max())


def _engine_models(eg):
    tc = spx.ModelConfig(num_layers=6, seed=eg["target_seed"])
    dc = spx.ModelConfig(num_layers=2, seed=eg["draft_seed"])
    return spx.init_model(tc, dtype="bf16"), spx.init_model(dc, dtype="bf16")


def _rec_tuple(r):
    return (r.token, r.exit_layer, r.predictor_fired, r.verified, list(r.active),
            r.full_head_count, r.predictor_evals)


def test_engine_golden_traces_strict(golden, oracle):
    """Every policy / schedule of engine_tiny.json reproduced record for
    record by the graph-captured device engine."""
    eg = golden.json("engine_tiny.json")
    t, d = _engine_models(eg)
    bank = {l: spx.init_predictor(4, 512, oracle.derive(eg["bank_seed"], l)) for l in range(5)}
    prof = spx.OfflineProfile(6, np.asarray(eg["exit_counts"]), 0)
    with numerics.using("strict"):
        for tr in eg["traces"]:
            pol = {"never": E.NeverExitPolicy(), "always": E.AlwaysExitPolicy()}.get(
                tr["policy"]) or E.PredictorPolicy(bank)
            cfg = E.EngineConfig(k=4, threshold=tr["threshold"], schedule_mode=tr["mode"])
            eng = E.ExitEngine(t, d, pol, cfg, prof,
                               spx.ScheduleConfig(tr["queue_len"], tr["radius"], tr["top_k"]))
            assert eng.device_resident()
            toks, trace = eng.generate(tr["prompt"], len(tr["tokens"]))
            assert toks == tr["tokens"], tr["policy"]
            for rec, ref in zip(trace, tr["records"]):
                assert _rec_tuple(rec) == (ref["token"], ref["exit_layer"], ref["predictor_fired"],
                                           ref["verified"], ref["active"], ref["full_head_count"],
                                           ref["predictor_evals"]), tr["policy"]


def test_engine_host_path_matches_device_path(golden, oracle):
    """The host-decision loop (used for custom policies) and the device graph
    agree record for record."""
    eg = golden.json("engine_tiny.json")
    t, d = _engine_models(eg)
    bank = {l: spx.init_predictor(4, 512, oracle.derive(eg["bank_seed"], l)) for l in range(5)}
    prof = spx.OfflineProfile(6, np.asarray(eg["exit_counts"]), 0)

    class Wrapped(E.PredictorPolicy):       # a user subclass -> host path
        pass

    with numerics.using("strict"):
        cfg = E.EngineConfig(k=4, threshold=0.5, schedule_mode="two-level")
        dev = E.ExitEngine(t, d, E.PredictorPolicy(bank), cfg, prof, spx.ScheduleConfig(5, 1, 2))
        host = E.ExitEngine(t, d, Wrapped(bank), cfg, prof, spx.ScheduleConfig(5, 1, 2))
        assert dev.device_resident() and not host.device_resident()
        a = dev.generate(PROMPT, 12)
        b = host.generate(PROMPT, 12)
        assert a[0] == b[0]
        assert [_rec_tuple(r) for r in a[1]] == [_rec_tuple(r) for r in b[1]]


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_never_exit_equals_greedy(golden, mode):
    """engine tests: test_never_exit_equals_greedy (tests/test_engine.py:14-20)."""
    eg = golden.json("engine_tiny.json")
    t, d = _engine_models(eg)
    with numerics.using(mode):
        base, _ = E.greedy_generate(t, PROMPT, 24)
        toks, trace = E.ExitEngine(t, d, E.NeverExitPolicy()).generate(PROMPT, 24)
    assert toks == base
    assert all(r.exit_layer == 5 for r in trace)
    assert not any(r.predictor_fired for r in trace)


def test_oracle_policy_lossless(golden):
    """tests/test_engine.py:23-38: the oracle policy with the full-vocabulary
    speculative set reproduces greedy output and the oracle exit layers."""
    eg = golden.json("engine_tiny.json")
    t, d = _engine_models(eg)
    base, layers = E.greedy_generate(t, PROMPT, 12)
    eng = E.ExitEngine(t, d, E.OraclePolicy(t), E.EngineConfig(spec_full_vocab=True))
    assert not eng.device_resident()
    toks, trace = eng.generate(PROMPT, 12)
    assert toks == base
    assert [r.exit_layer for r in trace] == layers


def test_always_exit_soundness(golden):
    """tests/test_engine.py:53-68: a verified exit token equals the full-head
    argmax at the exit layer (replayed from scratch)."""
    eg = golden.json("engine_tiny.json")
    t, d = _engine_models(eg)
    toks, trace = E.ExitEngine(t, d, E.AlwaysExitPolicy()).generate(PROMPT, 16)
    ctx = list(PROMPT)
    for rec in trace:
        st = DecodeState(t)
        st.begin(ctx)
        for l in range(rec.exit_layer + 1):
            st.launch_layer(l)
        tok, _, _ = spx.head_argmax(t, st.cur_hidden)
        if rec.verified or rec.exit_layer == 5:
            assert rec.token == int(tok[0].item())
        ctx.append(rec.token)


def test_predictor_policy_requires_layer_coverage(golden):
    """tests/test_engine.py:71-75."""
    eg = golden.json("engine_tiny.json")
    t, d = _engine_models(eg)
    bank = {0: spx.init_predictor(4, 8, seed=0)}
    eng = E.ExitEngine(t, d, E.PredictorPolicy(bank))
    with pytest.raises(KeyError):
        eng.generate(PROMPT, 2)


def test_context_overflow_raises(golden):
    eg = golden.json("engine_tiny.json")
    t, d = _engine_models(eg)
    eng = E.ExitEngine(t, d, E.NeverExitPolicy())
    with pytest.raises(ValueError):
        eng.generate(PROMPT, t.config.max_context)


def _corpus_prompts(corpus, n, plen, seed, oracle):
    data = np.frombuffer(corpus, dtype=np.uint8)
    starts = oracle.splitmix64(seed, n) % np.uint64(data.size - plen + 1)
    return [[int(b) for b in data[int(s):int(s) + plen]] for s in starts]


def test_tiny_pipeline_trace_on_device(oracle):
    """The reference pipeline's bench stage (pipeline.py:193-242) on the
    device engine: greedy stream, then generate_forced with the trained
    predictors, two-level scheduling (thr 0.7, ScheduleConfig(5, 1, 4)) --
    the shipped trace.jsonl reproduced record for record (f32 weights)."""
    d = os.path.join(GOLDEN, "tiny_pipeline")
    t = spx.load_weights(os.path.join(d, "target.spxw"))
    dm = spx.load_weights(os.path.join(d, "draft.spxw"))
    bank = spx.load_predictors(os.path.join(d, "predictors.spxp"))
    prof = spx.load_profile(os.path.join(d, "profile.spxs"))
    with open(os.path.join(d, "fixture_corpus.txt"), "rb") as fh:
        prompts = _corpus_prompts(fh.read(), 16, 16, 606, oracle)
    with open(os.path.join(d, "trace.jsonl")) as fh:
        golden = [json.loads(line) for line in fh if line.strip()]
    out = []
    with numerics.using("strict"):
        pol = E.PredictorPolicy(bank)
        for prompt in prompts:
            # one engine per prompt, as the reference pipeline does
            # (pipeline.py:220-223): each starts with an empty online window
            eng = E.ExitEngine(t, dm, pol,
                               E.EngineConfig(k=4, threshold=0.7, schedule_mode="two-level"),
                               prof, spx.ScheduleConfig(5, 1, 4))
            assert eng.device_resident()
            base, _ = E.greedy_generate(t, prompt, 48)
            out.extend(eng.generate_forced(prompt, base))
    assert len(out) == len(golden) == 768
    for i, (rec, ref) in enumerate(zip(out, golden)):
        assert (rec.token, rec.exit_layer, rec.predictor_fired, rec.verified, rec.active) == (
            ref["token"], ref["exit_layer"], ref["predictor_fired"], ref["verified"],
            ref["active"]), i


def test_device_step_graph_replays_without_host_sync(golden):
    """generate() of N tokens replays the captured token graph N times; the
    graph is captured once per (mode, forced) and reused across calls."""
    eg = golden.json("engine_tiny.json")
    t, d = _engine_models(eg)
    eng = E.ExitEngine(t, d, E.AlwaysExitPolicy())
    a, _ = eng.generate(PROMPT, 8)
    g = dict(eng._dev.graphs)
    b, _ = eng.generate(PROMPT, 8)
    assert a == b
    assert eng._dev.graphs == g and len(g) == 1


def _inject_flags(seed, n, p=0.8):
    u = (spx.rng.splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return [bool(x < p) for x in u]


def _oracle_engine(oracle, eg_or_cfgs, bank, thr, mode, counts, sc, k=4):
    tcfg, dcfg = eg_or_cfgs
    t = oracle.init_model(tcfg, bf16=True)
    d = oracle.init_model(dcfg, bf16=True)
    ob = {l: oracle.PredictorWeights(w.w1, w.b1, w.w2, w.b2) for l, w in bank.items()}
    return oracle.ExitEngineOracle(tcfg, t, dcfg, d, ob, k=k, threshold=thr, schedule_mode=mode,
                                   exit_counts=counts,
                                   schedule_config=oracle.ScheduleConfig(*sc))


def _orec(r):
    return (r.token, r.exit_layer, r.predictor_fired, r.verified, list(r.active),
            r.full_head_count, r.predictor_evals)


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_injected_spec_forced_matches_oracle(golden, oracle, mode):
    """The injected-spec hook (at 80% of the steps the
    target's final argmax joins the draft ids) on the device graph vs the
    oracle engine with the same hook, record for record."""
    eg = golden.json("engine_tiny.json")
    t, d = _engine_models(eg)
    bank = {l: spx.init_predictor(4, 512, oracle.derive(eg["bank_seed"], l)) for l in range(5)}
    counts = np.asarray(eg["exit_counts"])
    prof = spx.OfflineProfile(6, counts, 0)
    n = 20
    with numerics.using(mode):
        base, _ = E.greedy_generate(t, PROMPT, n)
        flags = _inject_flags(31, n)
        eng = E.ExitEngine(t, d, E.PredictorPolicy(bank),
                           E.EngineConfig(k=4, threshold=0.5, schedule_mode="two-level"), prof,
                           spx.ScheduleConfig(5, 1, 2))
        got = eng.generate_forced(PROMPT, base, inject=flags)
        host = E.ExitEngine(t, d, type("P", (E.PredictorPolicy,), {})(bank),
                            E.EngineConfig(k=4, threshold=0.5, schedule_mode="two-level"), prof,
                            spx.ScheduleConfig(5, 1, 2))
        assert not host.device_resident()
        got_host = host.generate_forced(PROMPT, base, inject=flags)
    oe = _oracle_engine(oracle, (oracle.ModelConfig(num_layers=6, seed=eg["target_seed"]),
                                 oracle.ModelConfig(num_layers=2, seed=eg["draft_seed"])),
                        bank, 0.5, "two-level", counts, (5, 1, 2))
    want = oe.generate_forced(PROMPT, base, inject=flags)
    assert [_rec_tuple(r) for r in got] == [_orec(r) for r in want]
    assert [_rec_tuple(r) for r in got_host] == [_orec(r) for r in want]


@pytest.mark.slow
def test_engine_7b_dims_fast_matches_oracle(oracle):
    """A 4-layer target / 2-layer draft at Llama2-7B widths (d=4096,
    ffn=11008, V=32000) in FAST mode (certified predictor decisions, the
    persistent layer kernel) against the oracle engine: 8 tokens, two-level,
    thr 0.5, every ExitRecord field equal."""
    tc = spx.ModelConfig(32000, 4096, 4, 32, 11008, 64, 1234)
    dc = spx.ModelConfig(32000, 4096, 2, 32, 11008, 64, 1235)
    t, d = spx.init_model(tc, dtype="bf16"), spx.init_model(dc, dtype="bf16")
    bank = {l: spx.init_predictor(4, 512, spx.rng.derive(1234, l)) for l in range(3)}
    counts = np.asarray([5, 1, 3, 0], np.uint64)
    prof = spx.OfflineProfile(4, counts, 0)
    prompt = [int(x) % 32000 for x in spx.rng.splitmix64(1234, 6)]
    with numerics.using("fast"):
        eng = E.ExitEngine(t, d, E.PredictorPolicy(bank),
                           E.EngineConfig(k=4, threshold=0.5, schedule_mode="two-level"), prof,
                           spx.ScheduleConfig(5, 1, 2))
        assert eng.device_resident()
        toks, got = eng.generate(prompt, 8)
    del t, d
    torch.cuda.empty_cache()
    oc = lambda c: oracle.ModelConfig(c.vocab_size, c.hidden_dim, c.num_layers,  # noqa: E731
                                      c.num_heads, c.ffn_dim, c.max_context, c.seed)
    oe = _oracle_engine(oracle, (oc(tc), oc(dc)), bank, 0.5, "two-level", counts, (5, 1, 2))
    _, want = oe.generate(prompt, 8)
    assert [_rec_tuple(r) for r in got] == [_orec(r) for r in want]


@pytest.mark.parametrize("dims", [(4096, 11008, 32), (1024, 2816, 8), (5120, 13824, 40)])
def test_tcgen05_layers_match_strict(dims):
    """Calls advancing >= 16 rows take the tensor-core layer path
    (spx_layer_tc.cuh: tcgen05.mma GEMMs over exact bf16 parts of the rows):
    a 40-row prefill, then single rows, vs the STRICT reference-order kernels
    (FAST tolerance 1e-3 as for the other FAST layer kernels)."""
    d, f, nh = dims
    cfg = spx.ModelConfig(vocab_size=512, hidden_dim=d, num_layers=2, num_heads=nh, ffn_dim=f,
                          max_context=64, seed=19)
    m = spx.init_model(cfg, dtype="bf16")
    outs = {}
    for mode in ("strict", "fast"):
        with numerics.using(mode):
            st = DecodeState(m)
            res = []
            for toks, depth in [(list(range(3, 43)), 2), ([6], 1), (list(range(50, 70)), 2),
                                ([7], 2)]:
                st.begin(toks)
                for l in range(depth):
                    res.append(st.run_layer(l).cpu().numpy())
            st.check()
            res.append(st.pending[:st.n].cpu().numpy())
            outs[mode] = res
    for a, b in zip(outs["strict"], outs["fast"]):
        np.testing.assert_allclose(b, a, rtol=1e-3, atol=1e-3 * np.abs(a).max())


@pytest.mark.parametrize("name", ["target.spxw", "draft.spxw"])
def test_save_weights_byte_identical(tmp_path, name):
    """SPXW writer (model.py:408-417): loading the reference pipeline's weight
    files into device layouts and writing them back reproduces the files byte
    for byte; a bf16 device model round-trips its (exactly widened) values."""
    src = os.path.join(GOLDEN, "tiny_pipeline", name)
    m = spx.load_weights(src)
    out = tmp_path / name
    spx.save_weights(m, out)
    with open(src, "rb") as a, open(out, "rb") as b:
        assert a.read() == b.read()
    mb = spx.init_model(spx.ModelConfig(num_layers=2, seed=7), dtype="bf16")
    spx.save_weights(mb, tmp_path / "b.spxw")
    back = spx.load_weights(tmp_path / "b.spxw", dtype="bf16")
    ta, tb = spx.to_tensors(mb), spx.to_tensors(back)
    assert ta.keys() == tb.keys()
    for k in ta:
        assert np.array_equal(ta[k], tb[k]), k


def test_engine_reuse_keeps_online_window(golden, oracle):
    """Two generate() calls on ONE engine in two-level mode: the online window
    carries over (the reference creates it in __init__ and never resets it,
    engine.py:122-160), so the second call's active layers, exits and tokens
    follow the first call's exits -- as the oracle engine reused the same way."""
    eg = golden.json("engine_tiny.json")
    tr = [x for x in eg["traces"] if x["mode"] == "two-level"][0]
    t, d = _engine_models(eg)
    bank = {l: spx.init_predictor(4, 512, oracle.derive(eg["bank_seed"], l)) for l in range(5)}
    prof = spx.OfflineProfile(6, np.asarray(eg["exit_counts"]), 0)
    tc = oracle.ModelConfig(num_layers=6, seed=eg["target_seed"])
    dc = oracle.ModelConfig(num_layers=2, seed=eg["draft_seed"])
    obank = {l: oracle.init_predictor(4, 512, oracle.derive(eg["bank_seed"], l)) for l in range(5)}
    ora = oracle.ExitEngineOracle(tc, oracle.init_model(tc, bf16=True), dc,
                                  oracle.init_model(dc, bf16=True), obank, k=4,
                                  threshold=tr["threshold"], schedule_mode="two-level",
                                  exit_counts=np.asarray(eg["exit_counts"]),
                                  schedule_config=oracle.ScheduleConfig(tr["queue_len"], tr["radius"],
                                                                        tr["top_k"]))
    with numerics.using("strict"):
        eng = E.ExitEngine(t, d, E.PredictorPolicy(bank),
                           E.EngineConfig(k=4, threshold=tr["threshold"], schedule_mode="two-level"),
                           prof, spx.ScheduleConfig(tr["queue_len"], tr["radius"], tr["top_k"]))
        for prompt in (tr["prompt"], [7, 9, 11, 13, 15]):
            toks, trace = eng.generate(prompt, 10)
            otoks, otrace = ora.generate(prompt, 10)
            assert toks == otoks
            for rec, ref in zip(trace, otrace):
                assert (rec.token, rec.exit_layer, rec.predictor_fired, rec.verified,
                        list(rec.active)) == (ref.token, ref.exit_layer, ref.predictor_fired,
                                              ref.verified, list(ref.active))


@pytest.mark.parametrize("k", [1, 4, 25, 64])
def test_topk_matches_stable_argsort(k):
    """spx_topk (speculation.py:57-60: np.argsort(-x, kind="stable")[:k]) for
    k up to 64, with exact ties, on one row and on many rows at once."""
    from paper_2504_08850_b200 import _native as N
    from paper_2504_08850_b200.speculation import topk_from_logits
    rs = np.random.default_rng(k)
    x = rs.integers(-50, 50, size=(6, 4000)).astype(np.float32) / 8   # many exact ties
    for r in range(x.shape[0]):
        ids = np.asarray(topk_from_logits(x[r], k))
        assert np.array_equal(ids, np.argsort(-x[r], kind="stable")[:k])
    xs = torch.as_tensor(x, device="cuda")
    out = torch.empty((x.shape[0], k), dtype=torch.int32, device="cuda")
    N.check(N.lib().spx_topk_rows(N.ptr(xs), x.shape[0], x.shape[1], k, N.ptr(out),
                                  N.stream_ptr()), "spx_topk_rows")
    assert np.array_equal(out.cpu().numpy(), np.argsort(-x, axis=1, kind="stable")[:, :k])


def test_tcgen05_layers_256_row_tiles_and_lazy_rows():
    """A 300-row prefill (three 128-row tiles; with SPX_TCL_N256=1 the
    256-row UMMA tiles over all 512 TMEM columns), then a call whose row set
    exceeds its expectation (20 new rows + 300 rows completing layer 2) makes
    CTAs walk extra row tiles.  FAST vs the STRICT reference-order kernels,
    FAST tolerance."""
    d, f, nh = 1024, 2816, 8
    cfg = spx.ModelConfig(vocab_size=512, hidden_dim=d, num_layers=3, num_heads=nh, ffn_dim=f,
                          max_context=400, seed=23)
    m = spx.init_model(cfg, dtype="bf16")
    outs = {}
    for mode in ("strict", "fast"):
        with numerics.using(mode):
            st = DecodeState(m)
            res = []
            st.begin([int(x) % 512 for x in range(7, 307)])
            res.append(st.run_layer(0).cpu().numpy())
            res.append(st.run_layer(1).cpu().numpy())
            # 20 new rows; layer 2 then also completes the 300 rows left at it
            st.begin(list(range(60, 80)))
            for l in range(3):
                res.append(st.run_layer(l).cpu().numpy())
            st.check()
            res.append(st.pending[:st.n].cpu().numpy())
            outs[mode] = res
    for a, b in zip(outs["strict"], outs["fast"]):
        assert a.shape == b.shape
        np.testing.assert_allclose(b, a, rtol=1e-3, atol=1e-3 * np.abs(a).max())
