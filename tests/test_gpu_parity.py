"""GPU parity of the sm_100a kernels against the oracle and the reference's
golden fixtures.  Every call goes through libspecexit_b200.so (C ABI).

Bars (BASELINE.json north_star): exit decisions and layer indices bit-exact,
probabilities within 1e-3 abs.  STRICT mode additionally reproduces logits,
features and the f32 pre-sigmoid bit-for-bit; FAST mode (production) is held
to bit-exact decisions, |prob diff| <= 1e-3, and logits within 1e-5 relative
(tolerance stated here), with the decision margin |z2 - z_cut| logged.
"""
import numpy as np
import pytest
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import _native as N
from paper_2504_08850_b200 import numerics

pytestmark = pytest.mark.gpu

LOGIT_RTOL_FAST = 1e-5
PROB_ATOL = 1e-3


def tiny_device_model(seed=3, layers=4):
    return spx.init_model(spx.ModelConfig(num_layers=layers, seed=seed), dtype="bf16")


def head_7b(seed=1234):
    cfg = spx.ModelConfig(vocab_size=32000, hidden_dim=4096, num_layers=32, num_heads=32,
                          ffn_dim=11008, max_context=512, seed=seed)
    return spx.init_model(cfg, dtype="bf16", head_only=True)


def run_fused(model, g, thr, mode):
    w = spx.PredictorWeights(g["w1"], g["b1"], g["w2"], float(g["b2"]))
    hidden = torch.as_tensor(g["hidden"], device="cuda")
    ids = torch.as_tensor(g["ids"].astype(np.int32), device="cuda")
    prev = torch.as_tensor(g["prev"], device="cuda").clone()
    feats = torch.empty((ids.shape[0], 3 * ids.shape[1]), device="cuda")
    out = spx.evaluate_batch(model, w, hidden, ids, prev, threshold=thr, mode=mode)
    # features come from the function-level operator on the same kernels
    torch.cuda.synchronize()
    N.raise_device_error(out.err.item())
    return out, prev


def _bits(t):
    return t.detach().cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("name", ["predictor_tiny.npz", "predictor_tiny_k20.npz",
                                  "predictor_tiny_h32.npz"])
def test_device_init_matches_reference_init(golden, oracle, name):
    m = tiny_device_model()
    t = oracle.init_model(oracle.ModelConfig(num_layers=4, seed=3), bf16=True)
    assert np.array_equal(m.lm_head.float().cpu().numpy(), t["lm_head"].T)
    assert np.array_equal(m.embedding.float().cpu().numpy(), t["embedding"])
    wq = m.layers[2]["wqkv"][:64].float().cpu().numpy()
    assert np.array_equal(wq, t["layers.2.attn.wq"].T)
    assert np.array_equal(m.layers[3]["ffn_w2"].float().cpu().numpy(), t["layers.3.ffn.w2"].T)


@pytest.mark.parametrize("name,thrs", [("predictor_tiny.npz", (0.5, 0.7)),
                                       ("predictor_tiny_k20.npz", (0.5,)),
                                       ("predictor_tiny_h32.npz", (0.5,))])
def test_fused_predictor_strict_bit_exact_tiny(golden, name, thrs):
    g = golden.npz(name)
    m = tiny_device_model()
    for thr in thrs:
        out, prev = run_fused(m, g, thr, N.SPX_MODE_STRICT)
        assert np.array_equal(_bits(out.logits), g["logits"].view(np.uint32))
        assert np.array_equal(_bits(prev), g["probs"].view(np.uint32))
        assert np.array_equal(_bits(out.z), g["z2"].view(np.uint32))
        assert np.max(np.abs(out.prob.cpu().numpy() - g["prob"])) <= 1e-6   # f32 sigmoid report
        assert np.array_equal(out.fired.cpu().numpy().astype(bool), g[f"fired_{thr}"])


@pytest.mark.parametrize("name,thrs", [("predictor_tiny.npz", (0.5, 0.7)),
                                       ("predictor_tiny_k20.npz", (0.5,))])
def test_fused_predictor_fast_decisions_exact_tiny(golden, name, thrs):
    g = golden.npz(name)
    m = tiny_device_model()
    for thr in thrs:
        out, prev = run_fused(m, g, thr, N.SPX_MODE_FAST)
        lg = out.logits.cpu().numpy()
        assert np.all(np.abs(lg - g["logits"]) <= LOGIT_RTOL_FAST * np.maximum(np.abs(g["logits"]), 1))
        assert np.max(np.abs(out.prob.cpu().numpy() - g["prob"])) <= PROB_ATOL
        assert np.array_equal(out.fired.cpu().numpy().astype(bool), g[f"fired_{thr}"])
        margin = np.min(np.abs(out.z.cpu().numpy().astype(np.float64) - spx.z_cut(thr)))
        print(f"[{name} thr={thr}] fast min |z2 - z_cut| = {margin:.3e}")


def test_fused_predictor_7b_head(golden, oracle):
    g = golden.npz("predictor_7b.npz")
    r = np.random.default_rng(int(g["hidden_seed"]))
    g["hidden"] = oracle.round_bf16(r.standard_normal((g["ids"].shape[0], 4096)).astype(np.float32))
    m = head_7b()
    for mode in (N.SPX_MODE_STRICT, N.SPX_MODE_FAST):
        for thr in (0.5, 0.7):
            out, prev = run_fused(m, g, thr, mode)
            assert np.array_equal(out.fired.cpu().numpy().astype(bool), g[f"fired_{thr}"])
            assert np.max(np.abs(out.prob.cpu().numpy() - g["prob"])) <= PROB_ATOL
            if mode == N.SPX_MODE_STRICT:
                assert np.array_equal(_bits(out.logits), g["logits"].view(np.uint32))
                assert np.array_equal(_bits(out.z), g["z2"].view(np.uint32))
    # verify kernel: argmax over 32000 vocab rows
    for mode in ("strict", "fast"):
        with numerics.using(mode):
            tok, _, _ = spx.head_argmax(m, torch.as_tensor(g["hidden"], device="cuda"))
        assert tok.cpu().numpy().tolist() == g["argmax"].tolist(), mode


def test_full_head_strict_bit_exact_and_fast_close(golden, oracle):
    g = golden.npz("predictor_tiny.npz")
    m = tiny_device_model()
    t = oracle.init_model(oracle.ModelConfig(num_layers=4, seed=3), bf16=True)
    for i in range(8):
        ref = oracle.full_head_logits(t, g["hidden"][i])
        with numerics.using("strict"):
            got = spx.full_head_logits(m, torch.as_tensor(g["hidden"][i], device="cuda"))
        assert np.array_equal(_bits(got), ref.view(np.uint32))
        fast = spx.full_head_logits(m, torch.as_tensor(g["hidden"][i], device="cuda")).cpu().numpy()
        assert np.all(np.abs(fast - ref) <= LOGIT_RTOL_FAST * np.maximum(np.abs(ref), 1))
        assert int(np.argmax(fast)) == int(g["argmax"][i])


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_slice_equals_full_head_gather_bitwise(golden, mode):
    """tests/test_model.py:148-152 of the reference, on device, both modes."""
    g = golden.npz("predictor_tiny.npz")
    m = tiny_device_model()
    with numerics.using(mode):
        for i in range(6):
            h = torch.as_tensor(g["hidden"][i], device="cuda")
            ids = [5, 77, 255, 0, 128]
            full = spx.full_head_logits(m, h)
            sl = spx.sliced_head_logits(m, h, ids)
            assert torch.equal(full[ids], sl)


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_grouped_logits(golden, mode):
    g = golden.npz("grouped_tiny.npz")
    m = tiny_device_model()
    lists = [x.tolist() for x in np.split(g["ids"], np.cumsum(g["sizes"])[:-1])]
    with numerics.using(mode):
        got = spx.grouped_speculative_logits(m, g["hidden"], lists)
        flat = torch.cat(got).cpu().numpy()
        if mode == "strict":
            assert np.array_equal(flat.view(np.uint32), g["logits"].view(np.uint32))
        else:
            assert np.allclose(flat, g["logits"], rtol=LOGIT_RTOL_FAST, atol=LOGIT_RTOL_FAST)
        for row in range(0, 40, 7):       # grouped == sliced exactly (test_tree.py:32-42)
            sl = spx.sliced_head_logits(m, torch.as_tensor(g["hidden"][row], device="cuda"), lists[row])
            assert torch.equal(got[row], sl)


def test_device_exp_matches_numpy():
    r = np.random.default_rng(1)
    x = np.concatenate([r.uniform(-104, 0, 4_000_000), r.uniform(-3, 0, 1_000_000),
                        np.linspace(-110, 1, 100_001)]).astype(np.float32)
    y = torch.empty(x.size, dtype=torch.float32, device="cuda")
    xd = torch.as_tensor(x, device="cuda")
    N.check(N.lib().spx_np_expf(N.ptr(xd), N.ptr(y), x.size, N.stream_ptr()), "spx_np_expf")
    with np.errstate(over="ignore", under="ignore"):
        ref = np.exp(x)
    bad = np.nonzero(y.cpu().numpy().view(np.uint32) != ref.view(np.uint32))[0]
    assert bad.size == 0, (x[bad[:5]], ref[bad[:5]])


def test_scheduler_stream_on_device(golden):
    for case in golden.json("scheduler_stream.json"):
        cfg = spx.ScheduleConfig(case["queue_len"], case["radius"], case["top_k"])
        prof = spx.OfflineProfile(case["L"], np.array(case["exit_counts"], np.uint64), 0)
        assert prof.ranked_layers == case["ranked"]
        st = spx.OnlineState(case["L"], cfg)
        for e, act, nbr in zip(case["exits"], case["active"], case["neighbor_counts"]):
            spx.update_online(st, e)
            assert st.neighbor_counts.tolist() == nbr
            assert spx.active_layers(prof, st, cfg) == act
        assert st.queue == case["queue"]


def test_scheduler_many_rows_at_once(golden):
    """All streams of the golden file advanced as rows of ONE device state."""
    cases = [c for c in golden.json("scheduler_stream.json") if c["queue_len"] == 5]
    from paper_2504_08850_b200.scheduler import update_online
    for c in cases[:1]:
        cfg = spx.ScheduleConfig(c["queue_len"], c["radius"], c["top_k"])
        st = spx.OnlineState(c["L"], cfg, rows=64)
        for step, e in enumerate(c["exits"]):
            update_online(st, torch.full((64,), e, dtype=torch.int32, device="cuda"))
            counts = st.counts.cpu().numpy()
            assert (counts == np.array(c["neighbor_counts"][step])).all()


def test_error_mapping():
    m = tiny_device_model()
    h = torch.randn(64, device="cuda")
    with pytest.raises(ValueError):
        spx.sliced_head_logits(m, h, [1, 256])
    with pytest.raises(ValueError):
        spx.sliced_head_logits(m, h, [])
    bad = h.clone()
    bad[3] = float("inf")
    with pytest.raises(ValueError):
        spx.sliced_head_logits(m, bad, [1, 2])
    with pytest.raises(ValueError):
        spx.extract_features(np.array([np.inf, 0], np.float32), spx.uniform_probs(2))
    with pytest.raises(ValueError):
        spx.extract_features(np.array([1, 2], np.float32), np.array([0.9, 0.3], np.float32))
    with pytest.raises(ValueError):
        spx.extract_features(np.array([1, 2, 3], np.float32), spx.uniform_probs(2))


def test_reference_predictor_unit_semantics():
    """tests/test_predictor.py:12-54 of the reference, against the drop-in."""
    fv = spx.extract_features(np.array([1, 2, 3, 4], np.float32), spx.uniform_probs(4))
    assert fv.k == 4 and tuple(fv.concat().shape) == (12,)
    logits = np.array([0.0, 1.0], np.float32)
    fv = spx.extract_features(logits, np.array([0.5, 0.5], np.float32))
    cat = fv.concat().cpu().numpy()
    assert np.array_equal(cat[:2], logits)
    assert abs(float(cat[2:4].sum()) - 1.0) < 1e-6
    assert np.allclose(cat[4:], cat[2:4] - 0.5)
    w = spx.init_predictor(4, 32, seed=0)
    f = np.linspace(-1, 1, 12).astype(np.float32)
    p = spx.predictor_forward(w, f)
    assert 0.0 < p < 1.0 and p == spx.predictor_forward(w, f)
    z = spx.PredictorWeights(w1=np.zeros((12, 8), np.float32), b1=np.zeros(8, np.float32),
                             w2=np.zeros(8, np.float32), b2=0.0)
    p = spx.predictor_forward(z, np.ones(12, np.float32))
    assert p == 0.5 and not spx.decide_exit(p, 0.5) and spx.decide_exit(0.51, 0.5)


def test_predictor_forward_matches_oracle(oracle):
    r = np.random.default_rng(3)
    for k in (1, 4, 16, 17, 64):
        w = spx.init_predictor(k, 512, seed=k)
        w.b1 = (r.standard_normal(512) * 0.05).astype(np.float32)
        ow = oracle.PredictorWeights(w.w1, w.b1, w.w2, w.b2)
        for _ in range(20):
            f = r.standard_normal(3 * k).astype(np.float32)
            assert spx.predictor_forward(w, f) == pytest.approx(oracle.predictor_forward(ow, f),
                                                                abs=1e-12)
