"""FAST-mode exit decisions are the reference's, bit for bit.

The production (FAST) predictor path computes logits in the canonical CDOT
order, not the reference's sequential sums; every decision is certified
against a stated error bound or re-evaluated by the STRICT chain in the same
spx_predictor_eval call.  These tests hold the result to the oracle
(oracle/specexit_oracle.py: the reference chain of model.py:298-314,
predictor.py:42-109) with NO margin exclusion:

* the bench configuration itself: Llama2-7B head (V=32000, d=4096), K=4,
  H=512, 31 layer launches chained through prev, B=1024 rows per launch, a
  256-row sample checked against the oracle at thresholds 0.5 and 0.7;
* K in {1, 8, 16, 64} at d in {4096, 8192} with a V=128000 head;
* the re-evaluation path forced for every row (bound inflated): FAST+recheck
  must then equal the STRICT kernel bit for bit.

Tolerances: decisions exact; probabilities 1e-3 absolute.
"""
import numpy as np
import pytest
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import numerics, rng

pytestmark = pytest.mark.gpu

PROB_ATOL = 1e-3
_MODELS = {}


def head(V, d, seed=1):
    key = (V, d, seed)
    if key not in _MODELS:
        cfg = spx.ModelConfig(vocab_size=V, hidden_dim=d, num_layers=1, num_heads=32,
                              ffn_dim=4 * d, max_context=64, seed=seed)
        _MODELS[key] = spx.init_model(cfg, dtype="bf16", head_only=True)
    return _MODELS[key]


def oracle_head(model, ids):
    """Oracle tensors for the ids used: the (d, U) f32 columns of the bf16 head
    (the strict dot reads one column per id, so a compact head gives the same
    bits) and ids remapped into it."""
    uniq, inv = np.unique(ids, return_inverse=True)
    rows = model.lm_head[torch.as_tensor(uniq, device="cuda", dtype=torch.long)]
    cols = np.ascontiguousarray(rows.float().cpu().numpy().T)
    t = {"lm_head": cols, "final_norm.g": model.final_g.cpu().numpy(),
         "final_norm.b": model.final_b.cpu().numpy()}
    return t, inv.reshape(ids.shape).astype(np.int64)


def distinct_ids(seed, B, K, V):
    out = np.empty((B, K), np.int32)
    for r in range(B):
        vals = rng.splitmix64(rng.derive(seed, r), 4 * K) % np.uint64(V)
        _, first = np.unique(vals, return_index=True)
        out[r] = vals[np.sort(first)[:K]].astype(np.int32)
    return out


def chain_gpu(model, bank, hidden, ids, thr, layers):
    """The bench's step: one certified FAST launch per layer, prev carried."""
    B, K = ids.shape[1], ids.shape[2]
    prev = torch.full((B, K), float(np.float32(1.0 / K)), device="cuda")
    fired, prob, logits = [], [], []
    with numerics.using("fast"):
        for l in range(layers):
            out = spx.evaluate_batch(model, bank, hidden[l], ids[l], prev, threshold=thr,
                                     layer=l)
            fired.append(out.fired.clone())
            prob.append(out.prob.clone())
            logits.append(out.logits.clone())
            assert out.err.item() == 0
    torch.cuda.synchronize()
    return (torch.stack(fired).cpu().numpy(), torch.stack(prob).cpu().numpy(),
            torch.stack(logits).cpu().numpy())


def chain_oracle(O, t, hid, ids, weights, thr, rows):
    K = ids.shape[2]
    fired = np.zeros((len(weights), len(rows)), bool)
    prob = np.zeros((len(weights), len(rows)))
    for j, r in enumerate(rows):
        prev = O.uniform_probs(K)
        for l, w in enumerate(weights):
            lg = O.sliced_head_logits(t, hid[l, r], ids[l, r])
            fv = O.extract_features(lg, prev)
            p = O.predictor_forward(w, fv)
            fired[l, j], prob[l, j] = p > thr, p
            prev = fv.local_probs
    return fired, prob


@pytest.fixture(scope="module")
def bench_case():
    """configs[1]/bench: 7B head, B=1024, K=4, H=512, 31 layers."""
    V, d, B, K, L = 32000, 4096, 1024, 4, 31
    model = head(V, d)
    gen = torch.Generator(device="cuda").manual_seed(5)
    hidden = torch.randn((L, B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids = np.stack([distinct_ids(rng.derive(9, l), B, K, V) for l in range(L)])
    weights = [spx.init_predictor(K, 512, rng.derive(11, l)) for l in range(L)]
    bank = spx.PredictorBank(dict(enumerate(weights)), L)
    return model, hidden, ids, weights, bank


@pytest.mark.parametrize("thr", [0.5, 0.7])
def test_bench_config_decisions_exact(bench_case, oracle, thr):
    model, hidden, ids, weights, bank = bench_case
    L, B = hidden.shape[0], hidden.shape[1]
    before = spx.recheck_stats()
    f_gpu, p_gpu, _ = chain_gpu(model, bank, hidden, torch.as_tensor(ids, device="cuda"), thr, L)
    after = spx.recheck_stats()
    rows = np.arange(0, B, B // 256)[:256]
    t, oid = oracle_head(model, ids[:, rows])
    hid = hidden[:, rows].cpu().numpy()
    ow = [oracle.PredictorWeights(w.w1, w.b1, w.w2, w.b2) for w in weights]
    f_ref, p_ref = chain_oracle(oracle, t, hid, oid, ow, thr, range(len(rows)))
    mism = int((f_gpu[:, rows].astype(bool) != f_ref).sum())
    assert mism == 0, f"{mism} decision mismatches at thr={thr}"
    assert np.abs(p_gpu[:, rows] - p_ref).max() <= PROB_ATOL
    rechecked = after[0] - before[0]
    print(f"thr={thr}: fire rate {f_gpu.mean():.3f}, rows re-evaluated {rechecked} of {L * B}, "
          f"unresolved {after[1] - before[1]}")


@pytest.mark.parametrize("d", [4096, 8192])
@pytest.mark.parametrize("K", [1, 8, 16, 64])
def test_k_sweep_decisions_exact(oracle, d, K):
    V, B, L = 128000, 96, 3
    model = head(V, d, seed=3)
    gen = torch.Generator(device="cuda").manual_seed(K + d)
    hidden = torch.randn((L, B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids = np.stack([distinct_ids(rng.derive(17 + K, l), B, K, V) for l in range(L)])
    weights = [spx.init_predictor(K, 512, rng.derive(21 + K, l)) for l in range(L)]
    bank = spx.PredictorBank(dict(enumerate(weights)), L)
    f_gpu, p_gpu, _ = chain_gpu(model, bank, hidden, torch.as_tensor(ids, device="cuda"), 0.5, L)
    t, oid = oracle_head(model, ids)
    ow = [oracle.PredictorWeights(w.w1, w.b1, w.w2, w.b2) for w in weights]
    f_ref, p_ref = chain_oracle(oracle, t, hidden.cpu().numpy(), oid, ow, 0.5, range(B))
    assert int((f_gpu.astype(bool) != f_ref).sum()) == 0
    assert np.abs(p_gpu - p_ref).max() <= PROB_ATOL


@pytest.mark.parametrize("K", [4, 16])
def test_forced_recheck_equals_strict(K):
    """Inflate the bound so that no row certifies: every row goes through the
    STRICT re-evaluation, whose outputs must equal the STRICT kernel's."""
    V, d, B, L = 32000, 4096, 200, 3
    model = head(V, d)
    gen = torch.Generator(device="cuda").manual_seed(99)
    hidden = torch.randn((L, B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids = torch.as_tensor(np.stack([distinct_ids(rng.derive(31, l), B, K, V) for l in range(L)]),
                          device="cuda")
    bank = spx.PredictorBank({l: spx.init_predictor(K, 512, rng.derive(41, l)) for l in range(L)}, L)
    kappa = model.cert_kappa
    res = {}
    try:
        for mode in ("strict", "fast"):
            model.cert_kappa = 1e30 if mode == "fast" else kappa
            prev = torch.full((B, K), float(np.float32(1.0 / K)), device="cuda")
            outs = []
            with numerics.using(mode):
                for l in range(L):
                    o = spx.evaluate_batch(model, bank, hidden[l], ids[l], prev, threshold=0.5,
                                           layer=l)
                    outs.append((o.fired.clone(), o.z.clone(), o.logits.clone()))
            torch.cuda.synchronize()
            res[mode] = (outs, prev.clone(), spx.prev_error(prev).clone())
    finally:
        model.cert_kappa = kappa
    for (fs, zs, ls), (ff, zf, lf) in zip(res["strict"][0], res["fast"][0]):
        assert torch.equal(fs, ff)
        assert torch.equal(zs.view(torch.int32), zf.view(torch.int32))
        assert torch.equal(ls.view(torch.int32), lf.view(torch.int32))
    assert torch.equal(res["strict"][1].view(torch.int32), res["fast"][1].view(torch.int32))
    assert float(res["fast"][2].abs().max()) == 0.0        # STRICT probabilities carried


def test_prev_error_bound_holds():
    """The carried bound prev_err covers the actual |prev_fast - prev_strict|."""
    V, d, B, K = 32000, 4096, 512, 4
    model = head(V, d)
    gen = torch.Generator(device="cuda").manual_seed(7)
    hidden = torch.randn((B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids = torch.as_tensor(distinct_ids(77, B, K, V), device="cuda")
    w = spx.init_predictor(K, 512, 5)
    got = {}
    for mode in ("strict", "fast"):
        prev = torch.full((B, K), 0.25, device="cuda")
        with numerics.using(mode):
            spx.evaluate_batch(model, w, hidden, ids, prev, threshold=0.7)
        torch.cuda.synchronize()
        got[mode] = (prev.clone(), spx.prev_error(prev).clone())
    diff = (got["fast"][0] - got["strict"][0]).abs().max(dim=1).values
    bound = got["fast"][1]
    assert bool((diff <= bound).all())
    assert float(bound.max()) < 1e-2
