"""The SPLIT predictor path (spx_predictor_gather + spx_predictor_tail,
csrc/spx_pred_split.cu) against the fused launch (spx_predictor_eval) and the
oracle: same arithmetic, so every output is compared BIT FOR BIT with the
fused FAST kernel over chained layers (prev carried), with skipped rows,
with the tail on a second stream, and with the STRICT re-evaluation forced
for every row; decisions against the oracle's reference chain on a sample.
"""
import numpy as np
import pytest
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import numerics, rng
from test_gpu_certify import chain_oracle, distinct_ids, head, oracle_head

pytestmark = pytest.mark.gpu


def _run(model, bank, hidden, ids, thr, split, tail_stream=None, row_done=None, mask=None,
         policy=None):
    L, B, K = ids.shape
    prev = torch.full((B, K), float(np.float32(1.0 / K)), device="cuda")
    prev_err = spx.prev_error(prev)
    prev_err.zero_()
    inter = torch.zeros((L, B, 2 * K + 2), dtype=torch.float32, device="cuda")
    evals = torch.zeros(B, dtype=torch.int32, device="cuda")
    res = []
    with numerics.using("fast"):
        for l in range(L):
            kw = dict(threshold=thr, layer=l, row_done=row_done, row_layer_mask=mask, evals=evals,
                      policy=policy)
            if split:
                o = spx.evaluate_batch_split(model, bank, hidden[l], ids[l], prev, inter[l],
                                             tail_stream=tail_stream, **kw)
            else:
                o = spx.evaluate_batch(model, bank, hidden[l], ids[l], prev, **kw)
            if tail_stream is not None:
                torch.cuda.current_stream().wait_stream(tail_stream)
            res.append([o.fired.clone(), o.z.clone(), o.prob.clone(), o.logits.clone(),
                        prev.clone(), prev_err.clone(), o.err.clone()])
    torch.cuda.synchronize()
    res.append([evals.clone()])
    return res


def _same(a, b):
    for ra, rb in zip(a, b):
        for x, y in zip(ra, rb):
            assert torch.equal(x.view(torch.uint8), y.view(torch.uint8))


@pytest.mark.parametrize("d,K,B", [(4096, 4, 1024), (4096, 4, 37), (2048, 8, 300),
                                   (8192, 4, 600), (4096, 1, 500), (4096, 2, 2000)])
def test_split_equals_fused(d, K, B):
    V, L = 32000, 3
    model = head(V, d)
    gen = torch.Generator(device="cuda").manual_seed(d + K + B)
    hidden = torch.randn((L, B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids = torch.as_tensor(np.stack([distinct_ids(rng.derive(3 + K, l), B, K, V)
                                    for l in range(L)]), device="cuda")
    bank = spx.PredictorBank({l: spx.init_predictor(K, 512, rng.derive(7, l)) for l in range(L)}, L)
    assert spx.predictor.split_supported(model, bank, hidden[0], ids[0],
                                         torch.zeros((B, K), device="cuda"))
    for thr in (0.5, 0.7):
        a = _run(model, bank, hidden, ids, thr, split=False)
        b = _run(model, bank, hidden, ids, thr, split=True)
        _same(a, b)
    side = torch.cuda.Stream()
    c = _run(model, bank, hidden, ids, 0.5, split=True, tail_stream=side)
    _same(_run(model, bank, hidden, ids, 0.5, split=False), c)


def test_split_skipped_rows_and_constant_policy():
    V, d, K, B, L = 32000, 4096, 4, 700, 3
    model = head(V, d)
    gen = torch.Generator(device="cuda").manual_seed(1)
    hidden = torch.randn((L, B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids = torch.as_tensor(np.stack([distinct_ids(rng.derive(5, l), B, K, V) for l in range(L)]),
                          device="cuda")
    bank = spx.PredictorBank({l: spx.init_predictor(K, 512, rng.derive(8, l)) for l in range(L)}, L)
    r = np.random.default_rng(0)
    done = torch.as_tensor((r.random(B) < 0.3).astype(np.uint8), device="cuda")
    mask = torch.as_tensor(r.integers(0, 8, B).astype(np.int64), device="cuda")
    for kw in (dict(row_done=done), dict(mask=mask), dict(row_done=done, mask=mask),
               dict(policy=1.0)):
        a = _run(model, bank, hidden, ids, 0.5, split=False, **kw)
        b = _run(model, bank, hidden, ids, 0.5, split=True, **kw)
        skipped = torch.zeros(B, dtype=torch.bool, device="cuda")
        if "row_done" in kw:
            skipped |= kw["row_done"].bool()
        # fired / prev / prev_err / evals are defined for every row; z, prob and
        # logits only for evaluated rows
        for l in range(L):
            live = ~skipped
            if "mask" in kw:
                live &= ((kw["mask"] >> l) & 1).bool()
            for j in (0, 4, 5):
                assert torch.equal(a[l][j].view(torch.uint8), b[l][j].view(torch.uint8))
            for j in (1, 2, 3):
                assert torch.equal(a[l][j][live].view(torch.uint8), b[l][j][live].view(torch.uint8))
        assert torch.equal(a[-1][0], b[-1][0])


def test_split_forced_recheck_equals_fused():
    """Bound inflated: every row takes the STRICT re-evaluation in the tail
    kernel's epilogue -- outputs equal the fused kernel's (which equal the
    STRICT kernel's, test_gpu_certify)."""
    V, d, K, B, L = 32000, 4096, 4, 150, 2
    model = head(V, d)
    gen = torch.Generator(device="cuda").manual_seed(2)
    hidden = torch.randn((L, B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids = torch.as_tensor(np.stack([distinct_ids(rng.derive(6, l), B, K, V) for l in range(L)]),
                          device="cuda")
    bank = spx.PredictorBank({l: spx.init_predictor(K, 512, rng.derive(9, l)) for l in range(L)}, L)
    kappa = model.cert_kappa
    try:
        model.cert_kappa = 1e30
        before = spx.recheck_stats()
        a = _run(model, bank, hidden, ids, 0.5, split=False)
        mid = spx.recheck_stats()
        b = _run(model, bank, hidden, ids, 0.5, split=True)
        after = spx.recheck_stats()
    finally:
        model.cert_kappa = kappa
    assert mid[0] - before[0] == after[0] - mid[0] == L * B
    _same(a, b)


def test_split_bench_shape_decisions_match_oracle(oracle):
    """The bench shape (7B head, B=1024, K=4, H=512) through the split path:
    decisions of a 128-row sample over 8 chained layers equal the oracle's."""
    V, d, K, B, L = 32000, 4096, 4, 1024, 8
    model = head(V, d)
    gen = torch.Generator(device="cuda").manual_seed(12)
    hidden = torch.randn((L, B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids_np = np.stack([distinct_ids(rng.derive(13, l), B, K, V) for l in range(L)])
    ids = torch.as_tensor(ids_np, device="cuda")
    weights = [spx.init_predictor(K, 512, rng.derive(14, l)) for l in range(L)]
    bank = spx.PredictorBank(dict(enumerate(weights)), L)
    side = torch.cuda.Stream()
    res = _run(model, bank, hidden, ids, 0.5, split=True, tail_stream=side)
    fired = torch.stack([r[0] for r in res[:L]]).cpu().numpy()
    prob = torch.stack([r[2] for r in res[:L]]).cpu().numpy()
    rows = np.arange(0, B, 8)
    t, inv = oracle_head(model, ids_np[:, rows])
    hid = hidden[:, rows].cpu().numpy()
    ow = [oracle.PredictorWeights(w.w1, w.b1, w.w2, w.b2) for w in weights]
    f_ref, p_ref = chain_oracle(oracle, t, hid, inv, ow, 0.5, np.arange(rows.size))
    assert np.array_equal(fired[:, rows].astype(bool), f_ref)
    assert np.abs(prob[:, rows] - p_ref).max() <= 1e-3


def _run_chain(model, bank, hidden, ids, thr, row_done=None, mask=None, policy=None):
    L, B, K = ids.shape
    prev = torch.full((B, K), float(np.float32(1.0 / K)), device="cuda")
    prev_err = spx.prev_error(prev)
    prev_err.zero_()
    inter = torch.zeros((L, B, 2 * K + 2), dtype=torch.float32, device="cuda")
    evals = torch.zeros(B, dtype=torch.int32, device="cuda")
    outs = []
    for l in range(L):
        o = spx.predictor.BatchResult(
            logits=torch.empty((B, K), device="cuda"), z=torch.empty(B, device="cuda"),
            prob=torch.empty(B, dtype=torch.float64, device="cuda"),
            fired=torch.empty(B, dtype=torch.uint8, device="cuda"),
            err=torch.zeros(1, dtype=torch.int32, device="cuda"))
        outs.append(o)
    with numerics.using("fast"):
        # the chain API has no per-layer snapshots of prev: compare the final
        # prev / prev_err and every layer's outputs
        spx.evaluate_chain(model, bank, hidden, ids, prev, inter, list(range(L)), threshold=thr,
                           outs=outs, policy=policy)
    torch.cuda.synchronize()
    return [[o.fired, o.z, o.prob, o.logits, o.err] for o in outs], prev, prev_err


@pytest.mark.parametrize("d,K,B", [(4096, 4, 1024), (4096, 4, 45), (2048, 8, 300),
                                   (8192, 4, 600), (4096, 2, 1500)])
def test_chain_equals_fused(d, K, B):
    """The pipelined chain (gather(l) + tail(l-1) per launch) vs one fused
    launch per layer: every output bit-identical."""
    V, L = 32000, 5
    model = head(V, d)
    gen = torch.Generator(device="cuda").manual_seed(d + 3 * K + B)
    hidden = torch.randn((L, B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids = torch.as_tensor(np.stack([distinct_ids(rng.derive(17 + K, l), B, K, V)
                                    for l in range(L)]), device="cuda")
    bank = spx.PredictorBank({l: spx.init_predictor(K, 512, rng.derive(19, l)) for l in range(L)}, L)
    for thr in (0.5, 0.7):
        a = _run(model, bank, hidden, ids, thr, split=False)
        b, prev, prev_err = _run_chain(model, bank, hidden, ids, thr)
        for l in range(L):
            for x, y in zip([a[l][0], a[l][1], a[l][2], a[l][3], a[l][6]], b[l]):
                assert torch.equal(x.view(torch.uint8), y.view(torch.uint8)), l
        assert torch.equal(a[L - 1][4].view(torch.uint8), prev.view(torch.uint8))
        assert torch.equal(a[L - 1][5].view(torch.uint8), prev_err.view(torch.uint8))


def test_chain_forced_recheck_equals_fused():
    """Bound inflated: every tail row is re-evaluated by the STRICT chain in
    the tail warps' epilogue (and in the final tail launch)."""
    V, d, K, B, L = 32000, 4096, 4, 150, 3
    model = head(V, d)
    gen = torch.Generator(device="cuda").manual_seed(21)
    hidden = torch.randn((L, B, d), device="cuda", generator=gen).to(torch.bfloat16).float()
    ids = torch.as_tensor(np.stack([distinct_ids(rng.derive(22, l), B, K, V) for l in range(L)]),
                          device="cuda")
    bank = spx.PredictorBank({l: spx.init_predictor(K, 512, rng.derive(23, l)) for l in range(L)}, L)
    kappa = model.cert_kappa
    try:
        model.cert_kappa = 1e30
        a = _run(model, bank, hidden, ids, 0.5, split=False)
        b0 = spx.recheck_stats()
        b, prev, _ = _run_chain(model, bank, hidden, ids, 0.5)
        b1 = spx.recheck_stats()
    finally:
        model.cert_kappa = kappa
    assert b1[0] - b0[0] == L * B
    for l in range(L):
        for x, y in zip([a[l][0], a[l][1], a[l][2], a[l][3]], b[l]):
            assert torch.equal(x.view(torch.uint8), y.view(torch.uint8)), l
    assert torch.equal(a[L - 1][4].view(torch.uint8), prev.view(torch.uint8))
