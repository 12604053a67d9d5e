"""K4 on the tensor cores (csrc/spx_verify_tc.cuh) against the CUDA-core
verify_kernel, which the parity tests pin to the oracle: for many gated rows
the tensor-core form must give bit-identical argmax tokens, max logits,
membership flags, exit flags / layers and full-head counters -- no tolerance,
including exact ties (duplicated LM-head rows: lowest index wins, engine.py:62)
and rows whose top two logits are closer than the tensor-core rounding.
Reference: verify_exit (engine.py:59-64), full_head_logits (model.py:289-295)."""
import numpy as np
import pytest
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import _native as N
from paper_2504_08850_b200 import numerics
from paper_2504_08850_b200.model import _VerifyScratch, launch_verify, verify_args

pytestmark = pytest.mark.gpu

_HEADS = {}


def _head(V, d, seed):
    key = (V, d, seed)
    if key not in _HEADS:
        _HEADS[key] = spx.init_model(spx.ModelConfig(V, d, 1, 8, 64, 16, seed), dtype="bf16",
                                     head_only=True)
    return _HEADS[key]


def _run(m, h, gate, done, spec_ptr, spec_ids, tc, layer=7):
    B = h.shape[0]
    out = {k: torch.full((B,), -1, dtype=torch.int32, device="cuda") for k in ("tok", "exit")}
    out["ver"] = torch.zeros(B, dtype=torch.uint8, device="cuda")
    out["mx"] = torch.zeros(B, dtype=torch.float32, device="cuda")
    out["done"] = done.clone()
    out["heads"] = torch.zeros(B, dtype=torch.int32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch, counter = _VerifyScratch.get(B)
    a = verify_args(m, h, B, out["tok"], scratch, counter, err, gate=gate, row_done=done,
                    spec_ptr=spec_ptr, spec_ids=spec_ids, verified_out=out["ver"],
                    maxlogit_out=out["mx"], done_out=out["done"], exit_layer_out=out["exit"],
                    full_heads=out["heads"], layer=layer, tensor_cores=tc,
                    mode=N.SPX_MODE_FAST)
    assert bool(a.tc_scratch) == tc
    launch_verify(a)
    torch.cuda.synchronize()
    assert err.item() == 0
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("V,d,B", [(32000, 4096, 8), (32000, 4096, 64), (32000, 5120, 37),
                                   (32000, 5120, 200), (4096, 8192, 130)])
def test_verify_tc_bit_identical_to_cuda_cores(V, d, B):
    m = _head(V, d, 11)
    g = torch.Generator(device="cuda").manual_seed(V + d + B)
    h = torch.randn((B, d), device="cuda", generator=g) * 3 + 0.5
    gate = (torch.rand(B, device="cuda", generator=g) < 0.7).to(torch.uint8)
    done = (torch.rand(B, device="cuda", generator=g) < 0.15).to(torch.uint8)
    # verify sets: 4 ids per row, one of them the row's true argmax half the time
    ref_tok = spx.head_argmax(m, h)[0].cpu().numpy()
    rs = np.random.default_rng(B)
    ids = rs.integers(0, V, size=(B, 4)).astype(np.int32)
    ids[::2, 0] = ref_tok[::2]
    sp = torch.as_tensor(np.arange(0, 4 * B + 1, 4, dtype=np.int32), device="cuda")
    si = torch.as_tensor(ids.reshape(-1), device="cuda")
    with numerics.using("fast"):
        a = _run(m, h, gate, done, sp, si, tc=False)
        b = _run(m, h, gate, done, sp, si, tc=True)
    on = (gate.cpu().numpy() != 0) & (done.cpu().numpy() == 0)
    assert on.sum() > 0
    for k in a:
        assert np.array_equal(a[k], b[k]), (k, np.nonzero(a[k] != b[k]))
    assert np.array_equal(a["tok"][on], ref_tok[on])
    assert (a["heads"][~on] == 0).all() and (a["heads"][on] == 1).all()
    assert a["ver"][on].sum() > 0


def test_verify_tc_exact_ties_and_near_ties():
    """Duplicated head rows tie exactly (lowest index must win); rows built so
    that their top logits differ by less than the tensor-core rounding."""
    V, d, B = 8192, 4096, 48
    m = spx.init_model(spx.ModelConfig(V, d, 1, 8, 64, 16, 5), dtype="bf16", head_only=True)
    src = torch.arange(0, 64, device="cuda")
    m.lm_head[V - 64:] = m.lm_head[src]            # rows V-64.. duplicate rows 0..63
    m.finalize()
    # hidden rows aligned with head rows 0..B-1: their logit is the max, tied
    # with the duplicate at V-64+i (lowest index = i must win)
    h = m.lm_head[:B].float() * 40 + 0.01 * torch.randn((B, d), device="cuda")
    gate = torch.ones(B, dtype=torch.uint8, device="cuda")
    done = torch.zeros(B, dtype=torch.uint8, device="cuda")
    sp = torch.as_tensor(np.arange(0, B + 1, dtype=np.int32), device="cuda")
    si = torch.as_tensor(np.arange(B, dtype=np.int32), device="cuda")
    with numerics.using("fast"):
        a = _run(m, h, gate, done, sp, si, tc=False)
        b = _run(m, h, gate, done, sp, si, tc=True)
    for k in a:
        assert np.array_equal(a[k], b[k]), k
    assert (a["tok"] == np.arange(B)).all() and (a["ver"] == 1).all()


@pytest.mark.parametrize("V,d,B,K", [(32000, 5120, 64, 4), (32000, 4096, 16, 16),
                                     (8192, 4096, 24, 64)])
def test_verify_tc_topk_equals_full_logits_topk(V, d, B, K):
    """The draft proposal's top-K from K4's tensor-core form equals the stable
    top-K (speculation.py:57-60) of the CUDA-core full logits, id for id."""
    m = _head(V, d, 3)
    g = torch.Generator(device="cuda").manual_seed(B * K)
    h = torch.randn((B, d), device="cuda", generator=g)
    if K == 64:                                   # exact ties inside the top-K
        m = spx.init_model(spx.ModelConfig(V, d, 1, 8, 64, 16, 9), dtype="bf16", head_only=True)
        m.lm_head[V - 64:] = m.lm_head[:64]
        m.finalize()
        h = m.lm_head[:B].float() * 30 + 0.01 * torch.randn((B, d), device="cuda", generator=g)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch, counter = _VerifyScratch.get(B)
    logits = torch.empty((B, V), dtype=torch.float32, device="cuda")
    tok_a = torch.empty(B, dtype=torch.int32, device="cuda")
    tok_b = torch.empty(B, dtype=torch.int32, device="cuda")
    ids_a = torch.empty((B, K), dtype=torch.int32, device="cuda")
    ids_b = torch.full((B, K), -1, dtype=torch.int32, device="cuda")
    with numerics.using("fast"):
        launch_verify(verify_args(m, h, B, tok_a, scratch, counter, err, logits_out=logits))
        N.check(N.lib().spx_topk_rows(N.ptr(logits), B, V, K, N.ptr(ids_a), N.stream_ptr()),
                "spx_topk_rows")
        a = verify_args(m, h, B, tok_b, scratch, counter, err, topk_out=ids_b, topk_k=K)
        assert a.tc_scratch
        launch_verify(a)
    torch.cuda.synchronize()
    assert err.item() == 0
    ia, ib = ids_a.cpu().numpy(), ids_b.cpu().numpy()
    assert np.array_equal(ia, ib)
    assert np.array_equal(tok_a.cpu().numpy(), tok_b.cpu().numpy())
    assert np.array_equal(ia[:, 0], tok_b.cpu().numpy())
    ref = np.argsort(-logits.cpu().numpy(), axis=1, kind="stable")[:, :K]
    assert np.array_equal(ref, ia)
