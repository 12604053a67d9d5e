"""GPU label collection and offline profiling -- drop-in for
the reference's ``collect_training_data`` (src/specexit/predictor.py:219-275)
and the counting run behind ``profile_offline`` (src/specexit/scheduler.py:
105-121, driven by pipeline.py:168-191).

Label collection reuses the hot-path kernels with exits disabled:

  per generated token (enqueued, no host sync):
    draft: embed -> Ld layers -> full head (K4, logits) -> stable top-K (spx_topk)
    target: embed -> every layer l, its hidden row copied to H[t, l]
    final argmax (K4) of H[t, L-1] -> next input token (device)
  after all prompts, batched over the T = num_prompts * max_new tokens:
    features: ONE K1-K3 launch per layer over T rows (constant policy, features
              written out, ``prev`` carried per row from layer to layer exactly
              as predictor.py:233-236 does)
    labels:   ONE K4 launch per requested layer over T rows (argmax at layer l
              == final argmax, predictor.py:237-238)

so the per-(token, layer) reference work -- a full 262 MB head GEMV per label
and a sliced gather per feature vector -- becomes L + |layers| batched
launches.  Offline profiling runs the device-resident ExitEngine (schedule
"all", the trained predictors) per prompt and histograms the exit layers on
the device; the counts come back once.
"""
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .decode import DecodeState
from .engine import EngineConfig, ExitEngine, PredictorPolicy
from .model import TransformerModel, _VerifyScratch, launch_verify, verify_args
from .predictor import evaluate_batch, prev_error
from .rng import splitmix64
from .scheduler import OfflineProfile


@dataclass
class TrainingExample:
    """predictor.py:112-116."""
    features: np.ndarray   # concatenated 3k vector
    label: bool            # early argmax at `layer` matches final argmax
    layer: int


def _prompt_starts(data, num_prompts, prompt_len, seed):
    """predictor.py:247-250 (note: max(size - prompt_len, 1), unlike
    pipeline.corpus_prompts)."""
    if data.size < prompt_len:
        raise ValueError("corpus shorter than prompt length")
    return splitmix64(seed, num_prompts) % np.uint64(max(data.size - prompt_len, 1))


class LayerTraces:
    """Device tensors of a batch of greedy generations: per token t the draft
    speculative ids spec[t] (K), every target layer's hidden row H[t, l] and
    the final argmax final[t]."""

    def __init__(self, spec, hidden, final):
        self.spec, self.hidden, self.final = spec, hidden, final


def generation_layer_traces(target: TransformerModel, draft: TransformerModel, corpus: bytes,
                            k: int, num_prompts: int, prompt_len: int, max_new: int,
                            seed: int) -> LayerTraces:
    """predictor.py:244-275 on the device (no host sync inside the loops)."""
    data = np.frombuffer(corpus, dtype=np.uint8)
    starts = _prompt_starts(data, num_prompts, prompt_len, seed)
    tc, dc = target.config, draft.config
    if prompt_len - 1 + max_new > min(tc.max_context, dc.max_context):
        raise ValueError("context overflow")
    if not 1 <= k <= min(64, dc.vocab_size):
        raise ValueError("k out of range")
    L, d, T = tc.num_layers, tc.hidden_dim, num_prompts * max_new
    lib = N.lib()
    spec = torch.zeros((T, k), dtype=torch.int32, device="cuda")
    hidden = torch.zeros((T, L, d), dtype=torch.float32, device="cuda")
    final = torch.zeros(T, dtype=torch.int32, device="cuda")
    dlogits = torch.zeros(dc.vocab_size, dtype=torch.float32, device="cuda")
    dtok = torch.zeros(1, dtype=torch.int32, device="cuda")
    nxt = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch, counter = _VerifyScratch.get(1)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    ts, ds = DecodeState(target), DecodeState(draft)
    for p, s in enumerate(starts):
        prompt = [int(b) for b in data[int(s):int(s) + prompt_len]]
        ts.reset()
        ds.reset()
        if len(prompt) > 1:
            for st, m in ((ts, target), (ds, draft)):
                st.begin(prompt[:-1])
                for l in range(m.config.num_layers):
                    st.launch_layer(l)
        nxt.fill_(prompt[-1])
        for i in range(max_new):
            t = p * max_new + i
            ds.embed_device(nxt, 1)
            for l in range(dc.num_layers):
                ds.launch_layer(l)
            launch_verify(verify_args(draft, ds.cur_hidden, 1, dtok, scratch, counter, err,
                                      logits_out=dlogits))
            N.check(lib.spx_topk(N.ptr(dlogits), dc.vocab_size, k, N._vp(spec[t].data_ptr()),
                                 N.stream_ptr()), "spx_topk")
            ts.embed_device(nxt, 1)
            for l in range(L):
                ts.launch_layer(l)
                hidden[t, l].copy_(ts.cur_hidden)
            launch_verify(verify_args(target, ts.cur_hidden, 1, final[t:t + 1], scratch, counter,
                                      err))
            nxt.copy_(final[t:t + 1])
            ts.n += 1
            ds.n += 1
    torch.cuda.synchronize()
    N.raise_device_error(int(err.item()) | int(ts.err.item()) | int(ds.err.item()))
    return LayerTraces(spec, hidden, final)


def layer_features_and_labels(target: TransformerModel, tr: LayerTraces, layers):
    """Features of every (token, layer) and labels of the requested layers:
    L feature launches + |layers| argmax launches over all T tokens.
    Returns (features (L, T, 3K) f32, labels {layer: (T,) bool}) on device."""
    T, L, d = tr.hidden.shape
    K = tr.spec.shape[1]
    feats = torch.empty((L, T, 3 * K), dtype=torch.float32, device="cuda")
    prev = torch.full((T, K), float(np.float32(1.0 / K)), dtype=torch.float32, device="cuda")
    prev_error(prev).zero_()
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    for l in range(L):
        # constant policy: features only (predictor.py:233-235; prev carried)
        out = evaluate_batch(target, None, tr.hidden[:, l], tr.spec, prev, layer=l,
                             outputs=False, policy=0.0, err=err, certify=False,
                             feat_out=feats[l])
        del out
    labels = {}
    toks = torch.empty(T, dtype=torch.int32, device="cuda")
    scratch, counter = _VerifyScratch.get(T)
    for l in layers:
        launch_verify(verify_args(target, tr.hidden[:, l], T, toks, scratch, counter, err))
        labels[l] = toks == tr.final
    torch.cuda.synchronize()
    N.raise_device_error(int(err.item()))
    return feats, labels


def collect_training_data(target: TransformerModel, draft: TransformerModel, corpus: bytes,
                          layers, k: int = 4, num_prompts: int = 8, prompt_len: int = 16,
                          max_new: int = 32, seed: int = 0):
    """predictor.py:219-241: greedy-generate from corpus prompts and record,
    per generated token and requested layer, the exit features and whether
    the layer's early argmax already matches the final argmax.  Same example
    order as the reference (prompt, token, layer ascending)."""
    if not corpus:
        raise ValueError("empty corpus")
    layers = sorted(int(l) for l in layers)
    L = target.config.num_layers
    if any(not 0 <= l < L for l in layers):
        raise ValueError("layer index out of range")
    tr = generation_layer_traces(target, draft, corpus, k, num_prompts, prompt_len, max_new, seed)
    feats, labels = layer_features_and_labels(target, tr, layers)
    T = tr.hidden.shape[0]
    if not layers:
        return []
    f = feats[layers].permute(1, 0, 2).cpu().numpy()               # (T, |layers|, 3K)
    lab = torch.stack([labels[l] for l in layers], 1).cpu().numpy()  # (T, |layers|)
    out = []
    for t in range(T):
        for j, l in enumerate(layers):
            out.append(TrainingExample(features=f[t, j].copy(), label=bool(lab[t, j]), layer=l))
    return out


def profile_offline_device(target: TransformerModel, draft: TransformerModel, bank: dict,
                           prompts, max_new: int, num_layers: int = None, fingerprint: int = 0,
                           k: int = 4, threshold: float = 0.5) -> OfflineProfile:
    """scheduler.py:105-121 with the engine of pipeline.py:178-186 (schedule
    "all", every predictor active): per prompt the device-resident token graph
    is replayed max_new times and its exit layers are histogrammed on the
    device; one host read at the end.  Tokens that never exit count at L-1."""
    L = target.config.num_layers if num_layers is None else num_layers
    eng = ExitEngine(target, draft, PredictorPolicy(bank),
                     EngineConfig(k=k, threshold=threshold, schedule_mode="all"))
    if not eng.device_resident():
        raise ValueError("profile_offline_device needs a predictor for every layer 0..L-2")
    if max_new < 1:
        raise ValueError("max_new must be >= 1")
    counts = torch.zeros(L, dtype=torch.int64, device="cuda")
    n_tok = 0
    for prompt in prompts:
        eng.start(prompt)
        eng.replay_device(max_new)
        counts += torch.bincount(eng._dev.rec_exit_layer[:max_new].long(), minlength=L)[:L]
        n_tok += max_new
    if n_tok == 0:
        raise ValueError("profiling produced no tokens (empty corpus?)")
    eng.sync_device()
    return OfflineProfile(num_layers=L, exit_counts=counts.cpu().numpy().astype(np.uint64),
                          fingerprint=fingerprint)
