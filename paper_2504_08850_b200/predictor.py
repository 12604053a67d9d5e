"""Exit features and the per-layer MLP exit predictor -- drop-in for the
reference's ``specexit.predictor`` (src/specexit/predictor.py), evaluated by
the sm_100a kernels of libspecexit_b200.so.

Same names, signatures and error behaviour as the reference:
``FeatureVector``, ``uniform_probs``, ``extract_features``,
``PredictorWeights``, ``init_predictor``, ``predictor_forward``,
``decide_exit``, ``predictor_param_count``, ``save_predictors`` /
``load_predictors`` (SPXP).  Arrays may be numpy arrays or torch tensors;
returned arrays are torch CUDA tensors.

``PredictorBank`` packs a ``{layer: PredictorWeights}`` dict into one device
buffer per field (the layout the fused kernel reads), and ``z_cut`` turns the
reference's float64 ``sigmoid(z) > threshold`` into the equivalent exact f32
comparison ``z >= z_cut`` evaluated in-kernel.
"""
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import numerics, rng


def _dev(x, dtype=torch.float32):
    if isinstance(x, torch.Tensor):
        return x.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device="cuda")


@dataclass(frozen=True)
class FeatureVector:
    """predictor.py:22-33: [spec_logits | local_probs | prob_variation]."""
    spec_logits: torch.Tensor
    local_probs: torch.Tensor
    prob_variation: torch.Tensor

    @property
    def k(self):
        return int(self.spec_logits.numel())

    def concat(self) -> torch.Tensor:
        return torch.cat([self.spec_logits, self.local_probs, self.prob_variation]).float()


def uniform_probs(k: int) -> torch.Tensor:
    """predictor.py:36-39."""
    return torch.full((k,), np.float32(1.0 / k).item(), dtype=torch.float32, device="cuda")


def extract_features(spec_logits, prev_local_probs) -> FeatureVector:
    """predictor.py:42-52 on device (spx_extract_features)."""
    N.require_cuda()
    lg = _dev(spec_logits).reshape(-1)
    pv = _dev(prev_local_probs).reshape(-1)
    if lg.numel() < 1 or tuple(np.shape(spec_logits)) != tuple(np.shape(prev_local_probs)):
        raise ValueError("bad feature input shapes")
    k = lg.numel()
    out = torch.empty(3 * k, dtype=torch.float32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().spx_extract_features(N.ptr(lg), N.ptr(pv), N.ptr(out), N.ptr(err), 1, k,
                                         N.stream_ptr()), "spx_extract_features")
    N.raise_device_error(err.item())
    return FeatureVector(spec_logits=lg, local_probs=out[k:2 * k], prob_variation=out[2 * k:])


@dataclass
class PredictorWeights:
    """predictor.py:55-75 (host arrays; validated like the reference)."""
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: float
    threshold: float = 0.5

    def __post_init__(self):
        if self.w1.shape[1] != np.size(self.b1) or self.w1.shape[1] != np.size(self.w2):
            raise ValueError("predictor weight shapes inconsistent")
        if not 0.0 < self.threshold < 1.0:
            raise ValueError("threshold must lie in (0, 1)")

    @property
    def k(self):
        return self.w1.shape[0] // 3

    @property
    def hidden(self):
        return self.w1.shape[1]


def init_predictor(k: int, hidden: int, seed: int, threshold: float = 0.5) -> PredictorWeights:
    """predictor.py:78-84 (same seeded values)."""
    d = 3 * k
    b = np.sqrt(6.0 / (d + hidden))
    w1 = rng.uniform(rng.derive(seed, 0), d * hidden, -b, b).reshape(d, hidden)
    b2 = np.sqrt(6.0 / (hidden + 1))
    w2 = rng.uniform(rng.derive(seed, 1), hidden, -b2, b2)
    return PredictorWeights(w1=w1, b1=np.zeros(hidden, np.float32), w2=w2, b2=0.0,
                            threshold=threshold)


def _sigmoid64(z):
    """predictor.py:87-94 (float64), host side, for the cut search."""
    z = np.asarray(z, dtype=np.float64)
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out


def _ord_to_f32(o):
    o = np.asarray(o, dtype=np.int64)
    bits = np.where(o >= 0, o, (-o) | 0x80000000).astype(np.uint32)
    return bits.view(np.float32)


_ZCUT_CACHE = {}


def z_cut(threshold: float) -> float:
    """Smallest float32 z with sigmoid(float64(z)) > threshold (the reference's
    decision, predictor.py:87-109, is monotone in the f32 logit, so
    ``prob > threshold`` == ``z >= z_cut``).  +inf/NaN edge cases: never fires
    returns NaN; always fires returns -inf."""
    thr = float(threshold)
    if thr in _ZCUT_CACHE:
        return _ZCUT_CACHE[thr]
    lo, hi = -0x7F800000, 0x7F800000        # ordered ints of -inf, +inf
    fires = lambda o: bool(_sigmoid64(_ord_to_f32(o).astype(np.float64)) > thr)  # noqa: E731
    if not fires(hi):
        cut = float("nan")
    elif fires(lo):
        cut = float("-inf")
    else:
        while hi - lo > 1:                  # invariant: !fires(lo), fires(hi)
            mid = (lo + hi) // 2
            if fires(mid):
                hi = mid
            else:
                lo = mid
        cut = float(_ord_to_f32(hi))
    _ZCUT_CACHE[thr] = cut
    return cut


def predictor_forward(w: PredictorWeights, features) -> float:
    """predictor.py:97-103 on device (spx_predictor_mlp); returns the float64
    probability as a Python float."""
    N.require_cuda()
    f = features.concat() if isinstance(features, FeatureVector) else _dev(features).reshape(-1)
    if tuple(f.shape) != (w.w1.shape[0],):
        raise ValueError(f"feature dimension {tuple(f.shape)} does not match predictor {w.w1.shape}")
    k, H = w.k, w.hidden
    dw = _DeviceWeights.of(w)
    prob = torch.empty(1, dtype=torch.float64, device="cuda")
    N.check(N.lib().spx_predictor_mlp(N.ptr(f.contiguous()), N.ptr(dw.w1), N.ptr(dw.b1),
                                      N.ptr(dw.w2), float(np.float32(w.b2)), float("nan"), None,
                                      N.ptr(prob), None, 1, k, H, N.stream_ptr()),
            "spx_predictor_mlp")
    return float(prob.item())


def decide_exit(prob: float, threshold: float) -> bool:
    """predictor.py:106-109 (strict >)."""
    return prob > threshold


def predictor_param_count(k: int, hidden: int, num_layers: int):
    """predictor.py:204-213: (4, 512, 32) -> (212992, 416.0)."""
    if min(k, hidden, num_layers) < 1:
        raise ValueError("arguments must be positive")
    per_layer = 3 * k * hidden + hidden
    return per_layer * num_layers, per_layer * num_layers * 2 / 1024


def _cert(w1, b1, w2, k, hidden):
    """Per-layer constants of the FAST-decision certification bound
    (spx_predictor_cert): M_i = sum_j |w2_j||W1_ij|, sum_j |w2_j b1_j|, sum |w2|."""
    out = torch.empty(3 * k + 2, dtype=torch.float32, device="cuda")
    N.check(N.lib().spx_predictor_cert(N.ptr(w1), N.ptr(b1), N.ptr(w2), k, hidden, N.ptr(out),
                                       N.stream_ptr()), "spx_predictor_cert")
    return out


class _DeviceWeights:
    """One PredictorWeights on device (cached per object identity)."""
    _cache = {}

    def __init__(self, w):
        self.w1 = _dev(np.asarray(w.w1, np.float32))
        self.b1 = _dev(np.asarray(w.b1, np.float32))
        self.w2 = _dev(np.asarray(w.w2, np.float32))
        self.cert = _cert(self.w1, self.b1, self.w2, w.k, w.hidden)

    @classmethod
    def of(cls, w):
        key = id(w)
        ent = cls._cache.get(key)
        if ent is None or ent[0] is not w:
            ent = (w, cls(w))
            cls._cache[key] = ent
        return ent[1]


class PredictorBank:
    """Device-packed per-layer predictors: w1 (L, 3K, H), b1 (L, H), w2 (L, H),
    b2 (L,) f32, plus the set of covered layers (PredictorPolicy raises
    KeyError for an active layer without a predictor, engine.py:90-91)."""

    def __init__(self, bank: dict, num_layers: int):
        if not bank:
            raise ValueError("empty predictor bank")
        ks = {w.k for w in bank.values()}
        hs = {w.hidden for w in bank.values()}
        if len(ks) != 1 or len(hs) != 1:
            raise ValueError("mixed predictor shapes in bank")
        self.k, self.hidden = ks.pop(), hs.pop()
        self.layers = frozenset(int(l) for l in bank)
        self.num_layers = num_layers
        n = 3 * self.k
        w1 = np.zeros((num_layers, n, self.hidden), np.float32)
        b1 = np.zeros((num_layers, self.hidden), np.float32)
        w2 = np.zeros((num_layers, self.hidden), np.float32)
        self.b2 = np.zeros(num_layers, np.float32)
        for l, w in bank.items():
            if not 0 <= l < num_layers:
                continue
            w1[l], b1[l], w2[l] = w.w1, w.b1, w.w2
            self.b2[l] = np.float32(w.b2)
        self.w1, self.b1, self.w2 = _dev(w1), _dev(b1), _dev(w2)
        self.cert = torch.stack([_cert(self.w1[l], self.b1[l], self.w2[l], self.k, self.hidden)
                                 for l in range(num_layers)])
        self.mask = sum(1 << l for l in self.layers if l < 64)


# --- SPXP persistence (predictor.py:284-342), same byte format -----------------

SPXP_MAGIC = b"SPXP"
SPXP_VERSION = 1


def save_predictors(bank: dict, path):
    if not bank:
        raise ValueError("empty predictor bank")
    ks = {w.k for w in bank.values()}
    hs = {w.hidden for w in bank.values()}
    if len(ks) != 1 or len(hs) != 1:
        raise ValueError("mixed predictor shapes in bank")
    k, hidden = ks.pop(), hs.pop()
    with open(path, "wb") as fh:
        fh.write(SPXP_MAGIC)
        fh.write(SPXP_VERSION.to_bytes(4, "little"))
        fh.write(k.to_bytes(4, "little"))
        fh.write(hidden.to_bytes(4, "little"))
        fh.write(len(bank).to_bytes(4, "little"))
        for layer in sorted(bank):
            w = bank[layer]
            fh.write(int(layer).to_bytes(4, "little"))
            fh.write(np.float32(w.threshold).tobytes())
            for arr in (w.w1, w.b1, w.w2, np.array([w.b2], np.float32)):
                fh.write(np.ascontiguousarray(arr, dtype="<f4").tobytes())


def load_predictors(path) -> dict:
    with open(path, "rb") as fh:
        data = fh.read()
    off = 0

    def read(n):
        nonlocal off
        if off + n > len(data):
            raise ValueError("truncated predictor file")
        b = data[off:off + n]
        off += n
        return b

    if read(4) != SPXP_MAGIC:
        raise ValueError("bad magic: not a predictor file")
    version = int.from_bytes(read(4), "little")
    if version != SPXP_VERSION:
        raise ValueError(f"unsupported predictor file version {version}")
    k = int.from_bytes(read(4), "little")
    hidden = int.from_bytes(read(4), "little")
    count = int.from_bytes(read(4), "little")
    bank = {}
    for _ in range(count):
        layer = int.from_bytes(read(4), "little")
        threshold = float(np.frombuffer(read(4), "<f4")[0])
        w1 = np.frombuffer(read(4 * 3 * k * hidden), "<f4").reshape(3 * k, hidden).copy()
        b1 = np.frombuffer(read(4 * hidden), "<f4").copy()
        w2 = np.frombuffer(read(4 * hidden), "<f4").copy()
        b2 = float(np.frombuffer(read(4), "<f4")[0])
        bank[layer] = PredictorWeights(w1=w1, b1=b1, w2=w2, b2=b2, threshold=threshold)
    return bank


class BatchResult:
    """Outputs of one fused launch (device tensors)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


_RECHECK = {}


def recheck_buffer(B: int, device=None):
    """The (5 + B) int32 work list of the STRICT re-evaluation, one per
    (stream, B); zeroed once, self-resetting (spx_predictor_args.recheck)."""
    key = (torch.cuda.current_stream().cuda_stream, int(B))
    buf = _RECHECK.get(key)
    if buf is None:
        buf = torch.zeros(5 + int(B), dtype=torch.int32, device=device or "cuda")
        _RECHECK[key] = buf
    return buf


def recheck_stats(buf=None):
    """(rows re-evaluated by the STRICT chain, rows whose STRICT decision was
    still inside the carried-prev bound) summed over the given buffer, or over
    every buffer of this process (synchronises)."""
    bufs = [buf] if buf is not None else list(_RECHECK.values())
    tot = [0, 0]
    for b in bufs:
        v = b[3:5].cpu().tolist()
        tot[0] += v[0]
        tot[1] += v[1]
    return tuple(tot)


def prev_error(prev: torch.Tensor) -> torch.Tensor:
    """The (B,) bound on |prev - prev_ref| carried with a prev tensor (created
    as zeros: a freshly filled prev -- the uniform prior or reference values --
    is exact).  Reset it with ``prev_error(prev).zero_()`` when prev is reset."""
    e = getattr(prev, "_spx_err", None)
    B = prev.shape[0] if prev.dim() > 1 else 1
    if e is None or e.numel() != B:
        e = torch.zeros(B, dtype=torch.float32, device=prev.device)
        prev._spx_err = e
    return e


def evaluate_batch(model, weights, hidden, ids, prev, threshold=0.5, layer=0, outputs=True, pdl=False,
                   row_layer_mask=None, row_done=None, evals=None, err=None, mode=None,
                   policy=None, out=None, prev_err=None, recheck=None, certify=True,
                   feat_out=None, fired_any=None):
    """K1+K2+K3 for B rows at one layer in ONE launch (spx_predictor_eval).

    model: TransformerModel (head + final norm used); weights: PredictorWeights
    or PredictorBank (row `layer` used); hidden (B, d) f32 CUDA; ids (B, K)
    int32 CUDA; prev (B, K) f32 CUDA, updated in place with the new local
    probabilities.  policy: None (MLP) or a constant probability (Never /
    Always policies).  Returns a BatchResult of device tensors (no sync).

    FAST mode certifies every decision against the reference's (DESIGN.md
    3.1): rows it cannot certify are re-evaluated by the STRICT chain in a
    follow-up launch of the same call, so ``fired`` is the reference's.
    prev_err (B,) is the error bound carried with ``prev`` (default: attached
    to the prev tensor, see prev_error); recheck the work list (default: one
    per stream and B, see recheck_buffer).  certify=False turns it off.
    feat_out: optional (B, 3K) f32 tensor receiving the feature vectors;
    fired_any: optional (B) u8 tensor, |= the decision (a token's predictor_fired)."""
    a, out = _batch_args(model, weights, hidden, ids, prev, threshold, layer, outputs, pdl,
                         row_layer_mask, row_done, evals, err, mode, policy, out, prev_err,
                         recheck, certify, feat_out)
    a.fired_any = N.ptr(fired_any)
    N.check(N.lib().spx_predictor_eval(a, N.stream_ptr()), "spx_predictor_eval")
    return out


def _batch_args(model, weights, hidden, ids, prev, threshold, layer, outputs, pdl, row_layer_mask,
                row_done, evals, err, mode, policy, out, prev_err, recheck, certify, feat_out):
    B, d = hidden.shape
    K = ids.shape[1]
    dev = hidden.device
    if out is None:
        out = BatchResult(
            logits=torch.empty((B, K), dtype=torch.float32, device=dev) if outputs else None,
            z=torch.empty(B, dtype=torch.float32, device=dev) if outputs else None,
            prob=torch.empty(B, dtype=torch.float64, device=dev) if outputs else None,
            fired=torch.empty(B, dtype=torch.uint8, device=dev),
            err=err if err is not None else torch.zeros(1, dtype=torch.int32, device=dev))
    a = N.PredictorArgs()
    a.hidden, a.hidden_stride = N.ptr(hidden), hidden.stride(0)
    a.norm_g, a.norm_b = N.ptr(model.final_g), N.ptr(model.final_b)
    a.head, a.head_dtype, a.head_bw = N.ptr(model.lm_head), model.spx_dtype, N.ptr(model.head_bw)
    a.ids, a.prev = N.ptr(ids), N.ptr(prev)
    cert = None
    if policy is None:
        if isinstance(weights, PredictorBank):
            a.w1 = N._vp(weights.w1[layer].data_ptr())
            a.b1 = N._vp(weights.b1[layer].data_ptr())
            a.w2 = N._vp(weights.w2[layer].data_ptr())
            a.b2 = float(weights.b2[layer])
            cert = weights.cert[layer]
            H = weights.hidden
        else:
            dw = _DeviceWeights.of(weights)
            a.w1, a.b1, a.w2, a.b2 = N.ptr(dw.w1), N.ptr(dw.b1), N.ptr(dw.w2), float(np.float32(weights.b2))
            cert = dw.cert
            H = weights.hidden
        a.policy = N.SPX_POLICY_MLP
        a.z_cut = z_cut(threshold)
    else:
        a.policy, a.const_prob, a.threshold, H = N.SPX_POLICY_CONST, float(policy), float(threshold), 0
    a.logits_out, a.z_out, a.prob_out = N.ptr(out.logits), N.ptr(out.z), N.ptr(out.prob)
    a.fired = N.ptr(out.fired)
    a.feat_out = N.ptr(feat_out)
    a.row_layer_mask, a.row_done, a.evals = N.ptr(row_layer_mask), N.ptr(row_done), N.ptr(evals)
    a.layer = layer
    a.mode = numerics.mode() if mode is None else mode
    a.pdl = 2 if (pdl == 2 and pdl is not True) else (1 if pdl else 0)
    a.err = N.ptr(out.err)
    a.B, a.d, a.V, a.K, a.H = B, d, model.config.vocab_size, K, H
    if certify and a.mode == N.SPX_MODE_FAST:
        out.recheck = recheck if recheck is not None else recheck_buffer(B)
        a.head_wmax, a.cert = N.ptr(model.head_wmax), N.ptr(cert)
        a.cert_kappa, a.cert_hnorm = model.cert_kappa, model.cert_hnorm
        a.prev_err = N.ptr(prev_err if prev_err is not None else prev_error(prev))
        a.recheck = N.ptr(out.recheck)
    elif a.mode == N.SPX_MODE_STRICT:
        a.prev_err = N.ptr(prev_err if prev_err is not None else prev_error(prev))
    return a, out


def split_supported(model, weights, hidden, ids, prev, policy=None, mode=None) -> bool:
    """True when the SPLIT form (spx_predictor_gather + spx_predictor_tail)
    serves this shape: FAST mode, bf16 head, K <= 8, d in {2048, 4096, 8192}."""
    a, _ = _batch_args(model, weights, hidden, ids, prev, 0.5, 0, False, False, None, None, None,
                       None, mode, policy, None, None, None, True, None)
    return bool(N.lib().spx_predictor_split_ok(a))


def evaluate_batch_split(model, weights, hidden, ids, prev, inter, threshold=0.5, layer=0,
                         outputs=True, pdl=3, tail_stream=None, row_layer_mask=None,
                         row_done=None, evals=None, err=None, policy=None, out=None,
                         prev_err=None, recheck=None, certify=True, feat_out=None):
    """evaluate_batch in its SPLIT form for large batches (same outputs, bit
    for bit): K1 (LayerNorm + gather + local logits) into ``inter`` (B, 2K+2)
    f32 on the current stream, then K2+K3 (features, MLP, decision,
    certification; carries ``prev``) on ``tail_stream`` (default: the current
    stream) after an event.  pdl=3: this layer's hidden rows and ids are not
    written by the kernel launched just before (e.g. the previous layer's
    gather), so consecutive gathers overlap.  No host sync; capturable."""
    a, out = _batch_args(model, weights, hidden, ids, prev, threshold, layer, outputs, False,
                         row_layer_mask, row_done, evals, err, N.SPX_MODE_FAST, policy, out,
                         prev_err, recheck, certify, feat_out)
    a.pdl = int(pdl)
    lib = N.lib()
    N.check(lib.spx_predictor_gather(a, N.ptr(inter), N.stream_ptr()), "spx_predictor_gather")
    if tail_stream is None:
        N.check(lib.spx_predictor_tail(a, N.ptr(inter), N.stream_ptr()), "spx_predictor_tail")
        return out
    ev = torch.cuda.Event()
    ev.record()
    tail_stream.wait_event(ev)
    with torch.cuda.stream(tail_stream):
        N.check(lib.spx_predictor_tail(a, N.ptr(inter), N.stream_ptr()), "spx_predictor_tail")
    return out


def evaluate_chain(model, weights, hidden, ids, prev, inter, layers, threshold=0.5, outs=None,
                   policy=None, prev_err=None, recheck=None, certify=True, feat_out=None):
    """Several layers' predictor evaluations over the same B rows, ``prev``
    carried from layer to layer (the token's layer loop of engine.py:192-207
    for B independent requests whose hidden rows of every listed layer are
    already resident), in the PIPELINED split form: gather(layers[0]), then
    per further layer ONE launch = that layer's gather + the previous layer's
    tail, then the last layer's tail -- so every LM-head gather overlaps its
    neighbours and no per-row MLP tail sits on the bandwidth-bound path.
    The last layer's tail runs on the same kernel's tail warps with an empty
    gather (spx_predictor_tail_pipelined).
    hidden[i] / ids[i] / inter[i] / outs[i] / feat_out[i] belong to
    layers[i]; inter: (len(layers), B, 2K+2) f32.  FAST mode, shapes of
    split_supported.  Same outputs, bit for bit, as evaluate_batch per layer.
    No host sync; capturable."""
    n = len(layers)
    if outs is None:
        outs = [None] * n
    args = []
    for i, l in enumerate(layers):
        a, o = _batch_args(model, weights, hidden[i], ids[i], prev, threshold, l, outs[i] is None,
                           False, None, None, None, None, N.SPX_MODE_FAST, policy, outs[i],
                           prev_err, recheck, certify, None if feat_out is None else feat_out[i])
        a.pdl = 3
        args.append(a)
        outs[i] = o
    lib = N.lib()
    st = N.stream_ptr()
    N.check(lib.spx_predictor_gather(args[0], N.ptr(inter[0]), st), "spx_predictor_gather")
    for i in range(1, n):
        N.check(lib.spx_predictor_gather_tail(args[i], N.ptr(inter[i]), args[i - 1],
                                              N.ptr(inter[i - 1]), st),
                "spx_predictor_gather_tail")
    N.check(lib.spx_predictor_tail_pipelined(args[-1], N.ptr(inter[n - 1]), st),
            "spx_predictor_tail_pipelined")
    return outs
