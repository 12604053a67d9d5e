"""ORACLE — CPU restatement of the SpecEE reference's speculative early-exit
predictor path.  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` leg may import this module, and only as the checker
(or the timed CPU baseline) -- never as the thing measured or shipped.  The
product package (paper_2504_08850_b200/) never imports it.

Every function restates the reference's algorithm (numpy + the strict-order
float32 kernels of oracle/strict.c) and cites the reference file:line it
follows; paths are relative to /root/reference/pkg/src/specexit/.  The
restatement is pinned against fixtures produced by the reference itself
(tests/golden/, made by tests/golden/make_golden.py) and against the
reference's shipped end-to-end golden trace (pkg/runs/default/trace.jsonl).

Arithmetic contract (reference kernels/__init__.py:57-71, model.py:140-152,
predictor.py:87-109): fp32 with strict ascending accumulation for layer norm,
head projections and softmax sums; numpy's float32 exp; numpy BLAS
(OpenBLAS sgemv/sdot) for the predictor MLP; float64 sigmoid; strict ``>``.
"""

import ctypes
import math
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LN_EPS = np.float32(1e-5)                      # model.py:27

# ---------------------------------------------------------------- strict kernels


def _load_strict():
    path = os.path.join(_HERE, "_lib", "libspx_oracle.so")
    if not os.path.exists(path):
        from . import build as _b  # noqa: F401  (builds on import if missing)
        _b.build()
    lib = ctypes.CDLL(path)
    f32p = ctypes.POINTER(ctypes.c_float)
    i64 = ctypes.c_int64
    lib.oracle_matmul_f32.argtypes = [f32p, f32p, f32p, i64, i64, i64]
    lib.oracle_seq_sum_f32.argtypes = [f32p, f32p, i64, i64]
    lib.oracle_gather_dot_f32.argtypes = [f32p, f32p, i64, ctypes.POINTER(ctypes.c_int64), i64,
                                          i64, f32p]
    return lib


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        _LIB = _load_strict()
    return _LIB


def _fp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def matmul(a, b):
    """kernels/__init__.py:57-63 + _ckern.pyx:16-31: strict k-ascending f32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise ValueError(f"matmul shape mismatch: {a.shape} @ {b.shape}")
    out = np.empty((a.shape[0], b.shape[1]), np.float32)
    _lib().oracle_matmul_f32(_fp(a), _fp(b), _fp(out), a.shape[0], a.shape[1], b.shape[1])
    return out


def seq_sum(x):
    """kernels/__init__.py:66-71 + _ckern.pyx:34-46: strict left-to-right."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim == 0:
        raise ValueError("seq_sum needs at least one axis")
    flat = np.ascontiguousarray(x.reshape(-1, x.shape[-1]))
    out = np.empty(flat.shape[0], np.float32)
    _lib().oracle_seq_sum_f32(_fp(flat), _fp(out), flat.shape[0], flat.shape[1])
    return out.reshape(x.shape[:-1])


def gather_matmul_row(h, w, ids):
    """matmul(h[None], ascontiguousarray(w[:, ids]))[0] without the copy
    (model.py:313-314); identical operation sequence."""
    h = np.ascontiguousarray(h, dtype=np.float32)
    ids = np.ascontiguousarray(ids, dtype=np.int64)
    out = np.empty(ids.size, np.float32)
    _lib().oracle_gather_dot_f32(_fp(h), _fp(w), w.shape[1],
                                 ids.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), ids.size,
                                 w.shape[0], _fp(out))
    return out


# ---------------------------------------------------------------- rng (rng.py)

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed, n):
    """rng.py:14-21."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + _GOLDEN * np.arange(1, n + 1, dtype=np.uint64)
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed, n, low, high):
    """rng.py:24-27."""
    u = (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return (low + (high - low) * u).astype(np.float32)


def derive(seed, index):
    """rng.py:30-32."""
    return int(splitmix64(seed, index + 1)[-1])


def round_bf16(x):
    """Round-to-nearest-even to bfloat16, returned as float32 (the parity
    recipe of SURVEY.md §8c step 2: both sides see identical values)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


# ---------------------------------------------------------------- model (model.py)


@dataclass(frozen=True)
class ModelConfig:
    """model.py:32-56."""
    vocab_size: int = 256
    hidden_dim: int = 64
    num_layers: int = 8
    num_heads: int = 4
    ffn_dim: int = 256
    max_context: int = 512
    seed: int = 0

    @property
    def head_dim(self):
        return self.hidden_dim // self.num_heads


def tensor_specs(cfg):
    """model.py:59-84 (declaration order fixes the per-tensor seed index)."""
    d, f, v = cfg.hidden_dim, cfg.ffn_dim, cfg.vocab_size
    specs = [("embedding", (v, d), "uniform")]
    for i in range(cfg.num_layers):
        p = f"layers.{i}"
        specs += [(f"{p}.ln1.g", (d,), "ones"), (f"{p}.ln1.b", (d,), "zeros"),
                  (f"{p}.attn.wq", (d, d), "uniform"), (f"{p}.attn.wk", (d, d), "uniform"),
                  (f"{p}.attn.wv", (d, d), "uniform"), (f"{p}.attn.wo", (d, d), "uniform"),
                  (f"{p}.ln2.g", (d,), "ones"), (f"{p}.ln2.b", (d,), "zeros"),
                  (f"{p}.ffn.w1", (d, f), "uniform"), (f"{p}.ffn.b1", (f,), "zeros"),
                  (f"{p}.ffn.w2", (f, d), "uniform"), (f"{p}.ffn.b2", (d,), "zeros")]
    specs += [("final_norm.g", (d,), "ones"), ("final_norm.b", (d,), "zeros"),
              ("lm_head", (d, v), "uniform")]
    return specs


def init_model(cfg, bf16=False, only=None):
    """model.py:121-137; ``bf16`` applies round_bf16 to every tensor (parity
    recipe), ``only`` restricts to a subset of tensor names (speed)."""
    tensors = {}
    for idx, (name, shape, kind) in enumerate(tensor_specs(cfg)):
        if only is not None and name not in only:
            continue
        if kind == "uniform":
            b = math.sqrt(6.0 / (shape[0] + shape[1]))
            t = uniform(derive(cfg.seed, idx), int(np.prod(shape)), -b, b).reshape(shape)
        elif kind == "zeros":
            t = np.zeros(shape, np.float32)
        else:
            t = np.ones(shape, np.float32)
        tensors[name] = round_bf16(t) if bf16 else t
    return tensors


def sinusoidal_encoding(max_len, dim):
    """model.py:112-118."""
    pe = np.zeros((max_len, dim), dtype=np.float64)
    pos = np.arange(max_len)[:, None]
    div = np.exp(np.arange(0, dim, 2) * (-math.log(10000.0) / dim))
    pe[:, 0::2] = np.sin(pos * div)
    pe[:, 1::2] = np.cos(pos * div)
    return pe.astype(np.float32)


def layer_norm(x, g, b):
    """model.py:140-146."""
    d = np.float32(x.shape[-1])
    mean = seq_sum(x) / d
    xc = x - mean[..., None]
    var = seq_sum(xc * xc) / d
    return xc / np.sqrt(var + LN_EPS)[..., None] * g + b


def softmax_1d(x):
    """model.py:149-152 (numpy's float32 exp)."""
    e = np.exp(x - np.max(x))
    return e / seq_sum(e[None, :])[0]


def _check_hidden(hidden):
    hidden = np.asarray(hidden, dtype=np.float32)
    if not np.all(np.isfinite(hidden)):
        raise ValueError("non-finite hidden state")
    return hidden


def full_head_logits(t, hidden):
    """model.py:289-295."""
    hidden = _check_hidden(hidden)
    h = layer_norm(hidden[None, :], t["final_norm.g"], t["final_norm.b"])
    return matmul(h, t["lm_head"])[0]


def sliced_head_logits(t, hidden, token_ids):
    """model.py:298-314."""
    token_ids = np.asarray(token_ids, dtype=np.int64)
    if token_ids.size == 0:
        raise ValueError("empty token id list")
    if token_ids.min() < 0 or token_ids.max() >= t["lm_head"].shape[1]:
        raise ValueError("token id out of range")
    hidden = _check_hidden(hidden)
    h = layer_norm(hidden[None, :], t["final_norm.g"], t["final_norm.b"])
    return gather_matmul_row(h[0], t["lm_head"], token_ids)


# ---------------------------------------------------------------- predictor.py


@dataclass
class FeatureVector:
    """predictor.py:22-33."""
    spec_logits: np.ndarray
    local_probs: np.ndarray
    prob_variation: np.ndarray

    def concat(self):
        return np.concatenate([self.spec_logits, self.local_probs,
                               self.prob_variation]).astype(np.float32)


def uniform_probs(k):
    """predictor.py:36-39."""
    return np.full(k, 1.0 / k, dtype=np.float32)


def extract_features(spec_logits, prev_local_probs):
    """predictor.py:42-52."""
    spec_logits = np.asarray(spec_logits, dtype=np.float32)
    prev_local_probs = np.asarray(prev_local_probs, dtype=np.float32)
    if spec_logits.size < 1 or spec_logits.shape != prev_local_probs.shape:
        raise ValueError("bad feature input shapes")
    if not np.all(np.isfinite(spec_logits)):
        raise ValueError("non-finite speculative logits")
    if abs(float(prev_local_probs.sum()) - 1.0) > 1e-5:
        raise ValueError("prev_local_probs must sum to 1")
    local = softmax_1d(spec_logits)
    return FeatureVector(spec_logits, local, local - prev_local_probs)


@dataclass
class PredictorWeights:
    """predictor.py:55-75."""
    w1: np.ndarray
    b1: np.ndarray
    w2: np.ndarray
    b2: float
    threshold: float = 0.5


def init_predictor(k, hidden, seed, threshold=0.5):
    """predictor.py:78-84."""
    d = 3 * k
    b = np.sqrt(6.0 / (d + hidden))
    w1 = uniform(derive(seed, 0), d * hidden, -b, b).reshape(d, hidden)
    b2 = np.sqrt(6.0 / (hidden + 1))
    w2 = uniform(derive(seed, 1), hidden, -b2, b2)
    return PredictorWeights(w1=w1, b1=np.zeros(hidden, np.float32), w2=w2, b2=0.0,
                            threshold=threshold)


def sigmoid(z):
    """predictor.py:87-94 (float64)."""
    z = np.asarray(z, dtype=np.float64)
    out = np.empty_like(z)
    pos = z >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-z[pos]))
    ez = np.exp(z[~pos])
    out[~pos] = ez / (1.0 + ez)
    return out if out.ndim else float(out)


def predictor_logit(w, features):
    """The f32 pre-sigmoid value of predictor.py:102-103 (numpy BLAS)."""
    f = features.concat() if isinstance(features, FeatureVector) else np.asarray(features)
    if f.shape != (w.w1.shape[0],):
        raise ValueError("feature dimension does not match predictor")
    h = np.maximum(f @ w.w1 + w.b1, 0)
    return h @ w.w2 + w.b2


def predictor_forward(w, features):
    """predictor.py:97-103."""
    return float(sigmoid(predictor_logit(w, features)))


def decide_exit(prob, threshold):
    """predictor.py:106-109 (strict >)."""
    return prob > threshold


# ---------------------------------------------------------------- scheduler.py


@dataclass(frozen=True)
class ScheduleConfig:
    """scheduler.py:17-27."""
    queue_len: int = 5
    radius: int = 2
    offline_top_k: int = 4


def ranked_layers(exit_counts, num_layers):
    """scheduler.py:41-46."""
    counts = np.asarray(exit_counts, np.uint64)[: num_layers - 1]
    return sorted(range(num_layers - 1), key=lambda i: (-int(counts[i]), i))


@dataclass
class OnlineState:
    """scheduler.py:49-58."""
    num_layers: int
    config: ScheduleConfig
    queue: list = field(default_factory=list)
    neighbor_counts: np.ndarray = None

    def __post_init__(self):
        if self.neighbor_counts is None:
            self.neighbor_counts = np.zeros(self.num_layers, dtype=np.int64)


def _neighborhood(layer, num_layers, radius):
    """scheduler.py:61-62."""
    return range(max(layer - radius, 0), min(layer + radius, num_layers - 1) + 1)


def update_online(state, exit_layer):
    """scheduler.py:65-79."""
    if not 0 <= exit_layer < state.num_layers:
        raise ValueError("exit layer out of range")
    r = state.config.radius
    if len(state.queue) == state.config.queue_len:
        ev = state.queue.pop(0)
        for i in _neighborhood(ev, state.num_layers, r):
            state.neighbor_counts[i] -= 1
    state.queue.append(exit_layer)
    for i in _neighborhood(exit_layer, state.num_layers, r):
        state.neighbor_counts[i] += 1
    return state


def active_layers(exit_counts, state, config):
    """scheduler.py:91-102."""
    L = state.num_layers
    if config.offline_top_k > L - 1:
        raise ValueError("offline_top_k exceeds predictor-capable layers")
    chosen = set(ranked_layers(exit_counts, L)[: config.offline_top_k])
    chosen.update(i for i in range(L - 1) if state.neighbor_counts[i] > 0)
    return sorted(l for l in chosen if l <= L - 2)


# ---------------------------------------------------------------- engine / tree


def verify_exit(t, hidden, spec_tokens):
    """engine.py:59-64 (np.argmax: lowest index on ties)."""
    tok = int(np.argmax(full_head_logits(t, hidden)))
    return tok if tok in tuple(spec_tokens) else None


def grouped_speculative_logits(t, hiddens, token_id_lists):
    """tree.py:92-113 (per-node bit-identical to sliced_head_logits)."""
    hiddens = np.asarray(hiddens, dtype=np.float32)
    if hiddens.ndim != 2 or hiddens.shape[0] < 1:
        raise ValueError("need at least one node hidden state")
    if len(token_id_lists) != hiddens.shape[0]:
        raise ValueError("one id list per node required")
    return [sliced_head_logits(t, hiddens[j], ids) for j, ids in enumerate(token_id_lists)]


def hypertoken_exit_decision(per_node_probs, threshold):
    """tree.py:116-122."""
    probs = list(per_node_probs)
    if not probs:
        raise ValueError("need at least one node probability")
    return all(decide_exit(p, threshold) for p in probs)


def topk_from_logits(logits, k):
    """speculation.py:57-60 (stable: ties by lower id)."""
    return np.argsort(-logits, kind="stable")[:k]


# ---------------------------------------------------------------- decode state


class DecodeState:
    """model.py:155-286 restated: lazy KV completion through per-position
    frontiers; tree rows with explicit ancestor lists, freezing, compaction."""

    def __init__(self, cfg, t, pos_encoding):
        self.cfg, self.t, self.pe = cfg, t, pos_encoding
        L, C, d = cfg.num_layers, cfg.max_context, cfg.hidden_dim
        self.k = np.zeros((L, C, d), np.float32)
        self.v = np.zeros((L, C, d), np.float32)
        self.pending = np.zeros((C, d), np.float32)
        self.frontier = np.zeros(C, np.int64)
        self.n = 0
        self.new_rows = []
        self.attn_index = {}
        self.frozen = set()

    def begin(self, tokens, pos_ids=None, attn_lists=None):
        """model.py:181-212 (pos_ids / attn_lists: tree rows, :201-211)."""
        rows = list(range(self.n, self.n + len(tokens)))
        if self.n + len(tokens) > self.cfg.max_context:
            raise ValueError("context overflow")
        pos = rows if pos_ids is None else list(pos_ids)
        self.pending[rows] = self.t["embedding"][np.asarray(tokens)] + self.pe[pos]
        self.frontier[rows] = 0
        for j, p in enumerate(rows):
            if attn_lists is not None and attn_lists[j] is not None:
                idx = np.asarray(sorted(set(attn_lists[j]) | {p}), dtype=np.int64)
                if idx.max() > p:
                    raise ValueError("attention index must not look ahead")
                self.attn_index[p] = idx
        self.n += len(tokens)
        self.new_rows = rows
        return rows

    def freeze(self, positions):
        """model.py:214-215."""
        self.frozen.update(positions)

    def unfreeze_all(self):
        """model.py:217-218."""
        self.frozen.clear()

    def run_layer(self, l):
        """model.py:220-233."""
        rows = [p for p in range(self.n) if self.frontier[p] == l and p not in self.frozen]
        if rows:
            self._advance(l, rows)
        return self.pending[self.new_rows].copy()

    def compact(self, keep_new_rows, n_committed):
        """model.py:272-286."""
        keep = list(keep_new_rows)
        dest = list(range(n_committed, n_committed + len(keep)))
        self.k[:, dest] = self.k[:, keep]
        self.v[:, dest] = self.v[:, keep]
        self.pending[dest] = self.pending[keep]
        self.frontier[dest] = self.frontier[keep]
        self.attn_index = {}
        self.n = n_committed + len(keep)
        self.new_rows = []
        self.frozen.clear()

    def _advance(self, l, rows):
        """model.py:235-270."""
        t, cfg = self.t, self.cfg
        p_ = f"layers.{l}"
        x = self.pending[rows]
        h = layer_norm(x, t[f"{p_}.ln1.g"], t[f"{p_}.ln1.b"])
        q = matmul(h, t[f"{p_}.attn.wq"])
        self.k[l, rows] = matmul(h, t[f"{p_}.attn.wk"])
        self.v[l, rows] = matmul(h, t[f"{p_}.attn.wv"])
        nh, dh = cfg.num_heads, cfg.head_dim
        scale = np.float32(1.0 / math.sqrt(dh))
        attn = np.empty_like(x)
        for j, p in enumerate(rows):
            ctx = self.attn_index.get(p)
            if ctx is None:
                ctx = np.arange(p + 1)
            kc, vc = self.k[l, ctx], self.v[l, ctx]
            out = np.empty(cfg.hidden_dim, np.float32)
            for hh in range(nh):
                s = slice(hh * dh, (hh + 1) * dh)
                scores = matmul(kc[:, s], q[j, s][:, None])[:, 0] * scale
                out[s] = matmul(softmax_1d(scores)[None, :], vc[:, s])[0]
            attn[j] = matmul(out[None, :], t[f"{p_}.attn.wo"])[0]
        x = x + attn
        h2 = layer_norm(x, t[f"{p_}.ln2.g"], t[f"{p_}.ln2.b"])
        f = np.maximum(matmul(h2, t[f"{p_}.ffn.w1"]) + t[f"{p_}.ffn.b1"], np.float32(0))
        x = x + matmul(f, t[f"{p_}.ffn.w2"]) + t[f"{p_}.ffn.b2"]
        self.pending[rows] = x
        self.frontier[rows] = l + 1


@dataclass
class ExitRecord:
    """engine.py:26-48."""
    token: int
    exit_layer: int
    predictor_fired: bool
    verified: bool
    active: list
    full_head_count: int = 0
    predictor_evals: int = 0
    probs: dict = field(default_factory=dict)      # layer -> predictor prob (diagnostic)
    logits: dict = field(default_factory=dict)     # layer -> f32 pre-sigmoid (diagnostic)


class ExitEngineOracle:
    """engine.py:122-246 restated for the PredictorPolicy / Never / Always
    policies; ``policy`` is a dict layer->PredictorWeights, or the strings
    "never" / "always"."""

    def __init__(self, target_cfg, target, draft_cfg, draft, policy, k=4, threshold=0.5,
                 schedule_mode="all", exit_counts=None, schedule_config=ScheduleConfig()):
        self.tc, self.t, self.dc, self.d = target_cfg, target, draft_cfg, draft
        self.policy, self.k, self.thr = policy, k, threshold
        self.mode, self.counts, self.sc = schedule_mode, exit_counts, schedule_config
        self.tpe = sinusoidal_encoding(target_cfg.max_context, target_cfg.hidden_dim)
        self.dpe = sinusoidal_encoding(draft_cfg.max_context, draft_cfg.hidden_dim)
        self.online = OnlineState(target_cfg.num_layers, schedule_config)

    def start(self, prompt):
        """engine.py:145-160."""
        prompt = list(prompt)
        self.ts = DecodeState(self.tc, self.t, self.tpe)
        self.ds = DecodeState(self.dc, self.d, self.dpe)
        if len(prompt) > 1:
            self.ts.begin(prompt[:-1])
            for l in range(self.tc.num_layers):
                self.ts.run_layer(l)
            self.ds.begin(prompt[:-1])
            for l in range(self.dc.num_layers):
                self.ds.run_layer(l)
        self.context = prompt
        self.next_in = prompt[-1]

    def _spec(self):
        """engine.py:162-168 + speculation.py:81-84."""
        self.ds.begin([self.next_in])
        for l in range(self.dc.num_layers):
            dout = self.ds.run_layer(l)
        logits = full_head_logits(self.d, dout[-1])
        return [int(i) for i in topk_from_logits(logits, self.k)]

    def _active(self):
        """engine.py:170-174."""
        L = self.tc.num_layers
        if self.mode == "all":
            return list(range(L - 1))
        return active_layers(self.counts, self.online, self.sc)

    def step(self, spec=None, drafted_already=False):
        """engine.py:176-217 (``spec`` overrides the draft proposal: the
        injected-spec hook of SURVEY.md §8d C2; drafted_already: the draft
        forward of this step has run)."""
        L = self.tc.num_layers
        drafted = None if drafted_already else self._spec()
        spec = drafted if spec is None else list(spec)
        active = self._active()
        aset = set(active)
        self.ts.begin([self.next_in])
        prev = uniform_probs(len(spec))
        token, exit_layer, fired, verified, heads, evals = None, L - 1, False, False, 0, 0
        rec = ExitRecord(0, 0, False, False, active)
        hidden = None
        for l in range(L):
            hidden = self.ts.run_layer(l)[-1]
            if l in aset:
                fv = extract_features(sliced_head_logits(self.t, hidden, spec), prev)
                prev = fv.local_probs
                if self.policy == "never":
                    prob = 0.0
                elif self.policy == "always":
                    prob = 1.0
                else:
                    if l not in self.policy:
                        raise KeyError(f"no predictor for active layer {l}")
                    z = predictor_logit(self.policy[l], fv)
                    prob = float(sigmoid(z))
                    rec.logits[l] = np.float32(z)
                rec.probs[l] = prob
                evals += 1
                if decide_exit(prob, self.thr):
                    fired = True
                    heads += 1
                    tok = verify_exit(self.t, hidden, spec)
                    if tok is not None:
                        token, exit_layer, verified = tok, l, True
                        break
        if token is None:
            heads += 1
            token = int(np.argmax(full_head_logits(self.t, hidden)))
        self.context.append(token)
        self.next_in = token
        update_online(self.online, exit_layer)
        rec.token, rec.exit_layer, rec.predictor_fired, rec.verified = token, exit_layer, fired, verified
        rec.full_head_count, rec.predictor_evals = heads, evals
        return rec

    def generate(self, prompt, max_new):
        """engine.py:219-225."""
        self.start(prompt)
        trace = [self.step() for _ in range(max_new)]
        return [r.token for r in trace], trace

    def generate_forced(self, prompt, forced, inject=None):
        """engine.py:227-246.  inject: per-step flags of the injected-spec hook
        (SURVEY.md §8d C2): at a flagged step the forced token replaces the
        last drafted id unless it is already among them."""
        self.start(prompt)
        trace = []
        for i, tok in enumerate(forced):
            spec = None
            if inject is not None and inject[i]:
                drafted = self._spec()
                if int(tok) not in drafted:
                    drafted[-1] = int(tok)
                spec = drafted
            trace.append(self.step(spec, drafted_already=spec is not None))
            self.context[-1] = int(tok)
            self.next_in = int(tok)
        return trace


# ---------------------------------------------------------------- tree mode


def propose_topk(cfg, t, pe, context, k):
    """speculation.py:62-84: a FRESH full draft forward over ``context``
    (:63-68), top-k with lower-id ties, probs = softmax_1d(logits)[ids]."""
    st = DecodeState(cfg, t, pe)
    st.begin(list(context))
    out = None
    for l in range(cfg.num_layers):
        out = st.run_layer(l)
    logits = full_head_logits(t, out[-1])
    ids = topk_from_logits(logits, k)
    probs = softmax_1d(logits)[ids]
    return tuple(int(i) for i in ids), tuple(float(p) for p in probs)


@dataclass
class TreeNodeO:
    """speculation.py:28-33."""
    token: int
    parent: int
    depth: int
    prob: float = 0.0


def build_token_tree(cfg, t, pe, context, branching):
    """speculation.py:87-125: depth-first expansion, then (depth, creation)
    order; node 0 is the root (last context token)."""
    nodes = [TreeNodeO(int(context[-1]), -1, 0)]
    context = list(context)

    def expand(idx, path_tokens, depth):
        if depth == len(branching):
            return
        toks, probs = propose_topk(cfg, t, pe, context + path_tokens, branching[depth])
        kids = []
        for tok, pr in zip(toks, probs):
            nodes.append(TreeNodeO(tok, idx, depth + 1, pr))
            kids.append(len(nodes) - 1)
        for cid, tok in zip(kids, toks):
            expand(cid, path_tokens + [tok], depth + 1)

    expand(0, [], 0)
    order = sorted(range(len(nodes)), key=lambda i: (nodes[i].depth, i))
    remap = {old: new for new, old in enumerate(order)}
    return [TreeNodeO(nodes[o].token, remap[nodes[o].parent] if nodes[o].parent >= 0 else -1,
                      nodes[o].depth, nodes[o].prob) for o in order]


def enumerate_paths(nodes):
    """speculation.py:36-54, :127-130: root-to-leaf paths (root excluded)."""
    parents = {n.parent for n in nodes}
    paths = []
    for leaf in (i for i in range(len(nodes)) if i not in parents):
        path, idx = [], leaf
        while idx != 0:
            path.append(idx)
            idx = nodes[idx].parent
        paths.append(path[::-1])
    return paths


def merge_paths(nodes, dcfg, draft, dpe, context, k):
    """tree.py:49-89 -> (paths, per-path verify specs, per-node feature ids).
    Feature ids = draft top-k at the node's own context (cached per node);
    verify spec = children for internal nodes, the feature ids for leaves."""
    paths = enumerate_paths(nodes)
    child_map = {}
    for j, n in enumerate(nodes):
        child_map.setdefault(n.parent, []).append(j)
    feat = {}
    specs = []
    for path in paths:
        ps = []
        for idx in path:
            if idx not in feat:
                upto = path[: path.index(idx) + 1]
                feat[idx] = propose_topk(dcfg, draft, dpe,
                                         list(context) + [nodes[i].token for i in upto], k)[0]
            kids = child_map.get(idx)
            ps.append(tuple(nodes[c].token for c in kids) if kids else feat[idx])
        specs.append(ps)
    return paths, specs, feat


@dataclass
class TreeStepO:
    """tree.py:37-46 (+ the per-call probability log of the golden)."""
    accepted_tokens: list
    correction_token: int
    path_exit_layers: list
    accepted_path: int
    predictor_evals: int
    num_paths: int
    max_path_len: int
    scheduled_layer_count: int
    probs: list = field(default_factory=list)


class TreeEngineOracle:
    """tree.py:133-302 restated; ``policy``: dict layer->PredictorWeights,
    "never" or "always" (engine.py:67-92)."""

    def __init__(self, target_cfg, target, draft_cfg, draft, policy, branching=(3, 2), k=4,
                 threshold=0.5, schedule_mode="all", exit_counts=None,
                 schedule_config=ScheduleConfig()):
        self.tc, self.t, self.dc, self.d = target_cfg, target, draft_cfg, draft
        self.policy, self.branching, self.k, self.thr = policy, tuple(branching), k, threshold
        self.mode, self.counts, self.sc = schedule_mode, exit_counts, schedule_config
        self.tpe = sinusoidal_encoding(target_cfg.max_context, target_cfg.hidden_dim)
        self.dpe = sinusoidal_encoding(draft_cfg.max_context, draft_cfg.hidden_dim)
        self.online = OnlineState(target_cfg.num_layers, schedule_config)

    def start(self, prompt):
        """tree.py:153-163."""
        prompt = list(prompt)
        self.ts = DecodeState(self.tc, self.t, self.tpe)
        if len(prompt) > 1:
            self.ts.begin(prompt[:-1])
            for l in range(self.tc.num_layers):
                self.ts.run_layer(l)
        self.context = prompt

    def _prob(self, l, fv):
        if self.policy == "never":
            return 0.0
        if self.policy == "always":
            return 1.0
        if l not in self.policy:
            raise KeyError(f"no predictor for active layer {l}")
        return predictor_forward(self.policy[l], fv)

    def _argmax(self, h):
        return int(np.argmax(full_head_logits(self.t, h)))

    def step(self):
        """tree.py:171-266."""
        L = self.tc.num_layers
        nodes = build_token_tree(self.dc, self.d, self.dpe, self.context, self.branching)
        paths, specs, feat = merge_paths(nodes, self.dc, self.d, self.dpe, self.context, self.k)
        n_nodes = len(nodes)
        m = len(self.context) - 1
        tokens = [n.token for n in nodes]
        pos_ids = [m + n.depth for n in nodes]
        attn, anc = [None], {0: [0]}
        for j in range(1, n_nodes):
            anc[j] = anc[nodes[j].parent] + [j]
            attn.append(list(range(m)) + [m + a for a in anc[j]])
        rows = self.ts.begin(tokens, pos_ids=pos_ids, attn_lists=attn)
        active = (list(range(L - 1)) if self.mode == "all"
                  else active_layers(self.counts, self.online, self.sc))
        aset = set(active)
        prev = {j: None for j in range(1, n_nodes)}
        live = set(range(len(paths)))
        exit_layer = [L - 1] * len(paths)
        preds = [None] * len(paths)
        evals, log, hidden = 0, [], None
        for l in range(L):
            hidden = self.ts.run_layer(l)
            if not live:
                break
            if l in aset and l <= L - 2:
                live_nodes = sorted({j for p in live for j in paths[p]})
                probs = {}
                for j in live_nodes:
                    lg = sliced_head_logits(self.t, hidden[j], feat[j])
                    pv = prev[j] if prev[j] is not None else uniform_probs(len(feat[j]))
                    fv = extract_features(lg, pv)
                    prev[j] = fv.local_probs
                    probs[j] = self._prob(l, fv)
                    log.append([l, probs[j]])
                    evals += 1
                for p in sorted(live):
                    if hypertoken_exit_decision([probs[j] for j in paths[p]], self.thr):
                        chain = [self._argmax(hidden[0])]
                        ok = True
                        for idx, spec in zip(paths[p], specs[p]):
                            am = self._argmax(hidden[idx])
                            if am not in spec:
                                ok = False
                                break
                            chain.append(am)
                        if ok:
                            exit_layer[p], preds[p] = l, chain
                            live.discard(p)
                keep = {j for p in live for j in paths[p]} | ({0} if live else set())
                self.ts.freeze(rows[j] for j in range(n_nodes) if j not in keep)
            if not live:
                break
        for p in list(live):
            preds[p] = [self._argmax(hidden[0])] + [self._argmax(hidden[j]) for j in paths[p]]
        self.ts.unfreeze_all()
        best_p, best_len = 0, -1
        for p, path in enumerate(paths):
            n_ok = 0
            for t_, idx in enumerate(path):
                if nodes[idx].token == preds[p][t_]:
                    n_ok += 1
                else:
                    break
            if n_ok > best_len:
                best_p, best_len = p, n_ok
        acc_nodes = paths[best_p][:best_len]
        acc = [nodes[j].token for j in acc_nodes]
        corr = preds[best_p][best_len]
        self.ts.compact([rows[0]] + [rows[j] for j in acc_nodes], m)
        self.context.extend(acc + [corr])
        for _ in range(len(acc) + 1):
            update_online(self.online, exit_layer[best_p])
        return TreeStepO(acc, corr, exit_layer, best_p, evals, len(paths),
                         max(len(p) for p in paths), max(len(aset), 1), log)


# ---------------------------------------------------------------- weight files


def load_spxw(path):
    """model.py:355-434 (SPXW reader) -> (ModelConfig, tensors)."""
    CONFIG_FIELDS = ("vocab_size", "hidden_dim", "num_layers", "num_heads", "ffn_dim",
                     "max_context")
    with open(path, "rb") as fh:
        data = fh.read()
    off = 0

    def take(n):
        nonlocal off
        if off + n > len(data):
            raise ValueError("truncated weight file")
        b = data[off:off + n]
        off += n
        return b

    if take(4) != b"SPXW":
        raise ValueError("bad magic: not a weight file")
    if int.from_bytes(take(4), "little") != 1:
        raise ValueError("unsupported weight file version")
    count = int.from_bytes(take(4), "little")
    tensors = {}
    for _ in range(count):
        nlen = int.from_bytes(take(2), "little")
        name = take(nlen).decode()
        rank = int.from_bytes(take(1), "little")
        shape = tuple(int.from_bytes(take(4), "little") for _ in range(rank))
        n = int(np.prod(shape)) if shape else 1
        tensors[name] = np.frombuffer(take(4 * n), "<f4").reshape(shape).astype(np.float32)
    vec = tensors.pop("config")
    fields = {f: int(v) for f, v in zip(CONFIG_FIELDS, vec)}
    seed = sum(int(v) << (16 * i) for i, v in enumerate(vec[len(CONFIG_FIELDS):]))
    return ModelConfig(seed=seed, **fields), tensors


def load_spxp(path):
    """predictor.py:316-342 (SPXP reader) -> {layer: PredictorWeights}."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != b"SPXP":
        raise ValueError("bad magic: not a predictor file")
    k, hidden, count = (int.from_bytes(data[o:o + 4], "little") for o in (8, 12, 16))
    off, bank = 20, {}
    for _ in range(count):
        layer = int.from_bytes(data[off:off + 4], "little")
        thr = float(np.frombuffer(data[off + 4:off + 8], "<f4")[0])
        off += 8
        n1 = 3 * k * hidden
        w1 = np.frombuffer(data[off:off + 4 * n1], "<f4").reshape(3 * k, hidden).copy()
        off += 4 * n1
        b1 = np.frombuffer(data[off:off + 4 * hidden], "<f4").copy()
        off += 4 * hidden
        w2 = np.frombuffer(data[off:off + 4 * hidden], "<f4").copy()
        off += 4 * hidden
        b2 = float(np.frombuffer(data[off:off + 4], "<f4")[0])
        off += 4
        bank[layer] = PredictorWeights(w1, b1, w2, b2, thr)
    return bank


def load_spxs(path):
    """scheduler.py:150-168 (SPXS reader) -> (num_layers, exit_counts)."""
    with open(path, "rb") as fh:
        data = fh.read()
    if data[:4] != b"SPXS":
        raise ValueError("bad magic: not a profile file")
    L = int.from_bytes(data[8:12], "little")
    counts = np.frombuffer(data[12:12 + 8 * L], "<u8").copy()
    return L, counts


# ---------------------------------------------------------------- CPU baseline


def reference_chain(t, hidden, ids, prev, w, threshold, kern=None):
    """One predictor evaluation exactly as the reference executes it
    (engine.py:196-200): sliced_head_logits (model.py:298-314, including the
    strided column gather copy of :313) -> extract_features -> predictor_forward
    -> decide_exit.  ``kern`` is a module exposing the reference's
    matmul_f32/seq_sum_f32 (the reference's own compiled _ckern from
    oracle/_ref when available, else this oracle's strict C kernels)."""
    mm = kern.matmul_f32 if kern is not None else (lambda a, b: matmul(a, b))
    ss = kern.seq_sum_f32 if kern is not None else (lambda x: seq_sum(x))
    h = np.asarray(hidden, np.float32)[None, :]
    d = np.float32(h.shape[-1])
    mean = ss(h) / d
    xc = h - mean[..., None]
    var = ss(xc * xc) / d
    hn = xc / np.sqrt(var + LN_EPS)[..., None] * t["final_norm.g"] + t["final_norm.b"]
    cols = np.ascontiguousarray(t["lm_head"][:, ids])
    logits = mm(np.ascontiguousarray(hn, np.float32), cols)[0]
    # extract_features' validation (predictor.py:47-50)
    if not np.all(np.isfinite(logits)):
        raise ValueError("non-finite speculative logits")
    if abs(float(prev.sum()) - 1.0) > 1e-5:
        raise ValueError("prev_local_probs must sum to 1")
    e = np.exp(logits - np.max(logits))
    local = e / ss(e[None, :])[0]
    f = np.concatenate([logits, local, local - prev]).astype(np.float32)
    z = np.maximum(f @ w.w1 + w.b1, 0) @ w.w2 + w.b2
    prob = float(sigmoid(z))
    return prob > threshold, local
