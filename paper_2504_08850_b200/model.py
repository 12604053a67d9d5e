"""Device-resident model weights in B200 layouts plus the head operators --
drop-in for the hot-path part of the reference's ``specexit.model``
(src/specexit/model.py).

Layouts in HBM (the reference keeps (in, out) f32 matrices):
  lm_head      (V, d)      vocab-row major, so a speculative gather reads K
                           contiguous rows (reference stores (d, V) and gathers
                           strided columns, model.py:82, :313)
  embedding    (V, d)
  wqkv         (3d, d)     out-row major [wq^T; wk^T; wv^T]
  wo           (d, d)      wo^T
  ffn_w1       (ffn, d)    ffn.w1^T
  ffn_w2       (d, ffn)    ffn.w2^T
  norms/biases f32
Weight storage is bf16 (production, ``dtype="bf16"``) or f32 (``dtype="f32"``,
exact for reference weights that are not bf16-representable).  Accumulation
is always fp32.
"""
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import numerics, rng

LN_EPS = np.float32(1e-5)                      # model.py:27
CONFIG_FIELDS = ("vocab_size", "hidden_dim", "num_layers", "num_heads", "ffn_dim", "max_context")
_TORCH_DTYPE = {"bf16": torch.bfloat16, "f32": torch.float32}
_SPX_DTYPE = {"bf16": N.SPX_DTYPE_BF16, "f32": N.SPX_DTYPE_F32}


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

    def validate(self):
        if self.vocab_size < 2:
            raise ValueError("vocab_size must be >= 2")
        if self.num_layers < 1:
            raise ValueError("num_layers must be >= 1")
        if min(self.hidden_dim, self.num_heads, self.ffn_dim, self.max_context) < 1:
            raise ValueError("all dimensions must be positive")
        if self.hidden_dim % self.num_heads != 0:
            raise ValueError("hidden_dim must be divisible by num_heads")
        if not 0 <= self.seed < 2 ** 64:
            raise ValueError("seed must fit in 64 bits")

    @property
    def head_dim(self):
        return self.hidden_dim // self.num_heads


def tensor_specs(config: ModelConfig):
    """model.py:59-84 -- declaration order fixes each tensor's seed index."""
    d, f, v = config.hidden_dim, config.ffn_dim, config.vocab_size
    specs = [("embedding", (v, d), "uniform")]
    for i in range(config.num_layers):
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


def sinusoidal_encoding(max_len: int, dim: int) -> np.ndarray:
    """model.py:112-118 (host, float64 then float32)."""
    pe = np.zeros((max_len, dim), dtype=np.float64)
    pos = np.arange(max_len)[:, None]
    div = np.exp(np.arange(0, dim, 2) * (-math.log(10000.0) / dim))
    pe[:, 0::2] = np.sin(pos * div)
    pe[:, 1::2] = np.cos(pos * div)
    return pe.astype(np.float32)


# name suffix -> (device attribute, transpose-to-out-major)
_LAYER_MAT = {"attn.wq": ("wqkv", 0), "attn.wk": ("wqkv", 1), "attn.wv": ("wqkv", 2),
              "attn.wo": ("wo", None), "ffn.w1": ("ffn_w1", None), "ffn.w2": ("ffn_w2", None)}
_LAYER_VEC = {"ln1.g": "ln1_g", "ln1.b": "ln1_b", "ln2.g": "ln2_g", "ln2.b": "ln2_b",
              "ffn.b1": "ffn_b1", "ffn.b2": "ffn_b2"}


CERT_LAMBDA = 8.0     # rounding-error model multiplier


class TransformerModel:
    """Immutable device weights of one model (target or draft).  Shareable
    across engines/streams (reference SPEC.md:112)."""

    def __init__(self, config: ModelConfig, dtype: str = "bf16", head_only: bool = False):
        config.validate()
        if dtype not in _TORCH_DTYPE:
            raise ValueError(f"unknown weight dtype {dtype!r}")
        if config.hidden_dim % 8:
            raise ValueError("hidden_dim must be a multiple of 8 on the B200 path")
        N.require_cuda()
        self.config, self.dtype, self.head_only = config, dtype, head_only
        self.spx_dtype = _SPX_DTYPE[dtype]
        td = _TORCH_DTYPE[dtype]
        d, f, v, L = config.hidden_dim, config.ffn_dim, config.vocab_size, config.num_layers
        dev = "cuda"
        self.lm_head = torch.empty((v, d), dtype=td, device=dev)
        self.final_g = torch.ones(d, dtype=torch.float32, device=dev)
        self.final_b = torch.zeros(d, dtype=torch.float32, device=dev)
        self.layers = []
        if not head_only:
            self.embedding = torch.empty((v, d), dtype=td, device=dev)
            self.pos_encoding = torch.as_tensor(sinusoidal_encoding(config.max_context, d),
                                                device=dev)
            for _ in range(L):
                self.layers.append({
                    "ln1_g": torch.ones(d, device=dev), "ln1_b": torch.zeros(d, device=dev),
                    "wqkv": torch.empty((3 * d, d), dtype=td, device=dev),
                    "wo": torch.empty((d, d), dtype=td, device=dev),
                    "ln2_g": torch.ones(d, device=dev), "ln2_b": torch.zeros(d, device=dev),
                    "ffn_w1": torch.empty((f, d), dtype=td, device=dev),
                    "ffn_b1": torch.zeros(f, device=dev),
                    "ffn_w2": torch.empty((d, f), dtype=td, device=dev),
                    "ffn_b2": torch.zeros(d, device=dev)})

    # -- construction -------------------------------------------------------

    def _target(self, name):
        """(tensor, transpose flag) receiving reference tensor `name`."""
        d = self.config.hidden_dim
        if name == "lm_head":
            return self.lm_head, True
        if name == "embedding":
            return (None if self.head_only else self.embedding), False
        if name == "final_norm.g":
            return self.final_g, False
        if name == "final_norm.b":
            return self.final_b, False
        _, i, rest = name.split(".", 2)
        if self.head_only:
            return None, False
        lay = self.layers[int(i)]
        if rest in _LAYER_VEC:
            return lay[_LAYER_VEC[rest]], False
        attr, part = _LAYER_MAT[rest]
        t = lay[attr]
        if part is not None:
            t = t[part * d:(part + 1) * d]
        return t, True

    def finalize(self):
        """Derived per-model constants once the weights are in place: the
        final-norm bias folded through the head, bw[v] = CDOT(b, head_v), used
        by the fast head kernels (logit = r * CDOT(xg, head_v) + bw[v])."""
        self.head_bw = torch.empty(self.config.vocab_size, dtype=torch.float32, device="cuda")
        N.check(N.lib().spx_head_bias(N.ptr(self.lm_head), self.spx_dtype, N.ptr(self.final_b),
                                      self.config.vocab_size, self.config.hidden_dim,
                                      N.ptr(self.head_bw), N.stream_ptr()), "spx_head_bias")
        # constants of the FAST-decision certification bound:
        # per-row max |W_v|, ||LN(h)|| <= max|g| sqrt(d) + ||b||, kappa = 2 lambda u sqrt(d)
        d = self.config.hidden_dim
        self.head_wmax = torch.empty(self.config.vocab_size, dtype=torch.float32, device="cuda")
        N.check(N.lib().spx_head_stats(N.ptr(self.lm_head), self.spx_dtype,
                                       self.config.vocab_size, d, N.ptr(self.head_wmax),
                                       N.stream_ptr()), "spx_head_stats")
        gmax = float(self.final_g.abs().max())
        bnorm = float(self.final_b.double().norm())
        self.cert_hnorm = (gmax * math.sqrt(d) + bnorm) * (1 + 1e-6)
        self.cert_kappa = 2.0 * CERT_LAMBDA * 2.0 ** -24 * math.sqrt(d)
        return self

    def numel(self):
        n = self.lm_head.numel() + 2 * self.config.hidden_dim
        if not self.head_only:
            n += self.embedding.numel() + sum(t.numel() for lay in self.layers for t in lay.values())
        return n

    def nbytes(self):
        tot = self.lm_head.numel() * self.lm_head.element_size()
        for lay in self.layers:
            tot += sum(t.numel() * t.element_size() for t in lay.values())
        return tot


def init_model(config: ModelConfig, dtype: str = "bf16", head_only: bool = False) -> TransformerModel:
    """model.py:121-137 evaluated on device (spx_init_uniform): the same
    splitmix64 stream per tensor in declaration order, uniform(+-sqrt(6/(fan_in+
    fan_out))), biases 0, gains 1 -- then stored as bf16 (RNE) or f32."""
    m = TransformerModel(config, dtype, head_only)
    L = N.lib()
    for idx, (name, shape, kind) in enumerate(tensor_specs(config)):
        if kind != "uniform":
            continue                         # ones/zeros already in place
        t, transpose = m._target(name)
        if t is None:
            continue
        b = math.sqrt(6.0 / (shape[0] + shape[1]))
        is_f32 = t.dtype == torch.float32
        assert t.is_contiguous()
        N.check(L.spx_init_uniform(N.ptr(t), int(is_f32), shape[0], shape[1], int(transpose),
                                   rng.derive(config.seed, idx), -b, b, N.stream_ptr()),
                "spx_init_uniform")
    m.finalize()
    return m


def from_tensors(config: ModelConfig, tensors: dict, dtype: str = "f32",
                 head_only: bool = False) -> TransformerModel:
    """Device model from reference-layout float32 tensors (e.g. a
    ``TransformerModel.tensors`` dict of the reference, or SPXW contents)."""
    expected = tensor_specs(config)
    for name, shape, _ in expected:
        if name not in tensors:
            if head_only and name.startswith("layers."):
                continue
            raise ValueError("tensor names do not match config")
        t = np.asarray(tensors[name])
        if t.shape != shape:
            raise ValueError(f"tensor {name}: bad shape/dtype {t.shape}/{t.dtype}")
        if not np.all(np.isfinite(t)):
            raise ValueError(f"tensor {name}: non-finite values")
    m = TransformerModel(config, dtype, head_only)
    for name, _, _ in expected:
        dst, transpose = m._target(name)
        if dst is None:
            continue
        src = torch.from_numpy(np.array(tensors[name], dtype=np.float32, order="C"))
        if transpose:
            src = src.t()
        dst.copy_(src.to(dst.dtype))
    m.finalize()
    return m


# --- SPXW (model.py:355-434) -----------------------------------------------------


def load_weights(path, dtype: str = "f32") -> TransformerModel:
    """Read a reference SPXW weight file into device layouts."""
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
    version = int.from_bytes(take(4), "little")
    if version != 1:
        raise ValueError(f"unsupported weight file version {version}")
    count = int.from_bytes(take(4), "little")
    tensors = {}
    for _ in range(count):
        nlen = int.from_bytes(take(2), "little")
        name = take(nlen).decode()
        rank = int.from_bytes(take(1), "little")
        shape = tuple(int.from_bytes(take(4), "little") for _ in range(rank))
        n = int(np.prod(shape)) if shape else 1
        tensors[name] = np.frombuffer(take(4 * n), "<f4").reshape(shape)
    if "config" not in tensors:
        raise ValueError("weight file missing config pseudo-tensor")
    vec = tensors.pop("config")
    if vec.size != len(CONFIG_FIELDS) + 4:
        raise ValueError("bad config pseudo-tensor length")
    fields = {f: int(v) for f, v in zip(CONFIG_FIELDS, vec)}
    seed = sum(int(v) << (16 * i) for i, v in enumerate(vec[len(CONFIG_FIELDS):]))
    return from_tensors(ModelConfig(seed=seed, **fields), tensors, dtype)


def to_tensors(model: TransformerModel) -> dict:
    """Reference-layout float32 tensors of a device model (the inverse of
    ``from_tensors``; bf16 weights widen exactly)."""
    if model.head_only:
        raise ValueError("head-only model has no decoder weights to export")
    out = {}
    for name, _, _ in tensor_specs(model.config):
        src, transpose = model._target(name)
        t = src.t() if transpose else src
        out[name] = t.to(torch.float32).cpu().numpy().copy()
    return out


def save_weights(model: TransformerModel, path):
    """SPXW writer (model.py:408-417): magic, u32 version 1, u32 count, the
    "config" pseudo-tensor (config fields + the seed as four 16-bit limbs),
    then every tensor in declaration order as u16 name length, name, u8 rank,
    u32 dims, f32 LE data."""
    cfg = model.config
    vec = np.array([getattr(cfg, f) for f in CONFIG_FIELDS]
                   + [(cfg.seed >> s) & 0xFFFF for s in (0, 16, 32, 48)], dtype=np.float32)
    tensors = to_tensors(model)

    def put(fh, name, arr):
        nb = name.encode()
        fh.write(len(nb).to_bytes(2, "little") + nb + arr.ndim.to_bytes(1, "little"))
        fh.write(b"".join(int(s).to_bytes(4, "little") for s in arr.shape))
        fh.write(np.ascontiguousarray(arr, dtype="<f4").tobytes())

    with open(path, "wb") as fh:
        fh.write(b"SPXW" + (1).to_bytes(4, "little") + (len(tensors) + 1).to_bytes(4, "little"))
        put(fh, "config", vec)
        for name, arr in tensors.items():
            put(fh, name, arr)


# --- head operators (the function-level drop-ins) --------------------------------


def _rows(hidden, d):
    h = hidden if isinstance(hidden, torch.Tensor) else torch.as_tensor(np.asarray(hidden, np.float32))
    h = h.to(device="cuda", dtype=torch.float32)
    if h.dim() == 1:
        h = h.reshape(1, -1)
    if h.shape[-1] != d:
        raise ValueError("hidden dimension mismatch")
    return h.contiguous()


def final_norm(model: TransformerModel, hidden) -> torch.Tensor:
    """Final LayerNorm of (N, d) rows (model.py:140-146 with final_norm.*)."""
    h = _rows(hidden, model.config.hidden_dim)
    out = torch.empty_like(h)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().spx_final_norm(N.ptr(h), h.shape[1], N.ptr(model.final_g),
                                   N.ptr(model.final_b), N.ptr(out), h.shape[0], h.shape[1],
                                   numerics.mode(), N.ptr(err), N.stream_ptr()), "spx_final_norm")
    N.raise_device_error(err.item())
    return out


def head_prep(model: TransformerModel, hidden):
    """(xg, r) of (N, d) rows for the fast head kernels (spx_head_prep); in
    strict mode xg is the reference LayerNorm and r = 1."""
    h = _rows(hidden, model.config.hidden_dim)
    xg = torch.empty_like(h)
    r = torch.empty(h.shape[0], dtype=torch.float32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().spx_head_prep(N.ptr(h), h.shape[1], N.ptr(model.final_g), N.ptr(model.final_b),
                                  N.ptr(xg), N.ptr(r), h.shape[0], h.shape[1], numerics.mode(),
                                  N.ptr(err), N.stream_ptr()), "spx_head_prep")
    N.raise_device_error(err.item())
    return xg, r


# K6 on the tensor cores when the merged node x unique-id tile is a real dense
# contraction (north-star (e)): at least TC_MIN_ROWS nodes and TC_MIN_UNIQUE
# unique ids with a requested fraction >= TC_MIN_DENSITY of the dense tile.
TC_MIN_ROWS, TC_MIN_UNIQUE, TC_MIN_DENSITY = 64, 64, 0.25
_TC_SCRATCH = {}


def _tc_scratch(nbytes):
    key = torch.cuda.current_device()
    buf = _TC_SCRATCH.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.zeros(max(nbytes, 1 << 20), dtype=torch.uint8, device="cuda")
        _TC_SCRATCH[key] = buf
    return buf


def use_tensor_cores(model, n_rows, n_unique, n_pairs) -> bool:
    """The dispatch rule of K6 (FAST mode, bf16 head)."""
    return (numerics.mode() == N.SPX_MODE_FAST and model.spx_dtype == N.SPX_DTYPE_BF16 and
            model.config.hidden_dim % 64 == 0 and n_rows >= TC_MIN_ROWS and
            n_unique >= TC_MIN_UNIQUE and n_pairs >= TC_MIN_DENSITY * n_rows * n_unique)


def merged_logits(model: TransformerModel, prep, id_lists, tensor_cores=None) -> list:
    """K6: logits of node j for id_lists[j], one HBM read per unique id.
    prep = head_prep(model, rows).  tensor_cores: None = the dispatch rule
    (use_tensor_cores), True / False to force the tcgen05 / CUDA-core kernel."""
    xg, rr = prep
    flat = np.concatenate([np.asarray(ids, np.int64).reshape(-1) for ids in id_lists])
    sizes = [len(ids) for ids in id_lists]
    node = np.repeat(np.arange(len(id_lists), dtype=np.int64), sizes)
    out_idx = np.arange(flat.size, dtype=np.int64)
    if flat.size and (flat.min() < 0 or flat.max() >= model.config.vocab_size):
        raise ValueError("token id out of range")
    uniq, inv = np.unique(flat, return_inverse=True)
    order = np.argsort(inv, kind="stable")
    counts = np.bincount(inv, minlength=uniq.size)
    uptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    dev = lambda a: torch.as_tensor(np.ascontiguousarray(a, np.int32), device="cuda")  # noqa: E731
    d_uniq, d_uptr = dev(uniq), dev(uptr)
    d_node, d_out = dev(node[order]), dev(out_idx[order])
    logits = torch.empty(flat.size, dtype=torch.float32, device="cuda")
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    if tensor_cores is None:
        tensor_cores = use_tensor_cores(model, xg.shape[0], uniq.size, flat.size)
    if tensor_cores and flat.size:
        lib = N.lib()
        nb = lib.spx_tree_tc_scratch_bytes(xg.shape[0], model.config.hidden_dim, uniq.size,
                                           flat.size)
        scratch = _tc_scratch(nb)
        d_uid = dev(inv[order])
        N.check(lib.spx_tree_merged_logits_tc(
            N.ptr(xg), N.ptr(rr), xg.shape[0], N.ptr(model.lm_head), model.spx_dtype,
            N.ptr(model.head_bw), model.config.vocab_size, model.config.hidden_dim,
            N.ptr(d_uniq), uniq.size, N.ptr(d_uptr), N.ptr(d_node), N.ptr(d_out), N.ptr(d_uid),
            flat.size,
            N.ptr(logits), N.ptr(scratch), N.ptr(err), N.stream_ptr()),
            "spx_tree_merged_logits_tc")
        N.raise_device_error(err.item())
        return list(torch.split(logits, sizes))
    N.check(N.lib().spx_tree_merged_logits(N.ptr(xg), N.ptr(rr), xg.shape[0], N.ptr(model.lm_head),
                                           model.spx_dtype, N.ptr(model.head_bw),
                                           model.config.vocab_size,
                                           model.config.hidden_dim, N.ptr(d_uniq), uniq.size,
                                           N.ptr(d_uptr), N.ptr(d_node), N.ptr(d_out),
                                           N.ptr(logits), numerics.mode(), N.ptr(err),
                                           N.stream_ptr()),
            "spx_tree_merged_logits")
    N.raise_device_error(err.item())
    return list(torch.split(logits, sizes))


def sliced_head_logits(model: TransformerModel, hidden, token_ids) -> torch.Tensor:
    """model.py:298-314: logits of selected vocabulary rows only (K1 order)."""
    ids = np.asarray(token_ids.cpu() if isinstance(token_ids, torch.Tensor) else token_ids,
                     dtype=np.int64).reshape(-1)
    if ids.size == 0:
        raise ValueError("empty token id list")
    if ids.min() < 0 or ids.max() >= model.config.vocab_size:
        raise ValueError("token id out of range")
    return merged_logits(model, head_prep(model, hidden), [ids])[0]


class _VerifyScratch:
    _per_device = {}

    @classmethod
    def get(cls, B):
        key = torch.cuda.current_device()
        s = cls._per_device.get(key)
        if s is None or s[0].numel() < B:
            s = (torch.zeros(max(B, 64), dtype=torch.int64, device="cuda"),
                 torch.zeros(1, dtype=torch.int32, device="cuda"))
            cls._per_device[key] = s
        return s


def verify_args(model: TransformerModel, hidden: torch.Tensor, B: int, token_out, scratch,
                counter, err, **kw) -> N.VerifyArgs:
    """spx_verify_args for B rows of `hidden` (row stride hidden.stride(0), or
    a (d) vector for B == 1); keyword arguments name the optional device
    pointers of the struct (gate, row_done, spec_ptr, spec_ids, verified_out,
    maxlogit_out, logits_out, done_out, exit_layer_out, full_heads) plus
    `layer` and `mode`.  Nothing is launched."""
    a = N.VerifyArgs()
    a.hidden = N.ptr(hidden)
    a.hidden_stride = hidden.stride(0) if hidden.dim() == 2 else model.config.hidden_dim
    a.norm_g, a.norm_b = N.ptr(model.final_g), N.ptr(model.final_b)
    a.head, a.head_dtype, a.head_bw = N.ptr(model.lm_head), model.spx_dtype, N.ptr(model.head_bw)
    for name in ("gate", "row_done", "spec_ptr", "spec_ids", "verified_out", "maxlogit_out",
                 "logits_out", "done_out", "exit_layer_out", "full_heads"):
        setattr(a, name, N.ptr(kw.get(name)))
    a.token_out = N.ptr(token_out)
    a.layer = int(kw.get("layer", 0))
    a.scratch, a.counter = N.ptr(scratch), N.ptr(counter)
    mode = kw.get("mode")
    a.mode, a.err = numerics.mode() if mode is None else mode, N.ptr(err)
    a.B, a.d, a.V = B, model.config.hidden_dim, model.config.vocab_size
    # many rows, bf16 head: the tensor-core form of K4 (spx_verify_tc.cuh) --
    # same tokens / flags; the library picks it only where it applies
    if (kw.get("tensor_cores", True)
            and (B >= N.SPX_VERIFY_TC_MIN_ROWS or kw.get("topk_out") is not None)
            and model.dtype == "bf16" and model.config.hidden_dim % 64 == 0
            and kw.get("logits_out") is None):
        a.head_wmax = N.ptr(model.head_wmax)
        a.tc_scratch = N.ptr(_verify_tc_scratch(B, model.config.hidden_dim, model.config.vocab_size))
        if kw.get("topk_out") is not None:
            a.topk_out, a.topk_k = N.ptr(kw["topk_out"]), int(kw["topk_k"])
    return a


_TC_VERIFY_SCRATCH = {}


def _verify_tc_scratch(B, d, V):
    key = (torch.cuda.current_device(), B, d, V)
    t = _TC_VERIFY_SCRATCH.get(key)
    if t is None:
        t = torch.empty(int(N.lib().spx_verify_tc_scratch_bytes(B, d, V)), dtype=torch.uint8,
                        device="cuda")
        _TC_VERIFY_SCRATCH[key] = t
    return t


def launch_verify(args: N.VerifyArgs, mode: int = None):
    """Enqueue one spx_verify on the current stream (no sync)."""
    if mode is not None:
        args.mode = mode
    N.check(N.lib().spx_verify(args, N.stream_ptr()), "spx_verify")


def head_argmax(model: TransformerModel, hidden, spec_lists=None, want_logits=False):
    """K4 on N rows: (tokens, verified, logits|None).  spec_lists: per-row
    verify sets (or None)."""
    h = _rows(hidden, model.config.hidden_dim)
    B, V = h.shape[0], model.config.vocab_size
    tok = torch.empty(B, dtype=torch.int32, device="cuda")
    ver = torch.zeros(B, dtype=torch.uint8, device="cuda")
    logits = torch.empty((B, V), dtype=torch.float32, device="cuda") if want_logits else None
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    scratch, counter = _VerifyScratch.get(B)
    d_ptr = d_ids = None
    if spec_lists is not None:
        ptr_ = np.concatenate([[0], np.cumsum([len(s) for s in spec_lists])]).astype(np.int32)
        ids = np.concatenate([np.asarray(s, np.int32).reshape(-1) for s in spec_lists]
                             ) if len(spec_lists) else np.zeros(0, np.int32)
        d_ptr = torch.as_tensor(ptr_, device="cuda")
        d_ids = torch.as_tensor(np.ascontiguousarray(ids, np.int32), device="cuda") \
            if ids.size else d_ptr
    a = verify_args(model, h, B, tok, scratch, counter, err, spec_ptr=d_ptr, spec_ids=d_ids,
                    verified_out=ver, logits_out=logits)
    launch_verify(a)
    N.raise_device_error(err.item())
    return tok, ver, logits


def full_head_logits(model: TransformerModel, hidden) -> torch.Tensor:
    """model.py:289-295: final norm then the full LM-head projection."""
    _, _, logits = head_argmax(model, hidden, want_logits=True)
    return logits[0] if (isinstance(hidden, torch.Tensor) and hidden.dim() == 1) or \
        np.ndim(hidden) == 1 else logits


def layer_norm(x, g, b) -> torch.Tensor:
    """model.py:140-146 for (n, d) rows with arbitrary gain/bias on device."""
    h = _rows(x, int(np.shape(x)[-1]))
    gt = torch.as_tensor(np.asarray(g, np.float32) if not isinstance(g, torch.Tensor) else g,
                         device="cuda", dtype=torch.float32).contiguous()
    bt = torch.as_tensor(np.asarray(b, np.float32) if not isinstance(b, torch.Tensor) else b,
                         device="cuda", dtype=torch.float32).contiguous()
    out = torch.empty_like(h)
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().spx_final_norm(N.ptr(h), h.shape[1], N.ptr(gt), N.ptr(bt), N.ptr(out),
                                   h.shape[0], h.shape[1], numerics.mode(), N.ptr(err),
                                   N.stream_ptr()), "spx_final_norm")
    return out
