"""Device-resident decode state with lazy KV completion -- drop-in for the
reference's ``specexit.model.DecodeState`` (src/specexit/model.py:155-286) and
the flag consumer of the early-exit path.

Rows carry a frontier (number of layers whose KV exist).  ``run_layer(l)``
advances every unfrozen row at frontier l -- the newest rows plus rows an
earlier early exit left behind -- through one decoder layer
(spx_layer_forward: 6 sm_100a launches), so positions skipped by an exit are
completed exactly when a later token needs their deeper KV.  All counters
(rows in use, newest row) also live on the device, so a token step can be
enqueued without host synchronisation and captured into a CUDA graph.
"""
import numpy as np
import torch

from . import _native as N
from . import numerics


class DecodeState:
    """KV cache plus lazy-completion bookkeeping for one generation stream."""

    def __init__(self, model, done_flag: torch.Tensor = None, max_context: int = None,
                 row_cap: int = 0, att_cap: int = 0):
        cfg = model.config
        if model.head_only:
            raise ValueError("DecodeState needs a model with decoder layers")
        self.model = model
        # max_context: rows of this state (default: the model's context);
        # row_cap / att_cap: per-call row-set and attention-list bounds for
        # states holding many interleaved streams (BatchedExitEngine)
        L, d, f = cfg.num_layers, cfg.hidden_dim, cfg.ffn_dim
        C = cfg.max_context if max_context is None else int(max_context)
        self.max_context = C
        self.row_cap, self.att_cap = int(row_cap), int(att_cap)
        dev = "cuda"
        self.kcache = torch.zeros((L, C, d), dtype=torch.float32, device=dev)
        self.vcache = torch.zeros_like(self.kcache)
        self.pending = torch.zeros((C, d), dtype=torch.float32, device=dev)
        self.frontier = torch.zeros(C, dtype=torch.int32, device=dev)
        self.frozen = torch.zeros(C, dtype=torch.uint8, device=dev)
        self.n_ctx = torch.zeros(1, dtype=torch.int32, device=dev)
        self.new_row = torch.full((1,), -1, dtype=torch.int32, device=dev)
        self.rows = torch.zeros(C, dtype=torch.int32, device=dev)
        self.nrows = torch.zeros(1, dtype=torch.int32, device=dev)
        self.s_q = torch.zeros((C, d), dtype=torch.float32, device=dev)
        self.s_att = torch.zeros((C, d), dtype=torch.float32, device=dev)
        self.s_f = torch.zeros((C, f), dtype=torch.float32, device=dev)
        self.cur_hidden = torch.zeros(d, dtype=torch.float32, device=dev)
        lib = N.lib()
        self.s_part = torch.zeros(max(1, lib.spx_layer_part_floats(d, f)), dtype=torch.float32,
                                  device=dev)
        self.s_flag = torch.zeros(max(1, lib.spx_layer_flag_ints(d, f)), dtype=torch.int32,
                                  device=dev)
        self.err = torch.zeros(1, dtype=torch.int32, device=dev)
        # tensor-core multi-row path (>= 16 rows per call, bf16 weights)
        self.tc_scratch = None
        if model.spx_dtype == N.SPX_DTYPE_BF16:
            nb = lib.spx_layer_tc_scratch_bytes(d, f, self.row_cap or C)
            if nb > 0:
                # zeroed once: the K-split tile counters at its end self-reset
                self.tc_scratch = torch.zeros(nb, dtype=torch.uint8, device=dev)
        self.attn_ptr = None
        self.attn_idx = None
        self.done = done_flag
        self.n = 0                       # host mirror of n_ctx
        self.new_rows = []
        self._tok_buf = torch.zeros(C, dtype=torch.int32, device=dev)
        self._pos_buf = torch.zeros(C, dtype=torch.int32, device=dev)
        self._any_frozen = False
        self._hint = 0                   # rows appended by the last begin / embed_device
        self._largs = [self._layer_args(l) for l in range(L)]

    @property
    def tokens_capacity_left(self):
        return self.max_context - self.n

    # -- begin (model.py:181-212) -----------------------------------------------

    def begin(self, tokens, pos_ids=None, attn_lists=None):
        cfg = self.model.config
        toks = np.asarray(tokens, dtype=np.int64)
        if toks.ndim != 1 or toks.size == 0:
            raise ValueError("tokens must be a non-empty 1-D sequence")
        if toks.min() < 0 or toks.max() >= cfg.vocab_size:
            raise ValueError("token id out of range")
        if self.n + toks.size > self.max_context:
            raise ValueError("context overflow")
        rows = list(range(self.n, self.n + toks.size))
        self._tok_buf[:toks.size].copy_(torch.as_tensor(toks.astype(np.int32)))
        pos = None
        if pos_ids is not None:
            self._pos_buf[:toks.size].copy_(torch.as_tensor(np.asarray(pos_ids, np.int32)))
            pos = self._pos_buf
        if attn_lists is not None:
            self._set_attn(rows, attn_lists)
        self.embed_device(self._tok_buf, toks.size, pos)
        self._hint = int(toks.size)
        self.n += toks.size
        self.new_rows = rows
        return rows

    def embed_device(self, tokens: torch.Tensor, T: int, pos: torch.Tensor = None):
        """Append T rows whose tokens live in device memory (graph-capturable)."""
        self._hint = int(T)
        m = self.model
        cfg = m.config
        N.check(N.lib().spx_embed(N.ptr(m.embedding), m.spx_dtype, N.ptr(m.pos_encoding),
                                  N.ptr(tokens), N.ptr(pos), T, cfg.hidden_dim, cfg.vocab_size,
                                  self.max_context, N.ptr(self.pending), N.ptr(self.frontier),
                                  N.ptr(self.n_ctx), N.ptr(self.new_row), N.ptr(self.err),
                                  N.stream_ptr()), "spx_embed")

    def _set_attn(self, rows, attn_lists):
        C = self.max_context
        if self.attn_ptr is None:
            self._attn_lists = {}
        for j, p in enumerate(rows):
            lst = attn_lists[j]
            if lst is not None:
                idx = sorted(set(int(a) for a in lst) | {p})
                if idx[-1] > p:
                    raise ValueError("attention index must not look ahead")
                self._attn_lists[p] = idx
        ptr = np.zeros(C + 1, np.int32)
        flat = []
        for p in range(C):
            ptr[p] = len(flat)
            flat.extend(self._attn_lists.get(p, []))
        ptr[C] = len(flat)
        self.attn_ptr = torch.as_tensor(ptr, device="cuda")
        self.attn_idx = torch.as_tensor(np.asarray(flat or [0], np.int32), device="cuda")
        self._largs = [self._layer_args(l) for l in range(self.model.config.num_layers)]

    def set_attention_csr(self, attn_ptr: torch.Tensor, attn_idx: torch.Tensor):
        """Static per-row attention lists (CSR over all max_context rows, each
        list ascending and ending at the row itself): rows of several
        interleaved streams attend only to their own stream's rows."""
        self.attn_ptr, self.attn_idx = attn_ptr, attn_idx
        self._attn_lists = None
        self._largs = [self._layer_args(l) for l in range(self.model.config.num_layers)]

    # -- run_layer (model.py:220-270) --------------------------------------------

    def _layer_args(self, l):
        m, cfg = self.model, self.model.config
        lay = m.layers[l]
        a = N.LayerArgs()
        a.ln1_g, a.ln1_b = N.ptr(lay["ln1_g"]), N.ptr(lay["ln1_b"])
        a.ln2_g, a.ln2_b = N.ptr(lay["ln2_g"]), N.ptr(lay["ln2_b"])
        a.wqkv, a.wo = N.ptr(lay["wqkv"]), N.ptr(lay["wo"])
        a.w1, a.w2 = N.ptr(lay["ffn_w1"]), N.ptr(lay["ffn_w2"])
        a.b1, a.b2 = N.ptr(lay["ffn_b1"]), N.ptr(lay["ffn_b2"])
        a.w_dtype = m.spx_dtype
        a.pending = N.ptr(self.pending)
        a.kcache = N._vp(self.kcache[l].data_ptr())
        a.vcache = N._vp(self.vcache[l].data_ptr())
        a.frontier, a.n_ctx, a.new_row = N.ptr(self.frontier), N.ptr(self.n_ctx), N.ptr(self.new_row)
        a.frozen = N.ptr(self.frozen)
        a.attn_ptr, a.attn_idx = N.ptr(self.attn_ptr), N.ptr(self.attn_idx)
        a.done = N.ptr(self.done)
        a.cur_hidden = N.ptr(self.cur_hidden)
        a.rows, a.nrows = N.ptr(self.rows), N.ptr(self.nrows)
        a.s_q, a.s_att, a.s_f = N.ptr(self.s_q), N.ptr(self.s_att), N.ptr(self.s_f)
        a.s_part, a.s_flag = N.ptr(self.s_part), N.ptr(self.s_flag)
        a.layer = l
        a.err = N.ptr(self.err)
        a.max_ctx, a.d, a.n_heads, a.ffn = self.max_context, cfg.hidden_dim, cfg.num_heads, cfg.ffn_dim
        a.row_cap, a.att_cap = self.row_cap, self.att_cap
        a.tc_scratch = N.ptr(self.tc_scratch)
        return a

    def launch_layer(self, l: int):
        """Enqueue layer l (no host sync; graph-capturable)."""
        a = self._largs[l]
        a.mode = numerics.mode()
        a.rows_hint = self._hint
        N.check(N.lib().spx_layer_forward(a, N.stream_ptr()), "spx_layer_forward")

    def run_layer(self, l: int):
        if not 0 <= l < self.model.config.num_layers:
            raise ValueError("layer index out of range")
        self.launch_layer(l)
        return self.pending[self.new_rows].clone()

    def freeze(self, positions):
        pos = list(positions)
        if pos:
            self.frozen[torch.as_tensor(pos, dtype=torch.long, device="cuda")] = 1

    def unfreeze_all(self):
        self.frozen.zero_()

    def compact(self, keep_new_rows, n_committed):
        """model.py:272-286."""
        keep = torch.as_tensor(list(keep_new_rows), dtype=torch.long, device="cuda")
        dest = torch.arange(n_committed, n_committed + len(keep_new_rows), device="cuda")
        if len(keep_new_rows):
            self.kcache[:, dest] = self.kcache[:, keep]
            self.vcache[:, dest] = self.vcache[:, keep]
            self.pending[dest] = self.pending[keep]
            self.frontier[dest] = self.frontier[keep]
        self.attn_ptr = self.attn_idx = None
        self._attn_lists = {}
        self.n = n_committed + len(keep_new_rows)
        self.n_ctx.fill_(self.n)
        self.new_rows = []
        self.new_row.fill_(-1)
        self.frozen.zero_()
        self._largs = [self._layer_args(l) for l in range(self.model.config.num_layers)]

    def reset(self):
        """Empty the state (buffers kept): n = 0, no rows, nothing frozen."""
        self.n = 0
        self.n_ctx.zero_()
        self.new_row.fill_(-1)
        self.frontier.zero_()
        self.frozen.zero_()
        self.new_rows = []
        if self.attn_ptr is not None and getattr(self, "_attn_lists", {}) is not None:
            self.attn_ptr = self.attn_idx = None
            self._attn_lists = {}
            self._largs = [self._layer_args(l) for l in range(self.model.config.num_layers)]

    def check(self):
        N.raise_device_error(self.err.item())


def forward_to_layer(model, tokens, stop_layer: int, state: DecodeState = None):
    """model.py:317-330: run layers 0..stop_layer for `tokens`."""
    if not 0 <= stop_layer < model.config.num_layers:
        raise ValueError("stop_layer out of range")
    if state is None:
        state = DecodeState(model)
    state.begin(tokens)
    out = None
    for l in range(stop_layer + 1):
        out = state.run_layer(l)
    return out[-1], state


def prefill(model, tokens) -> DecodeState:
    """model.py:344-352."""
    state = DecodeState(model)
    if len(tokens) > 1:
        state.begin(tokens[:-1])
        for l in range(model.config.num_layers):
            state.launch_layer(l)
    return state
