"""Early exiting under tree speculative decoding -- drop-in for the hot-path
part of the reference's ``specexit.tree`` (src/specexit/tree.py).

``grouped_speculative_logits`` is the context-aware merged mapping (K6): the
feature ids of all live nodes are de-duplicated and each unique LM-head row is
read from HBM once; ``path_conjunction`` is K7 (hyper-token AND over a CSR of
paths) on device.
"""
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from . import numerics
from .decode import DecodeState
from .model import (TransformerModel, _VerifyScratch, full_head_logits, head_prep, launch_verify,
                    merged_logits, verify_args)
from .predictor import decide_exit, extract_features, z_cut
from .scheduler import OfflineProfile, OnlineState, ScheduleConfig, active_layers, update_online
from .speculation import (SpeculativeSet, TokenTree, TreeNode, build_token_tree,
                          enumerate_paths, propose_topk, speculative_set_from_logits,
                          speculative_sets_from_rows)


def grouped_speculative_logits(model: TransformerModel, hiddens, token_id_lists):
    """tree.py:92-113: row j holds the logits of token_id_lists[j];
    bit-identical to sliced_head_logits on that node alone."""
    h = hiddens if isinstance(hiddens, torch.Tensor) else torch.as_tensor(
        np.asarray(hiddens, dtype=np.float32))
    if h.dim() != 2 or h.shape[0] < 1:
        raise ValueError("need at least one node hidden state")
    if len(token_id_lists) != h.shape[0]:
        raise ValueError("one id list per node required")
    v = model.config.vocab_size
    for ids in token_id_lists:
        if len(ids) == 0:
            raise ValueError("empty token id list")
        if min(ids) < 0 or max(ids) >= v:
            raise ValueError("token id out of range")
    return merged_logits(model, head_prep(model, h), token_id_lists)


def hypertoken_exit_decision(per_node_probs, threshold: float) -> bool:
    """tree.py:116-122: the slowest node gates the whole hyper-token."""
    probs = list(per_node_probs)
    if not probs:
        raise ValueError("need at least one node probability")
    return all(decide_exit(p, threshold) for p in probs)


def path_conjunction(node_fired: torch.Tensor, paths, live=None) -> torch.Tensor:
    """K7 on device: path_fire[p] = AND_j node_fired[paths[p][j]] (live paths)."""
    ptr_ = np.concatenate([[0], np.cumsum([len(p) for p in paths])]).astype(np.int32)
    nodes = np.concatenate([np.asarray(p, np.int32) for p in paths]).astype(np.int32)
    d_ptr = torch.as_tensor(ptr_, device="cuda")
    d_nodes = torch.as_tensor(nodes, device="cuda")
    d_live = None if live is None else torch.as_tensor(np.asarray(live, np.uint8), device="cuda")
    out = torch.empty(len(paths), dtype=torch.uint8, device="cuda")
    nf = node_fired.to(device="cuda", dtype=torch.uint8).contiguous()
    N.check(N.lib().spx_path_and(N.ptr(nf), N.ptr(d_ptr), N.ptr(d_nodes), N.ptr(d_live),
                                 len(paths), N.ptr(out), N.stream_ptr()), "spx_path_and")
    return out


# --------------------------------------------------------------------- engine


@dataclass
class HyperToken:
    """tree.py:23-34: one root-to-leaf path of the draft tree."""
    path: list
    per_node_spec: list
    per_node_feature_spec: list = None

    def feature_spec(self, pos):
        if self.per_node_feature_spec is None:
            return self.per_node_spec[pos]
        return self.per_node_feature_spec[pos]


@dataclass
class TreeStepResult:
    """tree.py:37-46."""
    accepted_tokens: list
    correction_token: int
    path_exit_layers: list
    accepted_path: int
    predictor_evals: int
    num_paths: int
    max_path_len: int
    scheduled_layer_count: int


def merge_paths(tree: TokenTree, draft: TransformerModel = None, context=None, k: int = 4,
                propose=None):
    """tree.py:49-89: one HyperToken per leaf; feature set = the draft's top-k
    at the node's own context (cached per node); verify set = the node's
    children for internal nodes, the feature set for leaves."""
    paths = enumerate_paths(tree)
    child_map = {}
    for j, n in enumerate(tree.nodes):
        child_map.setdefault(n.parent, []).append(j)
    cache = {}
    if propose is None and draft is not None:
        propose = lambda ctx, kk: propose_topk(draft, ctx, kk)  # noqa: E731

    def node_topk(idx, path):
        if idx not in cache:
            if propose is None or context is None:
                raise ValueError("speculative sets need the draft model and context")
            upto = path[: path.index(idx) + 1]
            cache[idx] = propose(list(context) + [tree.nodes[i].token for i in upto], k)
        return cache[idx]

    hts = []
    for path in paths:
        specs, fspecs = [], []
        for idx in path:
            kids = child_map.get(idx)
            fspecs.append(node_topk(idx, path))
            if kids:
                specs.append(SpeculativeSet(tokens=tuple(tree.nodes[c].token for c in kids),
                                            draft_probs=tuple(tree.nodes[c].prob for c in kids)))
            else:
                specs.append(fspecs[-1])
        hts.append(HyperToken(path=path, per_node_spec=specs, per_node_feature_spec=fspecs))
    return hts


def hypertoken_oracle_exit(target: TransformerModel, context, path_tokens) -> int:
    """tree.py:125-130: rearmost of the per-node oracle exit layers."""
    from .engine import oracle_exit_layer
    context = list(context)
    return max(oracle_exit_layer(target, context + list(path_tokens[:j]))
               for j in range(len(path_tokens)))


def _i32(a):
    return torch.as_tensor(np.ascontiguousarray(np.asarray(a, np.int64), np.int32), device="cuda")


class TreeEngine:
    """tree.py:133-302: tree speculative decoding with hyper-token exits.

    Per active layer the whole decision block runs as device launches and
    ONE host read-back (tree.py:199-232):
      spx_head_prep      final-norm statistics of every tree row
      K6 merged logits   the live nodes' feature ids de-duplicated: each unique
                         LM-head row read once (context-aware merged mapping)
      spx_tree_node_eval features vs each node's carried probabilities + MLP
                         (or the constant policy) -> fired[node]
      K7 spx_path_and    hyper-token conjunction over live paths
      K7b spx_tree_gate  rows whose full-head argmax is needed
      K4 spx_verify      gated argmax + membership in each node's verify set
      K7 spx_path_and    path verified = AND of its nodes' membership
    then path_ok / argmax tokens come back and the host retires exited paths
    and freezes rows no live path needs (the reference's control flow)."""

    def __init__(self, target: TransformerModel, draft: TransformerModel, policy,
                 branching=(3, 2), config=None, profile: OfflineProfile = None,
                 schedule_config: ScheduleConfig = ScheduleConfig()):
        from .engine import EngineConfig
        config = EngineConfig() if config is None else config
        if config.schedule_mode == "two-level" and profile is None:
            raise ValueError("two-level scheduling needs an offline profile")
        self.target, self.draft, self.policy = target, draft, policy
        self.branching = tuple(branching)
        self.config, self.profile, self.schedule_config = config, profile, schedule_config
        self.online = OnlineState(target.config.num_layers, schedule_config)
        self.tstate = None
        self._dstate = None
        self.context = None
        self.record_probs = False          # diagnostic: per-call (layer, prob) log
        self.prob_log = []

    # -- reference API -------------------------------------------------------------

    def start(self, prompt):
        prompt = [int(t) for t in prompt]
        if not prompt:
            raise ValueError("empty prompt")
        if self.tstate is None:
            self.tstate = DecodeState(self.target)
        else:
            self.tstate.reset()
        if self._dstate is None:
            self._dstate = DecodeState(self.draft)
        else:
            self._dstate.reset()
        if len(prompt) > 1:
            for st, m in ((self.tstate, self.target), (self._dstate, self.draft)):
                st.begin(prompt[:-1])
                for l in range(m.config.num_layers):
                    st.launch_layer(l)
        # the online window persists across generate() calls, as in the
        # reference (tree.py:133-170 creates it once, start() keeps it)
        self.context = prompt
        self.policy.start(prompt)

    def _draft_tree(self):
        """build_token_tree + the per-node draft top-k of merge_paths
        (speculation.py:87-125, tree.py:64-73) with a persistent draft KV cache:
        the draft state holds context[:-1]; the tree is drafted level by level,
        each level ONE batched forward of its nodes at positions m + depth with
        ancestor-only attention -- exactly the keys and positions of the
        reference's fresh full-context forward per node (speculation.py:63-68),
        so the node logits are the same.  Returns (tree, node logits)."""
        from .model import head_argmax
        ds, d = self._dstate, self.draft
        ctx = self.context
        m = len(ctx) - 1
        total, cnt = 1, 1
        for b in self.branching:
            cnt *= b
            total += cnt
        if len(ctx) + total > d.config.max_context:
            raise ValueError("tree exceeds max context")
        nodes = [TreeNode(token=int(ctx[-1]), parent=-1, depth=0)]
        anc = {0: [0]}
        level = [0]
        logits = {}
        K = self.config.k
        k_sets = {}
        kmax = max([K] + list(self.branching))
        fast_sets = (getattr(self, "tc_draft", True) and numerics.mode() != N.SPX_MODE_STRICT
                     and d.dtype == "bf16"
                     and d.config.hidden_dim % 64 == 0 and 1 <= kmax <= min(64, d.config.vocab_size))
        for depth in range(len(self.branching) + 1):
            toks = [nodes[j].token for j in level]
            if depth == 0:
                ds.begin(toks)
            else:
                ds.begin(toks, pos_ids=[m + depth] * len(level),
                         attn_lists=[list(range(m)) + [m + a for a in anc[j]] for j in level])
            for l in range(d.config.num_layers):
                ds.launch_layer(l)
            r0 = ds.n - len(level)
            last = depth == len(self.branching)
            if fast_sets:
                # FAST, bf16 draft: K4's tensor-core form gives each node's
                # exact stable top-max(K, b) ids (CDOT order, as the full
                # logits would) without writing the (n, V) logits; the
                # probabilities are the softmax of its tensor-core logits
                # (FAST tolerance).  The first K ids are the node's feature
                # set (merge_paths), the first b its children.
                b = 0 if last else self.branching[depth]
                kk = max(K, b)
                ids_h, pr_h = self._level_topk(ds.pending[r0:ds.n], len(level), kk)
                for i, j in enumerate(level):
                    k_sets[(j, K)] = SpeculativeSet(tokens=tuple(int(t) for t in ids_h[i, :K]),
                                                    draft_probs=tuple(float(p) for p in pr_h[i, :K]))
                if last:
                    break
                sets = [SpeculativeSet(tokens=tuple(int(t) for t in ids_h[i, :b]),
                                       draft_probs=tuple(float(p) for p in pr_h[i, :b]))
                        for i in range(len(level))]
            else:
                _, _, lg = head_argmax(d, ds.pending[r0:ds.n], want_logits=True)
                for i, j in enumerate(level):
                    logits[j] = lg[i]
                if last:
                    break
                sets = speculative_sets_from_rows(lg, self.branching[depth])    # one host read
            nxt = []
            for i, j in enumerate(level):
                spec = sets[i]
                for tok, pr in zip(spec.tokens, spec.draft_probs):
                    nodes.append(TreeNode(token=int(tok), parent=j, depth=depth + 1, prob=pr))
                    c = len(nodes) - 1
                    anc[c] = anc[j] + [c]
                    nxt.append(c)
            level = nxt
        return TokenTree(nodes=nodes, branching=self.branching), logits, k_sets

    def _level_topk(self, hidden, n, kk):
        """Exact stable top-kk ids of n draft rows (tensor-core K4 with
        candidate re-evaluation) and FAST softmax probabilities at those ids
        from the tensor-core logits; one host read."""
        from .model import _VerifyScratch, _verify_tc_scratch, launch_verify, verify_args
        d = self.draft
        V, D = d.config.vocab_size, d.config.hidden_dim
        ids = torch.empty((n, kk), dtype=torch.int32, device="cuda")
        tok = torch.empty(n, dtype=torch.int32, device="cuda")
        err = torch.zeros(1, dtype=torch.int32, device="cuda")
        scratch, counter = _VerifyScratch.get(n)
        a = verify_args(d, hidden, n, tok, scratch, counter, err, topk_out=ids, topk_k=kk,
                        mode=N.SPX_MODE_FAST)
        launch_verify(a)
        tl = _verify_tc_scratch(n, D, V)
        off = int(N.lib().spx_verify_tc_logits_offset(n, D, V))
        probs = torch.empty((n, kk), dtype=torch.float32, device="cuda")
        N.check(N.lib().spx_softmax_pick(tl.data_ptr() + off, n, V, N.ptr(ids), kk, N.ptr(probs),
                                         N.SPX_MODE_FAST, N.ptr(err), N.stream_ptr()),
                "spx_softmax_pick")
        hb = torch.cat([ids.to(torch.float64).view(-1), probs.to(torch.float64).view(-1),
                        err.to(torch.float64)]).cpu().numpy()
        N.raise_device_error(int(hb[-1]))
        return (hb[:n * kk].astype(np.int64).reshape(n, kk),
                hb[n * kk:2 * n * kk].reshape(n, kk))

    def _active_layers(self):
        L = self.target.config.num_layers
        if self.config.schedule_mode == "all":
            return list(range(L - 1))
        return active_layers(self.profile, self.online, self.schedule_config)

    def _policy_kind(self):
        from .engine import AlwaysExitPolicy, NeverExitPolicy, PredictorPolicy
        pol = self.policy
        if type(pol) in (NeverExitPolicy, AlwaysExitPolicy):
            return "const"
        if type(pol) is PredictorPolicy:
            return "mlp"
        return "host"

    def step(self) -> TreeStepResult:
        from .engine import PredictorPolicy  # noqa: F401
        cfg = self.target.config
        L, K = cfg.num_layers, self.config.k
        self._merge_cache = {}
        if K > self.draft.config.vocab_size:
            raise ValueError("k exceeds vocabulary size")
        tree, node_logits, k_sets = self._draft_tree()
        ctx_len = len(self.context)
        # every node's draft top-K at once (merge_paths' per-node feature / leaf
        # verify sets, tree.py:64-73): one batched top-K + softmax, one host
        # read (or already from the drafting levels)
        if not k_sets and 1 <= K <= 64:
            order = sorted(node_logits)
            batch = speculative_sets_from_rows(torch.stack([node_logits[j] for j in order]), K)
            k_sets = {(j, K): s_ for j, s_ in zip(order, batch)}

        def propose(context, k):                  # node context -> that node's own logits
            j = self._node_of_context[tuple(context[ctx_len:])]
            if (j, k) in k_sets:
                return k_sets[(j, k)]
            return speculative_set_from_logits(node_logits[j], k)
        self._node_of_context = {}
        for j, n in enumerate(tree.nodes):
            if j:
                self._node_of_context[tuple(tree.nodes[i].token for i in tree.path_to(j))] = j
        hts = merge_paths(tree, self.draft, self.context, K, propose=propose)
        paths = [ht.path for ht in hts]
        P, n_nodes = len(paths), len(tree.nodes)
        m = len(self.context) - 1

        tokens = [n.token for n in tree.nodes]
        pos_ids = [m + n.depth for n in tree.nodes]
        attn_lists, ancestors = [None], {0: [0]}
        for j in range(1, n_nodes):
            ancestors[j] = ancestors[tree.nodes[j].parent] + [j]
            attn_lists.append(list(range(m)) + [m + a for a in ancestors[j]])
        rows = self.tstate.begin(tokens, pos_ids=pos_ids, attn_lists=attn_lists)
        r0 = rows[0]

        # per-step device constants: node feature ids, path CSR, verify CSR
        fspec = {}
        for ht in hts:
            for pos, j in enumerate(ht.path):
                fspec.setdefault(j, ht.feature_spec(pos))
        vspec = {}
        for ht in hts:
            for pos, j in enumerate(ht.path):
                vspec.setdefault(j, ht.per_node_spec[pos])
        feat_ids = np.zeros((n_nodes, K), np.int64)
        for j, s in fspec.items():
            if len(s.tokens) != K:
                raise ValueError("feature set size differs from k")
            feat_ids[j] = s.tokens
        path_ptr = np.concatenate([[0], np.cumsum([len(p) for p in paths])])
        d_path_ptr, d_path_nodes = _i32(path_ptr), _i32(np.concatenate(paths))
        vlists = [[]] + [list(vspec[j].tokens) for j in range(1, n_nodes)]
        d_vptr = _i32(np.concatenate([[0], np.cumsum([len(v) for v in vlists])]))
        d_vids = _i32(np.concatenate([np.asarray(v, np.int64) for v in vlists]))
        dev = "cuda"
        prev = torch.full((n_nodes, K), float(np.float32(1.0 / K)), dtype=torch.float32, device=dev)
        fired = torch.zeros(n_nodes, dtype=torch.uint8, device=dev)
        prob = torch.zeros(n_nodes, dtype=torch.float64, device=dev)
        path_fire = torch.zeros(P, dtype=torch.uint8, device=dev)
        path_ok = torch.zeros(P, dtype=torch.uint8, device=dev)
        node_gate = torch.zeros(n_nodes, dtype=torch.uint8, device=dev)
        tok = torch.zeros(n_nodes, dtype=torch.int32, device=dev)
        ver = torch.zeros(n_nodes, dtype=torch.uint8, device=dev)
        live_mask = torch.ones(P, dtype=torch.uint8, device=dev)
        err = torch.zeros(1, dtype=torch.int32, device=dev)
        xg = torch.empty((n_nodes, cfg.hidden_dim), dtype=torch.float32, device=dev)
        rr = torch.empty(n_nodes, dtype=torch.float32, device=dev)
        scratch, counter = _VerifyScratch.get(n_nodes)
        hid = self.tstate.pending[r0:r0 + n_nodes]
        vargs = verify_args(self.target, hid, n_nodes, tok, scratch, counter, err,
                            gate=node_gate, spec_ptr=d_vptr, spec_ids=d_vids, verified_out=ver)
        kind = self._policy_kind()
        bank = self.policy.packed(L) if kind == "mlp" else None
        zc = z_cut(self.config.threshold) if kind == "mlp" else 0.0
        lib = N.lib()
        stream = N.stream_ptr()

        active_set = set(self._active_layers())
        live = set(range(P))
        exit_layer = [L - 1] * P
        preds = [None] * P
        evals = 0
        ran = False
        frozen_keep = None
        for l in range(L):
            self.tstate.launch_layer(l)
            ran = True
            if not live:
                break
            if l in active_set and l <= L - 2:
                live_nodes = sorted({j for p in live for j in paths[p]})
                n_live = len(live_nodes)
                if kind == "mlp" and l not in self.policy.bank:
                    raise KeyError(f"no predictor for active layer {l}")
                N.check(lib.spx_head_prep(N.ptr(hid), hid.stride(0), N.ptr(self.target.final_g),
                                          N.ptr(self.target.final_b), N.ptr(xg), N.ptr(rr),
                                          n_nodes, cfg.hidden_dim, numerics.mode(), N.ptr(err),
                                          stream), "spx_head_prep")
                logits = self._merged(xg, rr, live_nodes, feat_ids, err)
                d_live = self.last_live_idx
                fired.zero_()
                if kind == "host":
                    self._host_probs(l, live_nodes, logits, prev, hid, fired, prob)
                else:
                    if kind == "mlp":
                        w1, b1, w2 = (bank.w1[l], bank.b1[l], bank.w2[l])
                        if bank.k != K:
                            raise ValueError("feature dimension does not match predictor")
                        args = (N.ptr(w1), N.ptr(b1), N.ptr(w2), float(bank.b2[l]), zc,
                                N.SPX_POLICY_MLP, 0.0, 0.0)
                        H = bank.hidden
                    else:
                        args = (None, None, None, 0.0, 0.0, N.SPX_POLICY_CONST,
                                float(self.policy.const_prob), float(self.config.threshold))
                        H = 0
                    N.check(lib.spx_tree_node_eval(N.ptr(logits), N.ptr(d_live), n_live,
                                                   N.ptr(prev), *args, N.ptr(prob), N.ptr(fired),
                                                   N.ptr(err), K, H, stream), "spx_tree_node_eval")
                evals += n_live
                N.check(lib.spx_path_and(N.ptr(fired), N.ptr(d_path_ptr), N.ptr(d_path_nodes),
                                         N.ptr(live_mask), P, N.ptr(path_fire), stream),
                        "spx_path_and")
                N.check(lib.spx_tree_gate(N.ptr(path_fire), N.ptr(d_path_ptr), N.ptr(d_path_nodes),
                                          P, n_nodes, N.ptr(node_gate), stream), "spx_tree_gate")
                ver.zero_()
                launch_verify(vargs)
                N.check(lib.spx_path_and(N.ptr(ver), N.ptr(d_path_ptr), N.ptr(d_path_nodes),
                                         N.ptr(path_fire), P, N.ptr(path_ok), stream),
                        "spx_path_and")
                # one device->host read per active layer: error words, path
                # flags, node tokens (and probabilities when recorded)
                # (float64 holds every int32 word and the float64 probabilities exactly)
                parts = [err.to(torch.float64), self.tstate.err.to(torch.float64),
                         path_ok.to(torch.float64), tok.to(torch.float64)]
                if self.record_probs:
                    parts.append(prob)
                hb = torch.cat(parts).cpu()
                N.raise_device_error(int(hb[0]) | int(hb[1]))
                ok = hb[2:2 + P].numpy() != 0
                tk = hb[2 + P:2 + P + n_nodes].numpy().astype(np.int64)
                if self.record_probs:
                    pr = hb[2 + P + n_nodes:].numpy()
                    self.prob_log.extend([l, float(pr[j])] for j in live_nodes)
                if ok.any():
                    for p in sorted(live):
                        if ok[p]:
                            exit_layer[p] = l
                            preds[p] = [int(tk[0])] + [int(tk[j]) for j in paths[p]]
                            live.discard(p)
                    live_mask.copy_(torch.as_tensor(
                        np.asarray([1 if p in live else 0 for p in range(P)], np.uint8)))
                keep = {j for p in live for j in paths[p]} | ({0} if live else set())
                if keep != frozen_keep:                  # the frozen set only grows on exits
                    self.tstate.freeze([rows[j] for j in range(n_nodes) if j not in keep])
                    frozen_keep = keep
            if not live:
                break
        assert ran
        if live:
            gate = np.zeros(n_nodes, np.uint8)
            gate[0] = 1
            for p in live:
                gate[paths[p]] = 1
            node_gate.copy_(torch.as_tensor(gate))
            fargs = verify_args(self.target, hid, n_nodes, tok, scratch, counter, err,
                                gate=node_gate)
            launch_verify(fargs)
            tk = tok.cpu().numpy()
            N.raise_device_error(int(err.item()))
            for p in live:
                preds[p] = [int(tk[0])] + [int(tk[j]) for j in paths[p]]
        self.tstate.unfreeze_all()

        best_p, best_len = 0, -1
        for p, ht in enumerate(hts):
            n_ok = 0
            for t_, idx in enumerate(ht.path):
                if tree.nodes[idx].token == preds[p][t_]:
                    n_ok += 1
                else:
                    break
            if n_ok > best_len:
                best_p, best_len = p, n_ok
        acc_nodes = hts[best_p].path[:best_len]
        accepted = [tree.nodes[j].token for j in acc_nodes]
        correction = preds[best_p][best_len]
        self.tstate.compact([rows[0]] + [rows[j] for j in acc_nodes], m)
        self._dstate.compact([m] + [m + j for j in acc_nodes], m)
        self.context.extend(accepted + [correction])
        for _ in range(len(accepted) + 1):
            update_online(self.online, exit_layer[best_p])
        return TreeStepResult(accepted_tokens=accepted, correction_token=correction,
                              path_exit_layers=exit_layer, accepted_path=best_p,
                              predictor_evals=evals, num_paths=P,
                              max_path_len=max(len(p) for p in paths),
                              scheduled_layer_count=max(len(active_set), 1))

    def _merged(self, xg, rr, live_nodes, feat_ids, err):
        """K6 over the live nodes' feature ids: (n_live, K) logits in live
        order; each unique LM-head row is read from HBM once.  The merged
        mapping (unique ids + CSR) depends only on the live-node set, which
        changes only when a path exits, so it is built once per set and step
        (pinned host buffer, asynchronous copy: no stream synchronisation)."""
        K = feat_ids.shape[1]
        key = tuple(live_nodes)
        ent = self._merge_cache.get(key)
        if ent is None:
            sel = feat_ids[live_nodes]                   # (n_live, K)
            flat = sel.reshape(-1)
            uniq, inv = np.unique(flat, return_inverse=True)
            order = np.argsort(inv, kind="stable")
            uptr = np.concatenate([[0], np.cumsum(np.bincount(inv, minlength=uniq.size))])
            node = np.repeat(np.asarray(live_nodes, np.int64), K)
            out_idx = np.arange(flat.size)
            pack = np.concatenate([uniq, uptr, node[order], out_idx[order],
                                   np.asarray(live_nodes, np.int64)]).astype(np.int32)
            host = torch.from_numpy(pack).pin_memory()
            d = torch.empty(pack.size, dtype=torch.int32, device="cuda")
            d.copy_(host, non_blocking=True)
            ent = (d, host, uniq.size, flat.size)
            self._merge_cache[key] = ent
        d, _, U, n = ent
        self.last_live_idx = d[2 * U + 1 + 2 * n:]
        d_uniq, d_uptr = d[:U], d[U:2 * U + 1]
        d_node, d_out = d[2 * U + 1:2 * U + 1 + n], d[2 * U + 1 + n:2 * U + 1 + 2 * n]
        logits = torch.empty(n, dtype=torch.float32, device="cuda")
        m = self.target
        N.check(N.lib().spx_tree_merged_logits(N.ptr(xg), N.ptr(rr), xg.shape[0], N.ptr(m.lm_head),
                                               m.spx_dtype, N.ptr(m.head_bw), m.config.vocab_size,
                                               m.config.hidden_dim, N.ptr(d_uniq), U, N.ptr(d_uptr),
                                               N.ptr(d_node), N.ptr(d_out), N.ptr(logits),
                                               numerics.mode(), N.ptr(err), N.stream_ptr()),
                "spx_tree_merged_logits")
        self.last_unique_ids, self.last_pairs = U, n
        return logits.view(len(live_nodes), K)

    def _host_probs(self, l, live_nodes, logits, prev, hid, fired, prob):
        """Any other policy object: the reference's per-node calls
        (tree.py:213-220) with device features."""
        for i, j in enumerate(live_nodes):
            fv = extract_features(logits[i], prev[j])
            prev[j].copy_(fv.local_probs)
            p = float(self.policy.exit_prob(l, fv, hid[j]))
            prob[j] = p
            fired[j] = 1 if decide_exit(p, self.config.threshold) else 0

    def generate(self, prompt, max_new: int):
        """tree.py:290-302: commit at least max_new tokens."""
        if max_new < 1:
            raise ValueError("max_new must be >= 1")
        self.start(prompt)
        steps, produced = [], []
        while len(produced) < max_new:
            res = self.step()
            steps.append(res)
            produced.extend(res.accepted_tokens + [res.correction_token])
        return produced[:max_new], steps
