"""Early-exit decoding engine -- drop-in for the reference's ``specexit.engine``
(src/specexit/engine.py): ``ExitRecord``, ``EngineConfig``, ``verify_exit``,
the Never / Always / Predictor / Oracle policies, ``ExitEngine`` (``start`` /
``step`` / ``generate`` / ``generate_forced``), ``generate``,
``greedy_generate``, ``oracle_exit_layer``, ``write_trace`` / ``read_trace``.

B200 design.  For the built-in policies (Never, Always, Predictor with a
predictor for every layer 0..L-2) the WHOLE token step lives on the device and
is captured once into a CUDA graph (``_DeviceStep``):

  draft: embed next_in -> Ld flag-free layers -> full-head logits (spx_verify)
         -> stable top-K (spx_topk)                     = speculative ids
  spx_sched_active      (two-level or "all" bitmask, scheduler.py:95-102)
  spx_token_begin       (prev = f32(1/K), flags cleared, exit_layer = L-1)
  target: embed next_in; for l in 0..L-1:
         spx_layer_forward(l)        -- returns at once when done != 0
         l <= L-2: spx_predictor_eval (row_layer_mask=active, row_done=done;
                                      fired_any |= fired in-kernel)
                   spx_verify        (gate=fired, verify set = spec ids;
                                      on membership: done=1, exit_layer=l)
  spx_verify (row_done=done)         -- the final-layer argmax
  spx_token_end         (token choice, ExitRecord arrays, next_in, online window)
  [spx_force_next]      (generate_forced)

so no decision ever returns to the host inside a token: the predictor's
device flag gates the verify kernel, the verify kernel's exit flag stops the
remaining decoder layers.  ``generate`` replays the graph max_new times and
synchronises once.

Any other policy (OraclePolicy, user policies, a bank with missing layers,
spec_full_vocab) runs the reference's step loop on the host
(``_host_step``), calling the same device operators one by one.
"""
import gc
import json
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from . import numerics
from .decode import DecodeState
from .model import (TransformerModel, full_head_logits, head_argmax, launch_verify,
                    sliced_head_logits, verify_args)
from .predictor import (PredictorBank, decide_exit, extract_features, predictor_forward,
                        uniform_probs, z_cut)
from .scheduler import (OfflineProfile, OnlineState, ScheduleConfig, active_layers,
                        mask_to_layers, update_online)
from .speculation import SpeculativeSet, speculative_set_from_logits


@dataclass
class ExitRecord:
    """engine.py:26-48."""
    token: int
    exit_layer: int
    predictor_fired: bool
    verified: bool
    active: list = field(default_factory=list)
    full_head_count: int = 0
    predictor_evals: int = 0

    def to_json(self):
        return json.dumps({"token": self.token, "exit_layer": self.exit_layer,
                           "predictor_fired": self.predictor_fired, "verified": self.verified,
                           "active": list(self.active)})

    @classmethod
    def from_json(cls, line):
        d = json.loads(line)
        return cls(token=d["token"], exit_layer=d["exit_layer"],
                   predictor_fired=d["predictor_fired"], verified=d["verified"],
                   active=d["active"])


@dataclass(frozen=True)
class EngineConfig:
    """engine.py:51-56."""
    k: int = 4
    threshold: float = 0.5
    schedule_mode: str = "all"
    spec_full_vocab: bool = False


def verify_exit(model: TransformerModel, hidden, spec_set: SpeculativeSet):
    """engine.py:59-64: the global argmax if it lies in the speculative set."""
    tok, ver, _ = head_argmax(model, hidden, [list(spec_set.tokens)])
    return int(tok[0].item()) if int(ver[0].item()) else None


class NeverExitPolicy:
    """engine.py:67-76."""
    const_prob = 0.0

    def start(self, prompt):
        pass

    def observe(self, token):
        pass

    def exit_prob(self, layer, features, hidden):
        return 0.0


class AlwaysExitPolicy(NeverExitPolicy):
    """engine.py:79-81."""
    const_prob = 1.0

    def exit_prob(self, layer, features, hidden):
        return 1.0


class PredictorPolicy(NeverExitPolicy):
    """engine.py:83-92: trained per-layer MLP predictors."""
    const_prob = None

    def __init__(self, bank: dict):
        self.bank = bank
        self._packed = {}

    def packed(self, num_layers):
        pb = self._packed.get(num_layers)
        if pb is None:
            pb = self._packed[num_layers] = PredictorBank(self.bank, num_layers)
        return pb

    def exit_prob(self, layer, features, hidden):
        if layer not in self.bank:
            raise KeyError(f"no predictor for active layer {layer}")
        return predictor_forward(self.bank[layer], features)


class OraclePolicy:
    """engine.py:95-122: fires exactly when the layer's argmax equals the
    final argmax of a private full-depth forward of the same stream."""

    def __init__(self, target: TransformerModel):
        self.target = target
        self.state = None
        self.final_argmax = None

    def start(self, prompt):
        self.state = DecodeState(self.target)
        if len(prompt) > 1:
            self.state.begin(prompt[:-1])
            for l in range(self.target.config.num_layers):
                self.state.launch_layer(l)

    def observe(self, token):
        self.state.begin([token])
        for l in range(self.target.config.num_layers):
            self.state.launch_layer(l)
        tok, _, _ = head_argmax(self.target, self.state.cur_hidden)
        self.final_argmax = int(tok[0].item())

    def exit_prob(self, layer, features, hidden):
        tok, _, _ = head_argmax(self.target, hidden)
        return 1.0 if int(tok[0].item()) == self.final_argmax else 0.0


def _i32(n, fill=0):
    return torch.full((n,), fill, dtype=torch.int32, device="cuda")


def _u8(n):
    return torch.zeros(n, dtype=torch.uint8, device="cuda")


class _DeviceStep:
    """Device-resident token state + the captured token-step graph."""

    def __init__(self, eng):
        t, dm = eng.target.config, eng.draft.config
        self.eng = eng
        self.K = eng.config.k
        self.L = t.num_layers
        cap = t.max_context
        self.cap = cap
        self.prev = torch.zeros(self.K, dtype=torch.float32, device="cuda")
        self.prev_err = torch.zeros(1, dtype=torch.float32, device="cuda")
        self.recheck = torch.zeros(6, dtype=torch.int32, device="cuda")
        self.done, self.fired, self.fired_any = _u8(1), _u8(1), _u8(1)
        self.exit_layer, self.exit_token, self.final_token = _i32(1), _i32(1), _i32(1)
        self.evals, self.full_heads, self.next_in, self.step = _i32(1), _i32(1), _i32(1), _i32(1)
        self.active = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.rec_token, self.rec_exit_layer = _i32(cap), _i32(cap)
        self.rec_evals, self.rec_full_heads = _i32(cap), _i32(cap)
        self.rec_fired, self.rec_verified = _u8(cap), _u8(cap)
        self.rec_active = torch.zeros(cap, dtype=torch.int64, device="cuda")
        self.forced = _i32(cap)
        self.inject = _u8(cap)             # injected-spec flags (generate_forced)
        self.spec_ids = _i32(self.K)
        self.spec_ptr = torch.tensor([0, self.K], dtype=torch.int32, device="cuda")
        self.draft_logits = torch.zeros(dm.vocab_size, dtype=torch.float32, device="cuda")
        self.draft_tok = _i32(1)
        self.scratch = torch.zeros(4, dtype=torch.int64, device="cuda")
        self.counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.err = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.graphs = {}
        st = N.TokenStateC()
        for name in ("prev", "done", "fired", "fired_any", "exit_layer", "exit_token",
                     "final_token", "evals", "full_heads", "next_in", "step", "active",
                     "rec_token", "rec_exit_layer", "rec_evals", "rec_full_heads", "rec_fired",
                     "rec_verified", "rec_active", "prev_err"):
            setattr(st, name, N.ptr(getattr(self, name)))
        self.cst = st

    # -- argument structs, built once (pointers are stable) -------------------

    def _pred_args(self, l, mode):
        eng, m = self.eng, self.eng.target
        pol = eng.policy
        a = N.PredictorArgs()
        a.hidden, a.hidden_stride = N.ptr(eng.tstate.cur_hidden), m.config.hidden_dim
        a.norm_g, a.norm_b = N.ptr(m.final_g), N.ptr(m.final_b)
        a.head, a.head_dtype, a.head_bw = N.ptr(m.lm_head), m.spx_dtype, N.ptr(m.head_bw)
        a.ids, a.prev = N.ptr(self.spec_ids), N.ptr(self.prev)
        H = 0
        if pol.const_prob is None:
            pb = pol.packed(self.L)
            a.w1 = N._vp(pb.w1[l].data_ptr())
            a.b1 = N._vp(pb.b1[l].data_ptr())
            a.w2 = N._vp(pb.w2[l].data_ptr())
            a.b2 = float(pb.b2[l])
            a.z_cut = z_cut(eng.config.threshold)
            a.policy = N.SPX_POLICY_MLP
            H = pb.hidden
        else:
            a.policy, a.const_prob = N.SPX_POLICY_CONST, float(pol.const_prob)
            a.threshold = float(eng.config.threshold)
        a.fired, a.row_layer_mask = N.ptr(self.fired), N.ptr(self.active)
        a.fired_any = N.ptr(self.fired_any)      # the token's predictor_fired, in-kernel
        a.row_done, a.evals = N.ptr(self.done), N.ptr(self.evals)
        a.layer, a.mode, a.pdl, a.err = l, mode, 0, N.ptr(self.err)
        a.B, a.d, a.V, a.K, a.H = 1, m.config.hidden_dim, m.config.vocab_size, self.K, H
        a.prev_err = N.ptr(self.prev_err)
        if mode == N.SPX_MODE_FAST:        # certified FAST decisions
            a.head_wmax, a.recheck = N.ptr(m.head_wmax), N.ptr(self.recheck)
            a.cert_kappa, a.cert_hnorm = m.cert_kappa, m.cert_hnorm
            if pol.const_prob is None:
                a.cert = N._vp(pb.cert[l].data_ptr())
        return a

    def enqueue(self, mode, forced: bool, inject: bool = False):
        """Enqueue one token step on the current stream (capturable)."""
        eng = self.eng
        lib = N.lib()
        s = N.stream_ptr
        # draft proposal
        ds = eng.dstate
        ds.embed_device(self.next_in, 1)
        for l in range(eng.draft.config.num_layers):
            ds.launch_layer(l)
        launch_verify(verify_args(eng.draft, ds.cur_hidden, 1, self.draft_tok, self.scratch,
                                  self.counter, self.err, logits_out=self.draft_logits,
                                  mode=mode))
        N.check(lib.spx_topk(N.ptr(self.draft_logits), eng.draft.config.vocab_size, self.K,
                             N.ptr(self.spec_ids), s()), "spx_topk")
        if inject:
            N.check(lib.spx_inject_spec(N.ptr(self.spec_ids), self.K, N.ptr(self.forced),
                                        N.ptr(self.step), N.ptr(self.inject), self.cap, s()),
                    "spx_inject_spec")
        # schedule
        if eng.config.schedule_mode == "all":
            mask, m = 0, 0
        else:
            mask, m = eng.profile.offline_mask(eng.schedule_config.offline_top_k), 1
        N.check(lib.spx_sched_active(eng.online.cstate(), mask, 1, self.L, m, N.ptr(self.active),
                                     s()), "spx_sched_active")
        N.check(lib.spx_token_begin(self.cst, self.K, self.L, float(np.float32(1.0 / self.K)), s()),
                "spx_token_begin")
        # target layers with the exit machinery
        ts = eng.tstate
        ts.embed_device(self.next_in, 1)
        tm = eng.target
        for l in range(self.L):
            ts.launch_layer(l)
            if l <= self.L - 2:
                pa = self._pargs[l]
                N.check(lib.spx_predictor_eval(pa, s()), "spx_predictor_eval")
                launch_verify(verify_args(tm, ts.cur_hidden, 1, self.exit_token, self.scratch,
                                          self.counter, self.err, gate=self.fired,
                                          row_done=self.done, spec_ptr=self.spec_ptr,
                                          spec_ids=self.spec_ids, done_out=self.done,
                                          exit_layer_out=self.exit_layer,
                                          full_heads=self.full_heads, layer=l, mode=mode))
        launch_verify(verify_args(tm, ts.cur_hidden, 1, self.final_token, self.scratch,
                                  self.counter, self.err, row_done=self.done,
                                  full_heads=self.full_heads, layer=self.L - 1, mode=mode))
        sc = eng.schedule_config
        N.check(lib.spx_token_end(self.cst, eng.online.cstate(), self.L, sc.queue_len, sc.radius,
                                  self.cap, s()), "spx_token_end")
        if forced:
            N.check(lib.spx_force_next(N.ptr(self.forced), N.ptr(self.step), N.ptr(self.next_in),
                                       self.cap, s()), "spx_force_next")

    def graph(self, forced: bool, inject: bool = False):
        mode = numerics.mode()
        key = (mode, forced, inject)
        g = self.graphs.get(key)
        if g is None:
            # host-side preparation (weight packing, z_cut) before capture
            self._pargs = [self._pred_args(l, mode) for l in range(self.L - 1)]
            # dead engines are reference cycles (engine <-> _DeviceStep) that
            # may own CUDA graphs; collect them now -- a graph destroyed by a
            # GC pass DURING capture invalidates the capture
            gc.collect()
            g = torch.cuda.CUDAGraph()
            was = gc.isenabled()
            gc.disable()
            try:
                with torch.cuda.graph(g):
                    self.enqueue(mode, forced, inject)
            finally:
                if was:
                    gc.enable()
            self.graphs[key] = g
        return g

    def reset(self, next_in):
        self.step.zero_()
        self.next_in.fill_(int(next_in))
        self.err.zero_()

    def records(self, n):
        cols = [t[:n].cpu().numpy() for t in (self.rec_token, self.rec_exit_layer, self.rec_fired,
                                             self.rec_verified, self.rec_active,
                                             self.rec_full_heads, self.rec_evals)]
        out = []
        for i in range(n):
            out.append(ExitRecord(token=int(cols[0][i]), exit_layer=int(cols[1][i]),
                                  predictor_fired=bool(cols[2][i]), verified=bool(cols[3][i]),
                                  active=mask_to_layers(int(cols[4][i]), self.L),
                                  full_head_count=int(cols[5][i]),
                                  predictor_evals=int(cols[6][i])))
        return out


class ExitEngine:
    """engine.py:125-246: one generation stream; owns its KV caches and
    online schedule state."""

    def __init__(self, target: TransformerModel, draft: TransformerModel, policy,
                 config: EngineConfig = EngineConfig(), profile: OfflineProfile = None,
                 schedule_config: ScheduleConfig = ScheduleConfig()):
        if config.schedule_mode not in ("all", "two-level"):
            raise ValueError(f"unknown schedule mode {config.schedule_mode!r}")
        if config.schedule_mode == "two-level" and profile is None:
            raise ValueError("two-level scheduling needs an offline profile")
        self.target, self.draft, self.policy = target, draft, policy
        self.config, self.profile, self.schedule_config = config, profile, schedule_config
        self.online = OnlineState(target.config.num_layers, schedule_config)
        self.tstate = self.dstate = None
        self.context = None
        self.next_in = None
        self._dev = None
        self._steps = 0

    # -- which path ------------------------------------------------------------

    def device_resident(self) -> bool:
        """True when the token step runs as one captured device graph."""
        cfg, L = self.config, self.target.config.num_layers
        if cfg.spec_full_vocab or not 1 <= cfg.k <= 64 or L > 64:
            return False
        if cfg.k > self.draft.config.vocab_size or cfg.k > self.target.config.vocab_size:
            return False
        if self.draft.config.vocab_size != self.target.config.vocab_size:
            return False
        pol = self.policy
        if type(pol) in (NeverExitPolicy, AlwaysExitPolicy):
            return True
        if type(pol) is PredictorPolicy:
            ws = list(pol.bank.values())
            if not all(l in pol.bank for l in range(L - 1)):
                return False
            if any(w.k != cfg.k for w in ws) or len({w.hidden for w in ws}) != 1:
                return False
            return ws[0].hidden <= 1024
        return False

    # -- reference API -----------------------------------------------------------

    def start(self, prompt):
        prompt = [int(t) for t in prompt]
        if not prompt:
            raise ValueError("empty prompt")
        if self.config.schedule_mode == "two-level":
            self.schedule_config.validate(self.profile.num_layers)
        dev = self.device_resident()
        if dev and self._dev is None:
            # one set of device buffers per engine; graphs keep their pointers
            self.tstate = DecodeState(self.target)
            self.dstate = DecodeState(self.draft)
            self._dev = _DeviceStep(self)
            self.tstate.done = self._dev.done
            self.tstate._largs = [self.tstate._layer_args(l)
                                  for l in range(self.target.config.num_layers)]
        elif dev:
            self._reset_states()
        else:
            self.tstate = DecodeState(self.target)
            self.dstate = DecodeState(self.draft)
        if len(prompt) > 1:
            for st, m in ((self.tstate, self.target), (self.dstate, self.draft)):
                st.begin(prompt[:-1])
                for l in range(m.config.num_layers):
                    st.launch_layer(l)
        # the online window persists across generate() calls, as in the
        # reference (engine.py:122-160 creates it once, start() keeps it)
        self.context = prompt
        self.next_in = prompt[-1]
        self.policy.start(prompt)
        if dev:
            self._dev.reset(self.next_in)
        self._steps = 0

    def _reset_states(self):
        for st in (self.tstate, self.dstate):
            st.n = 0
            st.n_ctx.zero_()
            st.new_row.fill_(-1)
            st.frontier.zero_()
            st.frozen.zero_()
            st.new_rows = []

    def _check_capacity(self, n_steps):
        for st, m in ((self.tstate, self.target), (self.dstate, self.draft)):
            if st.n + n_steps > m.config.max_context:
                raise ValueError("context overflow")

    def _run_device(self, n, forced=None, inject=None):
        d = self._dev
        self._check_capacity(n)
        if forced is not None:
            d.forced[self._steps:self._steps + n].copy_(
                torch.as_tensor(np.asarray(forced, np.int32)))
        if inject is not None:
            d.inject[self._steps:self._steps + n].copy_(
                torch.as_tensor(np.asarray(inject, np.uint8)))
        self.replay_device(n, forced is not None, inject is not None)
        self.sync_device()
        recs = d.records(self._steps)[self._steps - n:]
        for r in recs:
            self.context.append(r.token)
        self.next_in = recs[-1].token
        if forced is not None:
            self.context[-n:] = [int(t) for t in forced]
            self.next_in = int(forced[-1])
        return recs

    def replay_device(self, n, forced: bool = False, inject: bool = False):
        """Enqueue n token steps (graph replays) without synchronising; the
        ExitRecord fields accumulate in the device record arrays."""
        self._check_capacity(n)
        g = self._dev.graph(forced, inject)
        for _ in range(n):
            g.replay()
        for st in (self.tstate, self.dstate):
            st.n += n
        self._steps += n

    def sync_device(self):
        """Synchronise and raise the reference's error for any device error word."""
        torch.cuda.synchronize()
        d = self._dev
        N.raise_device_error(int(d.err.item()) | int(self.tstate.err.item()) |
                             int(self.dstate.err.item()))

    def _speculative_set(self, inject_token=None):
        self.dstate.begin([self.next_in])
        for l in range(self.draft.config.num_layers):
            self.dstate.launch_layer(l)
        logits = full_head_logits(self.draft, self.dstate.cur_hidden)
        k = self.target.config.vocab_size if self.config.spec_full_vocab else self.config.k
        spec = speculative_set_from_logits(logits, k)
        if inject_token is not None and int(inject_token) not in spec.tokens:
            toks = list(spec.tokens)
            toks[-1] = int(inject_token)
            spec = SpeculativeSet(tokens=tuple(toks), draft_probs=spec.draft_probs)
        return spec

    def _active_layers(self):
        L = self.target.config.num_layers
        if self.config.schedule_mode == "all":
            return list(range(L - 1))
        return active_layers(self.profile, self.online, self.schedule_config)

    def _host_step(self, inject_token=None) -> ExitRecord:
        """engine.py:176-217 with device operators and host decisions."""
        L = self.target.config.num_layers
        spec = self._speculative_set(inject_token)
        active = self._active_layers()
        act = set(active)
        self.policy.observe(self.next_in)
        self.tstate.begin([self.next_in])
        prev = uniform_probs(len(spec.tokens))
        token, exit_layer = None, L - 1
        fired = verified = False
        full_heads = evals = 0
        hidden = None
        for l in range(L):
            self.tstate.launch_layer(l)
            hidden = self.tstate.cur_hidden.clone()
            if l in act:
                fv = extract_features(sliced_head_logits(self.target, hidden, spec.tokens), prev)
                prev = fv.local_probs
                prob = self.policy.exit_prob(l, fv, hidden)
                evals += 1
                if decide_exit(prob, self.config.threshold):
                    fired = True
                    full_heads += 1
                    tok = verify_exit(self.target, hidden, spec)
                    if tok is not None:
                        token, exit_layer, verified = tok, l, True
                        break
        if token is None:
            full_heads += 1
            t, _, _ = head_argmax(self.target, hidden)
            token = int(t[0].item())
        self.tstate.check()
        self.context.append(token)
        self.next_in = token
        update_online(self.online, exit_layer)
        return ExitRecord(token=token, exit_layer=exit_layer, predictor_fired=fired,
                          verified=verified, active=active, full_head_count=full_heads,
                          predictor_evals=evals)

    def step(self) -> ExitRecord:
        if self._dev is not None and self.device_resident():
            return self._run_device(1)[0]
        return self._host_step()

    def generate(self, prompt, max_new: int):
        """engine.py:219-225: (token list, ExitRecord trace)."""
        if max_new < 1:
            raise ValueError("max_new must be >= 1")
        self.start(prompt)
        if self._dev is not None and self.device_resident():
            trace = self._run_device(max_new)
        else:
            trace = [self._host_step() for _ in range(max_new)]
        return [r.token for r in trace], trace

    def generate_forced(self, prompt, forced_tokens, inject=None):
        """engine.py:227-246: position-aligned evaluation over a given
        continuation (normally the full model's greedy stream).

        inject (optional, one bool per step): the injected-spec hook of
        SURVEY.md §8d C2 on _speculative_set (engine.py:162-168) -- at a
        flagged step the forced token (the target's final argmax when the
        continuation is the greedy stream) replaces the last draft id unless
        it is already speculated.  Not part of the reference API; used to give
        random-init models a realistic exit-depth distribution."""
        forced_tokens = [int(t) for t in forced_tokens]
        if len(forced_tokens) == 0:
            raise ValueError("empty forced continuation")
        if inject is not None and len(inject) != len(forced_tokens):
            raise ValueError("inject needs one flag per forced token")
        self.start(prompt)
        if self._dev is not None and self.device_resident():
            return self._run_device(len(forced_tokens), forced_tokens, inject)
        trace = []
        for i, tok in enumerate(forced_tokens):
            trace.append(self._host_step(tok if inject is not None and inject[i] else None))
            self.context[-1] = tok
            self.next_in = tok
        return trace


def generate(target, draft, policy, prompt, max_new, config=EngineConfig(), profile=None,
             schedule_config=ScheduleConfig()):
    """engine.py:249-253."""
    return ExitEngine(target, draft, policy, config, profile, schedule_config).generate(prompt,
                                                                                     max_new)


def _layer_argmaxes(target, state):
    """Advance the newest row through every layer; argmax of the full head at
    each layer's hidden state (one K4 launch over the L stacked rows)."""
    L, d = target.config.num_layers, target.config.hidden_dim
    hs = torch.empty((L, d), dtype=torch.float32, device="cuda")
    for l in range(L):
        state.launch_layer(l)
        hs[l].copy_(state.cur_hidden)
    tok, _, _ = head_argmax(target, hs)
    return tok.cpu().numpy()


def _earliest(toks):
    final = int(toks[-1])
    for l, t in enumerate(toks):
        if int(t) == final:
            return l
    return len(toks) - 1


def greedy_generate(target: TransformerModel, prompt, max_new: int):
    """engine.py:256-274: plain full-depth greedy decoding; returns (tokens,
    per-token oracle exit layers)."""
    state = DecodeState(target)
    prompt = [int(t) for t in prompt]
    if len(prompt) > 1:
        state.begin(prompt[:-1])
        for l in range(target.config.num_layers):
            state.launch_layer(l)
    tokens, layers = [], []
    nxt = prompt[-1]
    for _ in range(max_new):
        state.begin([nxt])
        toks = _layer_argmaxes(target, state)
        nxt = int(toks[-1])
        tokens.append(nxt)
        layers.append(_earliest(toks))
    state.check()
    return tokens, layers


def oracle_exit_layer(target: TransformerModel, context) -> int:
    """engine.py:285-292."""
    state = DecodeState(target)
    state.begin(list(context))
    return _earliest(_layer_argmaxes(target, state))


def write_trace(trace, path):
    with open(path, "w") as fh:
        for rec in trace:
            fh.write(rec.to_json() + "\n")


def read_trace(path):
    with open(path) as fh:
        return [ExitRecord.from_json(line) for line in fh if line.strip()]
