"""B independent early-exit streams stepped together on one GPU -- the
batched decode behind BASELINE configs[3] (Llama2-13B, 1-256 requests per
GPU).  The reference runs one ExitEngine per stream (engine.py:122-246); this
is B of them sharing every weight read.

Layout: ONE DecodeState per model holds all B streams interleaved by
position -- row p*B + b is stream b's position p -- so each step appends B
contiguous rows (one launch per layer advances all of them, with the
lazily completed rows of earlier exits), and a static CSR of attention lists
(row p*B + b attends to q*B + b, q <= p) keeps the streams independent.
Per step (enqueued, one host sync at the end):

  draft:  embed B rows -> Ld layers -> K4 logits of the B rows -> top-K per row
  spx_sched_active   (B rows of the two-level / "all" schedule)
  target: embed B rows; per layer l: spx_layer_forward (all live rows), and for
          l <= L-2 the fused predictor over the B rows (row_layer_mask,
          row_done, fired_any in-kernel) -> gated K4 over the fired rows
          (done / exit_layer per row) -> exited rows frozen for the rest of
          the step (they are completed lazily by later tokens, model.py:220-270)
  final K4 of the rows still running, token choice, ExitRecord arrays,
  update_online of every stream (spx_sched_update), next inputs.

Every ExitRecord field of stream b equals a single-stream ExitEngine's on the
same prompt (tests/test_gpu_batched.py checks it against the oracle).
"""
import numpy as np
import torch

from . import _native as N
from . import numerics
from .decode import DecodeState
from .engine import (AlwaysExitPolicy, EngineConfig, ExitRecord, NeverExitPolicy,
                     PredictorPolicy)
from .model import _VerifyScratch, launch_verify, verify_args
from .predictor import BatchResult, evaluate_batch, prev_error, z_cut
from .scheduler import OnlineState, ScheduleConfig, mask_to_layers


def _interleaved_csr(B, C):
    """Attention lists of the interleaved layout: row p*B + b -> q*B + b, q <= p."""
    rows = np.arange(B * C, dtype=np.int64)
    p, b = rows // B, rows % B
    lens = p + 1
    ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    idx = np.empty(int(ptr[-1]), np.int32)
    for q in range(C):                       # vectorised per position
        sel = p >= q
        idx[ptr[:-1][sel] + q] = (q * B + b[sel]).astype(np.int32)
    return (torch.as_tensor(ptr.astype(np.int32), device="cuda"),
            torch.as_tensor(idx, device="cuda"))


class BatchedExitEngine:
    """ExitEngine semantics for `batch` streams at once (device policies:
    PredictorPolicy with every layer, NeverExitPolicy, AlwaysExitPolicy)."""

    def __init__(self, target, draft, policy, config: EngineConfig = EngineConfig(),
                 profile=None, schedule_config: ScheduleConfig = ScheduleConfig(), batch=1,
                 context=None, row_cap=None):
        if config.schedule_mode not in ("all", "two-level"):
            raise ValueError(f"unknown schedule mode {config.schedule_mode!r}")
        if config.schedule_mode == "two-level" and profile is None:
            raise ValueError("two-level scheduling needs an offline profile")
        if type(policy) not in (PredictorPolicy, NeverExitPolicy, AlwaysExitPolicy):
            raise ValueError("BatchedExitEngine runs the device policies only")
        if config.spec_full_vocab:
            raise ValueError("spec_full_vocab is not supported in batched mode")
        self.target, self.draft, self.policy = target, draft, policy
        self.config, self.profile, self.schedule_config = config, profile, schedule_config
        L, K, B = target.config.num_layers, config.k, int(batch)
        if type(policy) is PredictorPolicy and not all(l in policy.bank for l in range(L - 1)):
            raise KeyError("no predictor for some layer 0..L-2")
        C = int(context or target.config.max_context)
        if C > min(target.config.max_context, draft.config.max_context):
            raise ValueError("context exceeds the models' max_context")
        self.L, self.K, self.B, self.C = L, K, B, C
        rc = int(row_cap or min(B * C, 4 * B + 64))
        ptr, idx = _interleaved_csr(B, C)
        self.ts = DecodeState(target, max_context=B * C, row_cap=rc, att_cap=C)
        self.ds = DecodeState(draft, max_context=B * C, row_cap=rc, att_cap=C)
        for st in (self.ts, self.ds):
            st.set_attention_csr(ptr, idx)
        self.online = OnlineState(L, schedule_config, rows=B)
        dev = "cuda"
        z = lambda dt, *sh: torch.zeros(sh, dtype=dt, device=dev)  # noqa: E731
        self.next_in, self.pos = z(torch.int32, B), z(torch.int32, B)
        self.spec = z(torch.int32, B, K)
        self.spec_ptr = torch.arange(0, B * K + 1, K, dtype=torch.int32, device=dev)
        self.prev = z(torch.float32, B, K)
        self.done, self.fired_any = z(torch.uint8, B), z(torch.uint8, B)
        self.exit_layer, self.exit_token = z(torch.int32, B), z(torch.int32, B)
        self.final_token, self.evals, self.full_heads = (z(torch.int32, B), z(torch.int32, B),
                                                         z(torch.int32, B))
        self.active = z(torch.int64, B)
        self.dlogits = z(torch.float32, B, draft.config.vocab_size)
        self.dtok = z(torch.int32, B)
        self.err = z(torch.int32, 1)
        self.out = BatchResult(logits=None, z=None, prob=None, fired=z(torch.uint8, B),
                               err=self.err)
        self.recs = None
        self.steps = 0

    def start(self, prompts):
        """All prompts the same length (the interleaved layout advances every
        stream by one position per step)."""
        prompts = [[int(t) for t in p] for p in prompts]
        if len(prompts) != self.B or len({len(p) for p in prompts}) != 1 or not prompts[0]:
            raise ValueError("need `batch` non-empty prompts of equal length")
        P = len(prompts[0])
        self.P = P
        for st in (self.ts, self.ds):
            st.reset()
        # prefill position by position (B rows per call: the row set of a call
        # stays within row_cap; rows attend only to earlier, complete rows)
        for q in range(P - 1):
            toks = [prompts[b][q] for b in range(self.B)]
            for st, m in ((self.ts, self.target), (self.ds, self.draft)):
                st.begin(toks, pos_ids=[q] * self.B)
                for l in range(m.config.num_layers):
                    st.launch_layer(l)
        self.next_in.copy_(torch.as_tensor([p[-1] for p in prompts], dtype=torch.int32))
        self.p = P - 1
        self.steps = 0
        self.recs = []

    def _step_enqueue(self):
        B, L, K = self.B, self.L, self.K
        lib, s = N.lib(), N.stream_ptr
        mode = numerics.mode()
        if self.p >= self.C:
            raise ValueError("context overflow")
        n0 = self.p * B
        self.pos.fill_(self.p)
        scratch, counter = _VerifyScratch.get(B)
        # draft proposal (engine.py:162-168), B rows
        ds = self.ds
        ds.embed_device(self.next_in, B, self.pos)
        for l in range(self.draft.config.num_layers):
            ds.launch_layer(l)
        dh = ds.pending[n0:n0 + B]
        # the K draft ids straight from K4 (tensor-core form: stable top-K of
        # the CDOT logits, no full-logit round trip), else full logits + top-K
        a = verify_args(self.draft, dh, B, self.dtok, scratch, counter, self.err, mode=mode,
                        topk_out=self.spec, topk_k=K)
        if a.tc_scratch and mode != N.SPX_MODE_STRICT:
            launch_verify(a)
        else:
            launch_verify(verify_args(self.draft, dh, B, self.dtok, scratch, counter, self.err,
                                      logits_out=self.dlogits, mode=mode))
            N.check(lib.spx_topk_rows(N.ptr(self.dlogits), B, self.draft.config.vocab_size, K,
                                      N.ptr(self.spec), s()), "spx_topk_rows")
        # schedule (scheduler.py:95-102), all streams
        if self.config.schedule_mode == "all":
            mask, m = 0, 0
        else:
            mask, m = self.profile.offline_mask(self.schedule_config.offline_top_k), 1
        N.check(lib.spx_sched_active(self.online.cstate(), mask, B, L, m, N.ptr(self.active),
                                     s()), "spx_sched_active")
        # token start (engine.py:182-188)
        self.prev.fill_(float(np.float32(1.0 / K)))
        prev_error(self.prev).zero_()
        self.done.zero_()
        self.fired_any.zero_()
        self.exit_layer.fill_(L - 1)
        self.evals.zero_()
        self.full_heads.zero_()
        ts = self.ts
        ts.embed_device(self.next_in, B, self.pos)
        th = ts.pending[n0:n0 + B]
        pol = self.policy
        bank = pol.packed(L) if type(pol) is PredictorPolicy else None
        const = None if bank is not None else float(pol.const_prob)
        for l in range(L):
            ts.launch_layer(l)
            if l <= L - 2:
                evaluate_batch(self.target, bank, th, self.spec, self.prev,
                               threshold=self.config.threshold, layer=l, outputs=False,
                               row_layer_mask=self.active, row_done=self.done, evals=self.evals,
                               err=self.err, policy=const, out=self.out,
                               fired_any=self.fired_any)
                launch_verify(verify_args(self.target, th, B, self.exit_token, scratch, counter,
                                          self.err, gate=self.out.fired, row_done=self.done,
                                          spec_ptr=self.spec_ptr, spec_ids=self.spec,
                                          done_out=self.done, exit_layer_out=self.exit_layer,
                                          full_heads=self.full_heads, layer=l, mode=mode))
                ts.frozen[n0:n0 + B] |= self.done          # exited rows stop here
        launch_verify(verify_args(self.target, th, B, self.final_token, scratch, counter,
                                  self.err, row_done=self.done, full_heads=self.full_heads,
                                  layer=L - 1, mode=mode))
        # token end (engine.py:208-216)
        tok = torch.where(self.done.bool(), self.exit_token, self.final_token)
        self.recs.append((tok, self.exit_layer.clone(), self.fired_any.clone(),
                          self.done.clone(), self.active.clone(), self.evals.clone(),
                          self.full_heads.clone()))
        sc = self.schedule_config
        N.check(lib.spx_sched_update(self.online.cstate(), N.ptr(self.exit_layer), None, B, L,
                                     sc.queue_len, sc.radius, N.ptr(self.err), s()),
                "spx_sched_update")
        self.next_in.copy_(tok)
        ts.frozen[n0:n0 + B] = 0                            # lazy completion later
        for st in (self.ts, self.ds):
            st.n += B
        self.p += 1
        self.steps += 1

    def run(self, n):
        """Enqueue n steps (no host sync)."""
        for _ in range(n):
            self._step_enqueue()

    def sync(self):
        torch.cuda.synchronize()
        N.raise_device_error(int(self.err.item()) | int(self.ts.err.item()) |
                             int(self.ds.err.item()))

    def records(self):
        """Per stream: the list of ExitRecords of the steps run since start()."""
        self.sync()
        cols = [torch.stack(c).cpu().numpy() for c in zip(*self.recs)] if self.recs else []
        out = [[] for _ in range(self.B)]
        for t in range(len(self.recs)):
            for b in range(self.B):
                out[b].append(ExitRecord(
                    token=int(cols[0][t, b]), exit_layer=int(cols[1][t, b]),
                    predictor_fired=bool(cols[2][t, b]), verified=bool(cols[3][t, b]),
                    active=mask_to_layers(int(cols[4][t, b]), self.L),
                    predictor_evals=int(cols[5][t, b]), full_head_count=int(cols[6][t, b])))
        return out

    def generate(self, prompts, max_new):
        """engine.py:219-225 for every stream: (token lists, ExitRecord lists)."""
        if max_new < 1:
            raise ValueError("max_new must be >= 1")
        self.start(prompts)
        self.run(max_new)
        recs = self.records()
        return [[r.token for r in rs] for rs in recs], recs
