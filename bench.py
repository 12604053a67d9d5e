"""Benchmark of the B200-native SpecEE speculative early-exit predictor path.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]

Workload (Llama2-7B shape, BASELINE.json configs[1]/[4]): LM head V=32000 x
d=4096 (bf16 in HBM), K=4 speculative ids per request, a bank of 31 per-layer
MLP predictors (H=512, reference init_predictor), threshold 0.7.  One STEP is
one pass of the predictor path over every predictor-capable layer (31) for B
independent requests (default 1024 per GPU): 31 fused launches of K1+K2+K3
(LayerNorm + K-row gather + local logits + softmax/delta features + MLP +
sigmoid/threshold + device exit flag), each over that layer's own synthetic
hidden rows (31 x B x 4096 f32 = 520 MB > L2, so no L2 flush is needed).
``value`` = predictor evaluations/s over all ranks.  Requests shard across
GPUs with no collective on the hot path (weak scaling); one NCCL all_gather
of the per-rank fire counts after the timed region.

``e2e`` = the same step through the public drop-in API with HOST buffers:
each step copies its hidden rows/ids from pinned host memory to HBM and the
fired flags + probabilities back.

``--impl reference`` times the reference's CPU implementation of the same
chain (oracle port of sliced_head_logits -> extract_features ->
predictor_forward -> decide_exit with the reference's own compiled strict
kernel from oracle/_ref when present) on this host's cores, one forked
process per core.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

V, D, K, H, LAYERS = 32000, 4096, 4, 512, 32
PRED_LAYERS = LAYERS - 1
THRESHOLD = 0.7
SEED = 1234
# programmatic dependent launch; 2 = also "ids ready": the speculative ids of a
# token are fixed across its layer loop (written at token start by the draft),
# so each launch may start its LM-head row prefetch before the previous
# launch retires (include/specexit_b200.h, spx_predictor_args.pdl)
PDL = int(os.environ.get("SPX_PDL", "2"))
METRIC = "predictor evals/sec + early-exit decode tok/s, Llama2-7B shape, 1/2/4/8 B200"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=1024, help="requests per GPU")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--mode", default="fast", choices=["fast", "strict"])
    ap.add_argument("--no-decode", action="store_true")
    ap.add_argument("--no-tree", action="store_true")
    ap.add_argument("--no-c4", action="store_true", help="skip the Llama2-13B batch sweep")
    ap.add_argument("--decode-tokens", type=int, default=32)
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--fused", action="store_true",
                    help="one fused K1-K3 launch per layer instead of the split gather/tail form")
    ap.add_argument("--dry-run", action="store_true",
                    help="CPU/gloo rehearsal of the N-rank plumbing (no kernels)")
    return ap.parse_args()


def maybe_relaunch(args):
    """`bench.py --gpus N` outside torchrun: re-exec under torch.distributed.run
    with N ranks on this node (one process per GPU, 127.0.0.1 rendezvous) and
    exit with its status; rank 0 prints the JSON line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def distinct_ids(seed, B, K, V):
    """Per-request K distinct ids from the splitmix64 stream."""
    from paper_2504_08850_b200 import rng
    raw = rng.splitmix64(seed, B * K * 4) % np.uint64(V)
    ids = np.empty((B, K), np.int32)
    pos = 0
    for b in range(B):
        seen = []
        while len(seen) < K:
            v = int(raw[pos % raw.size]); pos += 1
            if v not in seen:
                seen.append(v)
        ids[b] = seen
    return ids


def launch_bytes(B, U):
    """Algorithmic HBM bytes of one fused launch."""
    return U * D * 2 + B * D * 4 + B * (3 * K * 4 + 5) + 2 * D * 4 + (3 * K * H + 2 * H + 1) * 4


# ------------------------------------------------------------------ clocks


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ CPU reference


def cpu_reference_rate(head_dv, final_g, final_b, bank, ids, seconds, seed=7):
    """evals/s of the reference chain on this host, one forked process per
    available core (OPENBLAS_NUM_THREADS=1), each running for `seconds`."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import specexit_oracle as O
    from oracle.build import load_ref_kernels
    kern = load_ref_kernels()
    kind = "port+reference-ckern" if kern is not None else "port"
    t = {"lm_head": head_dv, "final_norm.g": final_g, "final_norm.b": final_b}
    cores = sorted(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else [0]
    P = len(cores)
    r_fd, w_fd = os.pipe()
    pids = []
    for p in range(P):
        pid = os.fork()
        if pid == 0:
            try:
                os.sched_setaffinity(0, {cores[p]})
            except (AttributeError, OSError):
                pass
            rng = np.random.default_rng(seed + p)
            hidden = rng.standard_normal((64, D)).astype(np.float32)
            hb = hidden.view(np.uint32)                      # bf16-valued rows (RNE), as the GPU arm
            hidden = ((hb + 0x7FFF + ((hb >> 16) & 1)) & 0xFFFF0000).astype(np.uint32).view(np.float32)
            uni = np.full(K, np.float32(1.0 / K), np.float32)
            prev = uni
            n, t0 = 0, time.perf_counter()
            while time.perf_counter() - t0 < seconds:
                l = n % PRED_LAYERS
                if l == 0:
                    prev = uni                               # token start (engine.py:182-188)
                _, prev = O.reference_chain(t, hidden[n % 64], ids[(n * 7 + p) % ids.shape[0]],
                                            prev, bank[l], THRESHOLD, kern)
                n += 1
            el = time.perf_counter() - t0
            os.write(w_fd, f"{n} {el}\n".encode())
            os._exit(0)
        pids.append(pid)
    os.close(w_fd)
    data = b""
    with os.fdopen(r_fd, "rb") as fh:
        data = fh.read()
    for pid in pids:
        os.waitpid(pid, 0)
    rates = [int(a) / float(b) for a, b in (ln.split() for ln in data.decode().splitlines())]
    return sum(rates), P, kind, sum(int(ln.split()[0]) for ln in data.decode().splitlines())


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2504_08850_b200 import rng
    from oracle import specexit_oracle as O
    t0 = time.time()
    cfg = O.ModelConfig(vocab_size=V, hidden_dim=D, num_layers=LAYERS, num_heads=32, ffn_dim=11008,
                        max_context=512, seed=SEED)
    head = O.init_model(cfg, bf16=True, only={"lm_head", "final_norm.g", "final_norm.b"})
    bank = [O.init_predictor(K, H, rng.derive(SEED, 100 + l)) for l in range(PRED_LAYERS)]
    ids = distinct_ids(SEED + 1, 4096, K, V)
    per_step = max(0.5, min(args.cpu_seconds, 120.0 / max(args.steps + args.warmup, 1)))
    vals = []
    for s in range(args.warmup + args.steps):
        rate, P, kind, n = cpu_reference_rate(head["lm_head"], head["final_norm.g"],
                                              head["final_norm.b"], bank, ids, per_step, seed=s)
        if s >= args.warmup:
            vals.append(rate)
    value = statistics.median(vals)
    sample = (f"reference chain sliced_head_logits->extract_features->predictor_forward->"
              f"decide_exit at d={D}, V={V}, K={K}, H={H} on random bf16-valued rows, "
              f"{per_step:.1f}s per step per process, {P} processes x 1 core")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "evals/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * per_step, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": "predictor path, Llama2-7B head (V=32000,d=4096), K=4, H=512, "
                               "thr 0.7, CPU reference chain", "batch_per_gpu": None},
        "cpu_baseline": {"value": value, "unit": "evals/s", "cores": P, "kind": "port",
                         "sample": sample, "strict_kernel": kind},
        "e2e": {"value": value, "unit": "evals/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "wall_s": round(time.time() - t0, 1)}))


# ------------------------------------------------------------------ ours


def decode_bench(args, rank, ws, dev):
    """Early-exit decode at Llama2-7B shape, one stream per
    rank through the device-resident ExitEngine (one CUDA graph per token:
    2-layer draft + top-K, scheduler, 32 flag-guarded decoder layers, fused
    predictor evals on the active layers, gated verify GEMVs).  Device time of
    graph replays (max over ranks) and end-to-end ``generate()`` wall time
    (host prompt in, host tokens out)."""
    import torch
    import torch.distributed as dist

    import paper_2504_08850_b200 as spx
    from paper_2504_08850_b200 import engine as E
    from paper_2504_08850_b200 import rng
    seed = SEED + 1000 * rank
    tc = spx.ModelConfig(V, D, LAYERS, 32, 11008, 512, seed)
    dc = spx.ModelConfig(V, D, 2, 32, 11008, 512, seed + 1)
    t, d = spx.init_model(tc, dtype="bf16"), spx.init_model(dc, dtype="bf16")
    bank = {l: spx.init_predictor(K, H, rng.derive(seed, l)) for l in range(LAYERS - 1)}
    counts = np.asarray([int(x) % 97 for x in rng.splitmix64(seed + 7, LAYERS)], dtype=np.uint64)
    prof = spx.OfflineProfile(LAYERS, counts, 0)
    thr = 0.5
    eng = E.ExitEngine(t, d, E.PredictorPolicy(bank),
                       E.EngineConfig(k=K, threshold=thr, schedule_mode="two-level"), prof,
                       spx.ScheduleConfig(5, 2, 4))
    prompt = [int(x) % V for x in rng.splitmix64(seed, 16)]
    n = args.decode_tokens
    eng.generate(prompt, 4)                      # capture + warm
    eng.start(prompt)
    g = eng._dev.graph(False)
    for _ in range(3):
        g.replay()
    eng.start(prompt)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    recs = eng._dev.records(n)
    if ws > 1:
        # results gather after the timed region: every rank's
        # ExitRecord fields, one all_gather over NCCL
        from paper_2504_08850_b200 import shard
        packed = torch.as_tensor(shard.pack_records(recs), device=dev)
        gathered = [torch.empty_like(packed) for _ in range(ws)]
        dist.all_gather(gathered, packed)
    t0 = time.perf_counter()
    toks, trace = eng.generate(prompt, n)
    e2e_s = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    layer_bytes = (4 * D * D + 2 * D * 11008) * 2
    el = float(np.mean([r.exit_layer for r in recs]))
    heads = float(np.mean([r.full_head_count for r in recs]))
    ms_tok = float(ms.item()) / n
    # executed decoder layers = exit layer + 1; plus full-head GEMVs (262 MB)
    tok_bytes = (el + 1) * layer_bytes + heads * V * D * 2 + 2 * layer_bytes + V * D * 2
    # injected-spec variant: generate_forced over the greedy
    # stream with the target's final argmax put into the draft ids at 80% of
    # the steps, so verification succeeds and exits actually happen
    base, _ = E.greedy_generate(t, prompt, n)
    flags = (rng.splitmix64(seed + 99, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53 < 0.8
    dv = eng._dev

    def forced_start():
        eng.start(prompt)
        dv.forced[:n].copy_(torch.as_tensor(np.asarray(base, np.int32)))
        dv.inject[:n].copy_(torch.as_tensor(flags.astype(np.uint8)))

    gi = dv.graph(True, True)
    forced_start()
    for _ in range(3):
        gi.replay()
    forced_start()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(n):
        gi.replay()
    e1.record()
    torch.cuda.synchronize()
    ms_i = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(ms_i, op=dist.ReduceOp.MAX)
    irecs = dv.records(n)
    iel = float(np.mean([r.exit_layer for r in irecs]))
    iheads = float(np.mean([r.full_head_count for r in irecs]))
    ibytes = (iel + 1) * layer_bytes + iheads * V * D * 2 + 2 * layer_bytes + V * D * 2
    injected = {"tok_s": ws * n / (float(ms_i.item()) / 1e3), "unit": "tokens/s",
                "ms_per_token": float(ms_i.item()) / n, "p_inject": 0.8,
                "avg_exit_layer": iel, "full_heads_per_token": iheads,
                "fire_token_frac": float(np.mean([r.predictor_fired for r in irecs])),
                "verified_frac": float(np.mean([r.verified for r in irecs])),
                "hbm_bytes_per_token": ibytes,
                "hbm_GBps": ibytes / (float(ms_i.item()) / n * 1e-3) / 1e9,
                "tokens_match_greedy": [r.token for r in irecs] == list(base),
                "config": "generate_forced over the greedy stream; at 80% of the steps "
                          "(splitmix64 flags) the target's final argmax replaces the last "
                          "draft id (injected-spec hook on _speculative_set)"}
    tree = None
    if not args.no_tree:
        # configs[2]: EAGLE-like token tree, context-aware merged mapping
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import tree_bench
        tree = tree_bench.run(steps=3, seed=seed, models=(t, d))
    cpu_dec = None
    try:                     # reported CPU baseline of the same decode (one separate run)
        cpu_dec = json.load(open(os.path.join(ROOT, "profiles", "r02_cpu_decode.json")))
        cpu_dec = {"tok_s": cpu_dec["tok_s"], "cores": cpu_dec["cores"], "kind": "port",
                   "source": "profiles/r02_cpu_decode.json (scripts/cpu_decode_baseline.py on "
                             "the GPU box host: oracle ExitEngine, strict kernels, 3 tokens)"}
    except (OSError, KeyError, ValueError):
        pass
    return {"tok_s": ws * n / (float(ms.item()) / 1e3), "unit": "tokens/s", "tree": tree,
            "injected": injected, "cpu_baseline": cpu_dec,
            "ms_per_token": ms_tok, "streams": ws, "tokens_per_stream": n,
            "e2e_tok_s": ws * n / float(e2e_s.item()),
            "avg_exit_layer": el, "full_heads_per_token": heads,
            "fire_token_frac": float(np.mean([r.predictor_fired for r in recs])),
            "verified_frac": float(np.mean([r.verified for r in recs])),
            "evals_per_token": float(np.mean([r.predictor_evals for r in recs])),
            "hbm_bytes_per_token": tok_bytes,
            "hbm_GBps": tok_bytes / (ms_tok * 1e-3) / 1e9,
            "config": "Llama2-7B shape (reference architecture) random-init bf16, batch 1 per "
                      "GPU, 2-layer draft, K=4, H=512, thr 0.5, two-level (top-k 4, N=5, r=2), "
                      "16-token prompt"}



def parity_check(spx, model, bank, bank_w, hidden, ids_all, outs, stream, prev, prev0, B,
                 rows=64, inter=None):
    """Checker (untimed, rank 0): the decisions and probabilities of the
    benchmarked step against the oracle's reference chain (oracle/, the CPU
    restatement of model.py:298-314 + predictor.py:42-109) on a row sample,
    all 31 layers chained through prev -- at the bench threshold (the last
    timed replay's outputs) and at thr 0.5 (one extra untimed step)."""
    import torch
    from oracle import specexit_oracle as O
    from paper_2504_08850_b200 import numerics
    sel = np.linspace(0, B - 1, rows).astype(np.int64)
    ids_s = ids_all[:, sel]
    uniq, inv = np.unique(ids_s, return_inverse=True)
    cols = model.lm_head[torch.as_tensor(uniq, device=hidden.device, dtype=torch.long)]
    t = {"lm_head": np.ascontiguousarray(cols.float().cpu().numpy().T),
         "final_norm.g": model.final_g.cpu().numpy(), "final_norm.b": model.final_b.cpu().numpy()}
    oid = inv.reshape(ids_s.shape)
    hid = hidden[:, torch.as_tensor(sel, device=hidden.device)].cpu().numpy()
    ow = [O.PredictorWeights(bank_w[l].w1, bank_w[l].b1, bank_w[l].w2, bank_w[l].b2)
          for l in range(PRED_LAYERS)]
    res = {}
    for thr in (THRESHOLD, 0.5):
        if thr == THRESHOLD:
            torch.cuda.synchronize()
            fired = torch.stack([o.fired for o in outs]).cpu().numpy()[:, sel]
            prob = torch.stack([o.prob for o in outs]).cpu().numpy()[:, sel]
        else:
            with torch.cuda.stream(stream), numerics.using("fast"):
                prev.copy_(prev0)
                spx.prev_error(prev).zero_()
                fs, ps = [], []
                ids_d = torch.as_tensor(ids_all, device=hidden.device)
                if inter is not None:          # the benchmarked (pipelined) form
                    os_ = spx.evaluate_chain(model, bank, hidden, ids_d, prev, inter,
                                             list(range(PRED_LAYERS)), threshold=thr)
                    fs, ps = [o.fired for o in os_], [o.prob for o in os_]
                else:
                    for l in range(PRED_LAYERS):
                        o = spx.evaluate_batch(model, bank, hidden[l], ids_d[l], prev,
                                               threshold=thr, layer=l)
                        fs.append(o.fired)
                        ps.append(o.prob)
            torch.cuda.synchronize()
            fired = torch.stack(fs).cpu().numpy()[:, sel]
            prob = torch.stack(ps).cpu().numpy()[:, sel]
        mism, perr, margin = 0, 0.0, float("inf")
        for j in range(rows):
            pv = O.uniform_probs(K)
            for l in range(PRED_LAYERS):
                fv = O.extract_features(O.sliced_head_logits(t, hid[l, j], oid[l, j]), pv)
                p = O.predictor_forward(ow[l], fv)
                mism += int(bool(fired[l, j]) != (p > thr))
                perr = max(perr, abs(float(prob[l, j]) - p))
                margin = min(margin, abs(p - thr))
                pv = fv.local_probs
        res[str(thr)] = {"decision_mismatches": mism, "max_prob_err": perr, "min_margin": margin,
                         "fire_rate": float(fired.mean())}
    return {"checker": "oracle/specexit_oracle.py reference chain (CPU)", "rows": rows,
            "layers": PRED_LAYERS, "thresholds": res}


def dry_run(args):
    """CPU rehearsal of the N-rank plumbing with gloo: each rank takes its
    contiguous request shard, produces per-request records, and rank 0 prints
    the gathered shapes -- the same collectives the GPU run makes after its
    timed region, no kernels."""
    import torch
    import torch.distributed as dist
    from paper_2504_08850_b200 import shard
    ws, rank, _ = dist_env()
    if ws > 1:
        dist.init_process_group("gloo")
    total = args.batch * ws
    a, b = shard.shard_range(total, rank, ws)
    ids = np.arange(a, b)
    local = torch.as_tensor(np.stack([ids, ids % LAYERS, ids % 2, ids % 3 == 0, np.ones_like(ids),
                                      ids % 7], axis=1).astype(np.int32))
    full = shard.gather_rows(local, total) if ws > 1 else local
    tmax = shard.max_over_ranks(1.0 + rank, "cpu")
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": ws, "requests": total,
                          "gathered_shape": list(full.shape),
                          "gathered_ok": bool((full[:, 0] == torch.arange(total)).all()),
                          "max_over_ranks": tmax}))
    if ws > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    maybe_relaunch(args)
    if args.dry_run:
        dry_run(args)
        return
    if args.impl == "reference":
        run_reference(args)
        return
    import torch
    import torch.distributed as dist

    import paper_2504_08850_b200 as spx
    from paper_2504_08850_b200 import _native as N
    from paper_2504_08850_b200 import numerics, rng, shard

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    numerics.set_mode(args.mode)
    B = args.batch

    # ---- model head + predictor bank (reference init, bf16 head) ------------
    cfg = spx.ModelConfig(vocab_size=V, hidden_dim=D, num_layers=LAYERS, num_heads=32,
                          ffn_dim=11008, max_context=512, seed=SEED)
    model = spx.init_model(cfg, dtype="bf16", head_only=True)
    bank_w = {l: spx.init_predictor(K, H, rng.derive(SEED, 100 + l)) for l in range(PRED_LAYERS)}
    bank = spx.PredictorBank(bank_w, LAYERS)

    # ---- synthetic requests: this rank's shard ------------------------------
    g = torch.Generator(device=dev)
    g.manual_seed(SEED + 17 * rank)
    hidden = torch.randn((PRED_LAYERS, B, D), generator=g, device=dev, dtype=torch.float32)
    hidden = hidden.to(torch.bfloat16).float()            # bf16-valued rows
    # Distinct speculative ids per layer launch: in the engine the decoder layer
    # between two predictor launches streams ~315 MB and evicts the previous
    # launch's LM-head rows from the 126 MB L2; a predictor-only loop with one
    # id set would re-read the same 31 MB of head rows from L2 every launch.
    ids_all = np.stack([distinct_ids(SEED + 1 + 1000 * rank + l, B, K, V)
                        for l in range(PRED_LAYERS)])
    ids_np = ids_all[0]
    ids_l = torch.as_tensor(ids_all, device=dev)               # (layers, B, K)
    ids = ids_l[0]
    U = float(np.mean([np.unique(ids_all[l]).size for l in range(PRED_LAYERS)]))
    prev0 = torch.full((B, K), float(np.float32(1.0 / K)), device=dev)
    prev = prev0.clone()
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    outs = [spx.predictor.BatchResult(logits=None, z=None,
                                      prob=torch.empty(B, dtype=torch.float64, device=dev),
                                      fired=torch.empty(B, dtype=torch.uint8, device=dev), err=err)
            for _ in range(PRED_LAYERS)]

    prev_err = spx.prev_error(prev)
    recheck = spx.recheck_buffer(B)

    # PIPELINED split form (default when the shape allows): one
    # launch per layer = that layer's LM-head gather (K1) + the previous
    # layer's feature/MLP/decision tail (K2+K3, carries prev), programmatic
    # dependent launches that never wait for the preceding gather; a final
    # tail launch for the last layer.  --fused: one fused launch per layer.
    split = (not args.fused and args.mode == "fast" and
             spx.predictor.split_supported(model, bank, hidden[0], ids_l[0], prev))
    inter = torch.zeros((PRED_LAYERS, B, 2 * K + 2), dtype=torch.float32, device=dev)

    def step():
        prev.copy_(prev0)                                  # token start: uniform prior
        prev_err.zero_()                                   # ... which is exact
        if not split:
            for l in range(PRED_LAYERS):
                spx.evaluate_batch(model, bank, hidden[l], ids_l[l], prev, threshold=THRESHOLD,
                                   layer=l, outputs=False, out=outs[l], pdl=PDL)
            return
        spx.evaluate_chain(model, bank, hidden, ids_l, prev, inter, list(range(PRED_LAYERS)),
                           threshold=THRESHOLD, outs=outs, recheck=recheck)

    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        recheck = spx.recheck_buffer(B)                    # this stream's work list
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step()
    torch.cuda.synchronize()
    N.raise_device_error(err.item())

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            graph.replay()
    barrier()
    rc0 = recheck[3:5].cpu().tolist()
    clk = ClockSampler(local)
    clk.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(args.steps):
            graph.replay()
        e1.record(stream)
    e1.synchronize()
    clocks = clk.stop()
    barrier()
    ms = e0.elapsed_time(e1)
    rc1 = recheck[3:5].cpu().tolist()
    certified = {"rows_reevaluated_strict": rc1[0] - rc0[0], "unresolved": rc1[1] - rc0[1],
                 "evals": PRED_LAYERS * B * args.steps}
    ms_max = shard.max_over_ranks(ms, dev)                # device time, max over ranks
    evals_per_step = PRED_LAYERS * B * ws
    value = evals_per_step * args.steps / (ms_max / 1000.0)
    launches = (PRED_LAYERS + 1 if split else PRED_LAYERS) * args.steps
    t_launch = (ms / 1000.0) / (PRED_LAYERS * args.steps)    # per layer (the dominant launch)
    bytes_launch = launch_bytes(B, U)
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 6650.0))
    # ncu dram bytes per launch of the dominant kernel (profiles/, one --set full capture)
    kname = ("predictor_gather_kernel<d=4096, K=4, 1 team, 4 tail warps> (gather l + tail l-1)"
             if split else "predictor_stream_kernel<bf16, d=4096, K=4, H=512>")
    kkey = "predictor_gather_kernel" if split else "predictor_stream_kernel"
    traffic, traffic_src = None, None
    for fn in ("r02_ncu_summary.json", "r01_ncu_summary.json"):
        try:
            ncu = json.load(open(os.path.join(ROOT, "profiles", fn)))
            traffic = ncu[kkey]["traffic_bytes"]
            traffic_src = f"profiles/{fn} (ncu --set full, 1 launch)"
            break
        except (OSError, KeyError, ValueError):
            pass
    achieved = bytes_launch / t_launch / 1e9

    fired = torch.stack([o.fired for o in outs]).float().mean().item()
    fire_cnt = torch.tensor([fired], device=dev)
    if ws > 1:
        gathered = [torch.zeros_like(fire_cnt) for _ in range(ws)]
        dist.all_gather(gathered, fire_cnt)               # results gather (off the hot path)
        fired = float(torch.stack(gathered).mean().item())

    # ---- batch-1 latency of one fused launch (configs[1]: batch 1) ---------
    h1, i1, p1 = hidden[0, :1].contiguous(), ids[:1].contiguous(), prev0[:1].clone()
    o1 = spx.predictor.BatchResult(logits=None, z=None, prob=None,
                                   fired=torch.empty(1, dtype=torch.uint8, device=dev), err=err)
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.stream(stream):
        spx.evaluate_batch(model, bank, h1, i1, p1, threshold=THRESHOLD, layer=0, outputs=False, out=o1)
        torch.cuda.synchronize()
        with torch.cuda.graph(g1, stream=stream):
            for l in range(PRED_LAYERS):
                spx.evaluate_batch(model, bank, hidden[l, :1], i1, p1, threshold=THRESHOLD,
                                   layer=l, outputs=False, out=o1, pdl=PDL)
        for _ in range(5):
            g1.replay()
        torch.cuda.synchronize()
        b0, b1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        for _ in range(20):
            g1.replay()
        b1e.record(stream)
    b1e.synchronize()
    us_per_eval_b1 = b0.elapsed_time(b1e) * 1000.0 / (20 * PRED_LAYERS)

    # ---- e2e: public API with host buffers ---------------------------------
    e2e = None
    if not args.no_e2e:
        h_host = hidden.cpu().pin_memory()
        ids_host = ids_l.cpu().pin_memory()
        fired_host = torch.empty((PRED_LAYERS, B), dtype=torch.uint8).pin_memory()
        prob_host = torch.empty((PRED_LAYERS, B), dtype=torch.float64).pin_memory()
        hid_dev = torch.empty_like(hidden)
        ids_dev = torch.empty_like(ids_l)
        eo = [spx.predictor.BatchResult(logits=None, z=None,
                                        prob=torch.empty(B, dtype=torch.float64, device=dev),
                                        fired=torch.empty(B, dtype=torch.uint8, device=dev),
                                        err=err) for _ in range(PRED_LAYERS)]

        def e2e_step():
            hid_dev.copy_(h_host, non_blocking=True)
            ids_dev.copy_(ids_host, non_blocking=True)
            prev.copy_(prev0)
            for l in range(PRED_LAYERS):
                spx.evaluate_batch(model, bank, hid_dev[l], ids_dev[l], prev, threshold=THRESHOLD,
                                   layer=l, outputs=False, out=eo[l], pdl=PDL)
            for l in range(PRED_LAYERS):
                fired_host[l].copy_(eo[l].fired, non_blocking=True)
                prob_host[l].copy_(eo[l].prob, non_blocking=True)

        e2e_steps = max(3, min(args.steps, 10))
        with torch.cuda.stream(stream):
            for _ in range(2):
                e2e_step()
            barrier()
            x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            x0.record(stream)
            for _ in range(e2e_steps):
                e2e_step()
            x1.record(stream)
        x1.synchronize()
        xms = torch.tensor([x0.elapsed_time(x1)], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(xms, op=dist.ReduceOp.MAX)
        e2e = {"value": evals_per_step * e2e_steps / (float(xms.item()) / 1000.0),
               "unit": "evals/s",
               "h2d_bytes_per_step": int(hidden.numel() * 4 + ids_l.numel() * 4),
               "d2h_bytes_per_step": int(PRED_LAYERS * B * (1 + 8)),
               "path": "paper_2504_08850_b200.evaluate_batch -> spx_predictor_eval (C ABI)"}

    # ---- early-exit decode tok/s (configs[1]: 7B shape, batch 1 per rank) ---
    decode = None
    if not args.no_decode:
        decode = decode_bench(args, rank, ws, dev)
    # ---- configs[3]: Llama2-13B batch sweep (B requests per GPU) -----------
    c4 = None
    if not args.no_c4:
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        import batch_sweep
        numerics.set_mode("fast")
        c4 = {"per_gpu": batch_sweep.run([1, 16, 64, 256], steps=6, warmup=2),
              "note": "BatchedExitEngine, B independent requests per GPU, 13B random-init "
                      "bf16, 2-layer draft, K=4, thr 0.5, two-level; tok_s per GPU (device "
                      "time); with N GPUs the requests shard (B per GPU, no collective)"}
        for r in c4["per_gpu"]:
            r["tok_s_all_gpus"] = r["tok_s"] * ws
        numerics.set_mode(args.mode)

    # ---- CPU baseline (rank 0, N=1) ----------------------------------------
    cpu = None
    parity = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        head_dv = model.lm_head.float().t().contiguous().cpu().numpy()
        from oracle import specexit_oracle as O
        obank = [O.PredictorWeights(w.w1, w.b1, w.w2, w.b2) for w in
                 (bank_w[l] for l in range(PRED_LAYERS))]
        rate, P, kind, n = cpu_reference_rate(head_dv, model.final_g.cpu().numpy(),
                                              model.final_b.cpu().numpy(), obank, ids_np,
                                              args.cpu_seconds)
        cpu = {"value": rate, "unit": "evals/s", "cores": P, "kind": "port",
               "sample": f"{n} evals of the reference chain (sliced_head_logits->extract_features->"
                         f"predictor_forward->decide_exit, d={D}, V={V}, K={K}, H={H}) in "
                         f"{args.cpu_seconds:.0f}s on {P} forked single-core processes; "
                         f"strict kernel: {kind}"}
        del head_dv
    if rank == 0 and not args.no_parity:
        parity = parity_check(spx, model, bank, bank_w, hidden, ids_all, outs, stream, prev,
                              prev0, B, inter=inter if split else None)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "evals/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference splitmix64 init of the 7B head + predictors, bf16 head; "
                    "bf16-valued N(0,1) hidden rows; splitmix64 distinct ids)",
            "config": {"workload": f"predictor path step: {PRED_LAYERS} layers x {B} requests/GPU, "
                                   + ("pipelined: per layer one launch = K1 gather of layer l + "
                                      "K2-K3 tail of layer l-1 (+1 final tail launch)" if split else
                                      "one fused K1-K3 launch per layer")
                                   + f", Llama2-7B head V={V} d={D}, "
                                   f"K={K}, H={H}, thr={THRESHOLD}, mode={args.mode}",
                       "batch_per_gpu": B, "layers_per_step": PRED_LAYERS, "k": K,
                       "predictor_hidden": H, "unique_ids_per_launch": U,
                       "l2": "no flush: inputs exceed the 126 MB L2 (520 MB of hidden rows per step, "
                             "distinct speculative ids per layer launch over the 262 MB head)",
                       "parallelism": f"dp{ws} (request sharding, no hot-path collective)",
                       "cuda_graph": True, "pdl": 3 if split else PDL, "split": split},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic,
                         "traffic_source": traffic_src,
                         "kernel": kname,
                         "algorithmic_bytes_per_launch": bytes_launch,
                         "us_per_launch": t_launch * 1e6,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gpu_launches": launches,
            "clocks": clocks,
            "decode": decode,
            "c4_batch_sweep_13b": c4,
            "fire_rate": fired,
            "certified": certified,
            "parity": parity,
            "batch1_us_per_eval": us_per_eval_b1,
            "lib": N.version(),
        }
        print(json.dumps(line))
    if ws > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
