"""Early-exit decode at Llama2-7B shape, batch 1, through the
device-resident ExitEngine: tok/s of graph replays (device-timed) and of
generate() end to end.  Iteration tool; bench.py carries the contract line."""
import argparse
import os
import sys
import json
import time

import numpy as np
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import engine as E
from paper_2504_08850_b200 import numerics, rng


SHAPES = {"7b": (4096, 11008, 32, 32), "13b": (5120, 13824, 40, 40)}   # d, ffn, heads, layers


def c2_models(seed=1234, layers=32, draft_layers=2, d=4096, ffn=11008, heads=32, V=32000):
    tc = spx.ModelConfig(V, d, layers, heads, ffn, 512, seed)
    dc = spx.ModelConfig(V, d, draft_layers, heads, ffn, 512, seed + 1)
    return spx.init_model(tc, dtype="bf16"), spx.init_model(dc, dtype="bf16")


def c2_engine(t, d, seed=1234, thr=0.5, mode="two-level", k=4):
    L = t.config.num_layers
    bank = {l: spx.init_predictor(k, 512, rng.derive(seed, l)) for l in range(L - 1)}
    # seeded skewed offline profile
    counts = np.asarray([int(x) % 97 for x in rng.splitmix64(seed + 7, L)], dtype=np.uint64)
    prof = spx.OfflineProfile(L, counts, 0)
    return E.ExitEngine(t, d, E.PredictorPolicy(bank),
                        E.EngineConfig(k=k, threshold=thr, schedule_mode=mode), prof,
                        spx.ScheduleConfig(5, 2, 4))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="7b", choices=sorted(SHAPES))
    ap.add_argument("--layers", type=int, default=0, help="0: the model's own depth")
    ap.add_argument("--tokens", type=int, default=64)
    ap.add_argument("--thr", type=float, default=0.5)
    ap.add_argument("--mode", default="two-level")
    ap.add_argument("--numerics", default="fast")
    ap.add_argument("--profile", default=None, help="path: per-kernel table of 8 token replays")
    args = ap.parse_args()
    numerics.set_mode(args.numerics)
    t0 = time.time()
    dd, ff, hh, ll = SHAPES[args.model]
    t, d = c2_models(layers=args.layers or ll, d=dd, ffn=ff, heads=hh)
    eng = c2_engine(t, d, thr=args.thr, mode=args.mode)
    torch.cuda.synchronize()
    print(f"init {time.time() - t0:.1f}s", flush=True)
    prompt = [int(x) % 32000 for x in rng.splitmix64(1234, 16)]
    toks, trace = eng.generate(prompt, 8)             # capture + warm
    # timed: replay the captured step
    eng.start(prompt)
    g = eng._dev.graph(False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.tokens):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    recs = eng._dev.records(args.tokens)
    if args.profile:
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from kernel_table import kernel_table
        eng.start(prompt)
        kernel_table(lambda: [g.replay() for _ in range(8)], args.profile)
    el = np.mean([r.exit_layer for r in recs])
    fires = np.mean([r.predictor_fired for r in recs])
    ver = np.mean([r.verified for r in recs])
    evals = np.mean([r.predictor_evals for r in recs])
    heads = np.mean([r.full_head_count for r in recs])
    # e2e through the public API (host prompt in, host tokens out)
    t1 = time.perf_counter()
    toks, trace = eng.generate(prompt, args.tokens)
    e2e = args.tokens / (time.perf_counter() - t1)
    print(json.dumps({"tok_s": args.tokens / (ms / 1e3), "ms_per_tok": ms / args.tokens,
                      "e2e_tok_s": e2e, "avg_exit_layer": float(el), "fire_tok_frac": float(fires),
                      "verified_frac": float(ver), "evals_per_tok": float(evals),
                      "full_heads_per_tok": float(heads), "layers": t.config.num_layers,
                      "model": args.model}))


if __name__ == "__main__":
    main()
