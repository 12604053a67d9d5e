"""BASELINE configs[3]: Llama2-13B shape (40 layers, d=5120, ffn=13824,
V=32000), batch sweep of B independent requests per GPU through the
BatchedExitEngine (random-init bf16 weights, 2-layer draft, K=4, H=512,
thr 0.5, two-level).  One JSON line per B: tokens/s (device time of the timed
steps), ms per step, and the fraction of the HBM roofline if every weight were
read once per step (the multi-row layer path re-streams the weights per 8-row
slice, so that fraction falls with B -- see DESIGN.md §8)."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import engine as E
from paper_2504_08850_b200 import numerics, rng

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(batches, steps=8, warmup=3, layers=40, prompt=16, emit=None, profile=None):
    """The sweep; returns one dict per batch size (emit(d) is called as each
    finishes)."""
    numerics.set_mode("fast")
    seed = 1234
    V, d, ffn, nh = 32000, 5120, 13824, 40
    L = layers
    C = prompt + warmup + steps + 2
    t = spx.init_model(spx.ModelConfig(V, d, L, nh, ffn, 512, seed), dtype="bf16")
    dm = spx.init_model(spx.ModelConfig(V, d, 2, nh, ffn, 512, seed + 1), dtype="bf16")
    bank = {l: spx.init_predictor(4, 512, rng.derive(seed, l)) for l in range(L - 1)}
    counts = np.asarray([int(x) % 97 for x in rng.splitmix64(seed + 7, L)], np.uint64)
    prof = spx.OfflineProfile(L, counts, 0)
    peak = 6455.3
    try:
        peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except (OSError, KeyError, ValueError):
        pass
    layer_bytes = (4 * d * d + 2 * d * ffn) * 2
    out = []
    for B in batches:
        eng = spx.BatchedExitEngine(t, dm, E.PredictorPolicy(bank),
                                    E.EngineConfig(k=4, threshold=0.5, schedule_mode="two-level"),
                                    prof, spx.ScheduleConfig(5, 2, 4), batch=B, context=C)
        prompts = [[int(x) % V for x in rng.splitmix64(seed + 10 * b, prompt)] for b in range(B)]
        eng.start(prompts)
        eng.run(warmup)
        eng.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        eng.run(steps)
        e1.record()
        eng.sync()
        ms = e0.elapsed_time(e1)
        if profile:
            from kernel_table import kernel_table
            kernel_table(lambda: eng.run(1), f"{profile}_b{B}.txt")
        recs = eng.records()
        el = float(np.mean([r.exit_layer for rs in recs for r in rs[warmup:]]))
        heads = float(np.mean([r.full_head_count for rs in recs for r in rs[warmup:]]))
        # every weight once per step: the target layers, the draft, the full heads
        step_bytes = (L + 2) * layer_bytes + (1 + heads) * V * d * 2
        res = {"model": "Llama2-13B shape", "batch_per_gpu": B, "steps": steps,
               "ms_per_step": ms / steps, "tok_s": B * steps / (ms / 1e3),
               "avg_exit_layer": el, "full_heads_per_token": heads,
               "weights_once_GBps": step_bytes / (ms / steps * 1e-3) / 1e9,
               "weights_once_frac": step_bytes / (ms / steps * 1e-3) / 1e9 / peak,
               "mem_GB": round(torch.cuda.max_memory_allocated() / 1e9, 1)}
        out.append(res)
        if emit:
            emit(res)
        del eng
        torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batches", default="1,2,4,8,16,32,64,128,256")
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--layers", type=int, default=40)
    ap.add_argument("--prompt", type=int, default=16)
    ap.add_argument("--profile", default=None, help="path prefix: per-kernel table of one step")
    args = ap.parse_args()
    run([int(x) for x in args.batches.split(",")], args.steps, args.warmup, args.layers,
        args.prompt, emit=lambda r: print(json.dumps(r), flush=True), profile=args.profile)


if __name__ == "__main__":
    main()
