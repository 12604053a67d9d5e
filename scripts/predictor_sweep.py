"""Predictor microbench sweep (BASELINE configs[4]: vocab 32k/128k, K 1-64,
hidden 4096/8192, batch 1-1024) against the HBM roofline.  One JSON line per
configuration: device time per fused launch (CUDA graph of 8 launches over
distinct layers / id sets, warm-up first), algorithmic bytes, fraction of
MEASURED_PEAKS hbm_gbs, and which kernel served it (stream / team)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_08850_b200 as spx  # noqa: E402
from paper_2504_08850_b200 import numerics, rng  # noqa: E402

H, NL = 512, 8
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launch_bytes(B, U, K, d):
    return U * d * 2 + B * d * 4 + B * (3 * K * 4 + 5) + 2 * d * 4 + (3 * K * H + 2 * H + 1) * 4


def one(model, V, d, K, B, peak, chain=False):
    bank = spx.PredictorBank({l: spx.init_predictor(K, H, rng.derive(3, l)) for l in range(NL)}, NL)
    g = torch.Generator(device="cuda")
    g.manual_seed(B * 131 + K)
    hidden = torch.randn((NL, B, d), generator=g, device="cuda").to(torch.bfloat16).float()
    ids = torch.empty((NL, B, K), dtype=torch.int32, device="cuda")
    for l in range(NL):                    # K distinct ids per request, fresh set per layer
        ids[l] = torch.rand((B, V), generator=g, device="cuda").topk(K, dim=1).indices.to(torch.int32)
    U = float(np.mean([torch.unique(ids[l]).numel() for l in range(NL)]))
    prev0 = torch.full((B, K), float(np.float32(1.0 / K)), device="cuda")
    prev = prev0.clone()

    inter = torch.zeros((NL, B, 2 * K + 2), device="cuda")

    def step():
        prev.copy_(prev0)
        if chain:                          # pipelined split form (gather l + tail l-1)
            spx.evaluate_chain(model, bank, hidden, ids, prev, inter, list(range(NL)),
                               threshold=0.7)
            return
        for l in range(NL):
            spx.evaluate_batch(model, bank, hidden[l], ids[l], prev, threshold=0.7, layer=l,
                               outputs=False, pdl=2)

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=s):
            step()
        for _ in range(max(3, int(20000 / (NL * max(B, 64))))):   # clocks up, caches steady
            graph.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(s)
        for _ in range(reps):
            graph.replay()
        e1.record(s)
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (reps * NL)
    by = launch_bytes(B, U, K, d)
    kern = ("pipelined-chain" if chain else
            "stream" if (K <= 8 and d in (2048, 4096, 8192)) else
            "team-wide (2 teams)" if d * 2 * 2 * 4 * 2 > 227 * 1024 else "team")
    return {"V": V, "d": d, "K": K, "B": B, "U": U, "us_per_launch": us,
            "evals_per_s": B / (us * 1e-6), "GBps": by / (us * 1e-6) / 1e9,
            "frac": by / (us * 1e-6) / 1e9 / peak, "kernel": kern}


def main():
    numerics.set_mode("fast")
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6540.5) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6540.5
    for V in (32000, 128000):
        for d in (4096, 8192):
            cfg = spx.ModelConfig(vocab_size=V, hidden_dim=d, num_layers=NL + 1, num_heads=32,
                                  ffn_dim=4 * d, max_context=64, seed=11)
            model = spx.init_model(cfg, dtype="bf16", head_only=True)
            for K in (1, 4, 16, 64):
                for B in (1, 64, 1024):
                    print(json.dumps(one(model, V, d, K, B, peak)), flush=True)
                    if K <= 8 and B >= 64:
                        print(json.dumps(one(model, V, d, K, B, peak, chain=True)), flush=True)
            del model
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
