"""Minimal driver for ncu: a few fused predictor launches at the bench shape."""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import rng

B = int(os.environ.get("B", "1024"))
K = int(os.environ.get("K", "4"))
cfg = spx.ModelConfig(vocab_size=32000, hidden_dim=4096, num_layers=32, num_heads=32,
                      ffn_dim=11008, max_context=512, seed=1234)
m = spx.init_model(cfg, dtype="bf16", head_only=True)
bank = spx.PredictorBank({l: spx.init_predictor(K, 512, rng.derive(1234, 100 + l)) for l in range(4)}, 32)
hidden = torch.randn((4, B, 4096), device="cuda").to(torch.bfloat16).float()
ids = torch.randint(0, 32000, (B, K), device="cuda", dtype=torch.int32)
prev = torch.full((B, K), 1.0 / K, device="cuda")
inter = torch.zeros((4, B, 2 * K + 2), device="cuda")
ids4 = torch.stack([torch.randperm(32000, device="cuda")[:B * K].reshape(B, K).int()
                    for _ in range(4)])
for it in range(int(os.environ.get("ITERS", "6"))):
    prev.fill_(1.0 / K)
    if os.environ.get("CHAIN", "0") == "1":
        # the pipelined chain of the bench (gather l + tail l-1 per launch)
        out = spx.evaluate_chain(m, bank, hidden, ids4, prev, inter, [0, 1, 2, 3],
                                 threshold=0.7)[-1]
    else:
        out = spx.evaluate_batch(m, bank, hidden[it % 4], ids, prev, threshold=0.7,
                                 layer=it % 4, outputs=False)
torch.cuda.synchronize()
print("ok", out.err.item())
