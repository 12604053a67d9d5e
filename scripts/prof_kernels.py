"""Minimal drivers for ncu captures of single kernels at the 7B shape
(scripts/gpu.sh stages ncuverify / ncutree):

  verify  K4 spx_verify: 1 row, full 7B head (V=32000, d=4096, bf16), FAST
  tree    K6 spx_tree_merged_logits: 26 tree nodes x K=4 draft ids (configs[2])
          and a batched-tree tile (ROWS nodes x 4 ids, ROWS=256 by default)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200.model import head_prep, merged_logits

which = sys.argv[1] if len(sys.argv) > 1 else "verify"
cfg = spx.ModelConfig(vocab_size=32000, hidden_dim=4096, num_layers=32, num_heads=32,
                      ffn_dim=11008, max_context=512, seed=1234)
m = spx.init_model(cfg, dtype="bf16", head_only=True)
g = torch.Generator(device="cuda").manual_seed(0)
if which == "verify":
    h = torch.randn((4, 4096), device="cuda", generator=g).to(torch.bfloat16).float()
    for it in range(int(os.environ.get("ITERS", "6"))):
        tok, _, _ = spx.head_argmax(m, h[it % 4])
elif which == "tree":
    rows = int(os.environ.get("ROWS", "26"))
    k = int(os.environ.get("K", "4"))
    pool = int(os.environ.get("POOL", str(max(8, rows // 2))))
    tc = {"1": True, "0": False}.get(os.environ.get("TC", ""), None)
    rs = np.random.default_rng(0)
    h = torch.randn((rows, 4096), device="cuda", generator=g).to(torch.bfloat16).float()
    # tree-like id sets: siblings share most of their draft top-k
    base = rs.choice(32000, size=pool, replace=False)
    ids = [rs.choice(base, k, replace=False) for _ in range(rows)]
    prep = head_prep(m, h)
    for it in range(int(os.environ.get("ITERS", "6"))):
        out = merged_logits(m, prep, ids, tensor_cores=tc)
    torch.cuda.synchronize()
    if os.environ.get("TIME", "0") == "1":       # CUDA-event timing of both kernels
        for mode in (False, True):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(20):
                merged_logits(m, prep, ids, tensor_cores=mode)
            e1.record()
            torch.cuda.synchronize()
            print(f"rows={rows} U<={pool} k={k} tensor_cores={mode}: "
                  f"{e0.elapsed_time(e1) * 1000 / 20:.1f} us per call (incl. host CSR build)")
else:
    raise SystemExit(f"unknown kernel {which}")
torch.cuda.synchronize()
print("ok", which)
