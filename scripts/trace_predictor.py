"""Per-row phase timeline of the fused predictor kernel (debug hook
spx_debug_trace): where does a launch's time go?"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import _native as N
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
trace = torch.zeros((B, 16), dtype=torch.int64, device="cuda")
lib = N.lib()
lib.spx_debug_trace.argtypes = [ctypes.c_void_p]
# warm the clocks up (~0.3 s of launches) before the traced launch
for it in range(3000):
    spx.evaluate_batch(m, bank, hidden[it % 4], ids, prev, threshold=0.7, layer=it % 4, outputs=False)
for it in range(6):
    if it == 5:
        lib.spx_debug_trace(ctypes.c_void_p(trace.data_ptr()))
    if it < 5:
        prev.fill_(1.0 / K)
    spx.evaluate_batch(m, bank, hidden[it % 4], ids, prev, threshold=0.7, layer=it % 4, outputs=False)
torch.cuda.synchronize()
lib.spx_debug_trace(None)
t = trace.cpu().numpy().astype(np.int64)
t0 = t[:, 5].min()
t = t - t0
issue, tstart, data, p1, dots, done = t[:, 5], t[:, 0], t[:, 1], t[:, 2], t[:, 3], t[:, 4]
print(f"B={B} span(issue0->last done) = {done.max()/1e3:.2f} us")
wst = t[:, 6]
for name, v in [("issue->data ready", data - issue), ("compute wait start->data", data - wst),
                ("pass1 (data->barrier1)", p1 - data), ("pass2 (barrier1->release)", dots - p1),
                ("release->tail got logits", tstart - dots), ("tail compute", done - tstart),
                ("row total issue->done", done - issue),
                ("gap prev release->wait start", np.r_[0, wst[1:] - dots[:-1]])]:
    print(f"{name:30s} mean {v.mean()/1e3:7.3f} us  p50 {np.median(v)/1e3:7.3f}  max {v.max()/1e3:7.3f}")
for nm, a, b in [("softmax+features", 8, 9), ("tbar1", 9, 10), ("z1 quarter + tbar2", 10, 11),
                 ("z2 + outputs", 11, 12)]:
    dv = (t[:, b] - t[:, a]).astype(np.float64)
    print(f"tail {nm:20s} cycles p50 {np.median(dv):.0f} mean {dv.mean():.0f}")
rows0 = np.arange(0, B, 148)
print("CTA0 rows: issue", (issue[rows0] / 1e3).round(2), "\n data", (data[rows0] / 1e3).round(2),
      "\n release", (dots[rows0] / 1e3).round(2), "\n done", (done[rows0] / 1e3).round(2))
order = np.argsort(issue)
print("first issues (us):", (issue[order[:8]] / 1e3).round(3))
print("issue time quantiles (us):", np.percentile(issue, [0, 25, 50, 75, 100]) / 1e3)
print("done  time quantiles (us):", np.percentile(done, [0, 25, 50, 75, 100]) / 1e3)
