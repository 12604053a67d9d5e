"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
the stream predictor kernel (d=4096, K=4, two CTAs per SM), the team kernel
(tiny d), one device TreeEngine step and a few decode steps through the
persistent layer kernel; the round-2 kernels (pipelined chain, tcgen05 K6,
TMA-fed tcgen05 layer GEMMs, tensor-core K4 with top-K, head-dim-128
attention, softmax_pick through the tree step)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_08850_b200 as spx  # noqa: E402
from paper_2504_08850_b200 import engine as E  # noqa: E402
from paper_2504_08850_b200 import numerics, rng  # noqa: E402
from paper_2504_08850_b200 import tree as T  # noqa: E402

numerics.set_mode("fast")
# stream predictor kernel
cfg = spx.ModelConfig(vocab_size=2048, hidden_dim=4096, num_layers=2, num_heads=32, ffn_dim=8192,
                      max_context=32, seed=3)
m = spx.init_model(cfg, dtype="bf16", head_only=True)
w = spx.init_predictor(4, 512, 1)
B = 320
h = torch.randn((B, 4096), device="cuda")
ids = torch.randint(0, 2048, (B, 4), device="cuda", dtype=torch.int32)
ids[:, 1] = (ids[:, 0] + 1) % 2048
ids[:, 2] = (ids[:, 0] + 2) % 2048
ids[:, 3] = (ids[:, 0] + 3) % 2048
prev = torch.full((B, 4), 0.25, device="cuda")
out = spx.evaluate_batch(m, w, h, ids, prev, threshold=0.5, pdl=2)
torch.cuda.synchronize()
assert out.err.item() == 0
# tiny engine (team kernel + decode layers + device graph) and one tree step
t = spx.init_model(spx.ModelConfig(num_layers=4, seed=31), dtype="bf16")
d = spx.init_model(spx.ModelConfig(num_layers=2, seed=32), dtype="bf16")
bank = {l: spx.init_predictor(4, 512, rng.derive(77, l)) for l in range(3)}
eng = E.ExitEngine(t, d, E.PredictorPolicy(bank), E.EngineConfig(threshold=0.5))
print(eng.generate([84, 104, 101, 32], 3)[0])
te = T.TreeEngine(t, d, E.PredictorPolicy(bank), (2, 2))
te.start([84, 104, 101, 32])
print(te.step().accepted_tokens)
# persistent layer kernel at an LLM width (decode rows)
cfg2 = spx.ModelConfig(vocab_size=512, hidden_dim=1024, num_layers=2, num_heads=8, ffn_dim=2816,
                       max_context=32, seed=9)
m2 = spx.init_model(cfg2, dtype="bf16")
st = spx.DecodeState(m2)
st.begin([1, 2, 3])
for l in range(2):
    st.run_layer(l)
st.begin([4])
for l in range(2):
    st.run_layer(l)
st.check()
# round 2: the pipelined predictor chain, the tcgen05 K6 and the tcgen05
# multi-row layers (20 rows), the batched engine
L3 = 3
hh = torch.randn((L3, B, 4096), device="cuda").to(torch.bfloat16).float()
ids3 = torch.stack([ids, (ids + 7) % 2048, (ids + 13) % 2048])
bank3 = spx.PredictorBank({l: spx.init_predictor(4, 512, l) for l in range(L3)}, L3)
inter = torch.zeros((L3, B, 10), device="cuda")
prev3 = torch.full((B, 4), 0.25, device="cuda")
spx.evaluate_chain(m, bank3, hh, ids3, prev3, inter, [0, 1, 2], threshold=0.5)
from paper_2504_08850_b200.model import head_prep, merged_logits  # noqa: E402
rs = np.random.default_rng(0)
pool = rs.choice(2048, 96, replace=False)
rows_h = torch.randn((80, 4096), device="cuda")
merged_logits(m, head_prep(m, rows_h), [rs.choice(pool, 16, replace=False) for _ in range(80)],
              tensor_cores=True)
st2 = spx.DecodeState(m2)
st2.begin(list(range(1, 21)))
for l in range(2):
    st2.run_layer(l)
st2.check()
be = spx.BatchedExitEngine(t, d, E.PredictorPolicy(bank), E.EngineConfig(threshold=0.5),
                           batch=17, context=16)
be.generate([[84, 104, 101, 32]] * 17, 2)
# round 2, later: head dim 128 (warp-per-item attention writing Wo's parts),
# the TMA-fed tcgen05 GEMMs under PDL, the tensor-core K4 (+ draft top-K)
m3 = spx.init_model(spx.ModelConfig(vocab_size=1024, hidden_dim=1024, num_layers=3, num_heads=8,
                                    ffn_dim=2816, max_context=32, seed=11), dtype="bf16")
d3 = spx.init_model(spx.ModelConfig(vocab_size=1024, hidden_dim=1024, num_layers=1, num_heads=8,
                                    ffn_dim=2816, max_context=32, seed=12), dtype="bf16")
bank3b = {l: spx.init_predictor(4, 512, rng.derive(78, l)) for l in range(2)}
be3 = spx.BatchedExitEngine(m3, d3, E.PredictorPolicy(bank3b), E.EngineConfig(threshold=0.5),
                            batch=20, context=16)
be3.generate([[5, 6, 7, 8]] * 20, 2)
torch.cuda.synchronize()
print("sanitize workload ok")
