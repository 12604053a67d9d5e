"""A/B of the predictor step forms at the bench shape (7B head, B=1024, K=4,
H=512, 31 layers): fused launches, gathers alone, tails alone, and the
split step (gathers + tails on a second stream), each captured in a CUDA
graph and timed with events.  Iteration tool (bench.py carries the line)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2504_08850_b200 as spx
from paper_2504_08850_b200 import _native as N
from paper_2504_08850_b200 import rng

B = int(os.environ.get("B", "1024"))
K, L, V, D = 4, 31, 32000, 4096
cfg = spx.ModelConfig(vocab_size=V, hidden_dim=D, num_layers=32, num_heads=32, ffn_dim=11008,
                      max_context=512, seed=1234)
m = spx.init_model(cfg, dtype="bf16", head_only=True)
bank = spx.PredictorBank({l: spx.init_predictor(K, 512, rng.derive(1234, 100 + l))
                          for l in range(L)}, 32)
g = torch.Generator(device="cuda").manual_seed(0)
hidden = torch.randn((L, B, D), device="cuda", generator=g).to(torch.bfloat16).float()
ids = torch.stack([torch.randperm(V, device="cuda", generator=g)[:B * K].reshape(B, K).int()
                   for _ in range(L)])
prev0 = torch.full((B, K), 0.25, device="cuda")
prev = prev0.clone()
inter = torch.zeros((L, B, 2 * K + 2), device="cuda")
out = spx.predictor.BatchResult(logits=None, z=None, prob=None,
                                fired=torch.empty(B, dtype=torch.uint8, device="cuda"),
                                err=torch.zeros(1, dtype=torch.int32, device="cuda"))
tail_s = torch.cuda.Stream()
rc = spx.recheck_buffer(B)


def args_for(l):
    a, _ = spx.predictor._batch_args(m, bank, hidden[l], ids[l], prev, 0.7, l, False, False, None,
                                     None, None, None, N.SPX_MODE_FAST, None, out, None, rc, True,
                                     None)
    return a


A = [args_for(l) for l in range(L)]


def fused():
    prev.copy_(prev0)
    for l in range(L):
        A[l].pdl = 2
        N.check(N.lib().spx_predictor_eval(A[l], N.stream_ptr()), "eval")


def gathers(pdl=3):
    for l in range(L):
        A[l].pdl = pdl
        N.check(N.lib().spx_predictor_gather(A[l], N.ptr(inter[l]), N.stream_ptr()), "gather")


def tails():
    prev.copy_(prev0)
    for l in range(L):
        N.check(N.lib().spx_predictor_tail(A[l], N.ptr(inter[l]), N.stream_ptr()), "tail")


def split():
    prev.copy_(prev0)
    tail_s.wait_stream(torch.cuda.current_stream())
    for l in range(L):
        A[l].pdl = 3
        N.check(N.lib().spx_predictor_gather(A[l], N.ptr(inter[l]), N.stream_ptr()), "gather")
        ev = torch.cuda.Event()
        ev.record()
        tail_s.wait_event(ev)
        with torch.cuda.stream(tail_s):
            N.check(N.lib().spx_predictor_tail(A[l], N.ptr(inter[l]), N.stream_ptr()), "tail")
    torch.cuda.current_stream().wait_stream(tail_s)


def pipe():                          # pipelined: gather(l) + tail(l-1) per launch
    prev.copy_(prev0)
    for l in range(L):
        A[l].pdl = 3
    N.check(N.lib().spx_predictor_gather(A[0], N.ptr(inter[0]), N.stream_ptr()), "gather")
    for l in range(1, L):
        N.check(N.lib().spx_predictor_gather_tail(A[l], N.ptr(inter[l]), A[l - 1],
                                                  N.ptr(inter[l - 1]), N.stream_ptr()), "gt")
    N.check(N.lib().spx_predictor_tail_pipelined(A[L - 1], N.ptr(inter[L - 1]), N.stream_ptr()),
            "tailp")


def seq():                           # gather then tail, one stream
    prev.copy_(prev0)
    for l in range(L):
        A[l].pdl = 3
        N.check(N.lib().spx_predictor_gather(A[l], N.ptr(inter[l]), N.stream_ptr()), "gather")
        N.check(N.lib().spx_predictor_tail(A[l], N.ptr(inter[l]), N.stream_ptr()), "tail")


def timeit(fn, name, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            fn()
        for _ in range(3):
            gr.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for _ in range(reps):
            gr.replay()
        e1.record(s)
    e1.synchronize()
    us = e0.elapsed_time(e1) * 1000 / (reps * L)
    print(f"{name:10s} {us:7.2f} us/layer", flush=True)


for name in (os.environ.get("WHICH", "fused,gathers,pipe,split")).split(","):
    fn = {"fused": fused, "gathers": gathers, "gathers0": lambda: gathers(0), "tails": tails,
          "split": split, "seq": seq, "pipe": pipe}[name]
    timeit(fn, name)
print("err", out.err.item())
