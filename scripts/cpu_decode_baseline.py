"""Reference CPU early-exit decode at Llama2-7B shape (the e2e
baseline): the oracle restatement of ExitEngine (engine.py:122-246, reference
strict kernels compiled from the reference's own _ckern.c when present) on this
host, single process, batch 1 -- random-init bf16-valued weights, K=4, H=512,
thr 0.5, two-level schedule.  Prints one JSON line (tok/s over the timed
tokens, prefill excluded).  Test infrastructure / reported baseline only."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from oracle import specexit_oracle as O


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=3)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--prompt", type=int, default=8)
    args = ap.parse_args()
    t0 = time.time()
    seed = 1234
    tc = O.ModelConfig(32000, 4096, args.layers, 32, 11008, 64, seed)
    dc = O.ModelConfig(32000, 4096, 2, 32, 11008, 64, seed + 1)
    t = O.init_model(tc, bf16=True)
    d = O.init_model(dc, bf16=True)
    bank = {l: O.init_predictor(4, 512, O.derive(seed, l)) for l in range(args.layers - 1)}
    counts = np.asarray([int(x) % 97 for x in O.splitmix64(seed + 7, args.layers)], np.uint64)
    eng = O.ExitEngineOracle(tc, t, dc, d, bank, k=4, threshold=0.5, schedule_mode="two-level",
                             exit_counts=counts, schedule_config=O.ScheduleConfig(5, 2, 4))
    init_s = time.time() - t0
    prompt = [int(x) % 32000 for x in O.splitmix64(seed, args.prompt)]
    t1 = time.time()
    eng.start(prompt)
    prefill_s = time.time() - t1
    recs, times = [], []
    for _ in range(args.tokens):
        t2 = time.time()
        recs.append(eng.step())
        times.append(time.time() - t2)
    print(json.dumps({
        "what": "reference CPU early-exit decode (oracle ExitEngine, strict kernels), Llama2-7B "
                "shape random-init bf16-valued weights, batch 1, K=4, H=512, thr 0.5, two-level",
        "tok_s": len(times) / sum(times), "s_per_token": times, "tokens": len(times),
        "cores": 1, "strict_kernel": "oracle/strict.c (sequential f32, no FMA)",
        "avg_exit_layer": float(np.mean([r.exit_layer for r in recs])),
        "prompt_len": args.prompt, "prefill_s": prefill_s, "init_s": init_s}))


if __name__ == "__main__":
    main()
