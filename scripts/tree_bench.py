"""Tree speculative decoding with hyper-token exits at Llama2-7B shape
(BASELINE configs[2]: EAGLE-like tree, branching (5,2,1) = 26 nodes incl. the
root, 10 paths) through the device TreeEngine.  Prints one JSON line: committed
tokens/s (wall, end to end), per-step ms, merged-mapping statistics."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2504_08850_b200 as spx  # noqa: E402
from paper_2504_08850_b200 import engine as E  # noqa: E402
from paper_2504_08850_b200 import numerics, rng  # noqa: E402
from paper_2504_08850_b200 import tree as T  # noqa: E402


def run(steps=4, branching=(5, 2, 1), seed=1234, layers=32, thr=0.5, models=None, profile=None):
    V, D = 32000, 4096
    if models is None:
        tc = spx.ModelConfig(V, D, layers, 32, 11008, 512, seed)
        dc = spx.ModelConfig(V, D, 2, 32, 11008, 512, seed + 1)
        models = (spx.init_model(tc, dtype="bf16"), spx.init_model(dc, dtype="bf16"))
    t, d = models
    L = t.config.num_layers
    bank = {l: spx.init_predictor(4, 512, rng.derive(seed, l)) for l in range(L - 1)}
    counts = np.asarray([int(x) % 97 for x in rng.splitmix64(seed + 7, L)], dtype=np.uint64)
    prof = spx.OfflineProfile(L, counts, 0)
    eng = T.TreeEngine(t, d, E.PredictorPolicy(bank), branching,
                       E.EngineConfig(k=4, threshold=thr, schedule_mode="two-level"), prof,
                       spx.ScheduleConfig(5, 2, 4))
    prompt = [int(x) % V for x in rng.splitmix64(seed, 16)]
    eng.start(prompt)
    eng.step()                                    # warm-up (allocations, first launches)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = [eng.step() for _ in range(steps)]
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if profile:
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from kernel_table import kernel_table
        kernel_table(eng.step, profile)
    committed = sum(len(r.accepted_tokens) + 1 for r in res)
    return {"tok_s": committed / wall, "unit": "tokens/s", "ms_per_step": 1e3 * wall / steps,
            "steps": steps, "committed_tokens": committed, "branching": list(branching),
            "nodes": 1 + sum(int(np.prod(branching[:i + 1])) for i in range(len(branching))),
            "paths": int(np.prod(branching)),
            "predictor_evals_per_step": float(np.mean([r.predictor_evals for r in res])),
            "exits": int(sum(e != L - 1 for r in res for e in r.path_exit_layers)),
            "merged_unique_ids_last_layer": getattr(eng, "last_unique_ids", None),
            "merged_pairs_last_layer": getattr(eng, "last_pairs", None),
            "config": "Llama2-7B shape random-init bf16 target + 2-layer draft, K=4, thr "
                      f"{thr}, two-level, 16-token prompt, wall clock incl. host orchestration"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--layers", type=int, default=32)
    ap.add_argument("--profile", default=None, help="path: per-kernel table of one step")
    args = ap.parse_args()
    numerics.set_mode("fast")
    print(json.dumps(run(args.steps, layers=args.layers, profile=args.profile)))


if __name__ == "__main__":
    main()
