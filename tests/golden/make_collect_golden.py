"""Golden fixture for GPU label collection: the REFERENCE's
own ``collect_training_data`` (src/specexit/predictor.py:219-275) on the
tiny-pipeline artifacts (tests/golden/tiny_pipeline/, made by the reference
pipeline), written to tests/golden/collect_tiny.npz.

    python tests/golden/make_collect_golden.py [--ref /tmp/refcopy/src]

Use a writable copy with the Cython kernel built (see make_tiny_pipeline.sh)
for speed; /root/reference/pkg/src works too (pure-Python backend, same
results).  Only this container has the reference; the .npz is committed.
"""
import argparse
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
TP = os.path.join(HERE, "tiny_pipeline")

# the two configurations the GPU test replays (pipeline.py:42-43 defaults
# scaled down: every layer 0..L-2 requested, as the pipeline does)
CASES = {
    "a": dict(k=4, num_prompts=3, prompt_len=16, max_new=8, seed=303),
    "b": dict(k=4, num_prompts=2, prompt_len=8, max_new=6, seed=0),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/tmp/refcopy/src")
    args = ap.parse_args()
    ref = args.ref if os.path.isdir(args.ref) else "/root/reference/pkg/src"
    sys.path.insert(0, ref)
    from specexit.model import load_weights
    from specexit.predictor import collect_training_data

    t = load_weights(os.path.join(TP, "target.spxw"))
    d = load_weights(os.path.join(TP, "draft.spxw"))
    with open(os.path.join(TP, "fixture_corpus.txt"), "rb") as fh:
        corpus = fh.read()
    layers = list(range(t.config.num_layers - 1))
    out = {}
    for name, kw in CASES.items():
        ex = collect_training_data(t, d, corpus, layers, **kw)
        out[f"{name}_features"] = np.stack([e.features for e in ex]).astype(np.float32)
        out[f"{name}_labels"] = np.array([e.label for e in ex], np.uint8)
        out[f"{name}_layers"] = np.array([e.layer for e in ex], np.int32)
        out[f"{name}_args"] = np.array([kw["k"], kw["num_prompts"], kw["prompt_len"],
                                        kw["max_new"], kw["seed"]], np.int64)
        print(name, len(ex), "examples,", int(out[f"{name}_labels"].sum()), "positive")
    np.savez_compressed(os.path.join(HERE, "collect_tiny.npz"), **out)


if __name__ == "__main__":
    main()
