"""Generate tests/golden/tree_tiny.json by running the REFERENCE TreeEngine
(/root/reference/pkg/src/specexit/tree.py:133-302, imported read-only).

    python tests/golden/make_tree_golden.py [--ref /root/reference/pkg/src]

Inputs are the reference pipeline's own trained tiny artifacts
(tests/golden/tiny_pipeline/: 8-layer target, 2-layer draft, 7 trained
predictors, offline profile) and prompts drawn with the reference's
corpus_prompts.  Every exit_prob call is recorded (layer, node, prob) through
a thin policy wrapper, so a device run can be compared decision by decision,
and every TreeStepResult field is stored.
"""
import argparse
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PIPE = os.path.join(HERE, "tiny_pipeline")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--steps", type=int, default=8)
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from specexit.engine import AlwaysExitPolicy, EngineConfig, NeverExitPolicy, PredictorPolicy
    from specexit.model import load_weights
    from specexit.pipeline import corpus_prompts
    from specexit.predictor import load_predictors
    from specexit.scheduler import ScheduleConfig, load_profile
    from specexit.tree import TreeEngine

    target = load_weights(os.path.join(PIPE, "target.spxw"))
    draft = load_weights(os.path.join(PIPE, "draft.spxw"))
    bank = load_predictors(os.path.join(PIPE, "predictors.spxp"))
    profile = load_profile(os.path.join(PIPE, "profile.spxs"))
    with open(os.path.join(PIPE, "fixture_corpus.txt"), "rb") as fh:
        prompts = corpus_prompts(fh.read(), 3, 16, 707)

    class Recording:
        """Wraps a policy; logs every exit_prob call in call order."""

        def __init__(self, inner):
            self.inner, self.log = inner, []

        def start(self, prompt):
            self.inner.start(prompt)

        def observe(self, token):
            self.inner.observe(token)

        def exit_prob(self, layer, features, hidden):
            p = self.inner.exit_prob(layer, features, hidden)
            self.log.append([int(layer), float(p)])
            return p

    cases = [
        ("predictor_two_level_t07", lambda: PredictorPolicy(bank), 0.7, "two-level", (3, 2)),
        ("predictor_all_t05", lambda: PredictorPolicy(bank), 0.5, "all", (2, 2, 1)),
        ("predictor_two_level_t05", lambda: PredictorPolicy(bank), 0.5, "two-level", (5, 2, 1)),
        ("always_all", AlwaysExitPolicy, 0.5, "all", (3, 2)),
        ("never_all", NeverExitPolicy, 0.5, "all", (2, 2)),
    ]
    out = []
    for name, mk, thr, mode, branching in cases:
        for prompt in prompts:
            pol = Recording(mk())
            eng = TreeEngine(target, draft, pol, branching,
                             EngineConfig(k=4, threshold=thr, schedule_mode=mode),
                             profile=profile if mode == "two-level" else None,
                             schedule_config=ScheduleConfig(5, 1, 4))
            eng.start(prompt)
            steps = []
            for _ in range(args.steps):
                n0 = len(pol.log)
                r = eng.step()
                steps.append(dict(accepted_tokens=list(map(int, r.accepted_tokens)),
                                  correction_token=int(r.correction_token),
                                  path_exit_layers=list(map(int, r.path_exit_layers)),
                                  accepted_path=int(r.accepted_path),
                                  predictor_evals=int(r.predictor_evals),
                                  num_paths=int(r.num_paths), max_path_len=int(r.max_path_len),
                                  scheduled_layer_count=int(r.scheduled_layer_count),
                                  probs=pol.log[n0:]))
            out.append(dict(case=name, threshold=thr, mode=mode, branching=list(branching),
                            prompt=list(map(int, prompt)), context=list(map(int, eng.context)),
                            online_queue=list(map(int, eng.online.queue)), steps=steps))
            print(name, prompt[:4], [len(s["accepted_tokens"]) for s in steps],
                  [s["path_exit_layers"][s["accepted_path"]] for s in steps], flush=True)
    with open(os.path.join(HERE, "tree_tiny.json"), "w") as fh:
        json.dump(dict(source="reference TreeEngine on tests/golden/tiny_pipeline artifacts",
                       schedule=[5, 1, 4], k=4, cases=out), fh)
    print("wrote", os.path.join(HERE, "tree_tiny.json"))


if __name__ == "__main__":
    main()
