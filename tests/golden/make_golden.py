"""Generate the golden fixtures of tests/golden/ by running the REFERENCE
implementation (/root/reference/pkg/src/specexit, imported read-only).

    python tests/golden/make_golden.py [--ref /root/reference/pkg/src]

Only this container has /root/reference; the outputs are committed so the
tests (and the GPU box) never need it.  Every fixture records the inputs (or
the seeds that regenerate them) and the reference's outputs.

tiny_pipeline/ is produced separately by make_tiny_pipeline.sh (the
reference's own `Pipeline(load_config()).run_all()`, 5-6 min CPU); its
trace.jsonl is byte-identical to the reference's shipped
pkg/runs/default/trace.jsonl.
"""
import argparse
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


def f32bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


def round_bf16(x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg/src")
    ap.add_argument("--skip-7b", action="store_true")
    args = ap.parse_args()
    sys.path.insert(0, args.ref)
    from specexit import kernels, rng
    from specexit.engine import (AlwaysExitPolicy, EngineConfig, ExitEngine, NeverExitPolicy,
                                 PredictorPolicy)
    from specexit.model import (ModelConfig, TransformerModel, full_head_logits, init_model,
                                sliced_head_logits, tensor_specs)
    from specexit.predictor import (_sigmoid, extract_features, init_predictor,
                                    predictor_forward, uniform_probs)
    from specexit.scheduler import (OfflineProfile, OnlineState, ScheduleConfig, active_layers,
                                    update_online)
    from specexit.tree import grouped_speculative_logits
    print("reference kernels backend:", kernels.backend_name())

    # ---- 1. rng known answers (rng.py; tests/test_rng.py:7) -------------------
    kat = {
        "splitmix64_seed0": [int(v) for v in rng.splitmix64(0, 3)],
        "splitmix64_seed12345": [int(v) for v in rng.splitmix64(12345, 5)],
        "derive": [[s, i, int(rng.derive(s, i))] for s in (0, 7, 2 ** 63 + 5) for i in (0, 1, 5, 40)],
        "uniform_bits": f32bits(rng.uniform(99, 64, -0.25, 0.5)).tolist(),
    }
    with open(os.path.join(HERE, "rng_kat.json"), "w") as fh:
        json.dump(kat, fh)

    # ---- 2. predictor path at the tiny config (bf16-representable weights) ---
    def bf16_model(cfg):
        m = init_model(cfg)
        return TransformerModel(cfg, {k: round_bf16(v) for k, v in m.tensors.items()})

    def predictor_case(model, n_rows, K, H, seed, pred_seed, thr_list, hidden_scale=1.0):
        d, V = model.config.hidden_dim, model.config.vocab_size
        r = np.random.default_rng(seed)
        hidden = round_bf16(r.standard_normal((n_rows, d)).astype(np.float32) * hidden_scale)
        ids = np.stack([r.choice(V, size=K, replace=False) for _ in range(n_rows)]).astype(np.int64)
        w = init_predictor(K, H, pred_seed)
        w.b1 = (r.standard_normal(H) * 0.05).astype(np.float32)     # exercise +b1
        w.b2 = float(np.float32(r.standard_normal() * 0.01))
        prev = np.empty((n_rows, K), np.float32)
        out = {k: [] for k in ("logits", "probs", "feats", "z2", "prob", "argmax")}
        for i in range(n_rows):
            # alternate uniform prev and a carried prev (engine.py:184/:196)
            pv = uniform_probs(K) if i % 2 == 0 else out["probs"][-1]
            prev[i] = pv
            lg = sliced_head_logits(model, hidden[i], ids[i])
            fv = extract_features(lg, pv)
            f = fv.concat()
            h = np.maximum(f @ w.w1 + w.b1, 0)
            z2 = h @ w.w2 + w.b2
            p = predictor_forward(w, fv)
            assert p == float(_sigmoid(z2))
            out["logits"].append(lg)
            out["probs"].append(fv.local_probs)
            out["feats"].append(f)
            out["z2"].append(np.float32(z2))
            out["prob"].append(p)
            out["argmax"].append(int(np.argmax(full_head_logits(model, hidden[i]))))
        res = dict(hidden=hidden, ids=ids, prev=prev, w1=w.w1, b1=w.b1, w2=w.w2,
                   b2=np.float32(w.b2), logits=np.stack(out["logits"]),
                   probs=np.stack(out["probs"]), feats=np.stack(out["feats"]),
                   z2=np.array(out["z2"], np.float32), prob=np.array(out["prob"]),
                   argmax=np.array(out["argmax"], np.int64))
        for thr in thr_list:
            res[f"fired_{thr}"] = np.array([p > thr for p in out["prob"]])
        return res

    tiny = bf16_model(ModelConfig(num_layers=4, seed=3))
    np.savez_compressed(os.path.join(HERE, "predictor_tiny.npz"), seed=3, layers=4,
                        **predictor_case(tiny, 64, 4, 512, seed=11, pred_seed=404,
                                         thr_list=(0.5, 0.7)))
    # larger K (blocked sgemv order, 3K >= 51) and small H
    np.savez_compressed(os.path.join(HERE, "predictor_tiny_k20.npz"), seed=3, layers=4,
                        **predictor_case(tiny, 16, 20, 512, seed=12, pred_seed=405,
                                         thr_list=(0.5,)))
    np.savez_compressed(os.path.join(HERE, "predictor_tiny_h32.npz"), seed=3, layers=4,
                        **predictor_case(tiny, 16, 4, 32, seed=13, pred_seed=406,
                                         thr_list=(0.5,)))

    # ---- 3. 7B-shaped head (lm_head 4096 x 32000 + final norm), 8 rows --------
    if not args.skip_7b:
        cfg7 = ModelConfig(vocab_size=32000, hidden_dim=4096, num_layers=32, num_heads=32,
                           ffn_dim=11008, max_context=512, seed=1234)
        names = {"final_norm.g", "final_norm.b", "lm_head"}
        tensors = {}
        for idx, (name, shape, kind) in enumerate(tensor_specs(cfg7)):
            if name not in names:
                continue
            if kind == "uniform":
                b = np.sqrt(6.0 / (shape[0] + shape[1]))
                import math
                b = math.sqrt(6.0 / (shape[0] + shape[1]))
                t = rng.uniform(rng.derive(cfg7.seed, idx), int(np.prod(shape)), -b, b).reshape(shape)
            elif kind == "zeros":
                t = np.zeros(shape, np.float32)
            else:
                t = np.ones(shape, np.float32)
            tensors[name] = round_bf16(t)

        class _Head:           # duck-typed model: only what the head functions read
            config = cfg7

            def __getitem__(self, k):
                return tensors[k]

        head = _Head()
        case = predictor_case(head, 8, 4, 512, seed=21, pred_seed=rng.derive(1234, 7),
                              thr_list=(0.5, 0.7))
        case.pop("hidden")          # regenerated from seed (16 KB/row) by the tests
        np.savez_compressed(os.path.join(HERE, "predictor_7b.npz"), seed=1234, hidden_seed=21,
                            **case)

    # ---- 4. scheduler stream (scheduler.py:49-102) ----------------------------
    r = np.random.default_rng(5)
    sched = []
    for case_i in range(12):
        L = int(r.integers(2, 40))
        cfg = ScheduleConfig(queue_len=int(r.integers(1, 8)), radius=int(r.integers(0, 4)),
                             offline_top_k=int(r.integers(1, L)))
        counts = r.integers(0, 50, L).astype(np.uint64)
        prof = OfflineProfile(num_layers=L, exit_counts=counts, fingerprint=0)
        st = OnlineState(L, cfg)
        exits, actives, nbr = [], [], []
        for _ in range(60):
            e = int(r.integers(0, L))
            update_online(st, e)
            exits.append(e)
            actives.append(active_layers(prof, st, cfg))
            nbr.append(st.neighbor_counts.tolist())
        sched.append(dict(L=L, queue_len=cfg.queue_len, radius=cfg.radius,
                          top_k=cfg.offline_top_k, exit_counts=counts.tolist(),
                          ranked=prof.ranked_layers, exits=exits, active=actives,
                          neighbor_counts=nbr, queue=list(st.queue)))
    with open(os.path.join(HERE, "scheduler_stream.json"), "w") as fh:
        json.dump(sched, fh)

    # ---- 5. grouped logits (tree.py:92-113) ------------------------------------
    r = np.random.default_rng(0)
    hid = round_bf16(r.standard_normal((40, tiny.config.hidden_dim)).astype(np.float32))
    id_lists = [sorted(r.choice(256, size=int(r.integers(1, 9)), replace=False).tolist())
                for _ in range(40)]
    grouped = grouped_speculative_logits(tiny, hid, id_lists)
    flat = np.concatenate(grouped).astype(np.float32)
    np.savez_compressed(os.path.join(HERE, "grouped_tiny.npz"), hidden=hid,
                        ids=np.concatenate(id_lists).astype(np.int64),
                        sizes=np.array([len(x) for x in id_lists], np.int64), logits=flat)

    # ---- 6. engine traces at the tiny random-init config ----------------------
    target = bf16_model(ModelConfig(num_layers=6, seed=31))
    draft = bf16_model(ModelConfig(num_layers=2, seed=32))
    bank = {l: init_predictor(4, 512, rng.derive(77, l)) for l in range(5)}
    prof = OfflineProfile(num_layers=6, exit_counts=np.array([9, 3, 7, 1, 0, 20], np.uint64),
                          fingerprint=0)
    prompts = [[84, 104, 101, 32], [10, 200, 3, 3, 3, 77, 19], [65]]
    traces = []
    for pol_name, policy, econf, sc in [
            ("never", NeverExitPolicy(), EngineConfig(), ScheduleConfig()),
            ("always", AlwaysExitPolicy(), EngineConfig(), ScheduleConfig()),
            ("predictor_all", PredictorPolicy(bank), EngineConfig(threshold=0.5), ScheduleConfig()),
            ("predictor_two_level", PredictorPolicy(bank),
             EngineConfig(threshold=0.5, schedule_mode="two-level"),
             ScheduleConfig(queue_len=5, radius=1, offline_top_k=2))]:
        for prompt in prompts:
            eng = ExitEngine(target, draft, policy, econf,
                             profile=prof if econf.schedule_mode == "two-level" else None,
                             schedule_config=sc)
            toks, trace = eng.generate(prompt, 12)
            traces.append(dict(policy=pol_name, prompt=prompt, tokens=toks,
                               threshold=econf.threshold, mode=econf.schedule_mode,
                               queue_len=sc.queue_len, radius=sc.radius,
                               top_k=sc.offline_top_k,
                               records=[json.loads(t.to_json()) | {
                                   "full_head_count": t.full_head_count,
                                   "predictor_evals": t.predictor_evals} for t in trace]))
    with open(os.path.join(HERE, "engine_tiny.json"), "w") as fh:
        json.dump(dict(target_seed=31, draft_seed=32, bank_seed=77, exit_counts=[9, 3, 7, 1, 0, 20],
                       traces=traces), fh)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
