"""B200-native SpecEE speculative early-exit predictor path.

Drop-in for the hot path of the reference package ``specexit``: the same
function / class names, backed by hand-written sm_100a CUDA kernels in
libspecexit_b200.so (C ABI: include/specexit_b200.h).  No CPU fallback.
"""
from . import numerics  # noqa: F401
from .model import (LN_EPS, ModelConfig, TransformerModel, final_norm, from_tensors,  # noqa: F401
                    full_head_logits, head_argmax, init_model, layer_norm, load_weights,
                    save_weights, sliced_head_logits, tensor_specs, to_tensors)
from .predictor import (FeatureVector, PredictorBank, PredictorWeights, decide_exit,  # noqa: F401
                        evaluate_batch, evaluate_batch_split, evaluate_chain, extract_features, init_predictor,
                        load_predictors,
                        predictor_forward, predictor_param_count, prev_error,
                        recheck_buffer, recheck_stats, save_predictors, uniform_probs, z_cut)
from .scheduler import (OfflineProfile, OnlineState, ScheduleConfig, active_layers,  # noqa: F401
                        load_profile, online_hot_layers, profile_offline, recompute_counts,
                        save_profile, update_online, weight_fingerprint)
from .tree import (HyperToken, TreeEngine, TreeStepResult, grouped_speculative_logits,  # noqa: F401
                   hypertoken_exit_decision, hypertoken_oracle_exit, merge_paths)
from .decode import DecodeState, forward_to_layer, prefill  # noqa: F401
from .speculation import (SpeculativeSet, TokenTree, TreeNode, build_token_tree,  # noqa: F401
                          enumerate_paths, propose_topk, speculative_set_from_logits,
                          topk_from_logits)
from .engine import (AlwaysExitPolicy, EngineConfig, ExitEngine, ExitRecord,  # noqa: F401
                     NeverExitPolicy, OraclePolicy, PredictorPolicy, generate, greedy_generate,
                     oracle_exit_layer, read_trace, verify_exit, write_trace)

__version__ = "0.1.0"
from .profiling import (LayerTraces, TrainingExample, collect_training_data,  # noqa: F401
                        generation_layer_traces, profile_offline_device)
from .batched import BatchedExitEngine  # noqa: F401,E402
