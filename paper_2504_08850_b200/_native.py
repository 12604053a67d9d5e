"""ctypes binding of libspecexit_b200.so (the C ABI in include/specexit_b200.h).

There is no CPU fallback and no alternative backend: if the library is
missing or CUDA is unavailable, every operator raises.  All tensors handed to
the library are CUDA tensors owned by PyTorch; launches go to torch's current
stream (so they are captured by torch.cuda.graph like any torch op).
"""
import ctypes
import os

import torch

from . import build as _build

SPX_MODE_FAST, SPX_MODE_STRICT = 0, 1
SPX_DTYPE_BF16, SPX_DTYPE_F32 = 0, 1
SPX_POLICY_MLP, SPX_POLICY_CONST = 0, 1
SPX_VERIFY_TC_MIN_ROWS = 8               # include/specexit_b200.h
ERR_ID_RANGE, ERR_HIDDEN_NONFINITE, ERR_LOGIT_NONFINITE, ERR_PREV_SUM, ERR_BAD_LAYER = 1, 2, 4, 8, 16
ERR_ROW_CAP = 32
ERR_CAND_OVERFLOW = 64

# device error bits -> the reference's ValueError messages
ERR_MESSAGES = [
    (ERR_ID_RANGE, "token id out of range"),                      # model.py:307-308
    (ERR_HIDDEN_NONFINITE, "non-finite hidden state"),            # model.py:310-311
    (ERR_LOGIT_NONFINITE, "non-finite speculative logits"),       # predictor.py:47-48
    (ERR_PREV_SUM, "prev_local_probs must sum to 1"),             # predictor.py:49-50
    (ERR_BAD_LAYER, "exit layer out of range"),                   # scheduler.py:69-70
    (ERR_ROW_CAP, "layer call selected more rows than its row capacity"),
    (ERR_CAND_OVERFLOW, "tensor-core verify: too many near-maximal logits to re-evaluate"),
]

_vp = ctypes.c_void_p
_i32, _i64, _f32, _f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_double


class PredictorArgs(ctypes.Structure):
    _fields_ = [("hidden", _vp), ("hidden_stride", _i64), ("norm_g", _vp), ("norm_b", _vp),
                ("head", _vp), ("head_dtype", _i32), ("head_bw", _vp), ("ids", _vp),
                ("prev", _vp),
                ("w1", _vp), ("b1", _vp), ("w2", _vp), ("b2", _f32), ("z_cut", _f32),
                ("policy", _i32), ("const_prob", _f64), ("threshold", _f64),
                ("logits_out", _vp), ("feat_out", _vp), ("z_out", _vp), ("prob_out", _vp),
                ("fired", _vp), ("row_layer_mask", _vp), ("row_done", _vp), ("evals", _vp),
                ("layer", _i32), ("mode", _i32), ("pdl", _i32), ("err", _vp),
                ("B", _i64), ("d", _i64), ("V", _i64), ("K", _i64), ("H", _i64),
                ("head_wmax", _vp), ("cert", _vp), ("cert_kappa", _f32), ("cert_hnorm", _f32),
                ("prev_err", _vp), ("recheck", _vp), ("fired_any", _vp)]


class VerifyArgs(ctypes.Structure):
    _fields_ = [("hidden", _vp), ("hidden_stride", _i64), ("norm_g", _vp), ("norm_b", _vp),
                ("head", _vp), ("head_dtype", _i32), ("head_bw", _vp), ("gate", _vp),
                ("row_done", _vp),
                ("spec_ptr", _vp), ("spec_ids", _vp), ("token_out", _vp),
                ("verified_out", _vp), ("maxlogit_out", _vp), ("logits_out", _vp),
                ("done_out", _vp), ("exit_layer_out", _vp), ("full_heads", _vp),
                ("layer", _i32), ("scratch", _vp), ("counter", _vp), ("mode", _i32),
                ("err", _vp), ("B", _i64), ("d", _i64), ("V", _i64),
                ("head_wmax", _vp), ("tc_scratch", _vp), ("topk_out", _vp), ("topk_k", _i32)]


class OnlineStateC(ctypes.Structure):
    _fields_ = [("queue", _vp), ("head", _vp), ("len", _vp), ("counts", _vp)]


class LayerArgs(ctypes.Structure):
    """spx_layer_args (include/specexit_b200.h)."""
    _fields_ = [("ln1_g", _vp), ("ln1_b", _vp), ("ln2_g", _vp), ("ln2_b", _vp),
                ("wqkv", _vp), ("wo", _vp), ("w1", _vp), ("w2", _vp), ("b1", _vp), ("b2", _vp),
                ("w_dtype", _i32), ("pending", _vp), ("kcache", _vp), ("vcache", _vp),
                ("frontier", _vp), ("n_ctx", _vp), ("new_row", _vp), ("frozen", _vp),
                ("attn_ptr", _vp), ("attn_idx", _vp), ("done", _vp), ("cur_hidden", _vp),
                ("rows", _vp), ("nrows", _vp), ("s_q", _vp), ("s_att", _vp), ("s_f", _vp),
                ("s_part", _vp), ("s_flag", _vp),
                ("layer", _i32), ("mode", _i32), ("err", _vp),
                ("max_ctx", _i64), ("d", _i64), ("n_heads", _i64), ("ffn", _i64),
                ("rows_hint", _i32), ("row_cap", _i32), ("att_cap", _i32), ("tc_scratch", _vp)]


class TokenStateC(ctypes.Structure):
    """spx_token_state (include/specexit_b200.h)."""
    _fields_ = [("prev", _vp), ("done", _vp), ("fired", _vp), ("fired_any", _vp),
                ("exit_layer", _vp), ("exit_token", _vp), ("final_token", _vp), ("evals", _vp),
                ("full_heads", _vp), ("next_in", _vp), ("step", _vp), ("active", _vp),
                ("rec_token", _vp), ("rec_exit_layer", _vp), ("rec_evals", _vp),
                ("rec_full_heads", _vp), ("rec_fired", _vp), ("rec_verified", _vp),
                ("rec_active", _vp), ("prev_err", _vp)]


_LIB = None


def lib():
    """Load (building in-tree if needed) the CUDA library; raise if impossible."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = _build.LIB
    if not os.path.exists(path) or _build._stale():
        _build.build()
    L = ctypes.CDLL(path)
    L.spx_predictor_eval.argtypes = [ctypes.POINTER(PredictorArgs), _vp]
    L.spx_verify.argtypes = [ctypes.POINTER(VerifyArgs), _vp]
    L.spx_sched_update.argtypes = [OnlineStateC, _vp, _vp, _i64, _i32, _i32, _i32, _vp, _vp]
    L.spx_sched_active.argtypes = [OnlineStateC, ctypes.c_uint64, _i64, _i32, _i32, _vp, _vp]
    L.spx_tree_merged_logits.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp, _i64, _i64, _vp, _i64,
                                         _vp, _vp, _vp, _vp, _i32, _vp, _vp]
    L.spx_head_prep.argtypes = [_vp, _i64, _vp, _vp, _vp, _vp, _i64, _i64, _i32, _vp, _vp]
    L.spx_head_bias.argtypes = [_vp, _i32, _vp, _i64, _i64, _vp, _vp]
    L.spx_final_norm.argtypes = [_vp, _i64, _vp, _vp, _vp, _i64, _i64, _i32, _vp, _vp]
    L.spx_path_and.argtypes = [_vp, _vp, _vp, _vp, _i64, _vp, _vp]
    L.spx_tree_gate.argtypes = [_vp, _vp, _vp, _i64, _i64, _vp, _vp]
    L.spx_tree_node_eval.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp, _vp, _f32, _f32, _i32, _f64,
                                     _f64, _vp, _vp, _vp, _i64, _i64, _vp]
    L.spx_init_uniform.argtypes = [_vp, _i32, _i64, _i64, _i32, ctypes.c_uint64, _f64, _f64, _vp]
    L.spx_version.restype = ctypes.c_char_p
    L.spx_predictor_mlp.argtypes = [_vp, _vp, _vp, _vp, _f32, _f32, _vp, _vp, _vp, _i64, _i64,
                                    _i64, _vp]
    L.spx_extract_features.argtypes = [_vp, _vp, _vp, _vp, _i64, _i64, _vp]
    L.spx_np_expf.argtypes = [_vp, _vp, _i64, _vp]
    L.spx_layer_forward.argtypes = [ctypes.POINTER(LayerArgs), _vp]
    L.spx_layer_part_floats.argtypes = [_i64, _i64]
    L.spx_layer_part_floats.restype = _i64
    L.spx_layer_flag_ints.argtypes = [_i64, _i64]
    L.spx_layer_flag_ints.restype = _i64
    L.spx_embed.argtypes = [_vp, _i32, _vp, _vp, _vp, _i64, _i64, _i64, _i64, _vp, _vp, _vp,
                            _vp, _vp, _vp]
    L.spx_topk.argtypes = [_vp, _i64, _i32, _vp, _vp]
    L.spx_topk_rows.argtypes = [_vp, _i64, _i64, _i32, _vp, _vp]
    L.spx_token_begin.argtypes = [TokenStateC, _i32, _i32, _f32, _vp]
    L.spx_token_end.argtypes = [TokenStateC, OnlineStateC, _i32, _i32, _i32, _i64, _vp]
    L.spx_or_flag.argtypes = [_vp, _vp, _vp]
    L.spx_force_next.argtypes = [_vp, _vp, _vp, _i64, _vp]
    L.spx_predictor_split_ok.argtypes = [ctypes.POINTER(PredictorArgs)]
    L.spx_predictor_gather.argtypes = [ctypes.POINTER(PredictorArgs), _vp, _vp]
    L.spx_predictor_tail.argtypes = [ctypes.POINTER(PredictorArgs), _vp, _vp]
    L.spx_predictor_tail_pipelined.argtypes = [ctypes.POINTER(PredictorArgs), _vp, _vp]
    L.spx_predictor_gather_tail.argtypes = [ctypes.POINTER(PredictorArgs), _vp,
                                            ctypes.POINTER(PredictorArgs), _vp, _vp]
    L.spx_softmax_pick.argtypes = [_vp, _i64, _i64, _vp, _i32, _vp, _i32, _vp, _vp]
    L.spx_verify_tc_logits_offset.argtypes = [_i64, _i64, _i64]
    L.spx_verify_tc_logits_offset.restype = _i64
    L.spx_verify_tc_scratch_bytes.argtypes = [_i64, _i64, _i64]
    L.spx_verify_tc_scratch_bytes.restype = _i64
    L.spx_tree_tc_scratch_bytes.argtypes = [_i64, _i64, _i64, _i64]
    L.spx_tree_tc_scratch_bytes.restype = _i64
    L.spx_tree_merged_logits_tc.argtypes = [_vp, _vp, _i64, _vp, _i32, _vp, _i64, _i64, _vp, _i64,
                                            _vp, _vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp]
    L.spx_layer_tc_scratch_bytes.argtypes = [_i64, _i64, _i64]
    L.spx_layer_tc_scratch_bytes.restype = _i64
    L.spx_inject_spec.argtypes = [_vp, _i32, _vp, _vp, _vp, _i64, _vp]
    L.spx_predictor_cert.argtypes = [_vp, _vp, _vp, _i64, _i64, _vp, _vp]
    L.spx_head_stats.argtypes = [_vp, _i32, _i64, _i64, _vp, _vp]
    L.spx_debug_trace.argtypes = [_vp]
    L.spx_debug_trace.restype = None
    _LIB = L
    return L


def require_cuda(device=None):
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2504_08850_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    lib()


def stream_ptr():
    return _vp(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Device pointer of a CUDA tensor (or None)."""
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    return _vp(t.data_ptr())


def check(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed with code {rc}")


def raise_device_error(err_word):
    """Map the device error word to the reference's ValueError."""
    e = int(err_word)
    if e == 0:
        return
    for bit, msg in ERR_MESSAGES:
        if e & bit:
            raise ValueError(msg)
    raise ValueError(f"device error word {e:#x}")


def version():
    return lib().spx_version().decode()
