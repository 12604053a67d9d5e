"""Early exiting under tree speculative decoding -- drop-in for the hot-path
part of the reference's ``specexit.tree`` (src/specexit/tree.py).

``grouped_speculative_logits`` is the context-aware merged mapping (K6): the
feature ids of all live nodes are de-duplicated and each unique LM-head row is
read from HBM once; ``path_conjunction`` is K7 (hyper-token AND over a CSR of
paths) on device.
"""
import numpy as np
import torch

from . import _native as N
from .model import TransformerModel, head_prep, merged_logits
from .predictor import decide_exit


def grouped_speculative_logits(model: TransformerModel, hiddens, token_id_lists):
    """tree.py:92-113: row j holds the logits of token_id_lists[j];
    bit-identical to sliced_head_logits on that node alone."""
    h = hiddens if isinstance(hiddens, torch.Tensor) else torch.as_tensor(
        np.asarray(hiddens, dtype=np.float32))
    if h.dim() != 2 or h.shape[0] < 1:
        raise ValueError("need at least one node hidden state")
    if len(token_id_lists) != h.shape[0]:
        raise ValueError("one id list per node required")
    v = model.config.vocab_size
    for ids in token_id_lists:
        if len(ids) == 0:
            raise ValueError("empty token id list")
        if min(ids) < 0 or max(ids) >= v:
            raise ValueError("token id out of range")
    return merged_logits(model, head_prep(model, h), token_id_lists)


def hypertoken_exit_decision(per_node_probs, threshold: float) -> bool:
    """tree.py:116-122: the slowest node gates the whole hyper-token."""
    probs = list(per_node_probs)
    if not probs:
        raise ValueError("need at least one node probability")
    return all(decide_exit(p, threshold) for p in probs)


def path_conjunction(node_fired: torch.Tensor, paths, live=None) -> torch.Tensor:
    """K7 on device: path_fire[p] = AND_j node_fired[paths[p][j]] (live paths)."""
    ptr_ = np.concatenate([[0], np.cumsum([len(p) for p in paths])]).astype(np.int32)
    nodes = np.concatenate([np.asarray(p, np.int32) for p in paths]).astype(np.int32)
    d_ptr = torch.as_tensor(ptr_, device="cuda")
    d_nodes = torch.as_tensor(nodes, device="cuda")
    d_live = None if live is None else torch.as_tensor(np.asarray(live, np.uint8), device="cuda")
    out = torch.empty(len(paths), dtype=torch.uint8, device="cuda")
    nf = node_fired.to(device="cuda", dtype=torch.uint8).contiguous()
    N.check(N.lib().spx_path_and(N.ptr(nf), N.ptr(d_ptr), N.ptr(d_nodes), N.ptr(d_live),
                                 len(paths), N.ptr(out), N.stream_ptr()), "spx_path_and")
    return out
