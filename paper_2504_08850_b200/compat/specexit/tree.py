"""specexit.tree (src/specexit/tree.py) on the B200 library."""
import paper_2504_08850_b200.tree as _t
from paper_2504_08850_b200.tree import (HyperToken, TreeEngine, TreeStepResult,  # noqa: F401
                                        hypertoken_exit_decision, hypertoken_oracle_exit,
                                        merge_paths)

from ._conv import host_list


def grouped_speculative_logits(model, hiddens, token_id_lists):
    return host_list(_t.grouped_speculative_logits(model, hiddens, token_id_lists))
