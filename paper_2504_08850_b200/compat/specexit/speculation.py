"""specexit.speculation (src/specexit/speculation.py) on the B200 library."""
from paper_2504_08850_b200.speculation import (SpeculativeSet, TokenTree, TreeNode,  # noqa: F401
                                               build_token_tree, enumerate_paths, propose_topk,
                                               speculative_set_from_logits, topk_from_logits)
