"""specexit.model (src/specexit/model.py) on the B200 library.  Models are
device-resident (f32 weights, the reference's own values); functions return
numpy like the reference."""
import paper_2504_08850_b200 as _g
from paper_2504_08850_b200 import decode as _decode
from paper_2504_08850_b200 import model as _m

from ._conv import host

LN_EPS = _g.LN_EPS
ModelConfig = _g.ModelConfig
TransformerModel = _g.TransformerModel
tensor_specs = _g.tensor_specs


def init_model(config, dtype="f32"):
    """model.py:121-137 (f32: the reference's values exactly)."""
    return _g.init_model(config, dtype=dtype)


def load_weights(path):
    return _g.load_weights(path, dtype="f32")


def save_weights(model, path):
    """model.py:408-417."""
    _m.save_weights(model, path)


def full_head_logits(model, hidden):
    return host(_g.full_head_logits(model, hidden)).reshape(-1)


def sliced_head_logits(model, hidden, token_ids):
    return host(_g.sliced_head_logits(model, hidden, token_ids))


def layer_norm(x, g, b):
    return host(_g.layer_norm(x, g, b))


class DecodeState(_decode.DecodeState):
    """model.py:155-286: run_layer returns the new rows as numpy."""

    def run_layer(self, l):
        return host(super().run_layer(l))


def forward_to_layer(model, tokens, stop_layer, state=None):
    out, st = _decode.forward_to_layer(model, tokens, stop_layer,
                                       state if state is not None else DecodeState(model))
    return host(out), st


def prefill(model, tokens):
    st = DecodeState(model)
    if len(tokens) > 1:
        st.begin(tokens[:-1])
        for l in range(model.config.num_layers):
            st.launch_layer(l)
    return st
