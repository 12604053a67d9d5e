"""specexit.predictor (src/specexit/predictor.py) on the B200 library.
Training (predictor_loss_and_grads, train_predictor, PredictorTrainConfig) is
offline tooling outside the hot path: not provided here."""
from dataclasses import dataclass

import numpy as np

import paper_2504_08850_b200 as _g

from ._conv import host

PredictorWeights = _g.PredictorWeights
init_predictor = _g.init_predictor
predictor_param_count = _g.predictor_param_count
decide_exit = _g.decide_exit
save_predictors = _g.save_predictors
load_predictors = _g.load_predictors
TrainingExample = _g.TrainingExample
collect_training_data = _g.collect_training_data


@dataclass(frozen=True)
class FeatureVector:
    """predictor.py:22-33 with numpy fields."""
    spec_logits: np.ndarray
    local_probs: np.ndarray
    prob_variation: np.ndarray

    @property
    def k(self):
        return int(self.spec_logits.size)

    def concat(self):
        return np.concatenate([self.spec_logits, self.local_probs,
                               self.prob_variation]).astype(np.float32)


def uniform_probs(k):
    return host(_g.uniform_probs(k))


def extract_features(spec_logits, prev_local_probs):
    fv = _g.extract_features(spec_logits, prev_local_probs)
    return FeatureVector(host(fv.spec_logits), host(fv.local_probs), host(fv.prob_variation))


def predictor_forward(w, features):
    f = features.concat() if hasattr(features, "concat") else features
    return _g.predictor_forward(w, np.asarray(f, np.float32))


class _Unsupported:
    def __init__(self, name):
        self.name = name

    def __call__(self, *a, **kw):
        raise NotImplementedError(f"{self.name}: predictor training is offline tooling, not "
                                  "part of the B200 hot path (use the reference package)")


PredictorTrainConfig = _Unsupported("PredictorTrainConfig")
train_predictor = _Unsupported("train_predictor")
predictor_loss_and_grads = _Unsupported("predictor_loss_and_grads")
