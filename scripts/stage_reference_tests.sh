#!/usr/bin/env bash
# Stage the reference's own hot-path test modules so
# they can run against the B200 library through the `specexit` compatibility
# package (paper_2504_08850_b200/compat) on the GPU box, where /root/reference
# does not exist.  Copies into baseline/_ref/tests -- git-ignored (reference
# sources never enter the repository history), but shipped with the gpurun
# snapshot like the reference install in baseline/_ref.  Run here (this
# container has /root/reference):
#     bash scripts/stage_reference_tests.sh
# then on the GPU box: python -m pytest tests/test_gpu_reference_suite.py -m gpu
set -euo pipefail
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
SRC=/root/reference/pkg/tests
DST="$ROOT/baseline/_ref/tests"
mkdir -p "$DST"
for f in test_predictor.py test_scheduler.py test_engine.py test_tree.py; do
  cp "$SRC/$f" "$DST/$f"
done
: > "$DST/pytest.ini"
cat > "$DST/conftest.py" <<'PY'
"""Fixtures for the reference test modules run against the B200 library.

`import specexit` resolves to paper_2504_08850_b200/compat/specexit.  The
reference conftest trains its small_target / small_draft (train_lm, out of
scope here); these fixtures load the reference pipeline's own TRAINED tiny
target / draft instead (tests/golden/tiny_pipeline, made by the reference)."""
import os
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", "..", ".."))
sys.path.insert(0, ROOT)
from paper_2504_08850_b200 import compat  # noqa: E402

compat.install()
from specexit.model import ModelConfig, init_model, load_weights  # noqa: E402

TP = os.path.join(ROOT, "tests", "golden", "tiny_pipeline")


@pytest.fixture(scope="session")
def corpus():
    with open(os.path.join(TP, "fixture_corpus.txt"), "rb") as fh:
        return fh.read()


@pytest.fixture(scope="session")
def small_target():
    return load_weights(os.path.join(TP, "target.spxw"))


@pytest.fixture(scope="session")
def small_draft():
    return load_weights(os.path.join(TP, "draft.spxw"))


@pytest.fixture(scope="session")
def untrained_target():
    return init_model(ModelConfig(num_layers=4, seed=3))
PY
echo "staged $(ls "$DST" | wc -l) files into $DST"
