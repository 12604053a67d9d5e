"""The reference's OWN hot-path test modules (pkg/tests/test_predictor.py,
test_scheduler.py, test_engine.py, test_tree.py) run
against the B200 library through the `specexit` compatibility package
(paper_2504_08850_b200/compat, STRICT numerics), with fixtures from the
reference pipeline's trained tiny models.  Staged by
scripts/stage_reference_tests.sh into the git-ignored baseline/_ref/tests.

Deselected (documented skip list): predictor TRAINING, offline tooling
outside the hot path (train_predictor / predictor_loss_and_grads).
"""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref", "tests")

SKIP = [  # training (offline tooling, out of scope): test_predictor.py:80-137
    "test_predictor.py::test_trainable_on_separable_data",
    "test_predictor.py::test_loss_history_non_increasing",
    "test_predictor.py::test_training_deterministic",
    "test_predictor.py::test_gradients_match_finite_differences",
    "test_predictor.py::test_empty_examples_rejected",
]

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not os.path.isdir(REF), reason="stage with scripts/stage_reference_tests.sh")
@pytest.mark.parametrize("numerics", ["strict", "fast"])
def test_reference_suite_through_compat(numerics):
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", "-c",
           os.path.join(REF, "pytest.ini"), "--rootdir", REF]
    for s in SKIP:
        cmd += ["--deselect", s]
    cmd += ["test_predictor.py", "test_scheduler.py", "test_engine.py", "test_tree.py"]
    env = dict(os.environ, PYTHONPATH=ROOT + os.pathsep + os.environ.get("PYTHONPATH", ""),
               SPECEXIT_B200_NUMERICS=numerics)
    r = subprocess.run(cmd, cwd=REF, capture_output=True, text=True, timeout=1500, env=env)
    tail = (r.stdout + r.stderr)[-4000:]
    print(tail)
    assert r.returncode == 0, tail
