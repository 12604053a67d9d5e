"""``specexit`` compatibility package: the reference's import path
(src/specexit/__init__.py) backed by the B200 library.

Put ``paper_2504_08850_b200/compat`` first on ``sys.path`` (or
``paper_2504_08850_b200.compat.install()``) and ``import specexit`` /
``from specexit.engine import ExitEngine`` resolve here: the same names,
signatures, exceptions and result types as the reference (numpy arrays where
the reference returns numpy arrays, host lists / floats elsewhere), computed
by the sm_100a kernels.  Numerics default to STRICT -- the reference's own
operation order, bit-identical results on f32 reference weights (models are
created / loaded with dtype "f32").  ``numerics.set_mode("fast")`` switches
to the production order.

Out of scope (training, the offline pipeline, CLI, metrics): the training
entry points raise NotImplementedError; use the reference package for them.
"""
import os as _os

from paper_2504_08850_b200 import numerics as _numerics

# SPECEXIT_B200_NUMERICS=fast selects the production order for the whole package
_numerics.set_mode(_os.environ.get("SPECEXIT_B200_NUMERICS", "strict"))

from . import engine, model, predictor, rng, scheduler, speculation, tree  # noqa: E402,F401

__version__ = "b200-compat"
