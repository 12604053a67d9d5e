"""Numerics mode of the device kernels.

* ``"fast"`` (default, production): canonical 128-partial reductions with FMA
  (the CDOT order of csrc/spx_common.cuh).  Logits agree with the reference's
  strict fp32 within a few ulp; sliced == full-head == grouped bit-for-bit.
* ``"strict"`` (parity): the reference's own operation order -- sequential
  left-to-right sums from 0, products rounded before the add, no FMA
  (reference kernels/_ckern.pyx:16-46, model.py:140-152) -- so features and
  logits are bit-identical to the reference CPU path.

This is a numerics switch of the same kernels, not a backend registry.
"""
from . import _native as N

_MODES = {"fast": N.SPX_MODE_FAST, "strict": N.SPX_MODE_STRICT}
_mode = "fast"


def set_mode(name: str) -> str:
    """Select "fast" or "strict"; returns the previous mode."""
    global _mode
    if name not in _MODES:
        raise ValueError(f"unknown numerics mode {name!r}; have {sorted(_MODES)}")
    prev, _mode = _mode, name
    return prev


def mode_name() -> str:
    return _mode


def mode() -> int:
    return _MODES[_mode]


class using:
    """Context manager: ``with numerics.using("strict"): ...``."""

    def __init__(self, name):
        self.name = name

    def __enter__(self):
        self.prev = set_mode(self.name)

    def __exit__(self, *exc):
        set_mode(self.prev)
