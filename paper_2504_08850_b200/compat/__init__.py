"""Compatibility layer: ``install()`` makes ``import specexit`` resolve to the
B200-backed drop-in package in ``compat/specexit``."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def install():
    if HERE not in sys.path:
        sys.path.insert(0, HERE)
    for name in [m for m in sys.modules if m == "specexit" or m.startswith("specexit.")]:
        del sys.modules[name]
    import specexit  # noqa: F401
    return specexit
