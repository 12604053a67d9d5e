"""splitmix64 stream (host side), identical to the reference's rng.py:14-32.

Used to produce the same seeded random-init weights and synthetic inputs as
the reference (the device-side generator is spx_init_uniform).
"""
import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK = (1 << 64) - 1


def splitmix64(seed: int, n: int) -> np.ndarray:
    """First n outputs of the stream (rng.py:14-21)."""
    with np.errstate(over="ignore"):
        z = np.uint64(seed) + _GOLDEN * np.arange(1, n + 1, dtype=np.uint64)
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def splitmix64_at(seed: int, i: int) -> int:
    """Output i (1-based) alone, in Python integers."""
    z = (seed + 0x9E3779B97F4A7C15 * i) & _MASK
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
    return z ^ (z >> 31)


def uniform(seed: int, n: int, low: float, high: float) -> np.ndarray:
    """rng.py:24-27."""
    u = (splitmix64(seed, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return (low + (high - low) * u).astype(np.float32)


def derive(seed: int, index: int) -> int:
    """rng.py:30-32 (without materialising the prefix)."""
    return splitmix64_at(seed, index + 1)


def round_bf16(x: np.ndarray) -> np.ndarray:
    """RNE rounding of float32 values to bfloat16-representable float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return u.astype(np.uint32).view(np.float32).reshape(x.shape)
