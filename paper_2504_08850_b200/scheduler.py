"""Two-level predictor scheduling with the online state in device memory --
drop-in for the reference's ``specexit.scheduler`` (src/specexit/scheduler.py).

Offline: exit counts per layer -> ranked layers (count desc, id asc) -> the
top-k as a uint64 bitmask (``OfflineProfile.offline_mask``).  Online: a ring
of the last N exit layers plus per-layer neighbour counts, one per stream
(``OnlineState``; rows = independent streams), updated and turned into the
active-layer bitmask by the K5 kernels (spx_sched_update / spx_sched_active).
All integer -- exact by construction.
"""
import hashlib
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N


@dataclass(frozen=True)
class ScheduleConfig:
    """scheduler.py:17-27."""
    queue_len: int = 5
    radius: int = 2
    offline_top_k: int = 4

    def validate(self, num_layers):
        if self.queue_len < 1 or self.radius < 0:
            raise ValueError("bad schedule config")
        if self.offline_top_k > num_layers - 1:
            raise ValueError("offline_top_k exceeds predictor-capable layers")


@dataclass
class OfflineProfile:
    """scheduler.py:30-46."""
    num_layers: int
    exit_counts: np.ndarray
    fingerprint: int

    def __post_init__(self):
        self.exit_counts = np.asarray(self.exit_counts, dtype=np.uint64)
        if self.exit_counts.shape != (self.num_layers,):
            raise ValueError("exit_counts length must equal num_layers")

    @property
    def ranked_layers(self):
        counts = self.exit_counts[: self.num_layers - 1]
        return sorted(range(self.num_layers - 1), key=lambda i: (-int(counts[i]), i))

    def offline_mask(self, top_k: int) -> int:
        """Bitmask of the offline top-k layers (the device form of
        scheduler.py:100)."""
        m = 0
        for l in self.ranked_layers[:top_k]:
            m |= 1 << l
        return m


class OnlineState:
    """scheduler.py:49-58 with the queue and counts in device memory.

    ``rows`` independent streams share one allocation (row r = request r).
    ``queue`` / ``neighbor_counts`` read back row 0 (the reference's
    single-stream view) -- a synchronising convenience for tests."""

    def __init__(self, num_layers: int, config: ScheduleConfig, rows: int = 1):
        if num_layers > 64:
            raise ValueError("the device scheduler supports up to 64 layers")
        N.require_cuda()
        self.num_layers, self.config, self.rows = num_layers, config, rows
        self.q = torch.zeros((rows, config.queue_len), dtype=torch.int32, device="cuda")
        self.head = torch.zeros(rows, dtype=torch.int32, device="cuda")
        self.len = torch.zeros(rows, dtype=torch.int32, device="cuda")
        self.counts = torch.zeros((rows, num_layers), dtype=torch.int32, device="cuda")

    def cstate(self):
        return N.OnlineStateC(N.ptr(self.q), N.ptr(self.head), N.ptr(self.len), N.ptr(self.counts))

    def reset(self):
        for t in (self.q, self.head, self.len, self.counts):
            t.zero_()

    def queue_of(self, row=0):
        h, n = int(self.head[row]), int(self.len[row])
        q = self.q[row].tolist()
        return [q[(h + i) % self.config.queue_len] for i in range(n)]

    @property
    def queue(self):
        return self.queue_of(0)

    @property
    def neighbor_counts(self):
        return self.counts[0].to(torch.int64).cpu().numpy()


def update_online(state: OnlineState, exit_layer) -> OnlineState:
    """scheduler.py:65-79 on device.  ``exit_layer``: an int (row 0 / single
    stream) or a device int32 tensor of per-row exit layers."""
    if isinstance(exit_layer, torch.Tensor):
        e = exit_layer.to(device="cuda", dtype=torch.int32).contiguous()
        rows = e.numel()
    else:
        if not 0 <= int(exit_layer) < state.num_layers:
            raise ValueError("exit layer out of range")
        e = torch.full((1,), int(exit_layer), dtype=torch.int32, device="cuda")
        rows = 1
    err = torch.zeros(1, dtype=torch.int32, device="cuda")
    N.check(N.lib().spx_sched_update(state.cstate(), N.ptr(e), None, rows, state.num_layers,
                                     state.config.queue_len, state.config.radius, N.ptr(err),
                                     N.stream_ptr()), "spx_sched_update")
    if not isinstance(exit_layer, torch.Tensor):
        N.raise_device_error(err.item())
    return state


def recompute_counts(state: OnlineState, row: int = 0) -> np.ndarray:
    """scheduler.py:82-88: from-scratch oracle for the neighbour counts."""
    L, r = state.num_layers, state.config.radius
    counts = np.zeros(L, dtype=np.int64)
    for e in state.queue_of(row):
        counts[max(e - r, 0):min(e + r, L - 1) + 1] += 1
    return counts


def active_mask(profile, state: OnlineState, config: ScheduleConfig, mode: str = "two-level",
                out: torch.Tensor = None) -> torch.Tensor:
    """Per-row uint64 active-layer bitmask on device (spx_sched_active)."""
    L = state.num_layers
    if out is None:
        out = torch.empty(state.rows, dtype=torch.int64, device="cuda")
    if mode == "all":
        mask, m = 0, 0
    else:
        config.validate(profile.num_layers)
        mask, m = profile.offline_mask(config.offline_top_k), 1
    N.check(N.lib().spx_sched_active(state.cstate(), mask, state.rows, L, m, N.ptr(out),
                                     N.stream_ptr()), "spx_sched_active")
    return out


def mask_to_layers(mask: int, num_layers: int):
    mask &= (1 << 64) - 1
    return [i for i in range(num_layers) if (mask >> i) & 1]


def online_hot_layers(state: OnlineState):
    """scheduler.py:91-92."""
    c = state.neighbor_counts
    return [i for i in range(state.num_layers - 1) if c[i] > 0]


def active_layers(profile: OfflineProfile, state: OnlineState, config: ScheduleConfig):
    """scheduler.py:95-102: sorted union of offline top-k and hot layers."""
    config.validate(profile.num_layers)
    m = active_mask(profile, state, config)
    return mask_to_layers(int(m[0].item()), profile.num_layers)


def profile_offline(engine_generate, prompts, num_layers: int, fingerprint: int) -> OfflineProfile:
    """scheduler.py:105-121."""
    counts = np.zeros(num_layers, dtype=np.uint64)
    saw_any = False
    for prompt in prompts:
        for rec in engine_generate(prompt):
            saw_any = True
            counts[rec.exit_layer] += np.uint64(1)
    if not saw_any:
        raise ValueError("profiling produced no tokens (empty corpus?)")
    return OfflineProfile(num_layers=num_layers, exit_counts=counts, fingerprint=fingerprint)


def weight_fingerprint(path) -> int:
    """scheduler.py:124-130."""
    h = hashlib.sha256()
    with open(path, "rb") as fh:
        for chunk in iter(lambda: fh.read(1 << 16), b""):
            h.update(chunk)
    return int.from_bytes(h.digest()[:8], "little")


SPXS_MAGIC = b"SPXS"
SPXS_VERSION = 1


def save_profile(profile: OfflineProfile, path):
    """scheduler.py:141-147."""
    with open(path, "wb") as fh:
        fh.write(SPXS_MAGIC)
        fh.write(SPXS_VERSION.to_bytes(4, "little"))
        fh.write(int(profile.num_layers).to_bytes(4, "little"))
        fh.write(profile.exit_counts.astype("<u8").tobytes())
        fh.write(int(profile.fingerprint).to_bytes(8, "little"))


def load_profile(path, expect_fingerprint: int = None) -> OfflineProfile:
    """scheduler.py:150-168."""
    with open(path, "rb") as fh:
        data = fh.read()
    off = 0

    def read(n):
        nonlocal off
        if off + n > len(data):
            raise ValueError("truncated profile file")
        b = data[off:off + n]
        off += n
        return b

    if read(4) != SPXS_MAGIC:
        raise ValueError("bad magic: not a profile file")
    version = int.from_bytes(read(4), "little")
    if version != SPXS_VERSION:
        raise ValueError(f"unsupported profile version {version}")
    num_layers = int.from_bytes(read(4), "little")
    counts = np.frombuffer(read(8 * num_layers), dtype="<u8").copy()
    fingerprint = int.from_bytes(read(8), "little")
    if expect_fingerprint is not None and fingerprint != expect_fingerprint:
        raise ValueError("profile fingerprint does not match model weights")
    return OfflineProfile(num_layers=num_layers, exit_counts=counts, fingerprint=fingerprint)
