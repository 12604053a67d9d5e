"""Request sharding across GPUs: independent requests are
partitioned contiguously over the ranks of one node, every rank holds a full
replica of the model and predictor bank, and there is no collective on the
hot path.  After the timed region one all_gather collects the per-rank result
records (tokens, exit layers, predictor_fired / verified bits, counters) on
every rank, in global request order.

The helpers are backend-agnostic (NCCL on the B200 box, gloo in the CPU
tests); they never touch the device kernels.
"""
import numpy as np
import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int):
    """Contiguous [start, stop) of n requests owned by `rank` (sizes differ by
    at most one; lower ranks take the remainder)."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError("bad shard arguments")
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def gather_rows(local: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """All-gather per-rank row blocks (shape (rows_r, ...), rows_r from
    shard_range) into the global (n_total, ...) tensor on every rank.  Blocks
    are padded to the largest shard for the collective and trimmed after."""
    world = dist.get_world_size(group)
    sizes = [shard_range(n_total, r, world) for r in range(world)]
    cap = max(b - a for a, b in sizes)
    pad = torch.zeros((cap,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:b - a] for p, (a, b) in zip(parts, sizes)], dim=0)


def pack_records(records) -> np.ndarray:
    """ExitRecord list -> int32 (n, 6): token, exit_layer, fired, verified,
    full_head_count, predictor_evals (engine.py:26-48 fields that gather)."""
    return np.asarray([[r.token, r.exit_layer, int(r.predictor_fired), int(r.verified),
                        r.full_head_count, r.predictor_evals] for r in records],
                      dtype=np.int32).reshape(-1, 6)


def max_over_ranks(value: float, device, group=None) -> float:
    """Max of a per-rank scalar (device timings are reported as the max)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())
