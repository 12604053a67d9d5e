"""Multi-process host logic of the request-sharded path on CPU
with the gloo backend, world size 2: contiguous shards, the single
all_gather of per-rank result records in global request order, and the
max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2504_08850_b200 import shard


def test_shard_range_partitions_contiguously():
    for n in (0, 1, 7, 1024, 1031):
        for world in (1, 2, 3, 8):
            spans = [shard.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard.shard_range(4, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        a, b = shard.shard_range(n, rank, world)
        # per-request "records": a deterministic function of the global request id
        ids = np.arange(a, b)
        local = torch.as_tensor(np.stack([ids * 3 + 1, ids % 31, ids % 2, (ids // 2) % 2,
                                          np.ones_like(ids), ids % 5], axis=1).astype(np.int32))
        full = shard.gather_rows(local, n)
        tmax = shard.max_over_ranks(10.0 + rank, "cpu")
        np.save(os.path.join(out_dir, f"rank{rank}.npy"), full.numpy())
        with open(os.path.join(out_dir, f"rank{rank}.t"), "w") as fh:
            fh.write(str(tmax))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [7, 64])
def test_gather_records_world2_gloo(tmp_path, n):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    ids = np.arange(n)
    want = np.stack([ids * 3 + 1, ids % 31, ids % 2, (ids // 2) % 2, np.ones_like(ids), ids % 5],
                    axis=1).astype(np.int32)
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npy")
        assert np.array_equal(got, want)
        assert float((tmp_path / f"rank{r}.t").read_text()) == 11.0


def test_pack_records_layout():
    from paper_2504_08850_b200.engine import ExitRecord
    recs = [ExitRecord(token=5, exit_layer=3, predictor_fired=True, verified=False, active=[1, 3],
                       full_head_count=2, predictor_evals=4)]
    assert shard.pack_records(recs).tolist() == [[5, 3, 1, 0, 2, 4]]
