"""Multi-rank sharded apply on CPU: world_size 2 over gloo with the oracle
backend (tests/sharded_oracle.py) drives the SAME partitioning, phase and
exchange code the GPUs run (paper_2111_10743_b200.sharding) and must
reproduce the single-process apply."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLD


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2111_10743_b200.sharding import ShardedApply, partition_rows
    from sharded_oracle import OracleShardBackend
    g = dict(np.load(os.path.join(GOLD, "opset_torus_o3.npz")))
    nb = g["over_interp"].shape[1]
    n = g["nodes"].shape[0]
    parts = partition_rows(n // nb, nb, world)
    r0, nr = parts[rank]
    be = OracleShardBackend(g, r0, nr)
    drv = ShardedApply(be, parts, rank)
    out = torch.zeros(n, dtype=torch.float64)
    drv.apply(3, torch.from_numpy(g["tau"]), out)
    q.put((rank, out.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_a3_matches_single_process(world):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    g = np.load(os.path.join(GOLD, "opset_torus_o3.npz"))
    ref = oracle.OracleOperator(g, spp="combined").apply_a3(g["tau"])
    for r in range(world):
        assert np.abs(res[r] - ref).max() <= 1e-12 * np.abs(ref).max(), r
    assert np.array_equal(res[0], res[world - 1])  # every rank holds the same full result


def test_partition_rows_is_contiguous_and_patch_aligned():
    from paper_2111_10743_b200.sharding import partition_rows
    for world in (1, 2, 3, 8):
        parts = partition_rows(320, 28, world, cost=np.linspace(1, 3, 320))
        assert parts[0][0] == 0
        assert sum(nr for _, nr in parts) == 320 * 28
        for (a0, an), (b0, _) in zip(parts, parts[1:]):
            assert a0 + an == b0
        assert all(nr % 28 == 0 for _, nr in parts)
