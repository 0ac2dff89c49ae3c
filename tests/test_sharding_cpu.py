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


def test_partition_rejects_more_ranks_than_patches():
    """a rank without rows must never exist (it would reduce rows it
    never computed): every rank gets >= 1 patch, world > npatches raises."""
    from paper_2111_10743_b200.sharding import partition_rows
    parts = partition_rows(3, 10, 3)
    assert [nr for _, nr in parts] == [10, 10, 10]
    parts = partition_rows(8, 10, 4, cost=[100, 1, 1, 1, 1, 1, 1, 1])
    assert all(nr > 0 for _, nr in parts) and sum(nr for _, nr in parts) == 80
    with pytest.raises(ValueError):
        partition_rows(3, 10, 4)


def test_morton_patch_order_and_permutation():
    """Targets are partitioned by contiguous Morton range (north_star): the
    patch order sorts the centroids' Morton keys (the FMM's key function), so
    every rank's patches are one contiguous key range; the permuted geometry
    is a relabelling (node blocks move with their patch)."""
    from paper_2111_10743_b200.operators import Geometry
    from paper_2111_10743_b200.sharding import morton_patch_order, permute_geometry
    g = np.load(os.path.join(GOLD, "opset_torus_o3.npz"))
    geom = Geometry.from_arrays(g)
    nb = geom.nodes_per_patch
    order = morton_patch_order(geom.nodes, nb)
    assert sorted(order.tolist()) == list(range(geom.npatches))
    pg, ix = permute_geometry(geom, order)
    assert np.array_equal(pg.nodes, geom.nodes[ix])
    assert np.array_equal(pg.over_nodes.reshape(-1, pg.over_interp.shape[0], 3),
                          geom.over_nodes.reshape(-1, pg.over_interp.shape[0], 3)[order])
    assert np.array_equal(pg.coeffs_x, geom.coeffs_x[order])
    # consecutive patches in the new order are close: the mean centroid step
    # is far below the random-order step
    c = geom.nodes.reshape(-1, nb, 3).mean(1)
    step = np.linalg.norm(np.diff(c[order], axis=0), axis=1).mean()
    rnd = np.linalg.norm(np.diff(c[np.random.default_rng(0).permutation(len(c))], axis=0),
                         axis=1).mean()
    assert step < 0.6 * rnd


def test_rows_near_map_keeps_only_owned_rows():
    from paper_2111_10743_b200.quadrature import NearMap
    from paper_2111_10743_b200.sharding import _rows_near_map
    g = np.load(os.path.join(GOLD, "opset_torus_o3.npz"))
    near = NearMap(2.0, 128, g["near_offsets"], g["near_patches"])
    n = len(near.offsets) - 1
    r0, nr = n // 3, n // 3
    sub = _rows_near_map(near, r0, nr)
    cnt = np.diff(sub.offsets)
    assert cnt[:r0].sum() == 0 and cnt[r0 + nr:].sum() == 0
    assert np.array_equal(cnt[r0:r0 + nr], np.diff(near.offsets)[r0:r0 + nr])
    assert np.array_equal(sub.patches, near.patches[near.offsets[r0]:near.offsets[r0 + nr]])
