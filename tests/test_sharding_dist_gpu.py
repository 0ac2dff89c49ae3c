"""The real ShardedOperatorSet (device lb_opset handles on row ranges +
torch.distributed collectives between the apply's phases) with world size 2:
both ranks share cuda:0 and talk over gloo, so this checks the sharded code
path end to end on a one-GPU box (functional, not a timing).  Must reproduce
the unsharded LayerOperatorSet apply, exact sweeps and FMM far field."""

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import GOLD

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fixture, form, far, q, device_corr=False):
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    import datetime
    dist.init_process_group("gloo", rank=rank, world_size=world, timeout=datetime.timedelta(seconds=120))
    try:
        from paper_2111_10743_b200 import CorrectionSet, Geometry
        from paper_2111_10743_b200.sharding import ShardedOperatorSet
        g = dict(np.load(os.path.join(GOLD, fixture)))
        corr = None if device_corr else CorrectionSet.from_arrays(g)
        op = ShardedOperatorSet(Geometry.from_arrays(g), form, float(g["eps"]) if device_corr
                                else 1e-10, corr, far=far)
        y = op.apply(np.asarray(g["tau"]))
        q.put((rank, np.asarray(y), None))
    except Exception as exc:  # noqa: BLE001 - report to the parent
        q.put((rank, None, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fixture,form,far,device_corr", [
    ("opset_torus_o3.npz", "a3", "direct", False), ("opset_sphere_o3.npz", "a2", "direct", False),
    ("opset_torus_o3.npz", "a3", "fmm", False), ("opset_torus_o3.npz", "a3", "fmm", True),
    ("opset_torus_o3.npz", "a3", "direct", True)])
def test_sharded_operator_set_two_ranks(cuda, fixture, form, far, device_corr):
    """Morton-range target shards; per-rank corrections (device_corr: built on
    the device for the rank's rows only); with the FMM, the upward pass split
    by source range and all-reduced over the group between M2M and M2L."""
    from paper_2111_10743_b200 import CorrectionSet, Geometry, LayerOperatorSet
    g = dict(np.load(os.path.join(GOLD, fixture)))
    if device_corr:
        ref = LayerOperatorSet(Geometry.from_arrays(g), form, float(g["eps"]),
                               far=far).apply(g["tau"])
    else:
        ref = LayerOperatorSet(Geometry.from_arrays(g), form, 1e-10,
                               corrections=CorrectionSet.from_arrays(g), far=far).apply(g["tau"])
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fixture, form, far, q, device_corr))
             for r in range(world)]
    for p in procs:
        p.start()
    res = []
    try:
        for _ in range(world):
            r = q.get(timeout=300)
            res.append(r)
            assert r[2] is None, (r[0], r[2])  # a failing rank leaves the other in a collective
    finally:
        for p in procs:
            p.join(timeout=30 if len(res) == world else 1)
            if p.is_alive():
                p.terminate()
    for rank, y, err in res:
        rel = np.abs(y - ref).max() / np.abs(ref).max()
        # the distributed upward pass sums partial expansions in another order;
        # the surface representation (eps >= 3e-8) amplifies that roundoff
        # through its Tikhonov pseudo-inverse (measured 9.2e-11 at eps 1e-8)
        eps = float(g["eps"]) if device_corr else 1e-10
        bar = 1e-12 if far != "fmm" else (1e-9 if eps >= 3e-8 else 1e-11)
        assert rel < bar, (rank, rel)
