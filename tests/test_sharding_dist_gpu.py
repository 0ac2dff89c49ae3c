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


def _worker(rank, world, port, fixture, form, far, q):
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
        op = ShardedOperatorSet(Geometry.from_arrays(g), form, 1e-10,
                                CorrectionSet.from_arrays(g), far=far)
        y = op.apply(np.asarray(g["tau"]))
        q.put((rank, np.asarray(y), None))
    except Exception as exc:  # noqa: BLE001 - report to the parent
        q.put((rank, None, repr(exc)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fixture,form,far", [("opset_torus_o3.npz", "a3", "direct"),
                                              ("opset_sphere_o3.npz", "a2", "direct"),
                                              ("opset_torus_o3.npz", "a3", "fmm")])
def test_sharded_operator_set_two_ranks(cuda, fixture, form, far):
    from paper_2111_10743_b200 import CorrectionSet, Geometry, LayerOperatorSet
    g = dict(np.load(os.path.join(GOLD, fixture)))
    ref = LayerOperatorSet(Geometry.from_arrays(g), form, 1e-10,
                           corrections=CorrectionSet.from_arrays(g), far=far).apply(g["tau"])
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fixture, form, far, q))
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
        assert rel < 1e-12, (rank, rel)
