"""Projected multi-GPU strong scaling of the A3 apply measured
on ONE B200: the target rows are split into G shards exactly as
ShardedOperatorSet does (sharding.partition_rows, balanced by correction nnz
+ far rows); every shard is a real lb_opset handle on its row range with its
own copy of the FmmPlan (the reference's tree over all sources and targets,
owned target rows: lb_fmm_plan_set_target_range), and the apply runs phase by phase
(lb_opset_apply_phase) with the exchanges done by device copies, as in
tests/test_sharding_gpu.py.  Each shard's phase is timed alone with CUDA
events (shards never wait on one another: they run back to back), so

    projected apply(G) = sum over phases of max over shards (phase time)
                         + the exchange volume over NVLink (reported, not timed)

This is a projection, not a multi-GPU measurement: NCCL latency and any
contention are not in it.  Correction values are synthetic on the
reference's own near-map pattern (apply timing does not depend on them).
Usage: python scripts/shard_projection.py config3|config4 eps ncrit [G ...]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))
import apply_vs_n  # noqa: E402
from paper_2111_10743_b200 import Geometry  # noqa: E402
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402
from paper_2111_10743_b200.operators import FORMULATIONS, DeviceOperator  # noqa: E402
from paper_2111_10743_b200.sharding import partition_rows  # noqa: E402

name, eps, ncrit = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
worlds = [int(a) for a in sys.argv[4:]] or [1, 2, 4, 8]
g = dict(np.load(os.path.join(ROOT, "data", f"{name}_geom.npz")))
geom = Geometry.from_arrays(g)
cset = apply_vs_n.corrections(name, g, eps, True, 7)
n, nb = geom.nnodes, geom.nodes_per_patch
ip = cset.indptr.cpu().numpy() if hasattr(cset.indptr, "cpu") else cset.indptr
cost = (ip[nb::nb] - ip[:-1:nb]) + nb * geom.noversampled / 50.0
tau = torch.from_numpy(np.random.default_rng(2).standard_normal(n)).cuda()


def ev():
    return torch.cuda.Event(enable_timing=True)


for world in worlds:
    parts = partition_rows(n // nb, nb, world, cost)
    devs, plans = [], []
    for r0, nr in parts:
        d = DeviceOperator(geom, cset, list(FORMULATIONS["a3"]), row0=r0, nrows=nr)
        pl = FmmPlan(geom.over_nodes, geom.nodes, eps, ncrit=ncrit)  # replicated tree
        pl.set_target_range(r0, r0 + nr)                               # owned rows
        d.set_fmm(pl)
        devs.append(d)
        plans.append(pl)
    outs = [torch.zeros(n, dtype=torch.float64, device="cuda") for _ in devs]
    phase_ms = []
    for rep in range(2):  # first pass warms up (plans' device state, factors)
        phase_ms = []
        for p in range(3):
            ts = []
            for d, o in zip(devs, outs):
                e0, e1 = ev(), ev()
                e0.record()
                d.apply_phase(3, p, tau, o)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            phase_ms.append(ts)
            vecs, red = devs[0].phase_exchange(3, p)
            for k in vecs:
                full = torch.zeros(n, dtype=torch.float64, device="cuda")
                for d, (r0, nr) in zip(devs, parts):
                    full[r0:r0 + nr] = d.buffers()[0][k][r0:r0 + nr]
                for d in devs:
                    d.buffers()[0][k].copy_(full)
            if red:
                s = sum(d.buffers()[1].clone() for d in devs)
                for d in devs:
                    d.buffers()[1].copy_(s)
    # FMM stage split of the slowest shard's second far call (phase 1)
    worst = int(np.argmax(phase_ms[1]))
    plans[worst].set_timing(True)
    devs[worst].apply_phase(3, 1, tau, outs[worst])
    torch.cuda.synchronize()
    stages = plans[worst].stage_times()
    plans[worst].set_timing(False)
    proj = sum(max(ts) for ts in phase_ms)
    total = sum(sum(ts) for ts in phase_ms)
    print(json.dumps({"case": name, "eps": eps, "ncrit": ncrit, "world": world,
                      "rows": [nr for _, nr in parts],
                      "phase_ms_per_shard": phase_ms,
                      "projected_apply_ms": proj, "sum_over_shards_ms": total,
                      "worst_shard_call2_stages_ms": stages,
                      "exchange_bytes": 2 * 8 * n + 8 * world,
                      "exchange_note": "all-gather of S tau, S' tau (+ one scalar) per apply, "
                                       "and the result all-gather: 3*8*N bytes"}), flush=True)
    del devs, plans, outs
    torch.cuda.empty_cache()
