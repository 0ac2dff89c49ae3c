"""Projected multi-GPU strong scaling of the sharded A3 apply,
round-2 form, measured on ONE B200.  Every shard is set up exactly as
ShardedOperatorSet sets a rank up (sharding.py): patches in Morton order,
contiguous patch-aligned row ranges balanced by correction nnz + far rows,
the rank's OWN correction rows only, an FmmPlan over all sources / targets
with the rank's target range and, for G > 1, its source range (the upward
pass covers the rank's sources; the partial expansions are all-reduced by the
upward hook -- here a no-op, its volume is reported).  The shards of one G
are built, timed and freed ONE AT A TIME: each phase of each shard runs alone
under CUDA events (ranks never wait on one another), so

    projected apply(G) = sum over phases of max over shards (phase time)

NOT a multi-GPU measurement: the collectives (density all-gathers 3 x 8 N
bytes, one upward all-reduce of nbox x nd x nrep x 8 bytes per far call) are
reported as bytes, not timed.  Correction VALUES are seeded noise on the
device-built near-map pattern (apply timing does not depend on them).

Usage: python scripts/shard_projection_r2.py config3|config4 [ncrit] [G ...]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_10743_b200 import CorrectionSet, _build, shapes  # noqa: E402
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402
from paper_2111_10743_b200.operators import FORMULATIONS, DeviceOperator, _over_interp  # noqa: E402
from paper_2111_10743_b200.quadrature import build_near_map  # noqa: E402
from paper_2111_10743_b200.sharding import (_rows_near_map, morton_patch_order,  # noqa: E402
                                            partition_rows, permute_geometry)

_build.build(verbose=False)
name = sys.argv[1]
if name == "config3":
    disc = shapes.build_torus(7, 64, 32, 2.0, 1.0)
    eps, ncrit0 = 5e-8, 400
else:
    disc = shapes.wavy_torus(9, 82, 163)
    eps, ncrit0 = 1e-9, 400
ncrit = int(sys.argv[2]) if len(sys.argv) > 2 else ncrit0
worlds = [int(a) for a in sys.argv[3:]] or [1, 2, 4, 8]
oi = _over_interp(disc)
nbo, nb = oi.shape
n = disc.nodes.shape[0]
geom, _ = permute_geometry(disc, morton_patch_order(disc.nodes, nb))
near = build_near_map(geom, 2.0, cap=256)
nnz_patch = np.add.reduceat(np.diff(near.offsets), np.arange(0, n, nb)) * nb
cost = nnz_patch + nb * geom.over_nodes.shape[0] / 50.0
kinds = list(FORMULATIONS["a3"])
tau = torch.from_numpy(np.random.default_rng(2).standard_normal(n)).cuda()


def synthetic_rows(near_rows, seed):
    """CSR of compute_corrections' pattern (quadrature.py:693-698) for the
    rows `near_rows` keeps, seeded values."""
    off = torch.from_numpy(np.asarray(near_rows.offsets, dtype=np.int64)).cuda()
    pat = torch.from_numpy(np.asarray(near_rows.patches, dtype=np.int64)).cuda()
    cnt = off[1:] - off[:-1]
    row = torch.repeat_interleave(torch.arange(n, device="cuda"), cnt)
    pat = pat[torch.argsort(row * (int(pat.max()) + 1) + pat)]
    cols = (pat[:, None] * nb + torch.arange(nb, device="cuda")[None, :]).reshape(-1).to(torch.int32)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
    indptr[1:] = torch.cumsum(cnt * nb, 0)
    gen = torch.Generator(device="cuda").manual_seed(seed)
    vals = {k: 1e-4 * torch.randn(cols.numel(), dtype=torch.float64, device="cuda", generator=gen)
            for k in ("s", "sprime", "spp_plus_dprime")}
    return CorrectionSet(indptr, cols, vals)


def ev():
    return torch.cuda.Event(enable_timing=True)


for world in worlds:
    parts = partition_rows(n // nb, nb, world, cost)
    phase_ms = [[], [], []]
    stages2, up_bytes = [], 0
    for rank, (r0, nr) in enumerate(parts):
        cset = synthetic_rows(_rows_near_map(near, r0, nr), 7 + rank)
        dev = DeviceOperator(geom, cset, kinds, row0=r0, nrows=nr)
        plan = FmmPlan(geom.over_nodes, geom.nodes, eps, ncrit=ncrit, xw="direct")
        plan.set_target_range(r0, r0 + nr)
        if world > 1:
            plan.set_source_range(r0 // nb * nbo, (r0 + nr) // nb * nbo)

            def hook(up, nd, stream):
                global up_bytes
                up_bytes = max(up_bytes, up.numel() * 8)
            plan.set_upward_hook(hook)
        dev.set_fmm(plan)
        out = torch.zeros(n, dtype=torch.float64, device="cuda")
        for rep in range(2):  # the first pass warms up (device lists, factors)
            for p in range(3):
                e0, e1 = ev(), ev()
                e0.record()
                dev.apply_phase(3, p, tau, out)
                e1.record()
                torch.cuda.synchronize()
                if rep == 1:
                    phase_ms[p].append(e0.elapsed_time(e1))
                vecs, _ = dev.phase_exchange(3, p)
                for k in vecs:  # what the all-gather would bring: any finite data
                    dev.buffers()[0][k].copy_(tau)
        plan.set_timing(True)
        dev.apply_phase(3, 1, tau, out)
        torch.cuda.synchronize()
        stages2.append({k: round(v, 3) for k, v in plan.stage_times().items()})
        del dev, plan, cset, out
        torch.cuda.empty_cache()
    proj = sum(max(ts) for ts in phase_ms)
    worst = int(np.argmax(phase_ms[1]))
    print(json.dumps({"case": name, "eps": eps, "ncrit": ncrit, "world": world, "N": n,
                      "rows": [nr for _, nr in parts], "phase_ms_per_shard": phase_ms,
                      "projected_apply_ms": proj,
                      "sum_over_shards_ms": sum(sum(ts) for ts in phase_ms),
                      "worst_shard_call2_stages_ms": stages2[worst],
                      "allgather_bytes_per_apply": 3 * 8 * n,
                      "upward_allreduce_bytes_per_far_call": up_bytes}), flush=True)
