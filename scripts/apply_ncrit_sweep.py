"""BASELINE config 3 operator apply (A3, FMM far field, bench.py's step
without the MGS) against the FMM leaf capacity: one geometry / near map /
correction build, one LayerOperatorSet per ncrit, event-timed applies.
python scripts/apply_ncrit_sweep.py [ncrit ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2111_10743_b200 import LayerOperatorSet, _build  # noqa: E402

_build.build(verbose=False)
c = bench.CONFIG3
geom, near, cset, _ = bench.build_config3(torch)
n = geom.nnodes
tau = torch.from_numpy(np.random.default_rng(2).standard_normal(n)).cuda()
v = torch.empty(n, dtype=torch.float64, device="cuda")
ref = None
for ncrit in [int(a) for a in sys.argv[1:]] or [300, 400, 600, 800, 1000]:
    op = LayerOperatorSet(geom, "a3", c["eps"], corrections=cset, near=near, far="fmm",
                          fmm_ncrit=ncrit)
    for _ in range(3):
        op.apply_device(tau, out=v)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        op.apply_device(tau, out=v)
    e1.record()
    torch.cuda.synchronize()
    op.dev.set_timing(True)
    op.apply_device(tau, v)
    torch.cuda.synchronize()
    st = op.dev.stage_times()
    op.dev.set_timing(False)
    if ref is None:
        ref = v.clone()
    dev = float((v - ref).abs().max() / ref.abs().max())
    print(json.dumps({"ncrit": ncrit, "apply_ms": e0.elapsed_time(e1) / 5, "fmm1_ms": st[0],
                      "fmm2_ms": st[2], "spmv_ms": st[1] + st[3], "vs_first": dev}), flush=True)
    del op
