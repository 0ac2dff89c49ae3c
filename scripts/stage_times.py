"""Warm per-stage device times of the config-2 A3 apply (lb_opset_set_timing:
CUDA events between the stages, L2 flushed before each apply)."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2111_10743_b200 import LayerOperatorSet, _build, _lib  # noqa: E402

_build.build(verbose=False)
b = bench.load_bundle()
op = bench.with_corrections(b) or LayerOperatorSet.from_bundle(b, "a3")
tau = _lib.to_device(np.asarray(b["tau"]))
out = _lib.empty((tau.numel(),))
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(5):
    op.apply_device(tau, out=out)
op.dev.set_timing(True)
acc = None
reps = 50
for _ in range(reps):
    flush.zero_()
    op.apply_device(tau, out=out)
    torch.cuda.synchronize()
    t = np.asarray(op.dev.stage_times(), dtype=float)
    acc = t if acc is None else acc + t
print(json.dumps({"stage_ms": (acc / reps).round(4).tolist()}))
