"""One bench step (config 2, A3 apply + MGS k=4) inside an NVTX range
"step", after warm-up, for ncu launch lists / full captures:

  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum \
      --clock-control none --csv --log-file launches.csv \
      python scripts/profile_step.py
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2111_10743_b200 import LayerOperatorSet, _build, _lib  # noqa: E402
from paper_2111_10743_b200.solver import _bind  # noqa: E402

_build.build(verbose=False)
b = bench.load_bundle()
n = b["nodes"].shape[0]
op = bench.with_corrections(b) or LayerOperatorSet.from_bundle(b, "a3")
L = _bind()
st = _lib.stream_handle()
K = bench.K_ARNOLDI
rng = np.random.default_rng(2)
Q = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, K + 1)))[0].T.copy()).cuda()
hdev = torch.zeros(K + 2, dtype=torch.float64, device="cuda")
v = torch.empty(n, dtype=torch.float64, device="cuda")
tau = torch.from_numpy(np.asarray(b["tau"])).cuda()


def step():
    op.apply_device(tau, out=v)
    _lib.check(L.lb_arnoldi_mgs(_lib.ptr(Q), n, K - 1, n, _lib.ptr(v), _lib.ptr(hdev), st))


for _ in range(5):
    step()
torch.cuda.synchronize()
for _ in range(int(os.environ.get("PROFILE_STEPS", "1"))):
    torch.cuda.nvtx.range_push("step")
    step()
    torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("ok")
