"""One bench step (BASELINE config 3: A3 apply with the FMM far field +
MGS k=8, exactly bench.py's step) inside an NVTX range "step", after
warm-up, for ncu launch lists / full captures:

  ncu --nvtx --nvtx-include "step/" --metrics gpu__time_duration.sum \
      --clock-control none --csv --log-file launches.csv \
      python scripts/profile_step.py
  ncu --nvtx --nvtx-include "step/" --set full -k regex:m2l_fused \
      --clock-control none --import-source on -o m2l python scripts/profile_step.py

--config2 profiles bench.py's secondary config-2 line instead (exact sweeps).
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2111_10743_b200 import LayerOperatorSet, _build, _lib, shapes  # noqa: E402
from paper_2111_10743_b200.solver import _bind  # noqa: E402

_build.build(verbose=False)
if "--config2" in sys.argv:
    geom = shapes.icosphere(7)
    op = LayerOperatorSet(geom, "a3", 1e-10, far="direct")
    K = 4
else:
    c = bench.CONFIG3
    geom, near, cset, _ = bench.build_config3(torch)
    op = LayerOperatorSet(geom, "a3", c["eps"], corrections=cset, near=near, far="fmm",
                          fmm_ncrit=c["ncrit"])
    K = bench.K_ARNOLDI
n = geom.nnodes
L = _bind()
rng = np.random.default_rng(2)
Q = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, K + 1)))[0].T.copy()).cuda()
hdev = torch.zeros(K + 2, dtype=torch.float64, device="cuda")
v = torch.empty(n, dtype=torch.float64, device="cuda")
tau = torch.from_numpy(rng.standard_normal(n)).cuda()


def step():
    op.apply_device(tau, out=v)
    _lib.check(L.lb_arnoldi_mgs(_lib.ptr(Q), n, K - 1, n, _lib.ptr(v), _lib.ptr(hdev),
                                _lib.stream_handle()))


for _ in range(5):
    step()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("step")
step()
torch.cuda.nvtx.range_pop()
torch.cuda.synchronize()
print("profile_step: done", flush=True)
