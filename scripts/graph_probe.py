"""Config-2 bench step (A3 apply + MGS) eager vs captured in a CUDA graph:
how much of the step is launch gaps.  Usage: python scripts/graph_probe.py"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2111_10743_b200 import LayerOperatorSet, _lib  # noqa: E402
from paper_2111_10743_b200.solver import _bind  # noqa: E402

b = bench.load_bundle()
op = bench.with_corrections(b) or LayerOperatorSet.from_bundle(b, "a3")
n = b["nodes"].shape[0]
L = _bind()
K = bench.K_ARNOLDI
rng = np.random.default_rng(2)
Q = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, K + 1)))[0].T.copy()).cuda().contiguous()
hdev = torch.zeros(K + 2, dtype=torch.float64, device="cuda")
v = torch.empty(n, dtype=torch.float64, device="cuda")
tau = torch.from_numpy(np.asarray(b["tau"])).cuda()


def step():
    op.apply_device(tau, out=v)
    _lib.check(L.lb_arnoldi_mgs(_lib.ptr(Q), n, K - 1, n, _lib.ptr(v), _lib.ptr(hdev),
                                _lib.stream_handle()))


def timed(fn, k=200):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(k):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.mean(ts)), float(np.min(ts))


print("eager ms (mean, min)", timed(step))
ref = v.clone()
s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    for _ in range(3):
        step()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    step()
g.replay()
torch.cuda.synchronize()
print("graph replay matches eager:", torch.equal(v, ref))
print("graph ms (mean, min)", timed(g.replay))
