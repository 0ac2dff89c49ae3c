"""FP64 tensor-core GEMM of the FMM translations (lb_dgemm_cols, DMMA 8x8x4)
on the shapes the FMM uses: achieved TFLOP/s against the measured DMMA peak.
  python scripts/dgemm_probe.py"""
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_10743_b200 import _build, _lib  # noqa: E402

_build.build(verbose=False)
L = _lib.load()
P = ctypes.c_void_p


def run(M, K, n, gather=False, perm=False, reps=10):
    A = torch.randn(M, K, dtype=torch.float64, device="cuda")
    X = torch.randn(n + 7, K, dtype=torch.float64, device="cuda")  # column-major columns
    Y = torch.empty(n, M, dtype=torch.float64, device="cuda")
    cols = torch.randperm(n + 7, device="cuda")[:n].to(torch.int64) if gather else None
    kp_tab = torch.stack([torch.randperm(K, device="cuda") for _ in range(4)]).to(torch.int32) \
        if perm else None
    kp = torch.randint(0, 4, (n + 7,), device="cuda", dtype=torch.int32) if perm else None
    st = _lib.stream_handle()

    def go():
        _lib.check(L.lb_dgemm_cols(_lib.ptr(A), K, M, K, _lib.ptr(X), K, _lib.ptr(cols),
                                   _lib.ptr(kp_tab), _lib.ptr(kp), n, _lib.ptr(Y), M, 1.0, 0, st))
    go()
    torch.cuda.synchronize()
    Xg = X[cols] if gather else X[:n]
    if perm:
        kpg = kp[:n]
        Xg = torch.gather(Xg, 1, kp_tab[kpg.long()].long())
    ref = Xg @ A.T
    err = float((Y - ref).abs().max() / ref.abs().max())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        go()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    return {"M": M, "K": K, "n": n, "gather": gather, "perm": perm, "ms": t * 1e3,
            "TFLOPs": 2.0 * M * K * n / t / 1e12, "rel_err": err}


for case in [(488, 488, 20000), (488, 488, 2000), (729, 729, 20000), (64, 488, 20000),
             (104, 488, 20000), (488, 104, 20000), (488, 64, 20000), (64, 729, 20000),
             (729, 64, 20000)]:
    print(json.dumps(run(*case)), flush=True)
print(json.dumps(run(64, 488, 20000, gather=True, perm=True)), flush=True)
print(json.dumps(run(488, 488, 20000, gather=True)), flush=True)
