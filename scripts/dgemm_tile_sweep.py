"""Tile / pipeline sweep of lb_dgemm_cols on the FMM's config-3 translation shapes
(M = K = 488; one level's boxes x densities as columns).  The tile is gemm_cols' own choice (its wave model)."""
import ctypes, json, os, sys
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_10743_b200 import _lib
L = _lib.load()
names = {-1: "auto"}


def run(M, K, n, add, reps=20):
    A = torch.randn(M, K, dtype=torch.float64, device="cuda")
    X = torch.randn(n, K, dtype=torch.float64, device="cuda")
    Y = torch.zeros(n, M, dtype=torch.float64, device="cuda")
    st = _lib.stream_handle()
    def go():
        _lib.check(L.lb_dgemm_cols(_lib.ptr(A), K, M, K, _lib.ptr(X), K, None, None, None, n,
                                   _lib.ptr(Y), M, 1.0, add, st))
    for _ in range(3): go()
    torch.cuda.synchronize()
    if add == 0:
        err = float((Y - X @ A.T).abs().max())
        assert err < 1e-9, err
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): go()
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    return t * 1e6, 2.0 * M * K * n / t / 1e12


for n in (370, 740, 1500, 2200, 3000, 4380, 6000, 8760, 20000, 100000):
    out = []
    for f in names:
        if f < 0: os.environ.pop("LB_DG_FORCE", None)
        else: os.environ["LB_DG_FORCE"] = str(f)
        if n >= 3000 and f in (3, 13, 23, 33): continue
        us, tf = run(488, 488, n, 0)
        out.append(f"{names[f]} {us:.0f}us {tf:.1f}")
    print(f"n={n}: " + " | ".join(out), flush=True)
