"""Do DMMA (FP64 tensor) and DFMA (FP64 FMA pipe) overlap on B200?  Each
8-warp block runs nw_mma DMMA warps and 8 - nw_mma DFMA warps; the time of
the mix is compared with each half alone (same blocks, other half idle)."""
import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2111_10743_b200 import _lib
lib = _lib.load()


def run(blocks, it_mma, it_fma, nw):
    scr = torch.zeros(blocks, dtype=torch.float64, device="cuda")
    best = 1e9
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.lb_probe_mixed(_lib.ptr(scr), blocks, it_mma, it_fma, nw, _lib.stream_handle()))
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


for k in (1, 2, 4):
    blocks = 148 * k
    for nw in (4,):
        IM, IF = 4000, 1000
        tm = run(blocks, IM, 0, nw)
        tf = run(blocks, 0, IF, nw)
        tb = run(blocks, IM, IF, nw)
        fm = blocks * nw * IM * 8 * 512 / 1e9
        ff = blocks * (8 - nw) * 32 * IF * 256 / 1e9
        print(f"{k} blocks/SM nw_mma {nw}: dmma alone {tm:.3f} ms ({fm/tm:.1f} TF/s)  dfma alone {tf:.3f} ms "
              f"({ff/tf:.1f} TF/s)  mixed {tb:.3f} ms ({(fm+ff)/tb:.1f} TF/s; sum-of-times {tm+tf:.3f}, max {max(tm,tf):.3f})",
              flush=True)
