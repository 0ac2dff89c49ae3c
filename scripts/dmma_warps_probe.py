import sys, os
sys.path.insert(0, os.getcwd())
import torch
from paper_2111_10743_b200 import _lib
lib = _lib.load()
for k in (1, 2, 3, 4, 6, 8):
    blocks = 148 * k
    scr = torch.zeros(blocks, dtype=torch.float64, device="cuda")
    best = 0
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.lb_probe_dmma(_lib.ptr(scr), blocks, 4000, _lib.stream_handle()))
        e1.record(); torch.cuda.synchronize()
        best = max(best, blocks * 8 * 4000 * 8 * 512 / (e0.elapsed_time(e1) / 1e3) / 1e12)
    print(f"{k} blocks/SM = {2*k} warps/SMSP: {best:.1f} TF/s", flush=True)

for mode in (1, 2):
    for k in (1, 2, 4):
        blocks = 148 * k
        scr = torch.zeros(blocks, dtype=torch.float64, device="cuda")
        best = 0
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(lib.lb_probe_dmma_operands(_lib.ptr(scr), blocks, 4000, mode, _lib.stream_handle()))
            e1.record(); torch.cuda.synchronize()
            best = max(best, blocks * 8 * 4000 * 8 * 512 / (e0.elapsed_time(e1) / 1e3) / 1e12)
        print(f"operands mode {mode} ({'A' if mode == 1 else 'A and B'} change per DMMA), {2*k} warps/SMSP: {best:.1f} TF/s", flush=True)
