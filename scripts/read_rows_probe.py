"""HBM read ceiling in the correction SpMV's access shape (lb_probe_read_rows):
two value streams, one warp per row, against the copy bandwidth of
MEASURED_PEAKS.json and the SpMV's own 5.06 / 5.40 TB/s of actual bytes."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10743_b200 import _lib
L = _lib.load()
for rowlen, nrows in ((2808, 114688), (2808 * 8, 14336), (702, 458752), (2808, 458752)):
    n = rowlen * nrows
    a = torch.ones(n, dtype=torch.float64, device="cuda")
    b = torch.ones(n, dtype=torch.float64, device="cuda")
    out = torch.empty(nrows, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    best = 1e9
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.lb_probe_read_rows(_lib.ptr(a), _lib.ptr(b), nrows, rowlen, _lib.ptr(out), _lib.stream_handle()))
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    assert float(out[0]) == 2.0 * rowlen
    print(f"rows {nrows} x {rowlen} doubles x 2 streams: {2 * n * 8 / 1e9:.2f} GB in {best:.3f} ms = "
          f"{2 * n * 8 / best / 1e9:.2f} TB/s", flush=True)
    del a, b
