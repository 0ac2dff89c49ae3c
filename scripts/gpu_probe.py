"""Quick GPU measurements: FP64 FMA peak, MUFU rsqrt seed accuracy, P2P
throughput.  Prints JSON lines.  Usage: python scripts/gpu_probe.py"""

import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2111_10743_b200 import _build, _lib  # noqa: E402
import paper_2111_10743_b200 as b  # noqa: E402

_build.build(verbose=False)
L = _lib.load()
st = _lib.stream_handle()


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    return min(ts), float(np.median(ts))


sms = torch.cuda.get_device_properties(0).multi_processor_count
scr = torch.zeros(sms * 64, dtype=torch.float64, device="cuda")
for blocks_per_sm in (4, 8):
    blocks = sms * blocks_per_sm
    iters = 2000
    t, tm = timeit(lambda: _lib.check(L.lb_probe_dfma(_lib.ptr(scr), blocks, iters, st)))
    flops = blocks * 256 * iters * 256
    print(json.dumps({"probe": "dfma_peak", "blocks": blocks, "tflops_best": flops / t / 1e12,
                      "tflops_median": flops / tm / 1e12}))

rng = np.random.default_rng(0)
x = np.exp(rng.uniform(np.log(1e-30), np.log(1e30), 1 << 20))
x[:4] = [0.0, 1.0, 4.0, 1e-300]
xd = torch.from_numpy(x).cuda()
yd = torch.empty_like(xd)
for mode in (0, 1):
    _lib.check(L.lb_probe_rsqrt(_lib.ptr(xd), _lib.ptr(yd), len(x), mode, st))
    y = yd.cpu().numpy()
    ref = 1.0 / np.sqrt(x[4:].astype(np.longdouble))
    rel = np.abs((y[4:] - ref) / ref).astype(float)
    print(json.dumps({"probe": "rsqrt", "mode": ["seed", "refined"][mode],
                      "max_rel": float(rel.max()), "mean_rel": float(rel.mean()),
                      "at0": float(y[0]), "at1": float(y[1]), "at4": float(y[2])}))

for n_t, n_s, nm in ((8960, 35840, "config2-far1"), (100_000, 100_000, "1e5"),
                     (1_000_000, 1_000_000, "1e6")):
    xs = rng.standard_normal((n_s, 3))
    xs /= np.linalg.norm(xs, axis=1, keepdims=True)
    xt = xs[:n_t] if n_t <= n_s else None
    src = torch.from_numpy(xs).cuda()
    tgt = src[:n_t].contiguous()
    q = torch.from_numpy(rng.standard_normal((1, n_s))).cuda()
    pot = torch.empty((1, n_t), dtype=torch.float64, device="cuda")
    grad = torch.empty((1, n_t, 3), dtype=torch.float64, device="cuda")
    for level in (0, 1):
        fn = lambda: b.fmm.p2p_device(tgt, src, q, None, 1, 1, 0, level, pot, grad)
        t, tm = timeit(fn, reps=3 if n_t >= 10**6 else 10)
        pairs = n_t * n_s - min(n_t, n_s)
        print(json.dumps({"probe": "p2p", "case": nm, "level": level, "pairs": pairs,
                          "s": t, "pairs_per_s": pairs / t,
                          "tflops20": 20 * pairs / t / 1e12 if level == 1 else None}))
