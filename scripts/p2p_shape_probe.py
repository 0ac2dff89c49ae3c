"""Direct P2P (charge, pot+grad, sources == targets) device time at
N = 1e5 and 3e5 on seeded sphere points: the launch-shape probe for the
4-output pair functor (lb_p2p, csrc/p2p.cu).  Prints one JSON line."""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2111_10743_b200 as b  # noqa: E402

res = {}
for n in (100000, 300000):
    rng = np.random.default_rng(105)
    x = rng.standard_normal((n, 3))
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    q = rng.standard_normal((1, n))
    src = b.FmmSources(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())
    xt = torch.from_numpy(x).cuda()
    for _ in range(2):
        b.evaluate_direct(src, xt, ("pot", "grad"))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        b.evaluate_direct(src, xt, ("pot", "grad"))
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / reps / 1e3
    res[str(n)] = {"ms": t * 1e3, "pairs_per_s": n * n / t}
print(json.dumps(res))
