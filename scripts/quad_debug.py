"""Debug helper: run the device correction build on subsets of one golden case."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2111_10743_b200 import Geometry  # noqa: E402
from paper_2111_10743_b200.operators import KernelKind  # noqa: E402
from paper_2111_10743_b200.quadrature import NearMap, build_correction_set  # noqa: E402

g = dict(np.load(os.path.join(ROOT, "tests", "golden", sys.argv[1] + ".npz")))
geom = Geometry.from_arrays(g)
off, pat = g["near_offsets"], g["near_patches"]
n = geom.nnodes
for label, keep in (("target0-self", lambda t, j: t == 0 and j == 0),
                    ("target0-other", lambda t, j: t == 0 and j == 1),
                    ("target0-all", lambda t, j: t == 0),
                    ("all", lambda t, j: True)):
    lists = []
    for t in range(n):
        row = pat[off[t]:off[t + 1]]
        lists.append([p for j, p in enumerate(row) if keep(t, j)])
    cnt = np.array([len(x) for x in lists])
    nm = NearMap(2.0, 128, np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64),
                 np.concatenate([np.asarray(x, np.int32) for x in lists]).astype(np.int32))
    try:
        cs, tq = build_correction_set(geom, nm, [KernelKind.SINGLE_LAYER], float(g["eps"]))
        v = cs.values[KernelKind.SINGLE_LAYER].cpu().numpy()
        print(label, "ok", nm.offsets[-1], "pairs", np.abs(v).max(), flush=True)
    except Exception as e:  # noqa: BLE001
        print(label, "FAILED", e, flush=True)
        break
