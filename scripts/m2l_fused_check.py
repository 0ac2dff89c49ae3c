"""A/B check of the fused low-rank M2L against the staged one (same factors):
FMM outputs on the test_fmm cloud, written to gpurun_out/m2l_ab.npz."""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if len(sys.argv) > 1:
    sys.path.insert(0, ROOT)
    import paper_2111_10743_b200 as b
    g = np.load(os.path.join(ROOT, "tests", "golden", "fmm_apply.npz"))
    src = b.FmmSources(g["src"], g["ch"], g["dip"])
    out = {}
    for eps in (1e-3, 1e-6, 1e-9):
        r = b.evaluate_fmm(src, g["tgt"], eps, ("pot", "grad"), m2l="auto")
        out[f"{eps}"] = r.pot
    np.savez(sys.argv[1], **out)
    sys.exit(0)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
a = os.path.join(ROOT, "gpurun_out", "m2l_fused.npz")
s = os.path.join(ROOT, "gpurun_out", "m2l_staged.npz")
subprocess.run([sys.executable, __file__, a], check=True)
subprocess.run([sys.executable, __file__, s], check=True, env=dict(os.environ, LB_M2L_STAGED="1"))
A, S = np.load(a), np.load(s)
for k in A.files:
    print(k, float(np.abs(A[k] - S[k]).max() / np.abs(S[k]).max()))
