import sys, os, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/scripts")
import numpy as np
import apply_vs_n as A
g = dict(np.load("/root/repo/data/config3_geom.npz"))
cset = A.corrections("config3", g, 5e-8, True, 3)
for eps in (5e-8, 1e-9):
    for m2l in ("auto", "lowrank"):
        A.run("config3", g, cset, eps, "fmm", synthetic=True, ncrit=300, m2l=m2l)
