"""BASELINE config 5: seeded uniform points on the unit sphere, N(0,1)
charges; direct P2P at N = 1e4, 1e5, 1e6 and FMM at N = 1e6, 1e7 (eps 1e-6,
1e-9); pot+grad interactions/s, FMM stage breakdown, CPU oracle on a target
subsample (scaled linearly, all host threads).  Prints JSON lines."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402  (CPU baseline only)
import paper_2111_10743_b200 as b  # noqa: E402
from paper_2111_10743_b200 import _lib  # noqa: E402
from paper_2111_10743_b200.fmm_plan import FmmPlan  # noqa: E402

L = _lib.load()


def sphere(n, seed=105):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, 3))
    return x / np.linalg.norm(x, axis=1, keepdims=True), rng


def ev_time(fn, reps):
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    return best


def peak():
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    scr = torch.zeros(sms * 8, dtype=torch.float64, device="cuda")
    t = ev_time(lambda: _lib.check(L.lb_probe_dfma(_lib.ptr(scr), sms * 8, 4000,
                                                   _lib.stream_handle())), 3)
    return sms * 8 * 256 * 4000 * 256 / t / 1e12


pk = peak()
print(json.dumps({"fp64_peak_tflops_measured": pk}), flush=True)
threads = os.cpu_count()
for n in (10_000, 100_000, 1_000_000):
    x, rng = sphere(n)
    q = rng.standard_normal((1, n))
    xd = torch.from_numpy(x).cuda()
    qd = torch.from_numpy(q).cuda()
    pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
    grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
    t = ev_time(lambda: b.fmm.p2p_device(xd, xd, qd, None, 1, 1, 0, 1, pot, grad),
                3 if n >= 10**6 else 10)
    pairs = n * (n - 1)
    ns = min(n, 2000)
    t0 = time.perf_counter()
    oracle.p2p(x[:ns], x, q, level=1, nthreads=threads)
    tc = (time.perf_counter() - t0) * n / ns
    print(json.dumps({"case": f"p2p N={n}", "gpu_s": t, "interactions_per_s": pairs / t,
                      "tflops_20flop": 20 * pairs / t / 1e12,
                      "frac_of_measured_fp64": 20 * pairs / t / 1e12 / pk,
                      "cpu_oracle_s_scaled": tc, "cpu_threads": threads,
                      "cpu_sample": f"{ns} targets x {n} sources, scaled by {n / ns:.0f}",
                      "speedup_vs_cpu_oracle": tc / t}), flush=True)
for n, eps in ((1_000_000, 1e-6), (1_000_000, 1e-9), (10_000_000, 1e-6), (10_000_000, 1e-9)):
    x, rng = sphere(n)
    q = rng.standard_normal((1, n))
    t0 = time.perf_counter()
    plan = FmmPlan(x, x, eps)
    t_plan = time.perf_counter() - t0
    qd = torch.from_numpy(q).cuda()
    pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
    grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
    for xw in ("lists", "direct"):  # the reference's list evaluation, then lb_fmm_plan_set_xw(1)
        plan.set_xw(xw)
        plan.set_timing(False)
        t = ev_time(lambda: plan.apply_device(qd, None, 1, 1, 0, 1, pot, grad), 2)
        plan.set_timing(True)
        plan.apply_device(qd, None, 1, 1, 0, 1, pot, grad)
        st = plan.stage_times()
        idx = np.random.default_rng(7).choice(n, 200, replace=False)
        ref = b.evaluate_direct(b.FmmSources(x, q), x[idx], ("pot", "grad"))
        err = max(np.abs(pot.cpu().numpy()[:, idx] - ref.pot).max() / np.abs(ref.pot).max(),
                  np.abs(grad.cpu().numpy()[:, idx] - ref.grad).max() / np.abs(ref.grad).max())
        print(json.dumps({"case": f"fmm N={n} eps={eps}", "xw": xw, "rep": plan.rep, "m": plan.m,
                          "plan_s": t_plan, "apply_s": t,
                          "effective_interactions_per_s": n * (n - 1) / t,
                          "err_vs_direct_200_targets": err, "stages_ms": st,
                          "nbox": int(plan.tree.sizes[0]), "V": int(plan.tree.sizes[6]),
                          "U": int(plan.tree.sizes[7])}), flush=True)
    del plan
    torch.cuda.empty_cache()
