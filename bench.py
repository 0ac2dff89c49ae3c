"""Benchmark of the GMRES operator-apply hot path (BASELINE.json metric:
"fp64 Laplace pot+grad interactions/s; GMRES operator-apply time vs N").

Workload (N=1): BASELINE config 2 — icosphere, reference order 7 (N=8,960
nodes, 35,840 oversampled sources), A3 formulation (the reference default).
One step = one GMRES iteration of the device solver: the A3 operator apply
(oversample -> far sweep 1 -> 2 corrected SpMVs -> oversample -> far sweep 2 ->
4 corrected SpMVs + glue + W-average) followed by the modified Gram-Schmidt
Arnoldi update against K_ARNOLDI=4 basis vectors (the reference converges in
4 iterations here).  Interactions per step = sum over the two far sweeps of
(densities x N x N_over): 1 + 3 = 4 density-sweeps.

Geometry + corrections come from data/config2.npz (built by running the
reference, scripts/make_golden.py config2; git-ignored, travels with the
snapshot).  Without it the committed geometry bundle
tests/golden/config2_geom.npz (the reference's geometry arrays, near map, the
seeded tau and the reference's own A3 apply of it) is used and the
corrections are built on the device (csrc/quad.cu, eps 1e-10, the same
adaptive quadrature), which the JSON line then says.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
CONFIG2 = os.path.join(ROOT, "data", "config2.npz")
CONFIG2_GEOM = os.path.join(ROOT, "tests", "golden", "config2_geom.npz")
K_ARNOLDI = 4
METRIC = "fp64 Laplace pot+grad interactions/s; GMRES operator-apply time vs N"
UNIT = "interactions/s"
NOMINAL_FP64_TFLOPS = 37.2  # 148 SM x 64 DFMA/clk x 2 x 1.965 GHz


def _dist():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_bundle():
    """Config-2 bundle: the reference-built one when present, else the
    committed geometry bundle (corrections then come from the device build,
    see with_corrections)."""
    path = CONFIG2 if os.path.exists(CONFIG2) else CONFIG2_GEOM
    z = np.load(path)
    keys = [k for k in z.files if not k.startswith(("a2_", "a3_"))]
    b = {k: z[k] for k in keys} | {k: z[k] for k in z.files if k in ("a3_apply",)}
    b["_corrections"] = "reference" if "corr_indptr" in b else "device"
    return b


def with_corrections(b):
    """Fill corr_* from the device correction build (quadrature.py mirror,
    csrc/quad.cu) when the bundle carries none; returns the operator built on
    the way (None when the bundle had the reference's corrections)."""
    if "corr_indptr" in b:
        return None
    from paper_2111_10743_b200 import Geometry, LayerOperatorSet
    op = LayerOperatorSet(Geometry.from_arrays(b), "a3", float(b["eps"]))
    cs = op._cset

    def host(a):
        return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)
    b["corr_indptr"] = host(cs.indptr)
    b["corr_indices"] = host(cs.indices)
    for k, v in cs.values.items():
        b["corr_" + k.value] = host(v)
    return op


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line) through NVML every 5 ms; nvidia-smi when
    NVML is unavailable."""

    REASONS = {  # nvmlClocksEventReason bits
        0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown",
        0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
    }

    def __init__(self, index=0, period=0.005):
        self.index = index
        self.period = period
        self.sm = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                nv.nvmlDeviceGetCurrentClocksThrottleReasons
            while not self._stop.is_set():
                self.sm.append(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = get_r(h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
                self._stop.wait(self.period)
        except Exception:
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", f"--id={self.index}",
                         "--query-gpu=clocks.sm,clocks.max.sm",
                         "--format=csv,noheader,nounits"], capture_output=True,
                        text=True, timeout=5).stdout.strip().split(",")
                    self.sm.append(float(out[0]))
                    self.max_mhz = float(out[1])
                except Exception:
                    pass
                self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.sm)}


def fp64_peak_tflops(torch, lib, _lib):
    """Measured FP64 FMA-pipe peak (lb_probe_dfma), best of 3."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sms * 8, 4000
    scr = torch.zeros(blocks, dtype=torch.float64, device="cuda")
    st = _lib.stream_handle()
    best = 0.0
    for _ in range(4):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.lb_probe_dfma(_lib.ptr(scr), blocks, iters, st))
        e1.record()
        torch.cuda.synchronize()
        best = max(best, blocks * 256 * iters * 256 / (e0.elapsed_time(e1) / 1e3))
    return best / 1e12


def cpu_baseline_apply(b, nthreads, reps=1):
    """The oracle port (C restatement of the reference's direct sums + numpy
    glue, oracle/apply.py) timed on this host: full A3 applies."""
    import oracle
    op = oracle.OracleOperator(b, nthreads=nthreads)
    tau = np.asarray(b["tau"])
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        op.apply_a3(tau)
        ts.append(time.perf_counter() - t0)
    return min(ts), oracle.max_threads() if nthreads <= 0 else nthreads


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return
    b = load_bundle()
    if b["_corrections"] == "device":
        import torch
        torch.cuda.set_device(0)
        with_corrections(b)
    n, nover = b["nodes"].shape[0], b["over_nodes"].shape[0]
    inter = 4 * n * nover
    nthreads = os.cpu_count() or 1
    import oracle
    op = oracle.OracleOperator(b, nthreads=nthreads)
    tau = np.asarray(b["tau"])
    for _ in range(max(args.warmup, 1) if args.warmup < 3 else 1):
        op.apply_a3(tau)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        op.apply_a3(tau)
        ts.append(time.perf_counter() - t0)
    t = sum(ts) / len(ts)
    v = inter / t
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "config2-A3-operator-apply", "N": n,
                   "N_over": nover, "formulation": "a3",
                   "interactions_per_step": inter},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": nthreads,
                         "kind": "port",
                         "sample": "full A3 apply of config 2 per step (oracle/"
                                   "apply.py: C direct sums + numpy glue; corrections "
                                   f"built by the {b['_corrections']})"},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time the step without a CUDA graph")
    ap.add_argument("--no-fmm", action="store_true",
                    help="skip the secondary FMM line (config 5, N = 1e6 on the sphere)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    rank, world, local = _dist()
    # BENCH_SHARE_GPU=1: every rank on cuda:0 (a functional check of the sharded
    # path on a one-GPU box with BENCH_DIST_BACKEND=gloo; never a measurement)
    if os.environ.get("BENCH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")  # gloo: functional checks only
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2111_10743_b200 import _build, _lib
    _build.build(verbose=False)
    lib = _lib.load()
    from paper_2111_10743_b200 import LayerOperatorSet
    from paper_2111_10743_b200.solver import _bind

    b = load_bundle()
    op1 = with_corrections(b)
    n, nover = b["nodes"].shape[0], b["over_nodes"].shape[0]
    inter = 4 * n * nover  # density-sweeps x targets x sources per step
    if world > 1:
        # target rows sharded over the ranks, densities all-gathered between
        # the apply's phases over NCCL (sharding.py); GMRES replicated
        from paper_2111_10743_b200 import CorrectionSet, Geometry
        from paper_2111_10743_b200.sharding import ShardedOperatorSet
        op = ShardedOperatorSet(Geometry.from_arrays(b), "a3", float(b["eps"]),
                                CorrectionSet.from_arrays(b))
    else:
        op = op1 if op1 is not None else LayerOperatorSet.from_bundle(b, "a3")
    L = _bind()
    st = _lib.stream_handle()

    # Krylov state for the Arnoldi part of the step
    rng = np.random.default_rng(2)
    Q = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, K_ARNOLDI + 1)))[0].T
                         .copy()).cuda().contiguous()
    hdev = torch.zeros(K_ARNOLDI + 2, dtype=torch.float64, device="cuda")
    v = torch.empty(n, dtype=torch.float64, device="cuda")
    tau = torch.from_numpy(np.asarray(b["tau"])).cuda()

    def step():
        op.apply_device(tau, out=v)
        _lib.check(L.lb_arnoldi_mgs(_lib.ptr(Q), n, K_ARNOLDI - 1, n, _lib.ptr(v),
                                    _lib.ptr(hdev), st))

    # apply: 2 x (oversample, far sweep, CSR+epilogue) [+ add_scalar unless the
    # second sweep is fused]; MGS: one single-CTA kernel (n <= 12288)
    launches_per_step = (6 if op.dev.keep.get("phi_eta") is not None else 7) + 1
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2

    # parity spot check against the reference's own A3 apply
    y = op.apply(np.asarray(b["tau"]))
    parity = float(np.abs(y - b["a3_apply"]).max() / np.abs(b["a3_apply"]).max()) \
        if "a3_apply" in b else None

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()

    # the device-resident step replayed as a CUDA graph (the same 6 + 1
    # launches per step, without the host launch gaps: -1.7% measured,
    # scripts/graph_probe.py, bit-identical results); eager if capture fails
    run_step, graphed = step, False
    if world == 1 and not args.eager:
        try:
            s_cap = torch.cuda.Stream()
            s_cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_cap):
                step()
            torch.cuda.current_stream().wait_stream(s_cap)
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                step()
            graph.replay()
            torch.cuda.synchronize()
            run_step, graphed = graph.replay, True
        except Exception as exc:  # noqa: BLE001 - report and time eagerly
            print(f"bench: CUDA graph capture failed ({exc}); timing eagerly", file=sys.stderr)
            torch.cuda.synchronize()

    def timed(fn, k):
        times = []
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as cs:
            for _ in range(k):
                flush.zero_()  # L2 flush between timed iterations (untimed)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) / 1e3)
        if world > 1:
            torch.distributed.barrier()
        return times, cs.summary()

    times, clocks = timed(run_step, args.steps)
    t_step = sum(times) / len(times)
    if world > 1:
        tt = torch.tensor([t_step], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_step = float(tt.item())
    value = inter / t_step  # one apply per step, shared by all ranks (strong scaling)

    # dominant kernel: far sweep 2, timed alone
    from paper_2111_10743_b200.operators import _bind_opset  # noqa: F401
    far_t = far2_time(torch, op, tau, lib, _lib)
    nloc = op.dev.nrows if world > 1 else n

    # e2e through the public API with host buffers: H2D tau, apply, D2H result
    tau_h = torch.from_numpy(np.asarray(b["tau"])).pin_memory()
    out_h = torch.empty(n, dtype=torch.float64).pin_memory()
    tau_d = torch.empty(n, dtype=torch.float64, device="cuda")

    def e2e_step():
        tau_d.copy_(tau_h, non_blocking=True)
        op.apply_device(tau_d, out=v)
        _lib.check(L.lb_arnoldi_mgs(_lib.ptr(Q), n, K_ARNOLDI - 1, n, _lib.ptr(v),
                                    _lib.ptr(hdev), st))
        out_h.copy_(v, non_blocking=True)
    e2e_times, _ = timed(e2e_step, args.steps)
    e2e_t = sum(e2e_times) / len(e2e_times)
    if world > 1:
        tt = torch.tensor([e2e_t], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_t = float(tt.item())

    peak = fp64_peak_tflops(torch, lib, _lib)
    # dominant kernel: the second far sweep.  Fused A3 (exact sweeps + Phi):
    # opfar_kernel<FarA3c>, 39 algorithmic flop per pair; otherwise
    # opfar_kernel<FarA3b>, 44 (DESIGN.md §3 tables)
    fused = op.dev.keep.get("phi_eta") is not None
    kname = "FarA3c" if fused else "FarA3b"
    flops_pair = 39.0 if fused else 44.0
    traffic = None  # dram read+write bytes per launch of that kernel (ncu --set full)
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "round1",
                                           "ncu_full_config2_far_csr.json")))
        for k in prof:
            if kname in k["kernel"]:
                tb = [float(k[m].split()[0]) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
                                                "Gbyte": 1e9}[k[m].split()[1]]
                      for m in ("dram__bytes_read.sum", "dram__bytes_write.sum")]
                traffic = sum(tb)
    except (OSError, KeyError, ValueError):
        pass
    far_flops = flops_pair * nloc * nover  # algorithmic flops per launch
    achieved = far_flops / far_t / 1e12

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t_cpu, cores = cpu_baseline_apply(b, os.cpu_count() or 1)
        cpu = {"value": inter / t_cpu, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": "one full A3 apply of config 2 (oracle/apply.py: C direct "
                         "sums + numpy glue; MGS excluded)"}

    fmm = None
    if rank == 0 and world == 1 and not args.no_fmm:
        fmm = fmm_config5(torch)

    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3),
            "ms_per_step": t_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (config 2 geometry + corrections built by the "
                    f"{'reference' if b['_corrections'] == 'reference' else 'device (csrc/quad.cu)'})",
            "config": {"workload": "config2-A3-operator-apply+MGS(k=4)",
                       "N": n, "N_over": nover, "formulation": "a3",
                       "interactions_per_step": inter,
                       "parallelism": f"target-shard{world}" if world > 1 else "single",
                       "l2": "flushed between timed steps (256 MB write)",
                       "cuda_graph": graphed,
                       "apply_parity_vs_reference": parity},
            "roofline": {"bound": "fp64", "kernel": f"opfar_kernel<{kname}>",
                         "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak,
                         "peak_source": "measured in-run (lb_probe_dfma); nominal "
                                        f"{NOMINAL_FP64_TFLOPS}",
                         "far2_ms": far_t * 1e3, "flops_per_pair": flops_pair,
                         "traffic": traffic,
                         "traffic_note": "bytes/launch from profiles/round1 ncu --set full: "
                                         "the kernel is FP64-bound, DRAM traffic is the "
                                         "2.3 MB packed source array plus outputs"},
            "cpu_baseline": cpu,
            "e2e": {"value": inter / e2e_t, "unit": UNIT,
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "ms_per_step": e2e_t * 1e3},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "fmm_config5": fmm,
        }), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def fmm_config5(torch, n=1_000_000, eps=1e-6, reps=5):
    """Secondary evidence for the 'apply time vs N' half of the metric:
    BASELINE config 5's FMM (N = 1e6 unit-sphere cloud, sources = targets,
    seed 105, charge pot+grad) through the device FmmPlan -- plan setup
    (device tree, lists, operators) and the event-timed apply."""
    import time
    from paper_2111_10743_b200.fmm_plan import FmmPlan
    rng = np.random.default_rng(105)
    x = rng.standard_normal((n, 3))
    x /= np.linalg.norm(x, axis=1)[:, None]
    q = torch.from_numpy(rng.standard_normal((1, n))).cuda()
    FmmPlan(x[:1000], x[:1000], eps)  # unit operators (cached), as a user's first plan
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = FmmPlan(x, x, eps)
    pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
    grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
    plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)  # builds the device state
    torch.cuda.synchronize()
    t_setup_first = time.perf_counter() - t0
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = sum(ts) / len(ts)
    return {"workload": "config5-fmm", "N": n, "eps": eps, "rep": plan.rep, "m": plan.m,
            "apply_ms": t * 1e3, "effective_interactions_per_s": n * (n - 1) / t,
            "plan_plus_first_apply_s": t_setup_first, "setup_ms": plan.setup_times()}


def far2_time(torch, op, tau, lib, _lib, which=2, reps=20):
    """Average device duration of one far sweep (default: A3 call 2,
    FarA3c when fused, else FarA3b) timed with CUDA events on its launching stream
    (lb_opset_time_far); the packed sources are the last apply's."""
    import ctypes
    op.apply_device(tau)
    torch.cuda.synchronize()
    sec = ctypes.c_double(0.0)
    _lib.check(lib.lb_opset_time_far(op.dev.handle, which, reps, ctypes.byref(sec),
                                     _lib.stream_handle()))
    return sec.value


if __name__ == "__main__":
    main()
