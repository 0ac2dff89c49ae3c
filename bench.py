"""Benchmark of the GMRES operator-apply hot path (BASELINE.json metric:
"fp64 Laplace pot+grad interactions/s; GMRES operator-apply time vs N").

Headline workload (N=1): BASELINE config 3 -- the torus build_torus(7, 64,
32, 2, 1) (reference order 7: N = 114,688 nodes, N_over = 458,752
oversampled sources), A3 (the reference default and config 3's Hodge
solves), FMM far field at eps 5e-8 (the paper's Hodge setting), near-field
corrections built ON THE DEVICE (eta 2, cap 256: 3.2e8 nnz per kind, 3 kinds).
Every input is generated on the box (paper_2111_10743_b200/shapes.py hands
the device geometry build the reference's own chart coefficients).

One step = one GMRES iteration of the device solver: the A3 operator apply
(oversample -> FMM call 1 -> 2 corrected SpMVs -> oversample -> FMM call 2
-> 3 corrected SpMVs + glue + W-average) and the modified Gram-Schmidt
Arnoldi update against K_ARNOLDI basis vectors.  Interactions per step
(effective, the metric's unit) = density-sweeps x N x N_over = (1 + 3) x N x
N_over: the reference's two far calls (operators.py:229-266).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--impl reference times the oracle port of the reference's CPU path on the
host cores (the reference is Python and does not travel to the GPU box):
the same config-3 step, row-sampled (every ROW_STRIDE-th target: both far
calls as exact fp64 sums over ALL sources at the sampled targets, the
sampled CSR rows, the full-length oversampling and MGS), scaled by
N / rows.  It never loads libb200lb.so.
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
METRIC = "fp64 Laplace pot+grad interactions/s; GMRES operator-apply time vs N"
UNIT = "interactions/s"
NOMINAL_FP64_TFLOPS = 37.2  # 148 SM x 64 DFMA/clk x 2 x 1.965 GHz
K_ARNOLDI = 8               # MGS basis size in the timed step
CONFIG3 = {"order": 7, "nu": 64, "nv": 32, "R": 2.0, "r": 1.0, "eps": 5e-8,
           "eta": 2.0, "cap": 256, "ncrit": 400}
M2L_DRAM_BYTES_NCU = 763.6e6  # first factor 89.3 + 73.0 MB, fused 102.0 + 202.6 MB, reduce 283.6 + 13.1 MB (ncu launch list)
ROW_STRIDE = 128            # CPU arms: every 128th target (896 rows of 114,688)
WORKLOAD = "config3-torus64x32-o7-A3-fmm5e-8-apply+MGS(k=8)"


def _dist():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def _peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except (OSError, ValueError):
        return {}


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region
    (B200_PROFILING.md clocks line) through NVML every 5 ms; nvidia-smi when
    NVML is unavailable."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown",
               0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index=0, period=0.005):
        self.index, self.period = index, period
        self.sm, self.reasons, self.max_mhz = [], set(), None
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
                        ["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip().split(",")
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


# ---------------------------------------------------------------------------
# CPU side (oracle port): the reference arm and the cpu_baseline leg


def cpu_config3_setup(nthreads, stride=ROW_STRIDE):
    """Config-3 geometry on the host (oracle/geometry.py over the chart
    coefficients of shapes.build_torus), the near lists of every
    stride-th target and seeded correction values on the reference's CSR
    pattern for those rows (timing only)."""
    import oracle
    from oracle import geometry as og
    from oracle.sampled import SampledA3, synthetic_rows
    from paper_2111_10743_b200.shapes import build_torus
    c = CONFIG3
    coeffs = build_torus(c["order"], c["nu"], c["nv"], c["R"], c["r"], coefficients_only=True)
    geo = og.evaluate(c["order"], *coeffs)
    n = geo["nodes"].shape[0]
    rows = np.arange(0, n, stride)
    near = og.near_patches(geo["nodes"], geo["npatches"], geo["nb"], geo["over_nodes"], rows,
                           c["eta"])
    corr = synthetic_rows(near, geo["nb"])
    op = SampledA3(geo, rows, corr, nthreads=nthreads)
    rng = np.random.default_rng(2)
    tau = rng.standard_normal(n)
    Q = np.linalg.qr(rng.standard_normal((n, K_ARNOLDI + 1)))[0].T.copy()
    return op, tau, Q, n, geo["over_nodes"].shape[0], oracle.max_threads() if nthreads <= 0 \
        else nthreads


def cpu_step(op, tau, Q):
    """One sampled step: pass 1 + pass 2 at the sampled rows (pass 2's
    full-length sources from tau-sized substitutes, same cost), then the
    MGS update of a full-length vector against K_ARNOLDI basis rows
    (solver.py:74-81)."""
    res, (s, sp) = op.step(tau, tau, tau, 0.0)
    v = tau.copy()
    v[op.rows] = res
    h = np.empty(Q.shape[0])
    for j in range(Q.shape[0] - 1):
        h[j] = Q[j] @ v
        v -= h[j] * Q[j]
    nrm = np.linalg.norm(v)
    return v / nrm


def cpu_time(op, tau, Q, reps):
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        cpu_step(op, tau, Q)
        ts.append(time.perf_counter() - t0)
    return ts


def run_reference(args):
    rank, world, _ = _dist()
    if rank != 0:
        return  # rank 0 alone times the host-core baseline
    nthreads = os.cpu_count() or 1
    op, tau, Q, n, nover, cores = cpu_config3_setup(nthreads)
    inter = 4 * n * nover
    scale = n / len(op.rows)
    cpu_time(op, tau, Q, max(args.warmup, 1))
    ts = cpu_time(op, tau, Q, args.steps)
    t = scale * sum(ts) / len(ts)
    v = inter / t
    sample = (f"every {ROW_STRIDE}th target ({len(op.rows)} of {n} rows): both A3 far calls as "
              "exact fp64 sums over all 458,752 sources (oracle C port, OpenMP), the sampled "
              "CSR rows (seeded values on the reference's pattern), full-length oversampling "
              f"and MGS(k={K_ARNOLDI}); time x N/rows")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": max(args.warmup, 1), "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (config-3 geometry from the chart; correction values seeded on the "
                "reference's sparsity pattern)",
        "config": {"workload": WORKLOAD, "N": n, "N_over": nover, "formulation": "a3",
                   "interactions_per_step": inter, "eps": CONFIG3["eps"]},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "the oracle has no FMM: this arm's far field is the exact sum (the reference's "
                "use_fmm=False path).  The reference's own Python FmmPlan far field at this "
                "config, timed in the build container on 8 vCPU: 59.7 s per apply "
                "(profiles/round2/reference_fmm_config3_cpu.json)",
    }), flush=True)


# ---------------------------------------------------------------------------
# GPU side


def fp64_peak_tflops(torch, lib, _lib):
    """Measured FP64 FMA-pipe peak (lb_probe_dfma), best of 4."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sms * 8, 4000
    scr = torch.zeros(blocks, dtype=torch.float64, device="cuda")
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.lb_probe_dfma(_lib.ptr(scr), blocks, iters, _lib.stream_handle()))
        e1.record()
        torch.cuda.synchronize()
        best = max(best, blocks * 256 * iters * 256 / (e0.elapsed_time(e1) / 1e3))
    return best / 1e12


def dmma_peak_tflops(torch, lib, _lib):
    """Measured FP64 tensor-core peak (lb_probe_dmma: DMMA 8x8x4 chains), best of 4."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, iters = sms * 4, 2000
    scr = torch.zeros(blocks, dtype=torch.float64, device="cuda")
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.lb_probe_dmma(_lib.ptr(scr), blocks, iters, _lib.stream_handle()))
        e1.record()
        torch.cuda.synchronize()
        best = max(best, blocks * 8 * iters * 8 * 512 / (e0.elapsed_time(e1) / 1e3))
    return best / 1e12


def build_config3(torch, corrections=True):
    """Geometry (device), near map (device, eta 2, cap 256), corrections
    (device, eps 5e-8, S / S' / S''+D'; skipped for a sharded run, whose
    ranks build their own rows)."""
    from paper_2111_10743_b200 import shapes
    from paper_2111_10743_b200.operators import KernelKind
    from paper_2111_10743_b200.quadrature import build_correction_set, build_near_map
    c = CONFIG3
    t0 = time.perf_counter()
    geom = shapes.build_torus(c["order"], c["nu"], c["nv"], c["R"], c["r"])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    near = build_near_map(geom, c["eta"], cap=c["cap"])
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    if not corrections:
        return geom, near, None, {"geometry_s": t1 - t0, "near_map_s": t2 - t1}
    kinds = [KernelKind.SINGLE_LAYER, KernelKind.SPRIME, KernelKind.SPP_PLUS_DPRIME]
    cset, t_q = build_correction_set(geom, near, kinds, c["eps"])
    torch.cuda.synchronize()
    return geom, near, cset, {"geometry_s": t1 - t0, "near_map_s": t2 - t1, "t_q_s": t_q}


class Timer:
    def __init__(self, torch, world, local, flush):
        self.torch, self.world, self.local, self.flush = torch, world, local, flush

    def __call__(self, fn, k):
        torch = self.torch
        times = []
        if self.world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        with ClockSampler(self.local) as cs:
            for _ in range(k):
                self.flush.zero_()  # L2 flush between timed iterations (untimed)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) / 1e3)
        if self.world > 1:
            torch.distributed.barrier()
        return times, cs.summary()

    def max_over_ranks(self, t):
        if self.world == 1:
            return t
        tt = self.torch.tensor([t], dtype=self.torch.float64, device="cuda")
        self.torch.distributed.all_reduce(tt, op=self.torch.distributed.ReduceOp.MAX)
        return float(tt.item())


def capture(torch, step, lib, _lib):
    """The step as a CUDA graph (same launches, no host gaps) and its kernel
    count (lb_graph_kernel_nodes); eager with a count of None if capture fails."""
    import ctypes
    try:
        s_cap = torch.cuda.Stream()
        s_cap.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s_cap):
            step()
        torch.cuda.current_stream().wait_stream(s_cap)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph(keep_graph=True)
        with torch.cuda.graph(g):
            step()
        nk, nn = ctypes.c_int64(), ctypes.c_int64()
        raw = g.raw_cuda_graph()
        _lib.check(lib.lb_graph_kernel_nodes(ctypes.c_void_p(raw), ctypes.byref(nk),
                                             ctypes.byref(nn)), "lb_graph_kernel_nodes")
        g.instantiate()
        g.replay()
        torch.cuda.synchronize()
        return g.replay, True, int(nk.value)
    except Exception as exc:  # noqa: BLE001 - report and time eagerly
        print(f"bench: CUDA graph capture failed ({exc}); timing eagerly", file=sys.stderr)
        torch.cuda.synchronize()
        return step, False, None


def count_sharded_launches(torch, op, mgs, lib, _lib):
    """Kernel launches of one sharded step on this rank: every local phase of
    the apply (lb_opset_apply_phase) and the MGS are captured into throw-away
    CUDA graphs and their kernel nodes counted (lb_graph_kernel_nodes).  The
    collectives between the phases are not ours and are not counted; the
    FMM's upward hook (an all-reduce) is replaced by a no-op while capturing."""
    import ctypes
    from paper_2111_10743_b200.sharding import ShardedApply
    plan = op._plan
    fn0 = getattr(plan, "_hook_fn", None) if plan is not None else None
    if fn0 is not None:
        plan.set_upward_hook(lambda up, nd, stream: None)
    total = 0
    try:
        steps = [lambda p=p: op.dev.apply_phase(op._code, p, op._tau_p, op._out_p)
                 for p in range(ShardedApply.NPHASES[op._code])] + [mgs]
        for fn in steps:
            g = torch.cuda.CUDAGraph(keep_graph=True)
            with torch.cuda.graph(g):
                fn()
            nk, nn = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(lib.lb_graph_kernel_nodes(ctypes.c_void_p(g.raw_cuda_graph()),
                                                 ctypes.byref(nk), ctypes.byref(nn)),
                       "lb_graph_kernel_nodes")
            total += int(nk.value)
    except Exception as exc:  # noqa: BLE001 - the count is a report, not the measurement
        print(f"bench: launch count by capture failed ({exc})", file=sys.stderr)
        total = None
    finally:
        if fn0 is not None:
            plan.set_upward_hook(fn0)
        torch.cuda.synchronize()
    return total


def read_rows_gbs(torch, _lib, nrows, rowlen):
    """Best of 5 runs of lb_probe_read_rows (two streams of nrows x rowlen
    doubles, L2 flushed before each run), GB/s."""
    lib = _lib.load()
    nrows = int(min(nrows, (3 << 30) // (8 * rowlen)))  # <= 3 GB per stream
    a = torch.ones(nrows * rowlen, dtype=torch.float64, device="cuda")
    b = torch.ones(nrows * rowlen, dtype=torch.float64, device="cuda")
    out = torch.empty(nrows, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    best = None
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(lib.lb_probe_read_rows(_lib.ptr(a), _lib.ptr(b), nrows, rowlen, _lib.ptr(out),
                                          _lib.stream_handle()))
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return 2.0 * nrows * rowlen * 8 / best / 1e6


def stage_rooflines(torch, op, plan, n, nover, nnz, peak_tf, hbm_gbs, _lib, peak_tc=None):
    """Per-stage device times of one apply (lb_opset stage events) and of one
    pot+grad FMM call (lb_fmm stage events) with their rooflines: SpMV passes
    against HBM (algorithmic bytes = nnz x (kinds x 8 + 4) + 8 (N + 1)), the
    FMM's pairwise stages against the FP64 pipe (20 flop per pot+grad pair:
    SURVEY §8(d)), the M2L against FP64 by its algorithmic flops."""
    tau = torch.from_numpy(np.random.default_rng(2).standard_normal(n)).cuda()
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    op.dev.set_timing(True)
    op.apply_device(tau, out)
    torch.cuda.synchronize()
    st = op.dev.stage_times()
    op.dev.set_timing(False)
    # SURVEY §8(d) accounting: 8 B per value and kind + 4 B column index per
    # nnz + 8 B per row offset (+ x gathers in L2); the kernels read the
    # block-CSR index instead (4 / nb B per nnz): the bytes reported
    nb = int(op.disc.nodes_per_patch) if hasattr(op.disc, "nodes_per_patch") else 28
    b1 = nnz * (2 * 8 + 4) + 8 * (n + 1)
    b2 = nnz * (3 * 8 + 4) + 8 * (n + 1)
    a1 = nnz * (2 * 8 + 4.0 / nb) + 8 * (n + 1)
    a2 = nnz * (3 * 8 + 4.0 / nb) + 8 * (n + 1)
    # pure two-stream read in the SpMV's row shape (lb_probe_read_rows): the
    # read-only ceiling beside MEASURED_PEAKS.json's copy bandwidth
    read_gbs = read_rows_gbs(torch, _lib, n, max(nnz // max(n, 1), 1))

    def spmv(ms, actual, formula):
        # the kernels move the block-CSR bytes (ncu: 5.24 GB DRAM read for pass
        # 1 at config 3); the SURVEY formula charges a 4-byte
        # column index per nnz that they do not read, so its GB/s is a derived
        # figure that can exceed the copy bandwidth
        return {"ms": ms, "bytes": actual, "GBps": actual / ms / 1e6,
                "frac_hbm": actual / ms / 1e6 / hbm_gbs,
                "frac_of_read_ceiling": actual / ms / 1e6 / read_gbs if read_gbs else None,
                "survey_formula_bytes": formula, "survey_formula_GBps": formula / ms / 1e6}
    stages = {
        "fmm_call1_ms": st[0], "fmm_call2_ms": st[2],
        "spmv1": spmv(st[1], a1, b1), "spmv2_glue": spmv(st[3], a2, b2),
        "hbm_read_ceiling_GBps": read_gbs,
        "apply_ms": st[7]}
    # one charge pot+grad call of the plan (the metric's unit), stage split
    w = torch.from_numpy(np.random.default_rng(3).standard_normal((1, nover))).cuda()
    pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
    grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
    plan.set_timing(True)
    plan.apply_device(w, None, 1, 1, 0, 1, pot, grad)
    torch.cuda.synchronize()
    fs = plan.stage_times()
    plan.set_timing(False)
    wc = plan.work_counts()
    leaf_pairs = wc["u_pairs"] + wc["w_pairs"] + wc["de_pairs"]

    def fp(ms, flops, peak=peak_tf, pipe="fp64"):
        tf = flops / (ms / 1e3) / 1e12 if ms > 0 else None
        return {"ms": ms, "flops": flops, "TFLOPs": tf, "pipe": pipe,
                "frac": tf / peak if tf else None}
    fmm = {"p2m": fp(fs["p2m"], 11.0 * wc["p2m_pairs"]),
           "m2m_ms": fs["m2m"],
           "m2l": fp(fs["m2l"], wc["m2l_flops"], peak_tc or peak_tf, "fp64 tensor (DMMA)"),
           "x_list": fp(fs["x"], 11.0 * wc["x_pairs"]), "l2l_ms": fs["l2l"],
           "leaf": fp(fs["leaf"], 20.0 * leaf_pairs), "total_ms": fs["total"],
           "pairs": {k: wc[k] for k in ("u_pairs", "w_pairs", "de_pairs", "x_pairs",
                                         "p2m_pairs", "v_pairs")},
           "flop_convention": "pairwise 1/r: 20 flop per pot+grad pair (leaf), 11 per pot-only "
                              "lattice pair (P2M, X); M2L 4 nrep r_k per V pair (low-rank)"}
    stages["fmm_call1_stages"] = fmm
    return stages


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--eager", action="store_true", help="time the step without a CUDA graph")
    ap.add_argument("--no-extra", action="store_true",
                    help="skip the secondary lines (config 2 exact sweeps, config 5 FMM)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    rank, world, local = _dist()
    if os.environ.get("BENCH_SHARE_GPU") == "1":  # functional multi-rank check on one GPU
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator / NVLS lines in the log
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    from paper_2111_10743_b200 import _build, _lib
    _build.build(verbose=False)
    lib = _lib.load()
    from paper_2111_10743_b200 import LayerOperatorSet
    from paper_2111_10743_b200.solver import _bind

    peaks = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6547.2))
    geom, near, cset, setup = build_config3(torch, corrections=world == 1)
    n, nover = geom.nnodes, geom.noversampled
    inter = 4 * n * nover
    c = CONFIG3
    t0 = time.perf_counter()
    if world > 1:
        # Morton-range target shards, per-rank corrections, distributed
        # upward pass (sharding.py); GMRES replicated on full vectors
        from paper_2111_10743_b200.sharding import ShardedOperatorSet
        op = ShardedOperatorSet(geom, "a3", c["eps"], None, far="fmm", eta=c["eta"],
                                cap=c["cap"], fmm_ncrit=c["ncrit"])
        cset = type("C", (), {"nnz": int(np.asarray(near.offsets)[-1]) * int(geom.nodes_per_patch)})
    else:
        op = LayerOperatorSet(geom, "a3", c["eps"], corrections=cset, near=near, far="fmm",
                              fmm_ncrit=c["ncrit"])
    torch.cuda.synchronize()
    setup["plan_s"] = time.perf_counter() - t0
    L = _bind()
    nloc = n  # GMRES vectors are full length on every rank
    rng = np.random.default_rng(2)
    Q = torch.from_numpy(np.linalg.qr(rng.standard_normal((nloc, K_ARNOLDI + 1)))[0].T
                         .copy()).cuda().contiguous()
    hdev = torch.zeros(K_ARNOLDI + 2, dtype=torch.float64, device="cuda")
    v = torch.empty(nloc, dtype=torch.float64, device="cuda")
    tau_h = rng.standard_normal(n)
    tau = torch.from_numpy(tau_h).cuda()

    def mgs():
        _lib.check(L.lb_arnoldi_mgs(_lib.ptr(Q), nloc, K_ARNOLDI - 1, nloc, _lib.ptr(v),
                                    _lib.ptr(hdev), _lib.stream_handle()))

    def step():
        op.apply_device(tau, out=v)
        mgs()

    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    ref_v = v.clone()
    run_step, graphed, nkern = (step, False, None)
    if world == 1 and not args.eager:
        run_step, graphed, nkern = capture(torch, step, lib, _lib)
        if graphed:  # the replay must reproduce the eager step
            op.apply_device(tau, out=v)
            mgs()
            eager_v = v.clone()
            run_step()
            torch.cuda.synchronize()
            if not torch.equal(v, eager_v):
                print("bench: graph replay differs from the eager step; timing eagerly",
                      file=sys.stderr)
                run_step, graphed = step, False
    if world > 1:  # the rank's own kernels per step, counted from throw-away captures
        nkern = count_sharded_launches(torch, op, mgs, lib, _lib)
    timer = Timer(torch, world, local, flush)
    times, clocks = timer(run_step, args.steps)
    t_step = timer.max_over_ranks(sum(times) / len(times))
    value = inter / t_step

    # e2e: the public API with host buffers (pinned tau in, result out)
    tau_pin = torch.from_numpy(np.ascontiguousarray(tau.cpu().numpy())).pin_memory()
    out_pin = torch.empty(nloc, dtype=torch.float64).pin_memory()
    tau_d = torch.empty_like(tau)

    def e2e_step():
        tau_d.copy_(tau_pin, non_blocking=True)
        op.apply_device(tau_d, out=v)
        mgs()
        out_pin.copy_(v, non_blocking=True)
    e2e_times, _ = timer(e2e_step, args.steps)
    e2e_t = timer.max_over_ranks(sum(e2e_times) / len(e2e_times))

    peak = fp64_peak_tflops(torch, lib, _lib)
    peak_tc = dmma_peak_tflops(torch, lib, _lib)
    stages = roofline = None
    if world == 1:
        stages = stage_rooflines(torch, op, op._plan, n, nover, cset.nnz, peak, hbm, _lib, peak_tc)
        f = stages["fmm_call1_stages"]
        cands = [("spmv", stages["spmv2_glue"]["ms"], "hbm"),
                 ("leaf", f["leaf"]["ms"], "fp64"), ("m2l", f["m2l"]["ms"], "fp64")]
        dom = max(cands, key=lambda x: x[1])[0]
        if dom == "spmv":
            s2 = stages["spmv2_glue"]
            roofline = {"bound": "hbm", "kernel": "csr_epi_kernel (A3 pass 2: 3 kinds + glue)",
                        "achieved": s2["GBps"], "peak": hbm, "unit": "GB/s",
                        "frac": s2["frac_hbm"], "traffic": s2["bytes"],
                        "traffic_note": "block-CSR bytes the kernel reads (= ncu dram__bytes_read, "
                                        "profiles/round2/config3_step_launches.md)",
                        "peak_source": "MEASURED_PEAKS.json hbm_gbs"}
        elif dom == "m2l":
            s = f["m2l"]
            roofline = {"bound": "tensor", "kernel": "FMM M2L (m2l1::first_kernel + m2lf::m2l_fused_kernel, "
                        "DMMA 8x8x4, + m2lf::reduce_kernel), pot+grad call", "achieved": s["TFLOPs"],
                        "peak": peak_tc, "unit": "TFLOP/s", "frac": s["frac"],
                        "traffic": M2L_DRAM_BYTES_NCU,
                        "traffic_note": "dram read+write of its 3 launches, ncu "
                                        "(profiles/round2/config3_step_launches.md); algorithmic: one "
                                        "488 x 8 B multipole per V pair = 0.83 GB",
                        "peak_source": "measured in-run (lb_probe_dmma: FP64 tensor-core DMMA "
                                       "chains); FP64 FMA pipe measured " + f"{peak:.1f}"}
        else:
            s = f["leaf"]
            roofline = {"bound": "fp64", "kernel": "leaf_kernel (FMM U/W/DE lists)",
                        "achieved": s["TFLOPs"], "peak": peak, "unit": "TFLOP/s",
                        "frac": s["frac"], "traffic": None,
                        "peak_source": f"measured in-run (lb_probe_dfma); nominal "
                                       f"{NOMINAL_FP64_TFLOPS}"}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cop, ctau, cQ, _, _, cores = cpu_config3_setup(os.cpu_count() or 1)
        cpu_time(cop, ctau, cQ, 1)
        ts = cpu_time(cop, ctau, cQ, 2)
        tc = n / len(cop.rows) * min(ts)
        cpu = {"value": inter / tc, "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"every {ROW_STRIDE}th target ({len(cop.rows)} rows): both far calls "
                         "as exact sums over all sources (oracle C port), sampled CSR rows, "
                         "full oversampling + MGS; time x N/rows (bench.py --impl reference)"}
    extra = {}
    if rank == 0 and world == 1 and not args.no_extra:
        extra["config2"] = config2_line(torch, lib, _lib, peak, flush)
        extra["config5_fmm"] = fmm_config5(torch)
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t_step * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (config-3 torus from its chart; near map and corrections built "
                    "on the device, csrc/quad.cu)",
            "config": {"workload": WORKLOAD, "N": n, "N_over": nover, "formulation": "a3",
                       "far_field": f"FMM eps {c['eps']} ncrit {c['ncrit']} (surface m=10, "
                                    "low-rank M2L)",
                       "nnz_per_kind": cset.nnz, "interactions_per_step": inter,
                       "parallelism": f"target-shard{world}" if world > 1 else "single",
                       "l2": "flushed between timed steps (256 MB write); CSR 11.6 GB > L2",
                       "cuda_graph": graphed, "setup_s": setup},
            "roofline": roofline, "stages": stages, "cpu_baseline": cpu,
            "e2e": {"value": inter / e2e_t, "unit": UNIT, "h2d_bytes_per_step": 8 * nloc,
                    "d2h_bytes_per_step": 8 * nloc, "ms_per_step": e2e_t * 1e3},
            "gpu_launches": nkern * args.steps if nkern is not None else None,
            "launches_per_step": nkern,
            "clocks": clocks, "fp64_peaks_tflops": {"dfma": peak, "dmma": peak_tc},
            **extra,
        }), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def config2_line(torch, lib, _lib, peak, flush, steps=20):
    """Secondary: BASELINE config 2 (icosphere order 7, N = 8,960) with exact
    fp64 far sweeps (the fused A3 path), device corrections at eps 1e-10; the
    apply + MGS(k=4) step as a CUDA graph; roofline of the dominant kernel
    (opfar_kernel<FarA3c>, 39 flop per pair)."""
    import ctypes
    from paper_2111_10743_b200 import LayerOperatorSet, shapes
    from paper_2111_10743_b200.solver import _bind
    geom = shapes.icosphere(7)
    op = LayerOperatorSet(geom, "a3", 1e-10, far="direct")
    n, nover = geom.nnodes, geom.noversampled
    L = _bind()
    rng = np.random.default_rng(2)
    Q = torch.from_numpy(np.linalg.qr(rng.standard_normal((n, 5)))[0].T.copy()).cuda()
    h = torch.zeros(6, dtype=torch.float64, device="cuda")
    v = torch.empty(n, dtype=torch.float64, device="cuda")
    tau = torch.from_numpy(rng.standard_normal(n)).cuda()

    def step():
        op.apply_device(tau, out=v)
        _lib.check(L.lb_arnoldi_mgs(_lib.ptr(Q), n, 3, n, _lib.ptr(v), _lib.ptr(h),
                                    _lib.stream_handle()))
    for _ in range(3):
        step()
    run, graphed, nk = capture(torch, step, lib, _lib)
    ts, _ = Timer(torch, 1, 0, flush)(run, steps)
    t = sum(ts) / len(ts)
    sec = ctypes.c_double(0.0)
    op.apply_device(tau)
    torch.cuda.synchronize()
    _lib.check(lib.lb_opset_time_far(op.dev.handle, 2, 20, ctypes.byref(sec),
                                     _lib.stream_handle()))
    achieved = 39.0 * n * nover / sec.value / 1e12
    return {"workload": "config2-icosphere-o7-A3-exact-sweeps+MGS(k=4)", "N": n,
            "N_over": nover, "ms_per_step": t * 1e3, "value": 4 * n * nover / t, "unit": UNIT,
            "cuda_graph": graphed, "launches_per_step": nk,
            "roofline": {"bound": "fp64", "kernel": "opfar_kernel<FarA3c>", "achieved": achieved,
                         "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                         "far2_ms": sec.value * 1e3, "flops_per_pair": 39.0}}


def fmm_config5(torch, n=1_000_000, eps=1e-6, reps=5):
    """Secondary: BASELINE config 5's FMM (N = 1e6 unit-sphere cloud, sources
    = targets, seed 105, charge pot+grad) through the device FmmPlan."""
    from paper_2111_10743_b200.fmm_plan import FmmPlan
    from paper_2111_10743_b200.shapes import sphere_cloud
    x = sphere_cloud(n)
    q = torch.from_numpy(np.random.default_rng(5).standard_normal((1, n))).cuda()
    FmmPlan(x[:1000], x[:1000], eps)  # unit operators (cached), as a user's first plan
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = FmmPlan(x, x, eps)
    pot = torch.empty((1, n), dtype=torch.float64, device="cuda")
    grad = torch.empty((1, n, 3), dtype=torch.float64, device="cuda")
    plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = sum(ts) / len(ts)
    plan.set_timing(True)
    plan.apply_device(q, None, 1, 1, 0, 1, pot, grad)
    torch.cuda.synchronize()
    return {"workload": "config5-fmm", "N": n, "eps": eps, "rep": plan.rep, "m": plan.m,
            "apply_ms": t * 1e3, "effective_interactions_per_s": n * (n - 1) / t,
            "plan_plus_first_apply_s": t_setup, "stages_ms": plan.stage_times()}


if __name__ == "__main__":
    main()
