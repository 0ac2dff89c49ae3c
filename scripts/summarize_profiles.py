"""Summarise ncu outputs from gpurun_out/ into profiles/round1/ (tracked)."""
import csv
import json
import os
import re
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "profiles", "round1")
G = os.path.join(ROOT, "gpurun_out")
os.makedirs(OUT, exist_ok=True)


def launches(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            hdr, start = r, i
            break
    ki, mi, vi, ui, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                                    "Metric Unit", "ID"))
    recs = defaultdict(dict)
    names = {}
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3,
                 "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        recs[r[idi]][r[mi]] = v * scale
        names[r[idi]] = re.sub(r"\(.*", "", r[ki])[:80]
    return [(names[k], recs[k]) for k in sorted(recs, key=int)]


def step_summary():
    L = launches(os.path.join(G, "launches_step.csv"))
    tot = sum(m["gpu__time_duration.sum"] for _, m in L)
    lines = ["# Config 2 bench step (A3 apply + MGS k=4): ncu launch list",
             "", "Cold-cache, serialised (ncu); compare SHARES, not absolute times "
             "(bench.py times the step with CUDA events).", "",
             "| # | kernel | us | share | DRAM read MB | DRAM write MB |", "|---|---|---|---|---|---|"]
    for i, (nm, m) in enumerate(L):
        t = m["gpu__time_duration.sum"]
        lines.append(f"| {i} | `{nm}` | {t:.1f} | {100 * t / tot:.1f}% | "
                     f"{m.get('dram__bytes_read.sum', 0) / 1e6:.1f} | "
                     f"{m.get('dram__bytes_write.sum', 0) / 1e6:.1f} |")
    lines.append(f"| | total | {tot:.1f} | 100% | | |")
    open(os.path.join(OUT, "config2_step_launches.md"), "w").write("\n".join(lines) + "\n")
    return L


def bench_summary():
    """The launch list of `python bench.py --steps 2 --warmup 3 --no-cpu-baseline`
    (the bench command itself), aggregated by kernel."""
    L = launches(os.path.join(G, "launches_bench.csv"))
    agg = defaultdict(lambda: [0, 0.0])
    for nm, m in L:
        agg[nm.replace("void ", "").strip()][0] += 1
        agg[nm.replace("void ", "").strip()][1] += m["gpu__time_duration.sum"]
    tot = sum(v[1] for v in agg.values())
    lines = ["# `python bench.py --steps 2 --warmup 3 --no-cpu-baseline`: ncu launch list",
             "", "Every launch of the bench command (setup incl. the device correction build, parity apply, warm-up, timed "
             "steps, the far-sweep timing reps, e2e steps, the DFMA peak probe, the secondary config-5 FMM line), "
             "aggregated by kernel; cold-cache and serialised (shares, not absolutes).", "",
             "| kernel | launches | us | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {t:.1f} | {100 * t / tot:.1f}% |")
    lines.append(f"| total | {sum(v[0] for v in agg.values())} | {tot:.1f} | |")
    open(os.path.join(OUT, "bench_launches.md"), "w").write("\n".join(lines) + "\n")


def avn_summary():
    """profiles/round1/apply_vs_n.jsonl (scripts/apply_vs_n.py output) -> .md"""
    rows = [json.loads(l) for l in open(os.path.join(OUT, "apply_vs_n.jsonl"))]
    try:
        hbm = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        hbm = 6552.6
    L = ["# GMRES operator-apply time vs N (A3, B200, round 1)", "",
         "Second half of the BASELINE metric.  Corrections: config 2 built by the reference "
         "(eps 1e-10); configs 3 and 4 built ON THE DEVICE (`quadrature.build_correction_set`, "
         "csrc/quad.cu: the reference's adaptive quadrature; near map bit-exact against the "
         "reference's) because the reference's own build takes hours (config 3) to more than a "
         "day (config 4).  Stage times from `lb_opset_stage_times` (CUDA events).  Exact-sweep "
         "A3 runs the fused second sweep (FarA3c); the FMM path runs A3's second call on two FMM "
         "densities with a projected leaf stage.  `scripts/apply_vs_n.py`.", "",
         "| case | N | N_over | nnz/kind | far field | apply ms | far 1 ms | SpMV 1 ms (HBM frac) "
         "| far 2 ms | SpMV 2 + glue ms (HBM frac) |", "|---|---|---|---|---|---|---|---|---|---|"]
    builds = []
    for r in rows:
        if "apply_ms" not in r:
            builds.append(r)
            continue
        if r["far"] == "direct":
            far = "direct (exact fp64 sweeps, fused)"
        else:
            m2l = {0: "fp64 dense DGEMM", -1: "low-rank fp64"}.get(r["m2l_slices"], f"tcgen05 int8 S={r['m2l_slices']}")
            far = f"fmm eps={r['eps']:g} ncrit={r['fmm_ncrit']} M2L {m2l}"
        st = r["stages_ms"]
        L.append(f"| {r['case']} | {r['N']} | {r['N_over']} | {r['nnz_per_kind']:.3g} | {far} | "
                 f"{r['apply_ms']:.2f} | {st['far1']:.2f} | {st['spmv1']:.3f} "
                 f"({r['spmv1_GBps'] / hbm:.2f}) | {st['far2']:.2f} | {st['spmv2+glue']:.3f} "
                 f"({r['spmv2_GBps'] / hbm:.2f}) |")
    L += ["", "Device correction builds:", "",
          "| case | eps | pairs | near map s | t_q s | leaves evaluated |", "|---|---|---|---|---|---|"]
    for b in builds:
        bb = b["build"]
        L.append(f"| {b['case']} | {bb['eps']:g} | {bb['split']['pairs']} | {bb['t_near_s']:.2f} "
                 f"(bit-exact: {bb['near_equal_reference']}) | {bb['t_q_s']:.1f} | "
                 f"{bb['split']['leaves']:.3g} |")
    L += ["", "SpMV algorithmic bytes: pass 1 = nnz (2*8 + 4) + 8(N+1); pass 2 = nnz (k*8 + 4) + "
          "8(N+1) with k = 2 value arrays (fused: S', S''+D') or 3 (FMM path: S', S, S''+D'); x "
          f"gathers hit L2.  HBM peak = {hbm} GB/s (MEASURED_PEAKS.json).  Config 2's CSR "
          "(66 MB/kind) is L2-sized, so its passes are latency-bound.  Earlier rows of this round "
          "(3-density FMM, synthetic values): apply_vs_n_pre_fusion.jsonl.  Config-3 rows were "
          "re-measured after the leaf-pass fix (fmm_apply.cu); the config-4 rows predate it (its "
          "geometry file is too large to ship to the GPU box this session)."]
    open(os.path.join(OUT, "apply_vs_n.md"), "w").write("\n".join(L) + "\n")


def c5_summary():
    """profiles/round1/config5_sweep.jsonl (scripts/config5_sweep.py) -> .md"""
    rows = [json.loads(l) for l in open(os.path.join(OUT, "config5_sweep.jsonl"))]
    pk = rows[0]["fp64_peak_tflops_measured"]
    L = ["# BASELINE config 5 sweep (B200, round 1)", "",
         f"Measured FP64 FMA-pipe peak in the same run: {pk:.1f} TFLOP/s (lb_probe_dfma).", "",
         "## Direct P2P (charge, pot+grad, sources == targets, self skipped)", "",
         "| N | GPU time | interactions/s | TFLOP/s (20 flop) | frac of measured FP64 | "
         "CPU oracle, 16 threads (scaled sample) | speed-up |", "|---|---|---|---|---|---|---|"]
    for r in rows:
        if r.get("case", "").startswith("p2p"):
            L.append(f"| {r['case'].split('=')[1]} | {r['gpu_s'] * 1e3:.2f} ms | "
                     f"{r['interactions_per_s']:.3e} | {r['tflops_20flop']:.1f} | "
                     f"{r['frac_of_measured_fp64']:.2f} | {r['cpu_oracle_s_scaled']:.2f} s "
                     f"({r['cpu_sample']}) | {r['speedup_vs_cpu_oracle']:.0f}x |")
    L += ["", "## FMM (FmmPlan on the device; the reference's tree, lists and unit operators; "
          "M2L by the default low-rank factors)", "",
          "| case | rep | plan s | apply ms | N^2/t | err vs direct (200 targets) | M2L ms | "
          "X ms | leaf ms | reference apply (survey container, 8 vCPU) |",
          "|---|---|---|---|---|---|---|---|---|---|"]
    refs = {"N=1000000 eps=1e-06": "67.1 s", "N=1000000 eps=1e-09": "581.0 s"}
    for r in rows:
        if r.get("case", "").startswith("fmm"):
            c = r["case"][4:]
            st = r["stages_ms"]
            L.append(f"| {c} | {r['rep']} m={r['m']} | {r['plan_s']:.2f} | {r['apply_s'] * 1e3:.1f} | "
                     f"{r['effective_interactions_per_s']:.2e} | {r['err_vs_direct_200_targets']:.1e} | "
                     f"{st['m2l']:.1f} | {st['x']:.1f} | {st['leaf']:.1f} | "
                     f"{refs.get(c, 'not run (hours)')} |")
    L += ["", "`plan s` is FmmPlan construction including the unit operators' first "
          "(cached) host precompute (grid n=9: ~2 s, paid by the first 1e-9 row); the setup "
          "split without it is in plan_setup.md.",
          "", "Earlier rows of this round with the tcgen05 int8 M2L: config5_sweep_tc_m2l.jsonl "
          "(1e6 at 1e-9: 197 ms; 1e7 at 1e-9: 1.28 s)."]
    open(os.path.join(OUT, "config5_sweep.md"), "w").write("\n".join(L) + "\n")


def fmm_summary():
    L = launches(os.path.join(G, "launches_fmm.csv"))
    agg = defaultdict(lambda: [0, 0.0])
    for nm, m in L:
        key = re.sub(r"<.*", "", nm.replace("void ", "")).strip()
        agg[key][0] += 1
        agg[key][1] += m["gpu__time_duration.sum"]
    tot = sum(v[1] for v in agg.values())
    lines = ["# FMM apply, N = 1e6 uniform on the sphere, eps 1e-6 (surface m=8), nd=1 pot+grad",
             "", "ncu launch list aggregated by kernel (cold-cache, serialised).", "",
             "| kernel | launches | ms | share |", "|---|---|---|---|"]
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"| `{k}` | {c} | {t / 1e3:.2f} | {100 * t / tot:.1f}% |")
    lines.append(f"| total | {sum(v[0] for v in agg.values())} | {tot / 1e3:.2f} | |")
    open(os.path.join(OUT, "fmm_1e6_eps1e-6_launches.md"), "w").write("\n".join(lines) + "\n")


def full_summary(rep, out_name):
    raw = subprocess.run(["ncu", "-i", os.path.join(G, rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
            "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
            "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for w in want:
            if w in hdr:
                d[w] = r[hdr.index(w)] + " " + units[hdr.index(w)]
        res.append(d)
    json.dump(res, open(os.path.join(OUT, out_name), "w"), indent=1)
    return res


if __name__ == "__main__":
    what = sys.argv[1:] or ["step", "fmm", "full"]
    if "step" in what:
        step_summary()
    if "bench" in what:
        bench_summary()
    if "avn" in what:
        avn_summary()
    if "c5" in what:
        c5_summary()
    if "fmm" in what:
        fmm_summary()
    if "full" in what:
        full_summary("prof_step2.ncu-rep", "ncu_full_config2_far_csr.json")
    print("written to", OUT)
