#!/usr/bin/env python
"""Benchmark of the fast QMC matrix product X = Y·A on B200 (one process per
GPU; `--gpus N` without a torchrun environment re-launches itself under
torch.distributed.run with N ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]
                    [--scaling strong|weak]

A step is one pass of the whole hot path over the configured workload:
qmc_mean (or qmc_matmul) over this rank's contiguous column slab, X written
to HBM, plus the collective and finalize of the fused QMC mean.  BASELINE.json's
metric names no config, so the default is the largest single-GPU config,
configs[4] (C = 5: N = 786433, s = t = 8192, fused mean of exp X; its 51.5 GB
X fits one B200).  The other configs are parity cases and optional bench
lines (--config C).  --scaling strong (default) splits the config's t
columns over the N ranks in pair-aligned slabs; weak gives
every rank the config's t columns as its block of an N·t-column problem.
Prints ONE JSON line on rank 0.  See DESIGN.md §6 (measurement).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fast Y·A output entries/s (fp64) and % HBM roofline at 1/2/4/8 B200"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}
# fallback fp64 peak if profiles/fp64_peak.json is absent: 148 SM x 64 DFMA/clk x 2 x 1.965 GHz
FP64_FMA_PER_CLK_PER_SM = 64
N_SM = 148
F_NAMES = {None: "none", 0: "identity_mean", 1: "affine_mean", 2: "exp_mean", 3: "rowmean_relu"}
PHI_NAMES = {0: "identity", 1: "u-1/2", 2: "tent", 3: "invnorm(u+1/(2N))"}
# the paper's own best fast-method rate, Table 1, context only:
# Exp. 1, N = 16001, s = t = 1000, fast 0.741 s on a Xeon E5-2650v2 @ 2.6 GHz (Matlab R2013b)
PAPER_CONTEXT = {"paper_fast_entries_per_s": 16001 * 1000 / 0.741,
                 "workload": "Exp. 1, N=16001, s=t=1000, Phi^-1, random upper-triangular A (fast method)",
                 "hardware": "Intel Xeon E5-2650v2 @ 2.6 GHz, Matlab R2013b, mean of 5 runs",
                 "cite": "PAPER.md:779-781, 813-830 (Table 1)",
                 "note": "other hardware and workload: context, not a target (vs_baseline stays null)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--t", type=int, default=0, help="override the config's t (diagnostics only)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="strong",
                    help="N > 1: strong = the config's t columns split over the GPUs (pair-aligned "
                         "slabs); weak = every GPU runs the config's t columns (column block of a "
                         "G·t-column problem)")
    return ap.parse_args()


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        pk = {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
              "source": "measured (MEASURED_PEAKS.json)"}
    else:
        pk = dict(PEAKS_FALLBACK, source="fallback (B200_PROFILING.md)")
    f = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(f):
        with open(f) as fh:
            d = json.load(fh)
        pk["fp64_tflops"] = float(d["fp64_tflops_fma"])
        pk["fp64_instr_per_s"] = float(d["instr_peak_per_s"])
        pk["fp64_source"] = "measured (profiles/fp64_peak.json: DFMA-chain microbenchmark, all SMs, 1965 MHz)"
    else:
        pk["fp64_tflops"] = N_SM * FP64_FMA_PER_CLK_PER_SM * 2 * pk["sm_max_mhz"] * 1e6 / 1e12
        pk["fp64_instr_per_s"] = pk["fp64_tflops"] * 1e12 / 2
        pk["fp64_source"] = "derived: 148 SM x 64 DFMA/clk x 2 x sm_max_mhz"
    return pk


def cpu_info():
    """Host CPU model, sockets and the BLAS thread count the oracle uses."""
    info = {"cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            k, _, v = ln.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k.strip()] = v.strip()
    except Exception:  # noqa: BLE001
        pass
    try:
        from threadpoolctl import threadpool_info
        import numpy as np  # noqa: F401  (loads the BLAS)
        pools = threadpool_info()
        info["blas"] = [{"api": p.get("internal_api"), "threads": p.get("num_threads")} for p in pools]
    except Exception:  # noqa: BLE001
        pass
    return info


# ----------------------------------------------------------------- clocks
class ClockSampler:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- CPU oracle (baseline)
def cpu_oracle_rate(w, seconds: float, rows_per_block: int = 2048, seed: int = 0):
    """Entries/s of the oracle (Y by φ-table gather + NumPy GEMM) on the
    host, over random row blocks for about `seconds`; the φ table build is
    excluded.  The cost is linear in the rows, so the rate
    extrapolates to all N rows."""
    import numpy as np
    import oracle as O
    tab = O.phi_table(w.phi, w.N)
    if w.family == "poly":
        idx_fn = lambda r: O.polylattice_index_matrix(w.D, w.p, w.z, r)  # noqa: E731
    else:
        idx_fn = lambda r: O.lattice_index_matrix(w.N, w.z, r)  # noqa: E731
    rng = np.random.default_rng(seed)
    done, t0 = 0, time.perf_counter()
    while True:
        r0 = int(rng.integers(0, max(1, w.N - rows_per_block)))
        rows = np.arange(r0, min(w.N, r0 + rows_per_block))
        O.oracle_X_rows(tab, idx_fn(rows), w.A)
        done += len(rows)
        el = time.perf_counter() - t0
        if el >= seconds or done >= w.N:
            break
    try:
        from threadpoolctl import threadpool_info
        threads = max([i.get("num_threads", 1) for i in threadpool_info()] or [1])
    except Exception:
        threads = os.cpu_count()
    return done * w.t / el, done, el, threads


def cpu_baseline(w, seconds: float, repeats: int = 5):
    """BASELINE.md §4 protocol: `repeats` timed samples of random row blocks
    (each ~seconds/repeats), mean and median rate; host model and BLAS threads."""
    rates, rows_tot, el_tot, threads = [], 0, 0.0, 1
    for k in range(repeats):
        r, rows, el, threads = cpu_oracle_rate(w, seconds / repeats, seed=k)
        rates.append(r)
        rows_tot += rows
        el_tot += el
    return {"value": statistics.median(rates), "unit": "entries/s", "cores": threads, "kind": "oracle",
            "mean": statistics.fmean(rates), "median": statistics.median(rates), "repeats": repeats,
            "sample": f"{repeats} repeats of random 2048-row blocks x all {w.t} columns ({rows_tot} of "
                      f"N = {w.N} rows in {el_tot:.1f} s); rate extrapolated linearly to all N rows "
                      f"(phi-table gather + NumPy/OpenBLAS GEMM)",
            "extrapolated": rows_tot < w.N, "host": cpu_info()}


def slab(w, G, rank, scaling):
    """This rank's column slab [c0, c1) and the job's total columns."""
    from paper_1501_06286_b200.dist import shard_columns
    if scaling == "weak":  # every rank the config's t columns, block `rank` of a G·t-column problem
        return rank * w.t, (rank + 1) * w.t, G * w.t
    c0, c1 = shard_columns(w.t, G, rank)  # the config's t columns split over the ranks
    return c0, c1, w.t


def config_dict(w, G, scaling, tl):
    return {"workload": w.name, "family": w.family, "N": w.N, "s": w.s, "t": w.t,
            "t_total": G * w.t if scaling == "weak" else w.t, "t_per_gpu": tl,
            "phi": PHI_NAMES[w.phi], "f": F_NAMES[w.f], "parallelism": f"columns/{G}",
            "l2": "flushed between timed steps (256 MiB write, untimed)"}


def reference_arm(args, rank, world):
    """--impl reference: the oracle, as it stands, on the host cores (rank 0
    alone; other ranks exit without work)."""
    import qmc_workloads as W
    if rank != 0:
        return
    w = W.config(args.config, t_override=args.t or None)
    c0, c1, _ = slab(w, world, 0, args.scaling)
    rows = 1024
    # warmup + timed steps, each a bounded sample of `rows` rows × all t columns
    for _ in range(args.warmup):
        cpu_oracle_rate(w, 0.0, rows_per_block=rows, seed=1)
    t0 = time.perf_counter()
    done = 0
    threads = 1
    for k in range(args.steps):
        _, d, _, threads = cpu_oracle_rate(w, 0.0, rows_per_block=rows, seed=100 + k)
        done += d
    el = time.perf_counter() - t0
    value = done * w.t / el
    sample = (f"{rows} random contiguous rows x all {w.t} columns per step (of N={w.N}); rate "
              f"extrapolates linearly to all rows")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "entries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": args.scaling,
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": config_dict(w, world, args.scaling, c1 - c0),
        "cpu_baseline": {"value": value, "unit": "entries/s", "cores": threads, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- our arm
def k1_fp64_instr_per_item(L2):
    """fp64 instructions per thread per K1 item (row FFT forward + inverse,
    ×W, folded twiddles), counted from ncu smsp__sass_thread_inst_executed
    _op_{dadd,dmul,dfma} of the round-2 build (profiles/r02_fp64_audit.txt);
    None if not audited for this row length."""
    return {4096: 1658.0, 8192: 1871.0}.get(L2)


def ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1501_06286_b200 as q
    import qmc_workloads as W
    from paper_1501_06286_b200 import _abi as abi
    from paper_1501_06286_b200.dist import combine_means

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    w = W.config(args.config, t_override=args.t or None)
    G = world
    c0, c1, t_total = slab(w, G, rank, args.scaling)
    A_block = w.A if args.scaling == "weak" else w.A[:, c0:c1]
    tl = c1 - c0
    plan = q.Plan.from_workload(w, device=dev)
    A_host = np.ascontiguousarray(A_block.T)                 # (tl, s) row-major = A slab col-major
    A = torch.from_numpy(A_host).to(dev).t()
    X = q.x_empty(w.N, tl, dev)
    f, fp = w.f, w.f_param
    N = w.N
    if f == W.F_ROWMEAN_RELU:
        out = torch.empty(N, dtype=torch.float64, device=dev)
        res = torch.empty(1, dtype=torch.float64, device=dev)
    elif f is not None:
        out = torch.empty(max(tl, 1), dtype=torch.float64, device=dev)
    plan.call_workspace(tl, -1 if f is None else f)

    def step(Ain):
        """One pass of the hot path over this rank's column slab + the
        collective of the fused mean (dist.combine_means) + finalize."""
        if f is None:
            plan.matmul(Ain, X)
            return None
        plan.mean(Ain, f, fp, X=X, out=out)
        red = combine_means(out, f, t_total, c0, c1)
        if f == W.F_ROWMEAN_RELU:
            plan.finalize(f, red, t_total, out=res)
            return res
        return red

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    for _ in range(args.warmup):
        step(A)
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    stream = torch.cuda.current_stream(dev)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    # one untimed probe step with the library's per-launch events: when the
    # step is ONE launch of this library, the step's own events bracket
    # exactly that launch on the same stream, so the timed region runs without
    # the library's extra events (a few microseconds per step, most of a
    # one-row plan's step) and the kernel's time is the step time
    abi.qmc_profile_read()
    abi.qmc_profile_enable(True)
    l0 = abi.qmc_launch_count()
    step(A)
    torch.cuda.synchronize()
    probe_launches = abi.qmc_launch_count() - l0
    probe = {k: v for k, v in abi.qmc_profile_read().items() if v[0]}
    abi.qmc_profile_enable(False)
    single_launch = probe_launches == 1 and len(probe) == 1
    sampler = ClockSampler(local_rank)
    sampler.start()
    time.sleep(0.3)
    abi.qmc_profile_read()
    abi.qmc_profile_enable(not single_launch)
    l0 = abi.qmc_launch_count()
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    for k in range(args.steps):
        flush.zero_()                     # L2 flush between timed steps (untimed)
        evs[k][0].record(stream)
        step(A)
        evs[k][1].record(stream)
    torch.cuda.synchronize()
    if G > 1:
        dist.barrier()
    launches = abi.qmc_launch_count() - l0
    abi.qmc_profile_enable(False)
    prof = abi.qmc_profile_read()
    clocks = sampler.stop()
    ms_local = sum(a.elapsed_time(b) for a, b in evs)
    if single_launch:  # the step events are the kernel's own events
        prof = {next(iter(probe)): (args.steps, ms_local)}
    t_ms = torch.tensor([ms_local], dtype=torch.float64, device=dev)
    if G > 1:
        dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms_total = float(t_ms.item())
    ms_step = ms_total / args.steps
    entries = N * t_total
    value = entries * args.steps / (ms_total / 1e3)

    # ---- roofline of the dominant kernel (per-class CUDA events, this rank)
    peaks = load_peaks()
    info = plan.info
    L, L1, L2 = info["L"], info["L1"], info["L2"]
    npairs = (tl + 1) // 2
    kernels = {}
    tot_prof = sum(v[1] for v in prof.values()) or 1.0
    for name, (n, ms) in prof.items():
        if n:
            kernels[name] = {"launches": n, "ms_total": ms, "share": ms / tot_prof}
    dom = max(kernels, key=lambda k: kernels[k]["ms_total"]) if kernels else None
    fp64_peak = peaks["fp64_tflops"]
    roof = None
    if dom == "k_rows":
        dn, dms = kernels[dom]["launches"], kernels[dom]["ms_total"]
        items = args.steps * npairs * L1
        flops = items * 2 * 5.0 * L2 * math.log2(L2)
        achieved = flops / (dms / 1e3) / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": fp64_peak, "unit": "TFLOP/s",
                "frac": achieved / fp64_peak, "traffic": None, "kernel": dom,
                "work": "algorithmic fp64 flops per launch = K1 items (L1 rows x pairs) x 2 FFTs x "
                        "5 L2 log2 L2 (DESIGN.md §6)",
                "peak_source": peaks["fp64_source"]}
        ipi = k1_fp64_instr_per_item(L2)
        if ipi:  # the fp64-pipe view: audited instructions per item / measured instruction peak
            roof["fp64_instr_frac"] = items * (L2 // 16) * ipi / (dms / 1e3) / peaks["fp64_instr_per_s"]
    elif dom is not None:
        dn, dms = kernels[dom]["launches"], kernels[dom]["ms_total"]
        if dom == "k_cols":   # HBM: U read + X written per launch
            nbytes = args.steps * (16.0 * L * npairs + 8.0 * N * tl)
        elif dom == "k_pack":
            nbytes = args.steps * 8.0 * w.s * tl
        else:
            nbytes = args.steps * 8.0 * tl
        achieved = nbytes / (dms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"], "traffic": None, "kernel": dom}
    if roof is not None:
        roof["launches"] = dn
        roof["avg_launch_ms"] = dms / dn
        traffic_file = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(traffic_file):
            with open(traffic_file) as fh:
                tf = json.load(fh).get(f"c{args.config}", {})
            if dom in tf and tf.get("_batch_pairs") in (None, info["batch_pairs"]):
                roof["traffic"] = tf[dom]
    # whole-step HBM roofline (north star): compulsory bytes = read A + write X
    step_bytes = 8.0 * (N + w.s) * tl  # this rank's compulsory bytes (rank 0 reports)
    hbm_ach = step_bytes / (ms_step / 1e3) / 1e9
    hbm = {"bytes_per_step": step_bytes, "achieved_GBps": hbm_ach, "peak_GBps": peaks["hbm_gbs"],
           "frac": hbm_ach / peaks["hbm_gbs"], "frac_vs_8TBps_nominal": hbm_ach / 8000.0,
           "peak_source": peaks["source"]}

    # ---- e2e: host buffers in, result back to host, through the public API
    A_pin = torch.from_numpy(A_host).pin_memory()
    A_dev2 = torch.empty(A_host.shape, dtype=torch.float64, device=dev)
    if G == 1:
        f_e2e = f if f is not None else W.F_IDENTITY
        n_res = 1 if f_e2e == W.F_ROWMEAN_RELU else tl
        out_pin = torch.empty(n_res, dtype=torch.float64).pin_memory()
        out_dev = torch.empty(max(N, tl), dtype=torch.float64, device=dev)
        ws = plan.call_workspace(tl, f_e2e)
        st = stream.cuda_stream

        def e2e_step():
            abi.qmc_mean_host(plan.handle, A_pin, w.s, tl, f_e2e, fp, out_pin, A_dev2, X, max(tl, 1),
                              out_dev, ws, ws.numel(), st)
        for _ in range(max(1, args.warmup)):
            e2e_step()
        ee = []
        for k in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e2e_step()
            b.record(stream)
            torch.cuda.synchronize()
            ee.append(a.elapsed_time(b))
        e_ms = sum(ee)
        e2e = {"value": entries * args.steps / (e_ms / 1e3), "unit": "entries/s",
               "h2d_bytes_per_step": int(A_pin.numel() * 8), "d2h_bytes_per_step": int(n_res * 8),
               "ms_per_step": e_ms / args.steps, "ms_min": min(ee), "ms_median": sorted(ee)[len(ee) // 2],
               "ms_max": max(ee), "api": "qmc_mean_host (C ABI, pinned host A)"}
    else:
        A2 = A_dev2.t()  # the copied slab, column-major (s, tl): the step computes on it
        ee = []
        host = None
        for k in range(args.warmup + args.steps):
            flush.zero_()
            torch.cuda.synchronize()
            dist.barrier()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            A_dev2.copy_(A_pin, non_blocking=True)
            r = step(A2)
            host = r.cpu() if r is not None else X[0, :1].cpu()
            b.record(stream)
            torch.cuda.synchronize()
            if k >= args.warmup:
                ee.append(a.elapsed_time(b))
        t_e = torch.tensor([sum(ee)], dtype=torch.float64, device=dev)
        dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e_ms = float(t_e.item())
        e2e = {"value": entries * args.steps / (e_ms / 1e3), "unit": "entries/s",
               "h2d_bytes_per_step": int(A_pin.numel() * 8),
               "d2h_bytes_per_step": int(host.numel() * 8), "ms_per_step": e_ms / args.steps,
               "api": "Plan.mean + torch.distributed (pinned host A slab per rank, copied and "
                      "computed on every step)"}

    cpu = None
    if rank == 0 and G == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, args.cpu_seconds)

    if rank == 0:
        cfg = config_dict(w, G, args.scaling, tl)
        line = {
            "metric": METRIC, "value": value, "unit": "entries/s", "n_gpus": G,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": args.scaling if G > 1 else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "plan": {"L": L, "L1": L1, "L2": L2, "batch_pairs": info["batch_pairs"],
                     "k1_input": {1: "balanced", 0: "bucket order", 2: "dense"}.get(info["k1_order"])},
            "roofline": roof, "hbm_roofline_step": hbm, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clocks, "kernels": kernels,
            "kernel_timing": ("the step's own CUDA events (one launch of this library per step)"
                              if single_launch else "the library's per-launch CUDA events (qmc_profile_*)"),
            "paper_context": PAPER_CONTEXT,
        }
        print(json.dumps(line), flush=True)


def _free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    args = parse()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # no torchrun environment: re-launch under torch.distributed.run with one rank per GPU
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and rank == 0:
        print(f"bench.py: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        reference_arm(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    ours(args, rank, world, local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
