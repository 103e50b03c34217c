"""BASELINE.md §4 protocol on the host of the GPU box: the oracle (φ-table
gather + NumPy/OpenBLAS GEMM; table build excluded) timed
5 times, mean and median: full runs for configs 1, 2, 4; one 8192-row block
x all columns for configs 3 and 5, extrapolated linearly in N (labelled).
Prints one JSON line per config."""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import qmc_workloads as W  # noqa: E402
from bench import cpu_info  # noqa: E402


def run(c, reps=5):
    w = W.config(c)
    tab = O.phi_table(w.phi, w.N)
    idx = ((lambda r: O.polylattice_index_matrix(w.D, w.p, w.z, r)) if w.family == "poly"
           else (lambda r: O.lattice_index_matrix(w.N, w.z, r)))
    full = c in (1, 2, 4)
    rows = np.arange(w.N) if full else np.arange(8192)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for b in range(0, len(rows), 8192):
            O.oracle_X_rows(tab, idx(rows[b:b + 8192]), w.A)
        ts.append(time.perf_counter() - t0)
    scale = w.N / len(rows)
    ent = w.N * w.t
    return {"config": c, "workload": w.name, "rows_timed": int(len(rows)), "extrapolated": not full,
            "time_s_mean": statistics.fmean(ts) * scale, "time_s_median": statistics.median(ts) * scale,
            "entries_per_s_median": ent / (statistics.median(ts) * scale), "repeats": reps}


if __name__ == "__main__":
    print(json.dumps({"host": cpu_info()}), flush=True)
    for c in [int(x) for x in sys.argv[1:]] or [1, 2, 3, 4, 5]:
        print(json.dumps(run(c)), flush=True)
