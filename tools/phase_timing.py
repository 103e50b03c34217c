"""K1 phase timing (needs libqmc built with -DQMC_PHASE_TIMING): cycles per
item between QMC_TS marks: scatter (wait+stage), fwd FFT, xW, inv FFT, store."""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

import paper_1501_06286_b200 as q  # noqa: E402
import qmc_workloads as W  # noqa: E402

lib = q._abi._lib
lib.qmc_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
for bp in (32, 64):
    os.environ["QMC_BATCH_PAIRS"] = str(bp)
    os.environ["QMC_ONE_STREAM"] = "1"
    w = W.config(cfg, t_override=2 * bp)
    plan = q.Plan.from_workload(w)
    A = q.to_device_colmajor(w.A, "cuda")
    X = q.x_empty(plan.N, w.t, "cuda")
    for _ in range(3):
        plan.matmul(A, X)
    torch.cuda.synchronize()
    n = min(4096, plan.info["L1"] * bp)
    buf = np.zeros((n, 8), dtype=np.int64)
    lib.qmc_debug_phases(buf.ctypes.data, n)
    d = np.diff(buf[:, :6], axis=1)
    tot = buf[:, 5] - buf[:, 0]
    print(f"c{cfg} batch {bp}: items {n}: median cycles scatter/fwd/W/inv/store:",
          np.median(d, axis=0).astype(int), "total median", int(np.median(tot)), "max", int(tot.max()),
          "| of the scatter, chunk waits (mbarrier + barrier):", int(np.median(buf[:, 6])),
          "main loops:", int(np.median(buf[:, 7])))
