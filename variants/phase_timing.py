import ctypes, os, sys, numpy as np
sys.path.insert(0, os.getcwd())
import torch
import paper_1501_06286_b200 as q
import qmc_workloads as W
lib = q._abi._lib
lib.qmc_debug_phases.argtypes = [ctypes.c_void_p, ctypes.c_int]
for bp in (1, 8, 32):
    os.environ["QMC_BATCH_PAIRS"] = str(bp)
    w = W.config(2, t_override=2 * bp)
    plan = q.Plan.from_workload(w)
    A = q.to_device_colmajor(w.A, "cuda")
    X = q.x_empty(plan.N, w.t, "cuda")
    for _ in range(3):
        plan.matmul(A, X)
    torch.cuda.synchronize()
    n = 16 * bp
    buf = np.zeros((n, 8), dtype=np.int64)
    lib.qmc_debug_phases(buf.ctypes.data, n)
    d = np.diff(buf[:, :6], axis=1)
    tot = buf[:, 5] - buf[:, 0]
    print(f"batch {bp}: CTAs {n}: phase cycles median T/fwd/W/inv/store:", np.median(d, axis=0).astype(int), "total median", int(np.median(tot)), "max", int(tot.max()))
