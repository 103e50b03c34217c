"""Times Experiment 2 (Table 2 top row M = s = 2N) on the
GPU: X = Y·A by the fast path + N Thomas solves + mean, inputs resident,
CUDA events, after warm-up.  Prints one JSON line per N with the paper's
own "fast" time (Matlab on a CPU, context only)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1501_06286_b200 as q  # noqa: E402
import qmc_workloads as W  # noqa: E402

PAPER_FAST_S = {67: 0.035, 127: 0.042, 257: 0.114, 509: 0.462, 1021: 1.562, 2053: 5.591, 4001: 19.678,
                8009: 87.246, 16001: 342.615}


def main():
    Ns = [int(a) for a in sys.argv[1:]] or [257, 1021, 4001, 16001]
    for N in Ns:
        M = s = 2 * N
        w = W.pde1d_uniform(N, M, s, seed=N)
        pde = q.UniformPDE1D(w.N, w.z, w.A, w.extra["d0"], w.extra["e0"])
        for _ in range(3):
            pde.solve_mean()
        torch.cuda.synchronize()
        st = torch.cuda.current_stream()
        reps = 5
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            pde.solve_mean()
        b.record(st)
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / reps
        # solve + mean alone
        pde.plan.matmul(pde.A, pde.X)
        c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c.record(st)
        q._abi.qmc_tridiag_solve_mean(pde.N, pde.K, pde.d0, pde.e0, None, pde.X, pde.t, pde.mean, st.cuda_stream)
        d.record(st)
        torch.cuda.synchronize()
        print(json.dumps({"experiment": "exp2_uniform_pde1d", "N": N, "M": M, "s": s, "ms_total": ms,
                          "ms_solve_mean": c.elapsed_time(d), "entries": N * (2 * M - 3),
                          "paper_fast_s_matlab_cpu": PAPER_FAST_S.get(N),
                          "note": "GPU: fast X = Y·A + N Thomas solves + mean, inputs resident"}), flush=True)
        del pde
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
