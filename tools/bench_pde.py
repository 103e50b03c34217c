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
# Table 3 (log-normal), top row M = s = 2N, "fast"
PAPER_FAST_S_LOGN = {67: 0.040, 127: 0.033, 257: 0.094, 509: 0.326, 1021: 1.122, 2053: 4.296, 4001: 15.203,
                     8009: 60.546, 16001: 270.691}


def main():
    logn = "--lognormal" in sys.argv
    Ns = [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [257, 1021, 4001, 16001]
    for N in Ns:
        M = s = 2 * N
        if logn:
            w = W.pde1d_lognormal(N, M, s, seed=N)
            pde = q.LognormalPDE1D(w.N, w.z, w.A, w.extra["psi0"])
        else:
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
        c, d = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if logn:
            pde.plan.matmul(pde.Psi, pde.buf[:, :pde.M])
            c.record(st)
            q._abi.qmc_fe1d_lognormal_solve_mean(pde.N, pde.M, pde.psi0, None, pde.buf, pde.ldx, pde.mean,
                                                 st.cuda_stream)
        else:
            pde.plan.matmul(pde.A, pde.X)
            c.record(st)
            q._abi.qmc_tridiag_solve_mean(pde.N, pde.K, pde.d0, pde.e0, None, pde.X, pde.t, pde.mean,
                                          st.cuda_stream)
        d.record(st)
        torch.cuda.synchronize()
        print(json.dumps({"experiment": "exp3_lognormal_pde1d" if logn else "exp2_uniform_pde1d",
                          "N": N, "M": M, "s": s, "ms_total": ms,
                          "ms_solve_mean": c.elapsed_time(d), "entries": N * (M if logn else 2 * M - 3),
                          "paper_fast_s_matlab_cpu": (PAPER_FAST_S_LOGN if logn else PAPER_FAST_S).get(N),
                          "note": "GPU: fast X = Y·A + N Thomas solves + mean, inputs resident"}), flush=True)
        del pde
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
