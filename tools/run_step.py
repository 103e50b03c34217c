"""Minimal driver for profiling: one plan + `--steps` hot-path calls of a
config (no oracle, no timing).  Used under ncu / compute-sanitizer."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--t", type=int, default=0, help="override t (columns)")
    ap.add_argument("--nox", action="store_true", help="means only: X is not written")
    ap.add_argument("--matmul", action="store_true", help="qmc_matmul instead of the config's f")
    ap.add_argument("--poly", type=int, default=0, help="D: a polynomial-lattice workload of degree D instead "
                    "(smallest primitive p, s = 300, t = --t or 16)")
    a = ap.parse_args()
    import torch
    import paper_1501_06286_b200 as q
    import qmc_workloads as W
    if a.poly:
        # smallest primitive polynomials over F_2 by integer encoding
        p = {8: 285, 10: 1033, 12: 4179, 14: 16427, 16: 65581}[a.poly]
        w = W.custom_poly(a.poly, p, 300, a.t or 16, W.PHI_SHIFT_HALF, seed=a.poly)
    else:
        w = W.config(a.config, t_override=a.t or None)
    plan = q.Plan.from_workload(w)
    A = q.to_device_colmajor(w.A, "cuda")
    X = q.x_empty(plan.N, w.t, "cuda")
    for _ in range(a.steps):
        if w.f is None or a.matmul:
            plan.matmul(A, X)
        else:
            out = plan.mean(A, w.f, w.f_param, X=None if a.nox else X)
            if w.f == W.F_ROWMEAN_RELU:
                plan.finalize(w.f, out, w.t)
    torch.cuda.synchronize()
    print("ok", plan.info)


if __name__ == "__main__":
    main()
