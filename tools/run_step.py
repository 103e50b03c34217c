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
    a = ap.parse_args()
    import torch
    import paper_1501_06286_b200 as q
    import qmc_workloads as W
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
