"""Vendor comparator ("Comparator (out of product)"): the same
circulant correlation done with torch.fft (cuFFT Z2Z) at the same length L,
batched over the same column pairs, next to this build's qmc_matmul.

Not part of the product path: it only reads the plan's tables (qmc_plan_tables)
and runs stock torch ops. It checks that the cuFFT result agrees with the
library's X on every entry (so both compute the same thing), then times:
  * cuFFT core:   fft(a') * W -> ifft  (the part the hand-written K1/K2 replace)
  * cuFFT full:   scatter (index_add) + core + un-permutation gather into X
  * qmc_matmul:   the library call (K0 + K1 + K2), X written
Usage: python tools/cufft_compare.py [--config 2] [--iters 20]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    import torch
    import paper_1501_06286_b200 as q
    import qmc_workloads as W

    w = W.config(a.config)
    dev = "cuda"
    plan = q.Plan.from_workload(w)
    gen, P, L, e, zeta = plan.tables()
    m, N, t = plan.m, plan.N, w.t
    if L.shape[0] != N or t % 2:
        raise SystemExit("comparator supports the lattice/F2 configs with even t")
    e_d = torch.as_tensor(e.astype("int64"), device=dev)
    zeta_d = torch.as_tensor(zeta, device=dev, dtype=torch.float64)
    Wspec = torch.conj(torch.fft.fft(zeta_d.to(torch.complex128)))  # DFT(zeta)* ; ifft carries 1/m
    Lh = torch.as_tensor(L.astype("int64"), device=dev)
    r = torch.remainder(m - Lh[1:], m)  # reordered row of conventional row n >= 1

    A = q.to_device_colmajor(w.A, dev)  # (s, t) column-major
    Ac = torch.complex(A[:, 0::2].contiguous(), A[:, 1::2].contiguous())  # (s, t/2)
    AcT = Ac.t().contiguous()  # (t/2, s)
    npairs = t // 2
    ap_ = torch.zeros(npairs, m, dtype=torch.complex128, device=dev)
    Xc = torch.empty(N, t, dtype=torch.float64, device=dev)

    def core(x):
        return torch.fft.ifft(torch.fft.fft(x, dim=1) * Wspec, dim=1)

    def full():
        ap_.zero_()
        ap_.index_add_(1, e_d, AcT)
        B = core(ap_)
        Bs = B[:, r]  # (t/2, N-1)
        Xc[1:, 0::2] = Bs.real.t()
        Xc[1:, 1::2] = Bs.imag.t()
        Xc[0] = float(zeta0) * A.sum(dim=0)
        return Xc

    # phi(0): X[0,k] = phi(0) * sum_j A[j,k]; take it from the library's own X row 0.
    Xq = plan.matmul(A)
    torch.cuda.synchronize()
    colsum = A.sum(dim=0)
    k0 = int(torch.argmax(colsum.abs()))
    zeta0 = (Xq[0, k0] / colsum[k0]).item()

    Xf = full()
    torch.cuda.synchronize()
    diff = (Xf - Xq).abs().max().item()
    scale = Xq.abs().max().item()

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        s, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(a.iters):
            fn()
        en.record()
        torch.cuda.synchronize()
        return s.elapsed_time(en) / a.iters

    Xout = q.x_empty(N, t, dev)
    res = {
        "config": a.config, "L_cufft": m, "pairs": npairs,
        "max_abs_diff_vs_qmc": diff, "max_abs_X": scale,
        "ms_cufft_core": timeit(lambda: core(ap_)),
        "ms_cufft_full": timeit(full),
        "ms_qmc_matmul": timeit(lambda: plan.matmul(A, Xout)),
    }
    res["speedup_vs_cufft_full"] = res["ms_cufft_full"] / res["ms_qmc_matmul"]
    res["speedup_vs_cufft_core"] = res["ms_cufft_core"] / res["ms_qmc_matmul"]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
