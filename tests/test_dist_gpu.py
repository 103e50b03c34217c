"""The multi-GPU path on one GPU (the only GPU this pool gives a test):

- world size 1 over NCCL: dist.mean_sharded runs the library's qmc_mean on
  the slab, the NCCL all_reduce and qmc_mean_finalize (reading R10/R11);
- two column slabs computed separately (what two ranks compute), combined
  exactly as the all_reduce would (sum of the N partial row sums; the
  zero-padded per-column means) and finalised by qmc_mean_finalize: X and the
  means equal the unsharded call (X bitwise), Q within the R16 bound.
Both are checked against the oracle."""
import os
import socket

import numpy as np
import pytest

import oracle as O
import qmc_workloads as W
from _ref import X_full, col_tolerance

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def qmc():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    import paper_1501_06286_b200 as q
    return q


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _check_means(w, Xo, f, c, got):
    if f == W.F_ROWMEAN_RELU:
        Qo = O.rowmean_relu(Xo)
        assert abs(got - Qo) <= col_tolerance(w).sum() / w.t + 1e-14 * abs(Qo)
    else:
        mo = O.column_means(Xo, f, c)
        fprime = np.exp(Xo).max(axis=0) if f == W.F_EXP else 1.0
        assert np.all(np.abs(got - mo) <= col_tolerance(w) * fprime + 1e-14 * np.abs(mo) + 1e-15)


@pytest.mark.parametrize("f", [W.F_ROWMEAN_RELU, W.F_EXP, W.F_AFFINE])
def test_nccl_world1_mean_sharded(qmc, f):
    import torch
    import torch.distributed as dist
    from paper_1501_06286_b200.dist import mean_sharded
    w = W.custom_lattice(65537, 48, 32, W.PHI_INVNORM_MID, seed=71 + f)
    w.A = np.asfortranarray(w.A * 0.05)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        plan = qmc.Plan.from_workload(w)
        A = qmc.to_device_colmajor(w.A, "cuda")
        X = qmc.x_empty(plan.N, w.t, "cuda")
        out = mean_sharded(plan, A, f, 0.5, w.t, 0, X_local=X)
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()
    Xo = X_full(w)
    got = out.cpu().numpy()
    if f == W.F_AFFINE:
        Xg = X.cpu().numpy() - 0.5
    else:
        Xg = X.cpu().numpy()
    assert np.all(np.abs(Xg - Xo).max(axis=0) <= col_tolerance(w))
    _check_means(w, Xo, f, 0.5, float(got[0]) if f == W.F_ROWMEAN_RELU else got)


@pytest.mark.parametrize("f", [W.F_ROWMEAN_RELU, W.F_EXP])
def test_two_slabs_combined_and_finalized(qmc, f):
    import torch
    from paper_1501_06286_b200.dist import shard_columns
    w = W.custom_lattice(65537, 64, 64, W.PHI_INVNORM_MID, seed=91 + f)
    w.A = np.asfortranarray(w.A * 0.05)
    plan = qmc.Plan.from_workload(w)
    A = qmc.to_device_colmajor(w.A, "cuda")
    Xfull = qmc.x_empty(plan.N, w.t, "cuda")
    ref = plan.mean(A, f, 0.0, X=Xfull).clone()
    X2 = qmc.x_empty(plan.N, w.t, "cuda")
    locals_ = []
    for r in range(2):
        c0, c1 = shard_columns(w.t, 2, r)
        locals_.append((c0, c1, plan.mean(A[:, c0:c1], f, 0.0, X=X2[:, c0:c1]).clone()))
    torch.cuda.synchronize()
    assert torch.equal(Xfull, X2)            # X independent of the slab split, bitwise
    if f == W.F_ROWMEAN_RELU:
        red = locals_[0][2] + locals_[1][2]   # what all_reduce(SUM) of the partial row sums gives
        Q = float(plan.finalize(f, red, w.t).item())
        Qref = float(plan.finalize(f, ref, w.t).item())
        _check_means(w, X_full(w), f, 0.0, Q)
        assert abs(Q - Qref) <= 1e-14 * abs(Qref)
    else:
        full = torch.zeros(w.t, dtype=torch.float64, device="cuda")
        for c0, c1, loc in locals_:
            full[c0:c1] = loc[:c1 - c0]
        out = plan.finalize(f, full, w.t)
        assert torch.equal(out, ref[:w.t])
        _check_means(w, X_full(w), f, 0.0, out.cpu().numpy())


def test_empty_slab_rowsums_are_zero(qmc):
    """A rank with no columns (more ranks than column pairs) contributes zero
    row sums to the all-reduce (advisor finding, round 1)."""
    import torch
    w = W.custom_lattice(257, 20, 4, W.PHI_SHIFT_HALF, seed=5)
    plan = qmc.Plan.from_workload(w)
    A = qmc.to_device_colmajor(w.A, "cuda")
    out = torch.full((plan.N,), float("nan"), dtype=torch.float64, device="cuda")
    plan.mean(A[:, :0], W.F_ROWMEAN_RELU, 0.0, out=out)
    torch.cuda.synchronize()
    assert torch.count_nonzero(out).item() == 0
