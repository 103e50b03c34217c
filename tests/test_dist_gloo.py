"""Multi-rank host logic on CPU (gloo, world_size 2): column sharding,
the zero-padded allreduce of per-column means and the row-sum allreduce of
config 2's functional.  The per-rank local results come from the oracle (the
GPU kernels are covered by the -m gpu parity tests); what is checked here is
that the sharded pipeline reproduces the unsharded oracle result."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import qmc_workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _local_results(w, c0, c1, f, f_param, A=None):
    tab = O.phi_table(w.phi, w.N)
    A = w.A[:, c0:c1] if A is None else A
    X = O.oracle_X_full(lambda r: O.lattice_index_matrix(w.N, w.z, r), tab, w.N, A)
    if f == W.F_ROWMEAN_RELU:
        return X, torch.from_numpy(O.row_sums(X))
    return X, torch.from_numpy(O.column_means(X, f, f_param))


def _worker(rank, world, port, w, f, f_param, q, weak=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1501_06286_b200.dist import combine_means, shard_columns
    if weak:  # bench.py --scaling weak: every rank the full t columns, block `rank` of world·t
        c0, c1, t_total = rank * w.t, (rank + 1) * w.t, world * w.t
        X, local = _local_results(w, 0, w.t, f, f_param)
    else:
        c0, c1 = shard_columns(w.t, world, rank)
        t_total = w.t
        X, local = _local_results(w, c0, c1, f, f_param)
    red = combine_means(local, f, t_total, c0)
    if f == W.F_ROWMEAN_RELU:
        # finalize semantics of qmc_mean_finalize (reading R10), on the host
        r = red.numpy()
        out = math.fsum(max(0.0, x / t_total) for x in r) / w.N
    else:
        out = red.numpy().copy()
    q.put((rank, c0, c1, X, out))
    dist.barrier()
    dist.destroy_process_group()


def _run(world, w, f, f_param, weak=False):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, w, f, f_param, q, weak)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return sorted(res, key=lambda x: x[0])


def test_shard_columns_even_pairs():
    from paper_1501_06286_b200.dist import shard_columns
    for t in (1, 2, 7, 64, 1000, 1024, 2000, 65536):
        for world in (1, 2, 3, 4, 8):
            cuts = [shard_columns(t, world, r) for r in range(world)]
            assert cuts[0][0] == 0 and cuts[-1][1] == t
            for (a0, a1), (b0, b1) in zip(cuts, cuts[1:]):
                assert a1 == b0
            for c0, c1 in cuts:
                assert c1 == c0 or (c0 % 2 == 0 and ((c1 - c0) % 2 == 0 or c1 == t))
            pairs = [(c1 - c0 + 1) // 2 for c0, c1 in cuts]
            assert max(pairs) - min(pairs) <= 1


@pytest.mark.parametrize("f,f_param", [(W.F_ROWMEAN_RELU, 0.0), (W.F_AFFINE, 1.0), (W.F_EXP, 0.0)])
def test_gloo_world2_matches_unsharded(f, f_param):
    w = W.custom_lattice(257, 40, 10, W.PHI_INVNORM_MID, seed=17)
    w.A = np.asfortranarray(w.A * 0.05)
    res = _run(2, w, f, f_param)
    Xs = np.concatenate([r[3] for r in res], axis=1)
    tab = O.phi_table(w.phi, w.N)
    Xfull = O.oracle_X_full(lambda r: O.lattice_index_matrix(w.N, w.z, r), tab, w.N, w.A)
    np.testing.assert_allclose(Xs, Xfull, rtol=0, atol=1e-12)
    if f == W.F_ROWMEAN_RELU:
        want = O.rowmean_relu(Xfull)
        for r in res:
            assert abs(r[4] - want) <= 1e-14 * max(1.0, abs(want))
    else:
        want = O.column_means(Xfull, f, f_param)
        for r in res:
            np.testing.assert_allclose(r[4], want, rtol=0, atol=1e-14)
        assert np.array_equal(res[0][4], res[1][4])   # every rank holds the same vector


@pytest.mark.parametrize("f,f_param", [(W.F_ROWMEAN_RELU, 0.0), (W.F_EXP, 0.0)])
def test_gloo_world2_weak_blocks(f, f_param):
    """Weak scaling (bench.py --scaling weak): each rank runs all t columns as
    its block of a 2t-column problem [A, A]; the combined result equals the
    unsharded oracle on [A, A]."""
    w = W.custom_lattice(257, 40, 10, W.PHI_INVNORM_MID, seed=19)
    w.A = np.asfortranarray(w.A * 0.05)
    res = _run(2, w, f, f_param, weak=True)
    A2 = np.concatenate([w.A, w.A], axis=1)
    tab = O.phi_table(w.phi, w.N)
    Xfull = O.oracle_X_full(lambda r: O.lattice_index_matrix(w.N, w.z, r), tab, w.N, A2)
    np.testing.assert_allclose(np.concatenate([r[3] for r in res], axis=1), Xfull, rtol=0, atol=1e-12)
    if f == W.F_ROWMEAN_RELU:
        want = O.rowmean_relu(Xfull)
        for r in res:
            assert abs(r[4] - want) <= 1e-14 * max(1.0, abs(want))
    else:
        want = O.column_means(Xfull, f, f_param)
        for r in res:
            np.testing.assert_allclose(r[4], want, rtol=0, atol=1e-14)
