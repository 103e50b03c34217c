"""Parity of the CUDA path (through the C ABI) against the CPU oracle.

Bar (north_star, reading R16): per column k,
    max_n |X_gpu[n,k] - X_oracle[n,k]| <= 1e-11 · ||A[:,k]||_1 · max|φ|;
plan tables (generator, P, L, e) bit-exact.  Inputs are the seeded
workloads of qmc_workloads; expected values come only from oracle/.
"""
import numpy as np
import pytest

import oracle as O
import qmc_workloads as W
from _ref import X_full, X_rows, col_tolerance, index_fn, phi_tab, sample_rows

pytestmark = pytest.mark.gpu

PHIS = [W.PHI_IDENTITY, W.PHI_SHIFT_HALF, W.PHI_TENT, W.PHI_INVNORM_MID]


@pytest.fixture(scope="module")
def qmc():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    import paper_1501_06286_b200 as q
    return q


def dev_X(q, w, t=None):
    import torch
    plan = q.Plan.from_workload(w)
    A = q.to_device_colmajor(w.A if t is None else w.A[:, :t], "cuda")
    X = plan.matmul(A)
    torch.cuda.synchronize()
    return plan, X.cpu().numpy()


def check_X(w, Xg_s, Xo, cols=None):
    """Xg_s, Xo: the same rows and columns (cols names them for the tolerance)."""
    tol = col_tolerance(w, cols=cols)
    assert Xg_s.shape == Xo.shape
    err = np.abs(Xg_s - Xo).max(axis=0)
    assert np.all(np.isfinite(Xg_s))
    bad = np.nonzero(err > tol)[0]
    assert bad.size == 0, f"columns {bad[:5]} err {err[bad[:5]]} tol {tol[bad[:5]]}"
    return float((err / tol).max())


# ------------------------------------------------------------------ plan tables
def _oracle_tables(w):
    if w.family == "poly":
        P = O.gf2_power_table(w.p, w.D)
        L = O.gf2_log_table(w.D, P)
        gen = 2
    else:
        gen = O.primitive_root(w.N)
        P = O.power_table(w.N, gen)
        L = O.log_table(w.N, P)
    e = O.column_exponents(w.z, L) - 1
    return gen, P, L, e


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_plan_tables_bit_exact(qmc, c):
    w = W.config(c, t_override=2)
    plan = qmc.Plan.from_workload(w)
    gen, P, L, e, zeta = plan.tables()
    og, oP, oL, oe = _oracle_tables(w)
    assert gen == og
    np.testing.assert_array_equal(P, oP)
    np.testing.assert_array_equal(L, oL)
    np.testing.assert_array_equal(e, oe)
    tab = phi_tab(w)
    idx = oP if w.family == "lattice" else np.array([O.gf2_vd_index(int(r), w.p, w.D) for r in oP])
    np.testing.assert_allclose(zeta, tab[idx], rtol=1e-14, atol=1e-15)


def test_worked_example_gpu(qmc):
    """N=7, g=(1,5,3), φ = identity, a = (7,7,7) -> (0,9,11,6,15,10,12)."""
    import torch
    plan = qmc.Plan.lattice(7, [1, 5, 3], W.PHI_IDENTITY)
    gen, P, L, e, _ = plan.tables()
    assert gen == 3 and list(e + 1) == [1, 6, 2]
    A = qmc.to_device_colmajor(np.array([[7.0, 1.0], [7.0, 0.0], [7.0, 0.0]]), "cuda")
    X = plan.matmul(A).cpu().numpy()
    np.testing.assert_allclose(X[:, 0], [0, 9, 11, 6, 15, 10, 12], atol=1e-13)
    np.testing.assert_allclose(X[:, 1] * 7, [0, 1, 2, 3, 4, 5, 6], atol=1e-13)
    torch.cuda.synchronize()


# ------------------------------------------------------------------ small cases, full X
SMALL = [(7, 3, 2), (11, 20, 5), (13, 4, 1), (31, 100, 7), (61, 17, 8), (101, 300, 9), (257, 300, 64),
         (1021, 50, 6), (4001, 400, 10), (16001, 200, 4)]


@pytest.mark.parametrize("N,s,t", SMALL)
@pytest.mark.parametrize("phi", PHIS)
def test_small_lattice_full(qmc, N, s, t, phi):
    w = W.custom_lattice(N, s, t, phi, seed=N * 10 + phi)
    plan, Xg = dev_X(qmc, w)
    check_X(w, Xg, X_full(w))


@pytest.mark.parametrize("D", [2, 3, 4, 5, 6, 7, 8, 10, 12])
@pytest.mark.parametrize("phi", [W.PHI_SHIFT_HALF, W.PHI_INVNORM_MID])
def test_small_poly_full(qmc, D, phi):
    p = O.gf2_smallest_primitive(D)
    w = W.custom_poly(D, p, s=3 * D + 5, t=5, phi=phi, seed=D)
    plan, Xg = dev_X(qmc, w)
    check_X(w, Xg, X_full(w))


def test_config1_full(qmc):
    w = W.config(1)
    plan, Xg = dev_X(qmc, w)
    assert plan.info["L"] == 256 and plan.info["L1"] == 1
    ratio = check_X(w, Xg, X_full(w))
    assert ratio < 1e-2


# ------------------------------------------------------------------ edge cases
def test_edge_cases(qmc):
    import torch
    q = qmc
    # s = 1, t = 1 (odd, single column), all z equal, repeated z (s > m)
    for (N, z) in [(13, [5]), (13, [4] * 9), (11, list(range(1, 11)) * 3)]:
        w = W.custom_lattice(N, len(z), 1, W.PHI_TENT, seed=3)
        w.z = np.array(z, dtype=np.int64)
        plan, Xg = dev_X(q, w)
        check_X(w, Xg, X_full(w))
    # t = 0 is a no-op
    plan = q.Plan.lattice(13, [1, 2], W.PHI_SHIFT_HALF)
    A0 = torch.empty((0, 2), dtype=torch.float64, device="cuda").t()
    X0 = plan.matmul(A0)
    assert X0.shape == (13, 0)
    # lda > s and ldx > t: padding columns of X untouched; odd ldx (scalar stores)
    w = W.custom_lattice(101, 30, 6, W.PHI_SHIFT_HALF, seed=9)
    plan = q.Plan.from_workload(w)
    Abig = torch.zeros((6, 40), dtype=torch.float64, device="cuda")
    Abig[:, :30] = torch.from_numpy(np.ascontiguousarray(w.A.T)).cuda()
    A = Abig.t()[:30]                       # (30, 6), lda = 40
    for ldx in (16, 9):
        Xbig = torch.full((101, ldx), 7.5, dtype=torch.float64, device="cuda")
        X = Xbig[:, :6]                     # (101, 6), row-major, ldx
        plan.matmul(A, X)
        Xh = Xbig.cpu().numpy()
        assert np.all(Xh[:, 6:] == 7.5)
        check_X(w, Xh[:, :6], X_full(w))


def test_invalid_arguments(qmc):
    from paper_1501_06286_b200 import _abi as abi
    with pytest.raises(abi.QMCError) as e:
        qmc.Plan.lattice(15, [1, 2], W.PHI_IDENTITY)
    assert e.value.code == -1
    for z in ([0, 1], [1, 13]):
        with pytest.raises(abi.QMCError) as e:
            qmc.Plan.lattice(13, z, W.PHI_IDENTITY)
        assert e.value.code == -2
    with pytest.raises(abi.QMCError) as e:
        qmc.Plan.lattice(13, [1], 7)
    assert e.value.code == -5
    with pytest.raises(abi.QMCError) as e:     # x^4+x^2+1 = (x^2+x+1)^2 not primitive
        qmc.Plan.poly(4, 0b10101, [1, 2], W.PHI_IDENTITY)
    assert e.value.code == -3


def test_deterministic_and_shard_invariant(qmc):
    """Two runs are bitwise identical; computing columns [0,t) in two slabs
    with an even boundary gives bitwise the same X (columns are packed in
    pairs (2i, 2i+1), so an even split keeps every pair)."""
    import torch
    w = W.config(2, t_override=64)
    plan = qmc.Plan.from_workload(w)
    A = qmc.to_device_colmajor(w.A, "cuda")
    X1 = plan.matmul(A).clone()
    X2 = plan.matmul(A).clone()
    assert torch.equal(X1, X2)
    Xs = qmc.x_empty(plan.N, 64, "cuda")
    plan.matmul(A[:, :24], Xs[:, :24])
    plan.matmul(A[:, 24:], Xs[:, 24:])
    assert torch.equal(X1, Xs)


# ------------------------------------------------------------------ the five configs
def test_config2_full_and_rowmean_relu(qmc):
    """Config 2 at full size in bench.py's launch configuration (qmc_mean,
    f = ROWMEAN_RELU, X written): full X and the scalar Q (reading R10)."""
    import torch
    w = W.config(2)
    plan = qmc.Plan.from_workload(w)
    A = qmc.to_device_colmajor(w.A, "cuda")
    X = qmc.x_empty(plan.N, w.t, "cuda")
    rs = plan.mean(A, W.F_ROWMEAN_RELU, 0.0, X=X)
    Q = plan.finalize(W.F_ROWMEAN_RELU, rs, w.t)
    Xg = X.cpu().numpy()
    Xo = X_full(w, block=8192)
    check_X(w, Xg, Xo)
    Qo = O.rowmean_relu(Xo)
    # |ΔQ| <= (1/t) Σ_k tol_k + 1e-14·Q  (reading R16)
    tolQ = col_tolerance(w).sum() / w.t + 1e-14 * abs(Qo)
    assert abs(float(Q.item()) - Qo) <= tolQ
    rs_o = O.row_sums(Xo)
    np.testing.assert_allclose(rs.cpu().numpy(), rs_o, rtol=0, atol=col_tolerance(w).sum())
    torch.cuda.synchronize()


def test_config3_sampled(qmc):
    """Config 3 full size (qmc_mean, f = AFFINE c=1, X receives 1+X): 260 sampled rows
    × all 65536 columns, two full columns and their means (closed form R8 too)."""
    import torch
    w = W.config(3)
    plan = qmc.Plan.from_workload(w)
    A = qmc.to_device_colmajor(w.A, "cuda")
    X = qmc.x_empty(plan.N, w.t, "cuda")
    means = plan.mean(A, W.F_AFFINE, 1.0, X=X)
    rows = sample_rows(w.N, 256, seed=3)
    idx = torch.from_numpy(rows).cuda()
    Xs = X.index_select(0, idx).cpu().numpy()
    Xo = 1.0 + X_rows(w, rows)
    check_X(w, Xs, Xo)
    cols = [0, 1, 33333, w.t - 1]
    Xc = X[:, cols].cpu().numpy()
    Xoc = 1.0 + X_full(w, cols=cols, block=2048)
    check_X(w, Xc, Xoc, cols=cols)
    m_g = means.cpu().numpy()
    m_o = O.column_means(Xoc, O.F_IDENTITY)
    np.testing.assert_allclose(m_g[cols], m_o, rtol=0, atol=1e-13)
    closed = 1.0 - w.A.sum(axis=0) / (2 * w.N)
    np.testing.assert_allclose(m_g, closed, rtol=0, atol=1e-12)


def test_config4_sampled(qmc):
    """Config 4 (F_2 polynomial lattice, zero-padded 2^17 correlation)."""
    import torch
    w = W.config(4)
    plan = qmc.Plan.from_workload(w)
    assert plan.info["L"] == 131072
    A = qmc.to_device_colmajor(w.A, "cuda")
    X = plan.matmul(A)
    rows = sample_rows(w.N, 512, seed=4)
    Xs = X.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
    check_X(w, Xs, X_rows(w, rows))
    cols = [0, 1, 1000, 1999]
    check_X(w, X[:, cols].cpu().numpy(), X_full(w, cols=cols), cols=cols)


def test_config5_sampled(qmc):
    """Config 5 full size (qmc_mean, f = EXP, X written): sampled rows × all
    columns and one full column pair with its mean of exp(X)."""
    import torch
    w = W.config(5)
    plan = qmc.Plan.from_workload(w)
    A = qmc.to_device_colmajor(w.A, "cuda")
    X = qmc.x_empty(plan.N, w.t, "cuda")
    means = plan.mean(A, W.F_EXP, 0.0, X=X)
    rows = sample_rows(w.N, 256, seed=5)
    Xs = X.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
    check_X(w, Xs, X_rows(w, rows))
    cols = [0, 8191]
    Xc = X[:, cols].cpu().numpy()
    Xoc = X_full(w, cols=cols, block=8192)
    check_X(w, Xc, Xoc, cols=cols)
    m_o = O.column_means(Xoc, O.F_EXP)
    m_g = means.cpu().numpy()[cols]
    # Δ mean(exp X) <= tol · max exp(X) + 1e-14 · mean  (reading R16)
    tol = col_tolerance(w, cols=cols) * np.exp(Xoc).max(axis=0) + 1e-14 * np.abs(m_o)
    assert np.all(np.abs(m_g - m_o) <= tol)


# ------------------------------------------------------------------ fused epilogues on every K2 path
# (N, s, t, batch pairs or None): L1 = 16 pipelined K2 (t a multiple of 32),
# partial pair groups (t = 30, 6: k_cols_x), L1 = 10 (N = 40961), the
# two-stage column pass L1 = 96 (N = 786433), and several batches on two
# internal streams (batch 16 of 32 pairs); zero-padded lengths on the
# pipelined two-stage pass: N = 3079 (L = 6400 = 25·256, L1 = 5·5) and
# N = 65539 (L = 163840 = 20·8192, L1 = 2·10).
MEAN_CASES = [(65537, 64, 32, None), (65537, 64, 30, None), (40961, 50, 32, None), (65537, 40, 64, 16),
              (786433, 16, 6, None), (786433, 16, 32, None), (3079, 50, 32, None), (65539, 40, 32, None),
              # L1 = 96 takes 16-pair tiles: two whole groups (t = 64), and 24 pairs (t = 48: not whole
              # 16-pair groups, the general column pass)
              (786433, 16, 64, None), (786433, 16, 48, None),
              # one-row plans (the fused k_small): rows of 256 with s > m and odd t; rows of 32 (2 threads)
              (257, 300, 7, None), (13, 5, 4, None)]


@pytest.mark.parametrize("N,s,t,bp", MEAN_CASES)
@pytest.mark.parametrize("f", [W.F_IDENTITY, W.F_AFFINE, W.F_EXP, W.F_ROWMEAN_RELU])
def test_means_every_k2_path(qmc, monkeypatch, N, s, t, bp, f):
    import torch
    if bp:
        monkeypatch.setenv("QMC_BATCH_PAIRS", str(bp))
    phi = W.PHI_INVNORM_MID if f == W.F_EXP else W.PHI_SHIFT_HALF
    w = W.custom_lattice(N, s, t, phi, seed=N + s + t + f)
    plan = qmc.Plan.from_workload(w)
    A = qmc.to_device_colmajor(w.A, "cuda")
    X = qmc.x_empty(plan.N, t, "cuda")
    c = 0.75
    out = plan.mean(A, f, c, X=X)
    torch.cuda.synchronize()
    Xo = X_full(w)
    tol = col_tolerance(w)
    if f == W.F_AFFINE:
        check_X(w, X.cpu().numpy() - c, Xo)
    else:
        check_X(w, X.cpu().numpy(), Xo)
    if f == W.F_ROWMEAN_RELU:
        Q = float(plan.finalize(f, out, t).item())
        Qo = O.rowmean_relu(Xo)
        assert abs(Q - Qo) <= tol.sum() / t + 1e-14 * abs(Qo)
        np.testing.assert_allclose(out.cpu().numpy(), O.row_sums(Xo), rtol=0, atol=tol.sum())
    else:
        mo = O.column_means(Xo, f, c)
        mg = out.cpu().numpy()
        # reading R16: |Δmean| <= tol·max|f'| + 1e-14·mean|f|
        fprime = np.exp(Xo).max(axis=0) if f == W.F_EXP else 1.0
        assert np.all(np.abs(mg - mo) <= tol * fprime + 1e-14 * np.abs(mo) + 1e-15)


def test_mean_host_entry(qmc):
    """qmc_mean_host: host A in, device X, host result (the e2e path bench.py times)."""
    import torch
    from paper_1501_06286_b200 import _abi as abi
    w = W.custom_lattice(65537, 48, 32, W.PHI_SHIFT_HALF, seed=11)
    plan = qmc.Plan.from_workload(w)
    A_host = torch.from_numpy(np.ascontiguousarray(w.A.T)).pin_memory()   # col-major s×t, lda = s
    A_dev = torch.empty_like(A_host, device="cuda")
    X = qmc.x_empty(plan.N, w.t, "cuda")
    out_host = torch.empty(w.t, dtype=torch.float64).pin_memory()
    out_dev = torch.empty(max(plan.N, w.t), dtype=torch.float64, device="cuda")
    ws = plan.call_workspace(w.t, W.F_AFFINE)
    abi.qmc_mean_host(plan.handle, A_host, w.s, w.t, W.F_AFFINE, 1.0, out_host, A_dev, X, w.t, out_dev, ws,
                      ws.numel(), torch.cuda.current_stream().cuda_stream)
    Xo = X_full(w)
    check_X(w, X.cpu().numpy() - 1.0, Xo)
    np.testing.assert_allclose(out_host.numpy(), O.column_means(Xo, O.F_AFFINE, 1.0), rtol=0, atol=1e-13)


# ------------------------------------------------------------------ Korobov p-set (NEXT #1)
@pytest.mark.parametrize("K,s,t", [(5, 3, 1), (7, 9, 6), (31, 40, 33), (61, 20, 8), (257, 64, 16)])
@pytest.mark.parametrize("phi", [W.PHI_SHIFT_HALF, W.PHI_INVNORM_MID])
def test_korobov_pset(qmc, K, s, t, phi):
    """X = Y·A for the union of all Korobov lattices, N = (K-1)^2 rows in the
    conventional (g, n) order, against the oracle's plain definition."""
    import torch
    rng = np.random.default_rng(K * 100 + s + t)
    A = rng.standard_normal((s, t))
    ps = qmc.KorobovPSet(K, s, phi)
    X = ps.matmul(qmc.to_device_colmajor(A, "cuda"))
    torch.cuda.synchronize()
    tab = O.phi_table(phi, K)
    Xo = O.point_matrix_rows(tab, O.pset_index_matrix(K, s, np.arange((K - 1) ** 2))) @ A
    tol = 1e-11 * np.abs(A).sum(axis=0) * np.abs(tab).max()
    err = np.abs(X.cpu().numpy() - Xo).max(axis=0)
    assert X.shape == ((K - 1) ** 2, t)
    assert np.all(err <= tol), (err / tol).max()
    # the one-plan batched launch (qmc_pset_matmul) against one plan per block
    Xb = ps.matmul(qmc.to_device_colmajor(A, "cuda"), per_block=True)
    torch.cuda.synchronize()
    assert np.all(np.abs(Xb.cpu().numpy() - Xo).max(axis=0) <= tol)


@pytest.mark.parametrize("K,s,t", [(1021, 32, 8), (4001, 16, 4)])
def test_korobov_pset_large(qmc, K, s, t):
    """K = 1021 (N = 1,040,400 points; padded row of 2048, one launch for all
    1020 blocks) and K = 4001 (rows split L1 = 2: one plan per block), on
    sampled rows against the oracle's plain definition."""
    import torch
    rng = np.random.default_rng(K + s)
    A = rng.standard_normal((s, t))
    ps = qmc.KorobovPSet(K, s, W.PHI_SHIFT_HALF)
    X = ps.matmul(qmc.to_device_colmajor(A, "cuda"))
    torch.cuda.synchronize()
    rows = np.unique(np.concatenate([sample_rows((K - 1) ** 2, 400, seed=K), [0, K - 2, K - 1, (K - 1) ** 2 - 1]]))
    tab = O.phi_table(W.PHI_SHIFT_HALF, K)
    Xo = O.point_matrix_rows(tab, O.pset_index_matrix(K, s, rows)) @ A
    Xs = X.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
    tol = 1e-11 * np.abs(A).sum(axis=0) * np.abs(tab).max()
    assert np.all(np.abs(Xs - Xo).max(axis=0) <= tol)


# ------------------------------------------------------------------ Experiment 2 (NEXT #2)
@pytest.mark.parametrize("N,M,s", [(67, 134, 134), (127, 254, 254), (257, 514, 514), (1021, 32, 32)])
def test_pde1d_uniform_mean(qmc, N, M, s):
    """Mean FE coefficients of the paper's uniform ODE:
    fast X = Y·A, N Thomas solves and the mean on the GPU, against the oracle
    (direct product, LAPACK banded solves, fsum).  Tolerance: the R16 bound on
    X propagates through B^{-1} (condition number ≈ (M/π)^2); rtol 1e-8 is
    far above the observed error and far below any meaningful difference."""
    import torch
    w = W.pde1d_uniform(N, M, s, seed=N)
    pde = qmc.UniformPDE1D(w.N, w.z, w.A, w.extra["d0"], w.extra["e0"])
    ubar = pde.solve_mean().cpu().numpy()
    torch.cuda.synchronize()
    Xo = X_full(w)
    uo = O.pde1d_fe_mean(Xo, w.extra["d0"], w.extra["e0"])
    np.testing.assert_allclose(ubar, uo, rtol=1e-8, atol=0)


# ------------------------------------------------------------------ Experiment 3 (NEXT #3)
@pytest.mark.parametrize("N,M,s", [(67, 134, 134), (257, 514, 514), (1021, 33, 33), (127, 40, 254)])
def test_pde1d_lognormal_mean(qmc, N, M, s):
    """Mean FE coefficients of the paper's log-normal ODE:
    fast Θ = Y·Ψ, on-the-fly exp / midpoint assembly, N Thomas solves and the
    mean on the GPU, against the oracle (direct product, LAPACK banded
    solves).  rtol 1e-8 as for Experiment 2 (the exp adds a factor max a)."""
    import torch
    w = W.pde1d_lognormal(N, M, s, seed=N)
    pde = qmc.LognormalPDE1D(w.N, w.z, w.A, w.extra["psi0"])
    ubar = pde.solve_mean().cpu().numpy()
    torch.cuda.synchronize()
    Theta = X_full(w)
    uo = O.pde1d_lognormal_fe_mean(Theta, w.extra["psi0"])
    np.testing.assert_allclose(ubar, uo, rtol=1e-8, atol=0)


# ------------------------------------------------------------------ equal shift (NEXT #4)
@pytest.mark.parametrize("N,s,t,delta", [(13, 7, 3, 0.37), (257, 300, 64, 0.25), (65537, 64, 32, 0.0123456789),
                                         (4001, 100, 9, 0.999)])
@pytest.mark.parametrize("phi", [W.PHI_SHIFT_HALF, W.PHI_INVNORM_MID, W.PHI_TENT])
def test_shifted_lattice(qmc, N, s, t, delta, phi):
    import torch
    w = W.custom_lattice(N, s, t, phi, seed=N + t)
    plan = qmc.Plan.lattice(N, w.z, phi, delta=delta)
    X = plan.matmul(qmc.to_device_colmajor(w.A, "cuda")).cpu().numpy()
    torch.cuda.synchronize()
    tab = O.phi_table_shifted(phi, N, delta)
    Xo = O.oracle_X_full(index_fn(w), tab, N, w.A)
    tol = 1e-11 * np.abs(w.A).sum(axis=0) * np.abs(tab).max()
    assert np.all(np.abs(X - Xo).max(axis=0) <= tol)


def test_shifted_replicate_means(qmc):
    """R = 4 equally shifted replicates of config 3's affine mean (c + X), one
    base plan + qmc_plan_shift views: each replicate's fused column means
    against the oracle's, and the library's replicate mean / standard error
    (qmc_replicate_mean) against the oracle's estimate (R28)."""
    import torch
    N, s, t = 4001, 64, 8
    w = W.custom_lattice(N, s, t, W.PHI_SHIFT_HALF, seed=9)
    deltas = [0.1, 0.35, 0.6, 0.85]
    R, avg, err = qmc.shifted_means(N, w.z, W.PHI_SHIFT_HALF, qmc.to_device_colmajor(w.A, "cuda"),
                                    W.F_AFFINE, 1.0, deltas, return_stderr=True)
    torch.cuda.synchronize()
    Qo = []
    for r, d in enumerate(deltas):
        Xo = O.oracle_X_full(index_fn(w), O.phi_table_shifted(W.PHI_SHIFT_HALF, N, d), N, w.A)
        Qo.append(O.column_means(Xo, O.F_AFFINE, 1.0))
        np.testing.assert_allclose(R[r].cpu().numpy(), Qo[-1], rtol=0, atol=1e-12)
    mo, eo = O.replicate_estimate(np.array(Qo))
    np.testing.assert_allclose(avg.cpu().numpy(), mo, rtol=0, atol=1e-12)
    # the error is a difference of near-equal means: its absolute error is the means' (1e-12)
    np.testing.assert_allclose(err.cpu().numpy(), eo, rtol=0, atol=2e-12)
    # the fixed-order kernel equals the same-order sum of the replicates exactly
    Rh = R.cpu().numpy()
    np.testing.assert_array_equal(avg.cpu().numpy(), (((Rh[0] + Rh[1]) + Rh[2]) + Rh[3]) / 4)


@pytest.mark.parametrize("N,s,t,phi", [(13, 7, 3, W.PHI_SHIFT_HALF), (65537, 64, 32, W.PHI_INVNORM_MID),
                                       (4001, 100, 9, W.PHI_TENT)])
def test_plan_shift_matches_shifted_plan(qmc, N, s, t, phi):
    """A qmc_plan_shift view of an unshifted plan computes exactly (bitwise)
    what a plan created with the same Δ computes (same kernels, same tables),
    and against the oracle; the base plan is unchanged after the view."""
    import torch
    w = W.custom_lattice(N, s, t, phi, seed=N + 3 * t)
    A = qmc.to_device_colmajor(w.A, "cuda")
    base = qmc.Plan.lattice(N, w.z, phi)
    X0 = base.matmul(A).clone()
    for delta in (0.25, 0.7123):
        view = qmc.ShiftedPlan(base, delta)
        Xv = view.matmul(A).cpu().numpy()
        Xs = qmc.Plan.lattice(N, w.z, phi, delta=delta).matmul(A).cpu().numpy()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(Xv, Xs)
        tab = O.phi_table_shifted(phi, N, delta)
        Xo = O.oracle_X_full(index_fn(w), tab, N, w.A)
        tol = 1e-11 * np.abs(w.A).sum(axis=0) * np.abs(tab).max()
        assert np.all(np.abs(Xv - Xo).max(axis=0) <= tol)
    np.testing.assert_array_equal(base.matmul(A).cpu().numpy(), X0.cpu().numpy())


def test_replicate_mean_edges(qmc):
    """qmc_replicate_mean: R = 1 (stderr NaN), t = 0 (no-op), strided rows,
    bad dimensions rejected."""
    import torch
    Q = torch.tensor(np.random.default_rng(5).standard_normal((3, 10)), device="cuda")
    m, e = qmc.replicate_mean(Q[:1])
    assert torch.equal(m, Q[0]) and bool(torch.isnan(e).all())
    m, e = qmc.replicate_mean(Q[:, :4])   # rows strided by 10
    mo, eo = O.replicate_estimate(Q[:, :4].cpu().numpy())
    np.testing.assert_allclose(m.cpu().numpy(), mo, rtol=1e-15)
    np.testing.assert_allclose(e.cpu().numpy(), eo, rtol=1e-13)
    qmc._abi.qmc_replicate_mean(Q, 3, 0, 0, Q)   # t = 0: no-op
    with pytest.raises(qmc.QMCError):
        qmc._abi.qmc_replicate_mean(Q, 0, 4, 4, Q)
    with pytest.raises(qmc.QMCError):
        qmc._abi.qmc_replicate_mean(Q, 2, 4, 3, Q)


# ------------------------------------------------------------------ CBC (NEXT #4)
@pytest.mark.parametrize("N,s", [(101, 6), (1021, 12), (4001, 8)])
def test_cbc_lattice_gpu(qmc, N, s):
    """GPU fast CBC (qmc_matmul with φ = B_2 + qmc_cbc_step) is a valid CBC
    run: along the GPU's own choices, every z_d attains the minimum of the
    oracle's plain step-d criterion (to fp tolerance; exact ties z <-> z^{-1}
    make several choices valid), z_1 = 1, and the worst-case error matches the
    oracle's CBC vector's when the vectors coincide."""
    gam = [0.9 ** (j + 1) for j in range(s)]
    zg = qmc.cbc_lattice(N, s, gam)
    assert zg[0] == 1 and np.all((zg >= 1) & (zg <= (N - 1) // 2))
    B = O.cbc_criterion_table(N)
    n = np.arange(N, dtype=np.int64)
    cand = np.arange(1, (N - 1) // 2 + 1, dtype=np.int64)
    p = np.ones(N)
    for d in range(s):
        if d > 0:
            crit = B[(n[1:, None] * cand[None, :]) % N].T @ p[1:]
            assert crit[zg[d] - 1] <= crit.min() + 1e-12 * np.abs(crit).max()
        p = p * (1.0 + gam[d] * 2 * np.pi ** 2 * B[(n * int(zg[d])) % N])
    zo = O.cbc_lattice(N, s, gam)
    if np.array_equal(zo, zg):
        assert abs(O.cbc_error(N, zg, gam) - O.cbc_error(N, zo, gam)) == 0.0


# ------------------------------------------------------------------ K1 scatter-input orders
# (N, s, t): sparse buckets (s << L2), one chunk; dense (s = L2 = 4096, four
# chunks); dense rows of 8192 (s = L2, config 5's shape); heavy collisions
# (~15 entries per bucket: continuation rounds or the bucket-order fallback).
K1_ORDER_CASES = [(4001, 400, 10), (40961, 4096, 4), (786433, 8192, 2), (65537, 60000, 2)]


@pytest.mark.parametrize("N,s,t", K1_ORDER_CASES)
@pytest.mark.parametrize("heads", [False, True])
def test_k1_scatter_orders(qmc, monkeypatch, N, s, t, heads):
    """Both layouts of the row kernel's scatter input (plan.cu
    k1_balanced_order and the bucket-order fallback, forced by QMC_K1_HEADS)
    give X within the bar, on sampled rows and on one full column pair."""
    import torch
    if heads:
        monkeypatch.setenv("QMC_K1_HEADS", "1")
    w = W.custom_lattice(N, s, t, W.PHI_SHIFT_HALF, seed=N + s)
    plan = qmc.Plan.from_workload(w)
    if heads:
        assert plan.info["k1_order"] == 0 and plan.info["k1_slots"] == s
    elif s <= 8192:
        assert plan.info["k1_order"] == 1
    A = qmc.to_device_colmajor(w.A, "cuda")
    X = plan.matmul(A)
    rows = sample_rows(w.N, 128, seed=s)
    Xs = X.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
    check_X(w, Xs, X_rows(w, rows))
    if N * s <= 65537 * 60000:
        cols = [0, 1]
        check_X(w, X[:, cols].cpu().numpy(), X_full(w, cols=cols, block=8192), cols=cols)


@pytest.mark.parametrize("N,s,t", [(4001, 400, 10), (40961, 4096, 4)])
def test_k0_variants_bitwise(qmc, monkeypatch, N, s, t):
    """K0 through shared memory (s <= 4096) and the direct gather
    (QMC_PACK_GATHER) produce the same packed input, so X is bitwise equal."""
    import torch
    w = W.custom_lattice(N, s, t, W.PHI_SHIFT_HALF, seed=N + 3 * s)
    plan = qmc.Plan.from_workload(w)
    A = qmc.to_device_colmajor(w.A, "cuda")
    X1 = plan.matmul(A).clone()
    monkeypatch.setenv("QMC_PACK_GATHER", "1")        # read at plan creation
    plan2 = qmc.Plan.from_workload(w)
    X2 = plan2.matmul(A).clone()
    torch.cuda.synchronize()
    assert torch.equal(X1, X2)


def test_fused_reductions_closed_forms_gpu(qmc):
    """The fused means against closed forms (no oracle in the loop): equal z,
    φ = id -> mean exp(X[:,k]) = (1/N)(e^c - 1)/(e^{c/N} - 1), c = Σ_j A[j,k];
    A >= 0, φ = id -> Q = (N-1)/(2 N t)·Σ A (reading R8, no clipping)."""
    import torch
    N, s, t = 65537, 8, 32
    rng = np.random.default_rng(21)
    A = rng.uniform(-2.0, 2.0, size=(s, t))
    plan = qmc.Plan.lattice(N, np.ones(s, dtype=np.int64), W.PHI_IDENTITY)
    m = plan.mean(qmc.to_device_colmajor(A, "cuda"), W.F_EXP, 0.0).cpu().numpy()
    c = A.sum(axis=0)
    np.testing.assert_allclose(m, np.expm1(c) / np.expm1(c / N) / N, rtol=1e-12, atol=0)
    z = rng.integers(1, N, size=s)
    Ap = rng.uniform(0.0, 1.0, size=(s, t))
    plan2 = qmc.Plan.lattice(N, z, W.PHI_IDENTITY)
    rs = plan2.mean(qmc.to_device_colmajor(Ap, "cuda"), W.F_ROWMEAN_RELU, 0.0)
    Q = float(plan2.finalize(W.F_ROWMEAN_RELU, rs, t).item())
    want = (N - 1) / (2 * N * t) * Ap.sum()
    assert abs(Q - want) <= 1e-12 * want
    torch.cuda.synchronize()


@pytest.mark.parametrize("N,t", [(7681, 6), (40961, 4), (65537, 4), (25601, 4)])
def test_dense_input_all_generators(qmc, N, t):
    """The all-generators plan (z = 1..N-1, s = m, as in the CBC search) takes
    the dense first pass (k_pack_dense + k_dense_cols / k_dense_cols2 for
    L1 = 25 = 5·5 at N = 25601; plan info k1_order 2):
    X against the oracle on sampled rows (all rows for N = 7681), and against
    the bucket-order path (QMC_K1_HEADS) within the bar."""
    import os
    import torch
    s = N - 1
    w = W.custom_lattice(N, s, t, W.PHI_SHIFT_HALF, seed=N)
    w.z = np.arange(1, N, dtype=np.int64)
    plan = qmc.Plan.from_workload(w)
    assert plan.info["k1_order"] == 2 and plan.info["k1_slots"] == plan.info["L"]
    A = qmc.to_device_colmajor(w.A, "cuda")
    X = plan.matmul(A)
    if N <= 8000:
        check_X(w, X.cpu().numpy(), X_full(w))
    else:
        rows = sample_rows(w.N, 64, seed=N)
        Xs = X.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
        check_X(w, Xs, X_rows(w, rows))
    os.environ["QMC_K1_HEADS"] = "1"
    try:
        plan_h = qmc.Plan.from_workload(w)
    finally:
        del os.environ["QMC_K1_HEADS"]
    assert plan_h.info["k1_order"] == 0
    Xh = plan_h.matmul(A)
    check_X(w, X.cpu().numpy(), Xh.cpu().numpy())


@pytest.mark.parametrize("N,s,t", [(7681, 15360, 4), (65537, 70000, 2)])
def test_dense_input_with_collisions(qmc, monkeypatch, N, s, t):
    """Dense first pass with repeated columns (s > m, i.i.d. z): k_pack_dense
    sums the entries of each e in j order; X on sampled rows against the
    oracle and against the sparse path (QMC_NO_DENSE) within the bar."""
    import torch
    w = W.custom_lattice(N, s, t, W.PHI_SHIFT_HALF, seed=N + s)
    plan = qmc.Plan.from_workload(w)
    assert plan.info["k1_order"] == 2
    A = qmc.to_device_colmajor(w.A, "cuda")
    X = plan.matmul(A)
    rows = sample_rows(w.N, 64, seed=s)
    Xs = X.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy()
    check_X(w, Xs, X_rows(w, rows))
    monkeypatch.setenv("QMC_NO_DENSE", "1")
    plan_s = qmc.Plan.from_workload(w)
    assert plan_s.info["k1_order"] != 2
    check_X(w, X.cpu().numpy(), plan_s.matmul(A).cpu().numpy())


# ------------------------------------------------------------------ K1 staged first rounds, green mode
@pytest.mark.parametrize("N,s,t", [(40961, 4096, 4), (786433, 8192, 2)])
def test_k1_staged_rounds_bitwise(qmc, monkeypatch, N, s, t):
    """The direct scatter with its first rounds staged in shared memory
    (k1_srn, the default where room is left beside the row), with one staged
    round (QMC_K1_SR=1) and with none (QMC_K1_NOHYB) sums the same slots in
    the same order, so X is bitwise equal; and within the bar of the oracle."""
    import torch
    w = W.custom_lattice(N, s, t, W.PHI_INVNORM_MID, seed=N + 7 * s)
    A = qmc.to_device_colmajor(w.A, "cuda")
    plan = qmc.Plan.from_workload(w)
    nt = plan.info["L2"] // 16
    assert plan.info["k1_order"] == 1 and plan.info["k1_staged_slots"] >= nt
    assert plan.info["k1_staged_slots"] % nt == 0
    X0 = plan.matmul(A).clone()
    monkeypatch.setenv("QMC_K1_SR", "1")
    p1 = qmc.Plan.from_workload(w)
    assert p1.info["k1_staged_slots"] == nt
    X1 = p1.matmul(A).clone()
    monkeypatch.delenv("QMC_K1_SR")
    monkeypatch.setenv("QMC_K1_NOHYB", "1")
    p2 = qmc.Plan.from_workload(w)
    assert p2.info["k1_staged_slots"] == 0
    X2 = p2.matmul(A).clone()
    torch.cuda.synchronize()
    assert torch.equal(X0, X1) and torch.equal(X0, X2)
    rows = sample_rows(w.N, 128, seed=s + 1)
    check_X(w, X0.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy(), X_rows(w, rows))


@pytest.mark.parametrize("f", [W.F_EXP, W.F_ROWMEAN_RELU])
def test_green_partitions(qmc, monkeypatch, f):
    """Green mode (QMC_GREEN): K0/K1 on one SM partition and K2 on the other,
    batches handed over by per-set events; X and the fused reductions equal
    the single-stream results bitwise (same kernels, same order per column)
    across several batches, and the partition sizes add up to the device."""
    import torch
    N, s, t = 65537, 512, 96
    monkeypatch.setenv("QMC_BATCH_PAIRS", "16")  # three batches: both sets, reuse after the hand-off
    phi = W.PHI_INVNORM_MID if f == W.F_EXP else W.PHI_SHIFT_HALF
    w = W.custom_lattice(N, s, t, phi, seed=11 + f)
    if f == W.F_EXP:
        w.A = np.asfortranarray(w.A * 0.05)
    A = qmc.to_device_colmajor(w.A, "cuda")
    plan = qmc.Plan.from_workload(w)
    X0 = qmc.x_empty(plan.N, t, "cuda")
    m0 = plan.mean(A, f, 0.0, X=X0).clone()
    monkeypatch.setenv("QMC_GREEN", "24")
    pg = qmc.Plan.from_workload(w)
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    assert 24 <= pg.info["green_k2_sms"] < nsm
    X1 = qmc.x_empty(pg.N, t, "cuda")
    m1 = pg.mean(A, f, 0.0, X=X1).clone()
    torch.cuda.synchronize()
    assert torch.equal(X0, X1) and torch.equal(m0, m1)
    rows = sample_rows(w.N, 64, seed=3)
    check_X(w, X1.index_select(0, torch.from_numpy(rows).cuda()).cpu().numpy(), X_rows(w, rows))


def test_single_stream_batch_invariant(qmc, monkeypatch):
    """Plans with L1 > 16 run device calls on the caller's stream in one large
    batch (config 5: 1024 pairs); X is bitwise the same as with small batches
    (every pair's K1/K2 arithmetic is independent of the batching), the exp
    means agree to rounding, and the host entry (two streams, the two-stream
    batch) gives bitwise the same X out of the same workspace."""
    import torch
    N, s, t = 786433, 64, 40
    w = W.custom_lattice(N, s, t, W.PHI_INVNORM_MID, seed=7)
    A = qmc.to_device_colmajor(w.A, "cuda")
    res = {}
    for bp in (None, "4"):
        if bp:
            monkeypatch.setenv("QMC_BATCH_PAIRS", bp)
        plan = qmc.Plan.from_workload(w)
        assert plan.info["L1"] > 16
        X = qmc.x_empty(plan.N, t, "cuda")
        m = plan.mean(A, W.F_EXP, 0.0, X=X)
        torch.cuda.synchronize()
        res[bp] = (X.clone(), m.clone(), plan)
    monkeypatch.delenv("QMC_BATCH_PAIRS")
    from paper_1501_06286_b200 import _abi as abi
    (X1, m1, plan1), (X2, m2, _) = res[None], res["4"]
    assert plan1.info["batch_pairs"] >= 1024
    assert torch.equal(X1, X2)
    torch.testing.assert_close(m1, m2, rtol=1e-14, atol=0)
    # host entry on the large-batch plan: its own (two-stream) layout fits the
    # workspace the size query returns
    A_pin = torch.from_numpy(np.ascontiguousarray(w.A.T)).pin_memory()
    A_dev = torch.empty(A_pin.shape, dtype=torch.float64, device="cuda")
    Xh = qmc.x_empty(plan1.N, t, "cuda")
    out_pin = torch.empty(t, dtype=torch.float64).pin_memory()
    out_dev = torch.empty(max(plan1.N, t), dtype=torch.float64, device="cuda")
    ws = plan1.call_workspace(t, W.F_EXP)
    abi.qmc_mean_host(plan1.handle, A_pin, s, t, W.F_EXP, 0.0, out_pin, A_dev, Xh, t, out_dev, ws,
                      ws.numel(), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(X1, Xh)
    torch.testing.assert_close(out_pin.to("cuda"), m1, rtol=1e-14, atol=0)
