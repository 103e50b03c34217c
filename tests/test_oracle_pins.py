"""Pins of the CPU oracle against what the paper and the mathematics fix
(never against the oracle itself, never against the CUDA path).

Each test names the passage or fact it pins; see DESIGN.md §Oracle pins."""
import math
import statistics
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
import qmc_workloads as W
from conftest import load_golden

SMALL_PRIMES = [p for p in range(3, 102) if all(p % d for d in range(2, int(p ** 0.5) + 1))]


# ---------------------------------------------------------------- worked example
def test_worked_example_tables():
    g = load_golden("worked_example_n7.json")
    N = g["N"]
    beta = O.primitive_root(N)
    assert beta == g["beta"]
    assert (beta * g["beta_inv"]) % N == 1
    P = O.power_table(N, beta)
    L = O.log_table(N, P)
    c = O.column_exponents(g["g"], L)
    assert list(c) == g["c"]


def test_worked_example_points_and_factorisation():
    g = load_golden("worked_example_n7.json")
    N, z, beta, c = g["N"], g["g"], g["beta"], g["c"]
    conv = O.lattice_index_matrix(N, z, np.arange(N))
    assert conv.tolist() == g["conventional_numerators"]
    reord = [O.reordered_lattice_point(N, beta, c, n).tolist() for n in range(N)]
    assert reord == g["reordered_numerators"]
    # Z (phi = identity, numerators over 7) and P as printed; Y' = Z P (Eq. ZPa)
    zeta = O.power_table(N, beta).astype(float)              # z_k = {β^k/N}·N
    Z = O.circulant_Z(zeta)
    assert Z.astype(int).tolist() == g["Z_numerators"]
    Psel = O.selection_P(c, N - 1)
    assert Psel.astype(int).tolist() == g["P"]
    assert (Z @ Psel).astype(int).tolist() == g["reordered_numerators"][1:]


def test_worked_example_product_identity_phi():
    """X = Y·a with the paper's printed conventional points, a = (7,7,7)."""
    g = load_golden("worked_example_n7.json")
    N = g["N"]
    tab = O.phi_table(O.PHI_IDENTITY, N)
    idx = O.lattice_index_matrix(N, g["g"], np.arange(N))
    a = np.array([[7.0], [7.0], [7.0]])
    X = O.oracle_X_rows(tab, idx, a)[:, 0]
    printed = np.array(g["conventional_numerators"]).sum(axis=1)   # 7·(n_j/7)
    np.testing.assert_allclose(X, printed, rtol=0, atol=1e-13)
    assert np.round(X).astype(int).tolist() == [0, 9, 11, 6, 15, 10, 12]
    # the same values in the paper's reordered order
    spec = load_golden("spec_examples.json")
    # reordered row i is conventional row n_i; since g_1 = 1 its first
    # coordinate numerator is n_i itself
    order = [0] + [r[0] for r in g["reordered_numerators"][1:]]
    Xr = [X[0]] + [X[n] for n in order[1:]]
    assert np.round(Xr).astype(int).tolist() == spec["matvec_reordered_a777"]
    a1 = np.array([[1.0], [0.0], [0.0]])
    X1 = O.oracle_X_rows(tab, idx, a1)[:, 0] * 7
    assert np.round([X1[0]] + [X1[n] for n in order[1:]]).astype(int).tolist() == \
        spec["matvec_reordered_a100_times7"]


def test_spec_number_theory_examples():
    spec = load_golden("spec_examples.json")
    for b, e, n, want in spec["pow_mod"]:
        P = O.power_table(n, b % n) if O.is_prime(n) else None
        assert pow(b, e, n) == want
        if P is not None and e < n - 1:
            assert P[e] == want                            # repeated multiplication
    for n, want in spec["primitive_root"]:
        assert O.primitive_root(n) == want
    for a, n, want in spec["mod_inverse"]:
        assert (a * want) % n == 1
    # scatter: c = (1,6,2), a -> (a1, a3, 0, 0, 0, a2)
    c = spec["scatter_c"]
    a = np.array([1.5, -2.0, 3.25])
    sc = O.selection_P(c, 6) @ a
    np.testing.assert_array_equal(sc, [1.5, 3.25, 0, 0, 0, -2.0])
    # circulant first column
    Z = O.circulant_Z(O.power_table(7, 3).astype(float))
    assert Z[:, 0].astype(int).tolist() == spec["Z_first_column_times7"]


# ---------------------------------------------------------------- number theory
def _order(b, N):
    k, v = 1, b % N
    while v != 1:
        v = (v * b) % N
        k += 1
    return k


@pytest.mark.parametrize("N", SMALL_PRIMES)
def test_primitive_root_brute_force(N):
    beta = O.primitive_root(N)
    assert _order(beta, N) == N - 1
    assert all(_order(b, N) < N - 1 for b in range(2, beta))   # smallest (R1)
    P = O.power_table(N, beta)
    assert sorted(P.tolist()) == list(range(1, N))        # {β^k} = Z_N^*
    L = O.log_table(N, P)
    for r in range(1, N):                                  # brute-force discrete log
        assert pow(beta, int(L[r]), N) == r
    binv = pow(beta, N - 2, N)
    assert _order(binv, N) == N - 1


def test_config_primitive_roots():
    g = load_golden("primitive_roots.json")
    for Ns, want in g["roots"].items():
        N = int(Ns)
        assert O.primitive_root(N) == want
        qs = O.prime_factors(N - 1)
        assert all(pow(want, (N - 1) // q, N) != 1 for q in qs)
    assert pow(3, 128, 257) == 256 and pow(3, 32768, 65537) == 65536   # Pépin
    assert O.prime_factors(65535) == [3, 5, 17, 257]
    assert O.prime_factors(786432) == [2, 3] and O.prime_factors(40960) == [2, 5]


# ---------------------------------------------------------------- circulant invariance
@pytest.mark.parametrize("N", [5, 7, 11, 13, 31, 61, 101])
@pytest.mark.parametrize("phi", [O.PHI_IDENTITY, O.PHI_SHIFT_HALF, O.PHI_TENT, O.PHI_INVNORM_MID])
def test_circulant_invariance_lattice(N, phi):
    """Rows of the conventional Y, permuted to n_i = β^{-(i)}
    and with row 0 dropped, equal Z·P (Eq. ZPa), where Z is
    built from z_k = φ({β^k/N}).  z covers all of Z_N^* plus
    random repeats (P may then hold several 1s per row, reading R18)."""
    rng = np.random.default_rng(N)
    z = np.concatenate([np.arange(1, N), rng.integers(1, N, size=7)])
    beta = O.primitive_root(N)
    tab = O.phi_table(phi, N)
    Y = O.point_matrix_rows(tab, O.lattice_index_matrix(N, z, np.arange(N)))
    binv = pow(beta, N - 2, N)
    rows = [pow(binv, i, N) for i in range(N - 1)]         # n_i = β^{-i}, paper n = i+1
    Yp = Y[rows, :]
    zeta = tab[O.power_table(N, beta)]
    c = O.column_exponents(z, O.log_table(N, O.power_table(N, beta)))
    np.testing.assert_array_equal(Yp, O.circulant_Z(zeta) @ O.selection_P(c, N - 1))
    # y_0 = (φ(0), ..., φ(0))
    assert np.all(Y[0] == tab[0])


@pytest.mark.parametrize("N", SMALL_PRIMES)
def test_columns_are_permutations(N):
    """Each column of Y is a permutation of {φ(i/N)} (gcd(z_j, N) = 1)."""
    rng = np.random.default_rng(1000 + N)
    z = rng.integers(1, N, size=5)
    idx = O.lattice_index_matrix(N, z, np.arange(N))
    for j in range(len(z)):
        assert sorted(idx[:, j].tolist()) == list(range(N))


# ---------------------------------------------------------------- closed forms on X
@pytest.mark.parametrize("N,s,t", [(257, 300, 64), (65537, 64, 8), (40961, 128, 4)])
def test_column_sum_closed_form(N, s, t):
    """Σ_n {n z/N} = (N-1)/2 for gcd(z,N)=1 (north star; reading R8), so with
    φ = u - 1/2: Σ_n Y[n,j] = -1/2 and Σ_n X[n,k] = -1/2 Σ_j A[j,k]."""
    rng = np.random.default_rng(s)
    z = rng.integers(1, N, size=s)
    A = rng.standard_normal((s, t))
    tab = O.phi_table(O.PHI_SHIFT_HALF, N)
    X = O.oracle_X_full(lambda r: O.lattice_index_matrix(N, z, r), tab, N, A)
    colsum = np.array([math.fsum(X[:, k]) for k in range(t)])
    want = -0.5 * A.sum(axis=0)
    bound = 1e-15 * N * np.abs(A).sum(axis=0) * 0.5 * 8
    assert np.all(np.abs(colsum - want) <= bound + 1e-13)
    # identity φ: Σ_n Y[n,j] = (N-1)/2 exactly
    tabi = O.phi_table(O.PHI_IDENTITY, N)
    Yi = O.point_matrix_rows(tabi, O.lattice_index_matrix(N, z[:3], np.arange(N)))
    for j in range(3):
        assert abs(math.fsum(Yi[:, j]) - (N - 1) / 2) < 1e-9


def test_special_cases():
    N, s = 101, 12
    rng = np.random.default_rng(7)
    z = rng.integers(1, N, size=s)
    tab = O.phi_table(O.PHI_TENT, N)
    idx = O.lattice_index_matrix(N, z, np.arange(N))
    Y = O.point_matrix_rows(tab, idx)
    # A = I gives X = Y
    np.testing.assert_array_equal(O.oracle_X_rows(tab, idx, np.eye(s)), Y)
    # all z equal: X[n,k] = φ({n z/N}) Σ_j A[j,k]
    A = rng.standard_normal((s, 3))
    zz = np.full(s, 17)
    Xz = O.oracle_X_rows(tab, O.lattice_index_matrix(N, zz, np.arange(N)), A)
    want = tab[(np.arange(N) * 17) % N][:, None] * A.sum(axis=0)[None, :]
    np.testing.assert_allclose(Xz, want, rtol=0, atol=1e-13)
    # row 0: φ(0) Σ_j a_j
    X = O.oracle_X_rows(tab, idx, A)
    np.testing.assert_allclose(X[0], tab[0] * A.sum(axis=0), atol=1e-14)


def test_product_within_rounding_bound_exact_rational():
    """φ = identity, integer A: exact rational Y·A vs the fp64 oracle, within
    the fp64 dot-product error bound s·u·Σ|y||a|."""
    N, s, t = 61, 40, 3
    rng = np.random.default_rng(11)
    z = rng.integers(1, N, size=s)
    A = rng.integers(-50, 51, size=(s, t)).astype(float)
    tab = O.phi_table(O.PHI_IDENTITY, N)
    idx = O.lattice_index_matrix(N, z, np.arange(N))
    X = O.oracle_X_rows(tab, idx, A)
    Xf = O.oracle_X_rows_fsum(tab, idx, A)
    for n in range(N):
        for k in range(t):
            exact = sum(Fraction(int((n * int(z[j])) % N), N) * int(A[j, k]) for j in range(s))
            bound = s * 2.0 ** -53 * float(sum(abs(A[:, k]))) * 2
            assert abs(float(exact) - X[n, k]) <= bound
            assert abs(float(exact) - Xf[n, k]) <= 2e-14 * max(1.0, abs(float(exact)))


# ---------------------------------------------------------------- φ = Φ^{-1}(u + 1/(2N))
def test_invnorm_mid_round_trip_and_symmetry():
    """Φ(φ(i/N)) = (2i+1)/(2N) with Φ(x) = erfc(-x/√2)/2 (an independent
    routine), and the symmetry φ(i) = -φ(N-1-i)."""
    for N in (7, 257, 65537):
        tab = O.phi_table(O.PHI_INVNORM_MID, N)
        ii = np.unique(np.linspace(0, N - 1, 200).astype(int))
        for i in ii:
            u = 0.5 * math.erfc(-tab[i] / math.sqrt(2.0))
            assert abs(u - (2 * i + 1) / (2 * N)) <= 1e-14 * max(1.0, (2 * i + 1) / (2 * N)) + 1e-17
        np.testing.assert_allclose(tab, -tab[::-1], rtol=0, atol=1e-12)
    # R6: φ(0) values of configs 2 and 5
    scipy_special = pytest.importorskip("scipy.special")
    for N, want in ((65537, -4.324922404542677), (786433, -4.8441475519550155)):
        v = statistics.NormalDist().inv_cdf(1.0 / (2 * N))
        assert abs(v - want) < 1e-12
        assert abs(v - scipy_special.ndtri(1.0 / (2 * N))) < 1e-12
        assert O.phi_value(O.PHI_INVNORM_MID, 0, N) == v


def test_phi_definitions():
    """tent 1-|2x-1|, identity; shift u-1/2."""
    N = 8
    assert O.phi_value(O.PHI_TENT, 6, N) == 0.5           # tent(3/4) = 1/2
    assert O.phi_value(O.PHI_TENT, 4, N) == 1.0           # tent(1/2) = 1
    assert O.phi_value(O.PHI_TENT, 0, N) == 0.0
    assert O.phi_value(O.PHI_SHIFT_HALF, 0, N) == -0.5
    assert O.phi_value(O.PHI_IDENTITY, 3, N) == 3 / 8
    assert O.phi_value(O.PHI_INVNORM_MID, 3, 7) == 0.0    # Φ^{-1}(1/2)


# ---------------------------------------------------------------- F_2 polynomial lattice
def _gf2_order_of_x(p, D):
    v, k = 2, 1
    while v != 1:
        v <<= 1
        if v >> D:
            v ^= p
        k += 1
        if k > (1 << D):
            return None
    return k


def test_gf2_smallest_primitive_brute_force():
    g = load_golden("gf2_primitive.json")["smallest"]
    for Ds, p in g.items():
        D = int(Ds)
        assert O.gf2_smallest_primitive(D) == p if D <= 8 else O.gf2_is_primitive(p, D)
        assert _gf2_order_of_x(p, D) == (1 << D) - 1      # brute-force order of x
        if D <= 8:   # every smaller candidate of degree D fails by brute force
            for c in range((1 << D) | 1, p, 2):
                assert _gf2_order_of_x(c, D) != (1 << D) - 1
    assert O.gf2_smallest_primitive(16) == 65581


@pytest.mark.parametrize("D", [2, 3, 4, 5, 6, 7, 8])
def test_gf2_vd_index_is_polynomial_quotient(D):
    """v_D(r/p)·2^D is the quotient of r(x)·x^D by p(x) (long division, an
    independent algorithm from the digit recurrence), and is a bijection."""
    p = O.gf2_smallest_primitive(D)
    got = [O.gf2_vd_index(r, p, D) for r in range(1 << D)]
    for r in range(1 << D):
        q, _ = O.gf2_divmod(r << D, p)
        assert got[r] == q
    assert sorted(got) == list(range(1 << D))


def test_gf2_index_matrix_vectorised_matches_scalar():
    for D in (3, 5, 8):
        p = O.gf2_smallest_primitive(D)
        rng = np.random.default_rng(D)
        q = rng.integers(1, 1 << D, size=9)
        rows = np.arange(1 << D)
        M = O.polylattice_index_matrix(D, p, q, rows)
        for n in rows:
            for j, qj in enumerate(q):
                assert M[n, j] == O.gf2_vd_index(O.gf2_mulmod(int(n), int(qj), p), p, D)
        for j in range(len(q)):                          # column = permutation
            assert sorted(M[:, j].tolist()) == list(range(1 << D))
    # D = 16 (config 4): permutation property on 3 columns
    D, p = 16, 65581
    M = O.polylattice_index_matrix(D, p, [1, 12345, 65535], np.arange(1 << D))
    for j in range(3):
        assert np.array_equal(np.sort(M[:, j]), np.arange(1 << D))


@pytest.mark.parametrize("D", [2, 3, 4, 5, 6])
def test_circulant_invariance_poly_all_primitive(D):
    """Remark PAPER.md:456-459: the same factorisation holds for polynomial
    lattices over F_2 with x as generator; exhaustive over every primitive p of
    degree D and every nonzero q (reading R9)."""
    m = (1 << D) - 1
    prims = [p for p in range((1 << D) | 1, 1 << (D + 1), 2) if _gf2_order_of_x(p, D) == m]
    assert prims
    for p in prims:
        q = np.arange(1, m + 1)
        tab = O.phi_table(O.PHI_SHIFT_HALF, 1 << D)
        Y = O.point_matrix_rows(tab, O.polylattice_index_matrix(D, p, q, np.arange(1 << D)))
        P = O.gf2_power_table(p, D)
        assert sorted(P.tolist()) == list(range(1, m + 1))
        L = O.gf2_log_table(D, P)
        # n_i = x^{-i}
        rows = [int(P[(-i) % m]) for i in range(m)]
        zeta = np.array([tab[O.gf2_vd_index(int(P[k]), p, D)] for k in range(m)])
        c = L[q] + 1
        np.testing.assert_array_equal(Y[rows, :], O.circulant_Z(zeta) @ O.selection_P(c, m))


def test_lattice_and_poly_index_maps_agree_small():
    """Both maps k -> β^k mod N and k -> x^k mod p are bijections onto the
    nonzero residues whose inverse is the brute-force discrete log (R9)."""
    for N in SMALL_PRIMES[:12]:
        beta = O.primitive_root(N)
        P = O.power_table(N, beta)
        L = O.log_table(N, P)
        for k in range(N - 1):
            assert L[pow(beta, k, N)] == k
    for D in range(2, 9):
        p = O.gf2_smallest_primitive(D)
        P = O.gf2_power_table(p, D)
        L = O.gf2_log_table(D, P)
        v = 1
        for k in range((1 << D) - 1):
            assert L[v] == k
            v = O.gf2_mulmod(v, 2, p)


# ---------------------------------------------------------------- inputs module
def test_ar1_cholesky_closed_form_matches_lapack():
    A = W.ar1_upper_cholesky(256, 102.4)
    i = np.arange(256)
    Sigma = np.exp(-np.abs(i[:, None] - i[None, :]) / 102.4)
    np.testing.assert_allclose(A.T @ A, Sigma, atol=1e-13)
    np.testing.assert_allclose(A, np.linalg.cholesky(Sigma).T, atol=1e-12)


def test_config3_means_closed_form():
    """mean_n(1 + X[n,k]) = 1 + S_φ/N·colsum_k = 1 - colsum_k/(2N) for φ = u-1/2
    (reading R8), on two full columns of config 3."""
    N, s = 40961, 4096
    rng = np.random.default_rng(3)
    z = rng.integers(1, N, size=s)
    A = W.kl_sine_matrix(s, 65536, 2.0, 1.0, cols=[0, 40000])
    tab = O.phi_table(O.PHI_SHIFT_HALF, N)
    X = O.oracle_X_full(lambda r: O.lattice_index_matrix(N, z, r), tab, N, A, block=2048)
    means = O.column_means(X, O.F_AFFINE, 1.0)
    want = 1.0 - A.sum(axis=0) / (2 * N)
    np.testing.assert_allclose(means, want, rtol=0, atol=1e-13)


# ---------------------------------------------------------------- randomised QMC (R28)
def test_replicate_estimate_pins():
    """The replicate mean and standard error against the statistics module
    (fmean, sample stdev / sqrt(R)), the R = 2 closed form |Q0 - Q1| / 2,
    equal replicates (error 0) and R = 1 (NaN)."""
    rng = np.random.default_rng(28)
    Q = rng.standard_normal((7, 5))
    mean, err = O.replicate_estimate(Q)
    for k in range(5):
        col = [float(v) for v in Q[:, k]]
        assert math.isclose(mean[k], statistics.fmean(col), rel_tol=1e-15)
        assert math.isclose(err[k], statistics.stdev(col) / math.sqrt(7), rel_tol=1e-14)
    m2, e2 = O.replicate_estimate(Q[:2])
    np.testing.assert_allclose(e2, np.abs(Q[0] - Q[1]) / 2, rtol=1e-15)
    np.testing.assert_allclose(m2, (Q[0] + Q[1]) / 2, rtol=1e-15)
    m3, e3 = O.replicate_estimate(np.tile(Q[:1], (4, 1)))
    np.testing.assert_array_equal(m3, Q[0])
    np.testing.assert_array_equal(e3, np.zeros(5))
    m1, e1 = O.replicate_estimate(Q[:1])
    np.testing.assert_array_equal(m1, Q[0])
    assert np.all(np.isnan(e1))


# ---------------------------------------------------------------- the fused reductions
def test_rowmean_relu_pins():
    """Config 2's scalar Q = (1/N) Σ_n max(0, (1/t) Σ_k X[n,k]) (reading R10):
    (a) the paper's worked example (N = 7, z = (1,5,3),
    φ = id) with columns a = (7,7,7) and (-1,0,0): X = (0,9,11,6,15,10,12) and
    -(0,1,...,6)/7, every row sum >= 0, so Q = (1/14)(63 - 3) = 30/7;
    (b) A >= 0, φ = id: no clipping, Q = S_φ/(N t)·Σ A = (N-1)/(2 N t)·Σ A
    (reading R8); (c) A <= 0: every row sum <= 0, Q = 0."""
    g = load_golden("worked_example_n7.json")
    tab = O.phi_table(O.PHI_IDENTITY, 7)
    idx = O.lattice_index_matrix(7, g["g"], np.arange(7))
    X = O.oracle_X_rows(tab, idx, np.array([[7.0, -1.0], [7.0, 0.0], [7.0, 0.0]]))
    assert abs(O.rowmean_relu(X) - 30.0 / 7.0) <= 1e-15 * 30
    N, s, t = 101, 9, 5
    rng = np.random.default_rng(11)
    z = rng.integers(1, N, size=s)
    A = rng.uniform(0.0, 1.0, size=(s, t))
    tabN = O.phi_table(O.PHI_IDENTITY, N)
    X = O.oracle_X_full(lambda r: O.lattice_index_matrix(N, z, r), tabN, N, A)
    want = (N - 1) / (2 * N * t) * math.fsum(A.ravel())
    assert abs(O.rowmean_relu(X) - want) <= 1e-14 * want
    Xneg = O.oracle_X_full(lambda r: O.lattice_index_matrix(N, z, r), tabN, N, -A)
    assert O.rowmean_relu(Xneg) == 0.0


def test_exp_mean_pins():
    """Config 5's mean of exp(X) (PAPER.md:60-62 with f = exp): (a) A = 0 gives
    1; (b) all z_j equal to 1 and φ = id: X[n,k] = (n/N)·c_k with c_k = Σ_j
    A[j,k], so the mean is the geometric sum (1/N)(e^{c} - 1)/(e^{c/N} - 1)."""
    N, s, t = 257, 4, 6
    tab = O.phi_table(O.PHI_IDENTITY, N)
    z = np.ones(s, dtype=np.int64)
    fn = lambda r: O.lattice_index_matrix(N, z, r)  # noqa: E731
    X0 = O.oracle_X_full(fn, tab, N, np.zeros((s, t)))
    np.testing.assert_array_equal(O.column_means(X0, O.F_EXP), np.ones(t))
    A = np.random.default_rng(12).uniform(-2.0, 2.0, size=(s, t))
    X = O.oracle_X_full(fn, tab, N, A)
    c = A.sum(axis=0)
    want = (np.expm1(c) / np.expm1(c / N)) / N
    np.testing.assert_allclose(O.column_means(X, O.F_EXP), want, rtol=1e-13, atol=0)


# ---------------------------------------------------------------- Korobov p-set
@pytest.mark.parametrize("K", [5, 7, 11, 13, 31])
def test_pset_columns_are_uniform_multisets(K):
    """Every column of the p-set hits each nonzero residue exactly K-1 times:
    for fixed g, n -> n·g^j is a bijection of Z_K^* (PAPER.md:478-489), so the
    column sums of Y are (K-1)·Σ_{i=1}^{K-1} φ(i/K) (closed form)."""
    s = 6
    idx = O.pset_index_matrix(K, s, np.arange((K - 1) ** 2))
    for j in range(s):
        counts = np.bincount(idx[:, j], minlength=K)
        assert counts[0] == 0 and np.all(counts[1:] == K - 1)
    tab = O.phi_table(O.PHI_SHIFT_HALF, K)
    Y = O.point_matrix_rows(tab, idx)
    S = math.fsum(tab[1:])
    np.testing.assert_allclose(Y.sum(axis=0), (K - 1) * S, rtol=0, atol=1e-12 * K * K)


@pytest.mark.parametrize("K", [5, 7, 11, 13, 31, 61])
def test_pset_paper_reordering(K):
    """The paper's substitution n -> β^{-(n-1)}, g -> β^{(g-1)} turns x_{n,g}
    into ({β^{c_{g,j} - n}/K})_j with c_{g,j} = (j-1)(g-1)+1 mod (K-1)
    (PAPER.md:510-524): checked point by point against the conventional
    definition, exhaustively over n, g."""
    s = 5
    beta = O.primitive_root(K)
    binv = pow(beta, K - 2, K)
    for g in range(1, K):
        for n in range(1, K):
            nc = pow(binv, n - 1, K)            # conventional n
            gc = pow(beta, g - 1, K)            # conventional g
            r = (gc - 1) * (K - 1) + (nc - 1)
            conv = O.pset_index_matrix(K, s, [r])[0]
            assert np.array_equal(conv, O.pset_reordered_point(K, beta, s, n, g))


@pytest.mark.parametrize("K", [7, 11, 13])
def test_pset_blocks_are_circulant_with_one_Z(K):
    """Y'_g = Z·P_g for every block with the same circulant Z:
    all K-1 blocks share one spectrum, only the column map c_{g,·} changes."""
    s = K + 2                                    # repeats in c_{g,·} (reading R18)
    beta = O.primitive_root(K)
    tab = O.phi_table(O.PHI_TENT, K)
    Z = O.circulant_Z(tab[O.power_table(K, beta)])
    for g in range(1, K):
        Yp = np.array([tab[O.pset_reordered_point(K, beta, s, n, g)] for n in range(1, K)])
        np.testing.assert_array_equal(Yp, Z @ O.selection_P(O.pset_c(K, s, g), K - 1))


def test_pset_block_is_korobov_lattice():
    """Block g (rows (g-1)(K-1) .. g(K-1)-1) is the Korobov rank-1 lattice with
    z = (1, g, g^2, ...) mod K without its row n = 0."""
    K, s = 31, 8
    idx = O.pset_index_matrix(K, s, np.arange((K - 1) ** 2))
    for g in (1, 2, 3, 17, 30):
        z = [pow(g, j, K) for j in range(s)]
        blk = idx[(g - 1) * (K - 1): g * (K - 1)]
        np.testing.assert_array_equal(blk, O.lattice_index_matrix(K, z, np.arange(1, K)))


# ---------------------------------------------------------------- Experiment 2 (NEXT #2)
def test_pde1d_stiffness_closed_forms_by_quadrature():
    """The paper's closed forms of a_{j,k,l} = ∫ j^{-3/2} sin(2πjx) φ'_k φ'_l dx
    (PAPER.md:862-868), as restated by qmc_workloads.pde1d_uniform_matrix,
    against adaptive quadrature of the integral itself (φ'_k = ±M on the two
    elements of node k)."""
    from scipy.integrate import quad
    M, s = 9, 5
    A, d0, e0 = W.pde1d_uniform_matrix(M, s)
    K = M - 1
    assert d0 == 4 * M and e0 == -2 * M          # ∫ 2 φ'_k φ'_l: 2·2M, 2·(-M)
    for j in range(1, s + 1):
        psi = lambda x, j=j: j ** -1.5 * np.sin(2 * np.pi * j * x)  # noqa: E731
        for k in range(1, K + 1):                 # (k, k): M^2 ∫ over [x_{k-1}, x_{k+1}]
            v = M * M * quad(psi, (k - 1) / M, (k + 1) / M, epsabs=1e-13)[0]
            assert abs(A[j - 1, k - 1] - v) <= 1e-9 * max(1.0, abs(v))
        for k in range(1, K):                     # (k, k+1): -M^2 ∫ over [x_k, x_{k+1}]
            v = -M * M * quad(psi, k / M, (k + 1) / M, epsabs=1e-13)[0]
            assert abs(A[j - 1, K + k - 1] - v) <= 1e-9 * max(1.0, abs(v))


def test_pde1d_solve_closed_form_constant_coefficient():
    """y = 0 (no perturbation): B = 2M·tridiag(-1, 2, -1) and ĝ = 1, whose
    solution is û_k = k(K+1-k) / (4M) (discrete Poisson, closed form)."""
    M = 12
    K = M - 1
    X = np.zeros((3, 2 * K - 1))
    ubar = O.pde1d_fe_mean(X, 4.0 * M, -2.0 * M)
    k = np.arange(1, K + 1)
    np.testing.assert_allclose(ubar, k * (K + 1 - k) / (4.0 * M), rtol=1e-13)


def test_pde1d_solve_matches_dense():
    """The banded solves of the oracle against dense np.linalg.solve."""
    rng = np.random.default_rng(7)
    M, N = 10, 4
    K = M - 1
    X = 0.3 * rng.standard_normal((N, 2 * K - 1)) * M
    d0, e0 = 4.0 * M, -2.0 * M
    U = []
    for n in range(N):
        B = np.diag(d0 + X[n, :K]) + np.diag(e0 + X[n, K:], 1) + np.diag(e0 + X[n, K:], -1)
        U.append(np.linalg.solve(B, np.ones(K)))
    np.testing.assert_allclose(O.pde1d_fe_mean(X, d0, e0), np.mean(U, axis=0), rtol=1e-12)


# ---------------------------------------------------------------- Experiment 3 (NEXT #3)
def test_pde1d_lognormal_constant_coefficient_closed_form():
    """Θ = 0: a = e^{ψ0} everywhere, B̂ = e^{ψ0}·M·tridiag(-1, 2, -1), whose
    solution with ĝ = 1 is û_k = k(K+1-k) / (2 e^{ψ0} M)."""
    M = 10
    K = M - 1
    ubar = O.pde1d_lognormal_fe_mean(np.zeros((2, M)), 2.0)
    k = np.arange(1, K + 1)
    np.testing.assert_allclose(ubar, k * (K + 1 - k) / (2 * np.exp(2.0) * M), rtol=1e-13)


def test_pde1d_lognormal_midpoint_assembly_exact_for_affine_coefficient():
    """When a(x) is affine on every element the one-point midpoint rule of
    reading R25 is exact, so the oracle's assembled B̂ must equal the exact
    stiffness ∫ a φ'_k φ'_l dx (adaptive quadrature): checked through the
    solution ū for a(x) = 1 + x (log a at the midpoints supplied as Θ)."""
    from scipy.integrate import quad
    M = 8
    K = M - 1
    mids = (np.arange(M) + 0.5) / M
    Theta = np.log(1.0 + mids)[None, :] - 2.0          # exp(2 + Θ) = 1 + x at the midpoints
    ubar = O.pde1d_lognormal_fe_mean(Theta, 2.0)
    a = lambda x: 1.0 + x  # noqa: E731
    B = np.zeros((K, K))
    for k in range(1, K + 1):
        B[k - 1, k - 1] = M * M * quad(a, (k - 1) / M, (k + 1) / M)[0]
        if k < K:
            B[k - 1, k] = B[k, k - 1] = -M * M * quad(a, k / M, (k + 1) / M)[0]
    np.testing.assert_allclose(ubar, np.linalg.solve(B, np.ones(K)), rtol=1e-12)


def test_pde1d_lognormal_psi_matrix():
    """Ψ[j-1, i] = j^{-3/2} sin(2π j (i + 1/2)/M) (R25)."""
    Psi, psi0 = W.pde1d_lognormal_matrix(6, 4)
    assert psi0 == 2.0 and Psi.shape == (4, 6)
    assert abs(Psi[2, 1] - 3 ** -1.5 * math.sin(2 * math.pi * 3 * 1.5 / 6)) < 1e-15


# ---------------------------------------------------------------- equal shift (NEXT #4)
@pytest.mark.parametrize("N,delta", [(7, 0.3), (13, 0.9), (101, 0.123456789), (257, 1e-3)])
def test_shifted_column_sums_closed_form(N, delta):
    """u - 1/2 on a rule shifted by Δ: every column is a permutation of the
    shifted grid, so its sum is Σ_i (i/N + Δ) - #wraps - N/2 with
    #wraps = #{i : i/N + Δ >= 1} = N - ceil(N(1 - Δ)) (closed form)."""
    rng = np.random.default_rng(N)
    z = rng.integers(1, N, size=5)
    tab = O.phi_table_shifted(O.PHI_SHIFT_HALF, N, delta)
    Y = O.point_matrix_rows(tab, O.lattice_index_matrix(N, z, np.arange(N)))
    wraps = N - math.ceil(N * (1 - delta))
    closed = (N - 1) / 2 + N * delta - wraps - N / 2
    np.testing.assert_allclose(Y.sum(axis=0), closed, rtol=0, atol=1e-12 * N)


def test_shift_half_cell_is_the_midpoint_rule():
    """Δ = 1/(2N) with φ = identity gives the midpoints (2i+1)/(2N)."""
    N = 31
    tab = O.phi_table_shifted(O.PHI_IDENTITY, N, 1.0 / (2 * N))
    np.testing.assert_allclose(tab, (2 * np.arange(N) + 1) / (2 * N), rtol=0, atol=1e-16)


@pytest.mark.parametrize("N", [11, 61])
def test_shift_by_grid_step_permutes_rows(N):
    """Δ = k/N: column j of the shifted Y is column j of the unshifted Y with
    row n moved to n - k·z_j^{-1} mod N ({(n z_j + k)/N} = {(n + k z_j^{-1}) z_j / N})."""
    rng = np.random.default_rng(N + 5)
    z = rng.integers(1, N, size=4)
    k = 3
    Ys = O.point_matrix_rows(O.phi_table_shifted(O.PHI_TENT, N, k / N),
                             O.lattice_index_matrix(N, z, np.arange(N)))
    Y = O.point_matrix_rows(O.phi_table(O.PHI_TENT, N), O.lattice_index_matrix(N, z, np.arange(N)))
    for j, zj in enumerate(z):
        zinv = pow(int(zj), N - 2, N)
        perm = (np.arange(N) + k * zinv) % N
        np.testing.assert_allclose(Ys[:, j], Y[perm, j], rtol=0, atol=1e-15)


# ---------------------------------------------------------------- CBC (NEXT #4)
@pytest.mark.parametrize("N", [7, 101, 1021])
def test_cbc_error_one_dimension_closed_form(N):
    """d = 1, z = 1: Σ_i B_2(i/N) = 1/(6N), so e² = γ 2π²/(6N²) = γ π²/(3N²)."""
    g = 0.7
    assert abs(O.cbc_error(N, [1], g) - g * math.pi ** 2 / (3 * N * N)) <= 1e-14


def test_cbc_criterion_symmetry_exact():
    """B_2(1 - u) = B_2(u), so the criterion of z and N - z coincide exactly:
    the candidate range 1..(N-1)/2 loses nothing (exact rationals)."""
    N = 13
    rng = np.random.default_rng(1)
    p = [Fraction(int(v), 7) for v in rng.integers(1, 20, size=N)]
    def crit(z):
        return sum(p[n] * (Fraction(n * z % N, N) ** 2 - Fraction(n * z % N, N) + Fraction(1, 6)) for n in range(1, N))
    for z in range(1, N):
        assert crit(z) == crit(N - z)


@pytest.mark.parametrize("N,s", [(13, 4), (17, 5), (31, 4)])
def test_cbc_choices_are_exact_minimisers(N, s):
    """Each z_d of the oracle's CBC attains, in exact rational arithmetic, the
    minimum of the step-d criterion, for rational weights γ_j = 1/j².  (Exact
    ties occur: from step 2 the criterion is invariant under z -> z^{-1} mod N
    for the z_1 = 1 prefix, e.g. 12 and 13 for N = 31; any minimiser is a
    valid CBC choice.)"""
    gam = [Fraction(1, (j + 1) ** 2) for j in range(s)]
    z = O.cbc_lattice(N, s, [float(g) for g in gam])
    assert z[0] == 1
    B = [Fraction(i, N) ** 2 - Fraction(i, N) + Fraction(1, 6) for i in range(N)]
    pi2 = Fraction(math.pi ** 2)   # the update uses the float 2π²; its exact value cancels in the argmin
    p = [Fraction(1)] * N
    for d in range(s):
        if d > 0:
            crits = {zc: sum(p[n] * B[n * zc % N] for n in range(1, N)) for zc in range(1, (N - 1) // 2 + 1)}
            best = min(crits.values())
            assert crits[int(z[d])] == best
        p = [p[n] * (1 + gam[d] * 2 * pi2 * B[n * int(z[d]) % N]) for n in range(N)]
