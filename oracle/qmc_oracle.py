"""Plain, slow, obviously-correct CPU oracle (fp64).  TEST INFRASTRUCTURE ONLY.

Every function cites the PAPER.md passage it follows (file:line, section /
equation).  Where the paper is silent the reading is the one recorded in
DESIGN.md §Readings (R1..R20, taken from SURVEY.md §8(c)).

Contents
  number theory (lattice)   : is_prime, prime_factors, primitive_root,
                              power_table, log_table, column_exponents
  number theory (F_2[x])    : gf2_mul, gf2_mod, gf2_divmod, gf2_mulmod,
                              gf2_is_primitive, gf2_power_table,
                              gf2_log_table, gf2_vd_index
  point sets                : phi_table, lattice_index_matrix,
                              polylattice_index_matrix, point_matrix_rows,
                              reordered_lattice_point, circulant_Z,
                              selection_P
  the product and means     : oracle_X_rows, oracle_X_rows_fsum,
                              column_means, rowmean_relu
  randomised QMC            : replicate_estimate (reading R28)
Pins: tests/test_oracle_pins.py (``rowmean_relu`` and ``column_means``
with f=EXP by special cases: test_rowmean_relu_pins, test_exp_mean_pins).
"""
from __future__ import annotations

import math
from fractions import Fraction
import statistics

import numpy as np

__all__ = [
    "PHI_IDENTITY", "PHI_SHIFT_HALF", "PHI_TENT", "PHI_INVNORM_MID", "PHI_BERNOULLI2",
    "F_IDENTITY", "F_AFFINE", "F_EXP",
    "is_prime", "prime_factors", "primitive_root", "power_table", "log_table",
    "column_exponents",
    "gf2_mul", "gf2_mod", "gf2_divmod", "gf2_mulmod", "gf2_is_primitive",
    "gf2_smallest_primitive", "gf2_power_table", "gf2_log_table", "gf2_vd_index",
    "phi_value", "phi_table", "lattice_index_matrix", "polylattice_index_matrix",
    "point_matrix_rows", "reordered_lattice_point", "circulant_Z", "selection_P",
    "oracle_X_rows", "oracle_X_rows_fsum", "oracle_X_full", "column_means",
    "rowmean_relu", "row_sums", "replicate_estimate",
    "pset_index_matrix", "pset_c", "pset_reordered_point",
    "pde1d_fe_mean", "pde1d_lognormal_fe_mean", "phi_value_shifted", "phi_table_shifted",
    "cbc_criterion_table", "cbc_lattice", "cbc_error",
]

# φ enumeration (PAPER.md:295-302 names Φ^{-1}, the tent transform and the
# identity; SHIFT_HALF is config 1/3/4's u - 1/2; INVNORM_MID is
# Φ^{-1}(u + 1/(2N)), the paper's equal shift Δ = 1/(2N), PAPER.md:466-468,
# reading R6).  Values are this project's ABI numbering, restated here
# independently of the C header.
PHI_IDENTITY = 0
PHI_SHIFT_HALF = 1
PHI_TENT = 2
PHI_INVNORM_MID = 3
PHI_BERNOULLI2 = 4   # B_2(u) = u^2 - u + 1/6 (CBC worst-case error kernel)

# downstream f for the QMC mean (1/N) Σ_n f(b_n)
F_IDENTITY = 0
F_AFFINE = 1      # f(x) = c + x   (config 3's field 1 + X)
F_EXP = 2         # f(x) = exp(x)  (config 5's log-normal field)


# --------------------------------------------------------------------------
# number theory, rank-1 lattice (§2.1)
# --------------------------------------------------------------------------
def is_prime(n: int) -> bool:
    """Trial division.  PAPER.md:243 "Let N be a prime number"."""
    if n < 2:
        return False
    if n % 2 == 0:
        return n == 2
    d = 3
    while d * d <= n:
        if n % d == 0:
            return False
        d += 2
    return True


def prime_factors(m: int) -> list[int]:
    """Distinct prime factors of m by trial division (ascending)."""
    out = []
    d = 2
    while d * d <= m:
        if m % d == 0:
            out.append(d)
            while m % d == 0:
                m //= d
        d += 1
    if m > 1:
        out.append(m)
    return out


def primitive_root(N: int) -> int:
    """Smallest primitive element β of Z_N^* (reading R1:
    the paper says "let β be a primitive element", we take the smallest).
    β is primitive iff β^{(N-1)/q} != 1 mod N for every prime q | N-1."""
    if not is_prime(N) or N < 3:
        raise ValueError("N must be a prime >= 3")
    m = N - 1
    qs = prime_factors(m)
    for beta in range(2, N):
        if all(pow(beta, m // q, N) != 1 for q in qs):
            return beta
    raise AssertionError("unreachable: every prime has a primitive root")


def power_table(N: int, beta: int) -> np.ndarray:
    """P[k] = β^k mod N for k = 0..N-2, by repeated multiplication
    (PAPER.md:319-324 z_k = φ({β^k/N}); PAPER.md:256 {β^k mod N} = Z_N^*)."""
    m = N - 1
    P = np.empty(m, dtype=np.int64)
    v = 1
    for k in range(m):
        P[k] = v
        v = (v * beta) % N
    return P


def log_table(N: int, P: np.ndarray) -> np.ndarray:
    """Discrete log: L[P[k]] = k, L[0] = -1 (reading R5).
    PAPER.md:260-262 g_j ≡ β^{c_j - 1}."""
    L = np.full(N, -1, dtype=np.int64)
    L[P] = np.arange(len(P), dtype=np.int64)
    return L


def column_exponents(z, L: np.ndarray) -> np.ndarray:
    """c_j with z_j ≡ β^{c_j - 1} mod N, 1 <= c_j <= N-1."""
    z = np.asarray(z, dtype=np.int64)
    e = L[z]
    if np.any(e < 0):
        raise ValueError("z_j must be in Z_N^*")
    return e + 1


# --------------------------------------------------------------------------
# number theory, polynomial lattice over F_2 (
# reading R2/R3).  Polynomials are Python ints, bit i = coefficient of x^i.
# --------------------------------------------------------------------------
def gf2_mul(a: int, b: int) -> int:
    """Carry-less product in F_2[x]."""
    r = 0
    while b:
        if b & 1:
            r ^= a
        a <<= 1
        b >>= 1
    return r


def gf2_divmod(a: int, p: int) -> tuple[int, int]:
    """Polynomial long division in F_2[x]: a = q·p + r, deg r < deg p."""
    dp = p.bit_length() - 1
    q = 0
    while a and a.bit_length() - 1 >= dp:
        sh = a.bit_length() - 1 - dp
        q ^= 1 << sh
        a ^= p << sh
    return q, a


def gf2_mod(a: int, p: int) -> int:
    return gf2_divmod(a, p)[1]


def gf2_mulmod(a: int, b: int, p: int) -> int:
    return gf2_mod(gf2_mul(a, b), p)


def gf2_is_primitive(p: int, D: int) -> bool:
    """p of degree D is primitive iff x has multiplicative order 2^D - 1 in
    F_2[x]/p(x) (then F_2[x]/p is a field whose unit group x generates)."""
    if p.bit_length() - 1 != D or D < 2 or not (p & 1):
        return False
    m = (1 << D) - 1

    def xpow(e: int) -> int:
        r, b = 1, 2
        while e:
            if e & 1:
                r = gf2_mulmod(r, b, p)
            b = gf2_mulmod(b, b, p)
            e >>= 1
        return r

    if xpow(m) != 1:
        return False
    return all(xpow(m // q) != 1 for q in prime_factors(m))


def gf2_smallest_primitive(D: int) -> int:
    """Smallest primitive p of degree D by integer encoding (reading R2)."""
    for p in range((1 << D) | 1, 1 << (D + 1), 2):
        if gf2_is_primitive(p, D):
            return p
    raise AssertionError("unreachable")


def gf2_power_table(p: int, D: int) -> np.ndarray:
    """P[k] = x^k mod p(x), k = 0..2^D-2, by repeated multiplication by x."""
    m = (1 << D) - 1
    P = np.empty(m, dtype=np.int64)
    v = 1
    for k in range(m):
        P[k] = v
        v <<= 1
        if v >> D:
            v ^= p
    return P


def gf2_log_table(D: int, P: np.ndarray) -> np.ndarray:
    L = np.full(1 << D, -1, dtype=np.int64)
    L[P] = np.arange(len(P), dtype=np.int64)
    return L


def gf2_vd_index(r: int, p: int, D: int) -> int:
    """v_D(r(x)/p(x)) · 2^D as an integer (reading R3): the digits t_1..t_D of
    r/p = Σ_{i>=1} t_i x^{-i} by the long-division recurrence
    t_i = bit_{D-1}(r_{i-1}),  r_i = (r_{i-1} << 1) xor t_i·p;
    idx = Σ t_i 2^{D-i}, so v_D = idx / 2^D."""
    idx = 0
    for _ in range(D):
        t = (r >> (D - 1)) & 1
        r = (r << 1) ^ (p if t else 0)
        idx = (idx << 1) | t
    return idx


# --------------------------------------------------------------------------
# the transform φ and the point matrix
# --------------------------------------------------------------------------
_ND = statistics.NormalDist()


def phi_value(phi: int, i: int, N: int) -> float:
    """φ(i/N) for the four supported φ (reading R6 for INVNORM_MID:
    argument fl((2i+1)/(2N)), i.e. u + 1/(2N) with u = i/N)."""
    if phi == PHI_IDENTITY:
        return i / N
    if phi == PHI_SHIFT_HALF:
        return i / N - 0.5
    if phi == PHI_TENT:
        return 1.0 - abs(2.0 * (i / N) - 1.0)
    if phi == PHI_INVNORM_MID:
        return _ND.inv_cdf((2 * i + 1) / (2 * N))
    if phi == PHI_BERNOULLI2:
        u = Fraction(i, N)
        return float(u * u - u + Fraction(1, 6))
    raise ValueError("unknown phi")


def phi_value_shifted(phi: int, i: int, N: int, delta: float) -> float:
    """φ at the point i/N of a rule shifted by the equal shift Δ
    (PAPER.md:466-468): u = frac(i/N + Δ) (INVNORM_MID: frac(i/N + 1/(2N) +
    Δ), its own midpoint shift composed with Δ); Δ = 0 is phi_value."""
    if delta == 0.0:
        return phi_value(phi, i, N)
    u = Fraction(i, N) + (Fraction(1, 2 * N) if phi == PHI_INVNORM_MID else 0) + Fraction(delta)
    u = float(u - math.floor(u))
    if phi == PHI_IDENTITY:
        return u
    if phi == PHI_SHIFT_HALF:
        return u - 0.5
    if phi == PHI_TENT:
        return 1.0 - abs(2.0 * u - 1.0)
    if phi == PHI_INVNORM_MID:
        return _ND.inv_cdf(u)
    if phi == PHI_BERNOULLI2:
        return u * u - u + 1.0 / 6.0
    raise ValueError("unknown phi")


def phi_table_shifted(phi: int, N: int, delta: float) -> np.ndarray:
    """tab[i] = φ(frac(i/N + Δ)) (see phi_value_shifted)."""
    return np.array([phi_value_shifted(phi, i, N, delta) for i in range(N)], dtype=np.float64)


def phi_table(phi: int, N: int) -> np.ndarray:
    """tab[i] = φ(i/N), i = 0..N-1.  For the F_2 family N = 2^D (points lie on
    the grid i/2^D).  Building it is excluded from timings."""
    return np.array([phi_value(phi, i, N) for i in range(N)], dtype=np.float64)


def lattice_index_matrix(N: int, z, rows) -> np.ndarray:
    """idx[r, j] = (n_r · z_j) mod N: the conventional rank-1 lattice point
    {n z_j / N} = idx/N."""
    rows = np.asarray(rows, dtype=np.int64)
    z = np.asarray(z, dtype=np.int64)
    return (rows[:, None] * z[None, :]) % N


def polylattice_index_matrix(D: int, p: int, q, rows) -> np.ndarray:
    """idx[r, j] = 2^D · v_D((n_r(x) q_j(x) mod p(x)) / p(x)) (reading R3),
    vectorised over the (rows × s) grid; same recurrences as gf2_mul,
    gf2_mod and gf2_vd_index, applied bit by bit."""
    rows = np.asarray(rows, dtype=np.int64)
    q = np.asarray(q, dtype=np.int64)
    a = np.broadcast_to(q[None, :], (len(rows), len(q))).copy()
    prod = np.zeros_like(a)
    for b in range(D):                       # carry-less product n ⊗ q
        bit = ((rows >> b) & 1).astype(bool)
        prod[bit, :] ^= (a[bit, :] << b)
    for b in range(2 * D - 2, D - 1, -1):    # reduce mod p
        hit = ((prod >> b) & 1).astype(bool)
        prod[hit] ^= (np.int64(p) << (b - D))
    r = prod
    idx = np.zeros_like(r)
    for _ in range(D):                       # digits of r/p
        t = (r >> (D - 1)) & 1
        r = (r << 1) ^ (t * np.int64(p))
        idx = (idx << 1) | t
    return idx


def point_matrix_rows(tab: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Y[rows, :] = φ(idx / N) via the table (PAPER.md:288-294 y_n = φ(x_n))."""
    return tab[idx]


def reordered_lattice_point(N: int, beta: int, c, n: int) -> np.ndarray:
    """The paper's reordered point x_n as integer numerators over N
    (PAPER.md:271-283): x_0 = 0, x_n,j = {β^{c_j - n} / N} for n >= 1."""
    c = np.asarray(c, dtype=np.int64)
    if n == 0:
        return np.zeros(len(c), dtype=np.int64)
    m = N - 1
    return np.array([pow(beta, int((cj - n) % m), N) for cj in c], dtype=np.int64)


def circulant_Z(zeta: np.ndarray) -> np.ndarray:
    """Z with first row (z_0 .. z_{N-2}) and each row the cyclic right shift
    of the previous one: Z[i, k] = z_{(k - i) mod m}."""
    m = len(zeta)
    i = np.arange(m)[:, None]
    k = np.arange(m)[None, :]
    return zeta[(k - i) % m]


def selection_P(c, m: int) -> np.ndarray:
    """p_{k,j} = 1 if k = c_j else 0, 1 <= k <= N-1."""
    c = np.asarray(c, dtype=np.int64)
    P = np.zeros((m, len(c)), dtype=np.float64)
    P[c - 1, np.arange(len(c))] = 1.0
    return P


# --------------------------------------------------------------------------
# the product and the QMC means
# --------------------------------------------------------------------------
def oracle_X_rows(tab: np.ndarray, idx: np.ndarray, A: np.ndarray, cols=None) -> np.ndarray:
    """X[rows, cols] = Y[rows, :] · A[:, cols] (PAPER.md:151-153 YA = B).
    NumPy matmul (BLAS) is the library primitive for the sum."""
    Y = point_matrix_rows(tab, idx)
    Ac = A if cols is None else A[:, cols]
    return Y @ Ac


def oracle_X_rows_fsum(tab: np.ndarray, idx: np.ndarray, A: np.ndarray) -> np.ndarray:
    """Same product with math.fsum per entry (correctly rounded sums)."""
    Y = point_matrix_rows(tab, idx)
    out = np.empty((Y.shape[0], A.shape[1]))
    for r in range(Y.shape[0]):
        for k in range(A.shape[1]):
            out[r, k] = math.fsum(Y[r, :] * A[:, k])
    return out


def oracle_X_full(index_fn, tab: np.ndarray, N: int, A: np.ndarray, cols=None,
                  block: int = 8192) -> np.ndarray:
    """Full X (N × len(cols)), streaming Y in row blocks.  index_fn(rows) -> idx."""
    ncols = A.shape[1] if cols is None else len(cols)
    X = np.empty((N, ncols), dtype=np.float64)
    for r0 in range(0, N, block):
        rows = np.arange(r0, min(N, r0 + block))
        X[r0:r0 + len(rows)] = oracle_X_rows(tab, index_fn(rows), A, cols)
    return X


def column_means(Xcol: np.ndarray, f: int, param: float = 0.0) -> np.ndarray:
    """(1/N) Σ_{n=0}^{N-1} f(X[n, k]) per column (PAPER.md:60-62 eq_qmc,
    PAPER.md:154-157), math.fsum per column.  f=EXP pinned by special cases
    (A = 0; equal z: geometric sum)."""
    Xcol = np.asarray(Xcol)
    N = Xcol.shape[0]
    if f == F_IDENTITY:
        F = Xcol
    elif f == F_AFFINE:
        F = param + Xcol
    elif f == F_EXP:
        F = np.exp(Xcol)
    else:
        raise ValueError("unknown f")
    return np.array([math.fsum(F[:, k]) / N for k in range(F.shape[1])])


def replicate_estimate(Q: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Randomised-QMC estimate from R independently shifted replicates
    (reading R28; the shifts are the equal shifts PAPER.md:466-468 allows):
    Q̄_k = (1/R) Σ_r Q[r,k] and the standard error
    sqrt(Σ_r (Q[r,k] - Q̄_k)^2 / (R (R-1))) (NaN for R = 1), math.fsum.
    Pinned against statistics.fmean / statistics.stdev / sqrt(R) and the
    R = 2 closed form |Q_0 - Q_1| / 2 (test_replicate_estimate_pins)."""
    Q = np.asarray(Q, dtype=np.float64)
    R, t = Q.shape
    mean = np.array([math.fsum(Q[:, k]) / R for k in range(t)])
    if R < 2:
        return mean, np.full(t, np.nan)
    err = np.array([math.sqrt(math.fsum((Q[:, k] - mean[k]) ** 2) / (R * (R - 1))) for k in range(t)])
    return mean, err


def row_sums(X: np.ndarray) -> np.ndarray:
    """r_n = Σ_k X[n, k] (math.fsum per row)."""
    return np.array([math.fsum(X[n, :]) for n in range(X.shape[0])])


def rowmean_relu(X: np.ndarray, t_total: int | None = None) -> float:
    """Config 2's scalar (reading R10): Q = (1/N) Σ_n max(0, (1/t) Σ_k X[n,k]).
    Pinned by the worked example and the no-clipping / all-clipped cases."""
    N, t = X.shape
    t = t if t_total is None else t_total
    r = row_sums(X)
    return math.fsum(max(0.0, rn / t) for rn in r) / N


# ---------------------------------------------------------------- Korobov p-set
def pset_index_matrix(K: int, s: int, rows) -> np.ndarray:
    """The union of all Korobov lattice point sets (Hua–Wang):
    N = (K-1)^2 points x_{n,g} = ({n g^0/K}, {n g^1/K}, ..., {n g^{s-1}/K}),
    n, g = 1..K-1, K prime.  Conventional order (reading R24): row
    r = (g-1)(K-1) + (n-1).  Returns idx[r, j] = (n · g^j) mod K, so that
    x_{r,j} = idx / K."""
    rows = np.asarray(rows, dtype=np.int64)
    g = rows // (K - 1) + 1
    n = rows % (K - 1) + 1
    gj = np.ones((len(rows), s), dtype=np.int64)
    for j in range(1, s):                       # g^j mod K by repeated multiplication
        gj[:, j] = (gj[:, j - 1] * g) % K
    return (n[:, None] * gj) % K


def pset_c(K: int, s: int, g: int) -> np.ndarray:
    """c_{g,j} = (j-1)(g-1) + 1 mod (K-1), j = 1..s: the
    column map of block g in the paper's reordered indexing, with the residue
    0 read as K-1 (reading R5)."""
    j = np.arange(1, s + 1, dtype=np.int64)
    c = ((j - 1) * (g - 1) + 1) % (K - 1)
    c[c == 0] = K - 1
    return c


def pset_reordered_point(K: int, beta: int, s: int, n: int, g: int) -> np.ndarray:
    """The paper's reordered point x_{n,g} = ({β^{c_{g,j} - n} / K})_j
    (PAPER.md:510-521), as integer numerators over K; n, g = 1..K-1."""
    c = pset_c(K, s, g)
    return np.array([pow(beta, int((cj - n) % (K - 1)), K) for cj in c], dtype=np.int64)


# ---------------------------------------------------------------- Experiment 2
def pde1d_fe_mean(X: np.ndarray, d0: float, e0: float, rhs: np.ndarray | None = None) -> np.ndarray:
    """Mean FE coefficients ū = (1/N) Σ_n û^{(n)} where
    û^{(n)} solves B(y_n) û = ĝ, B(y_n) = A_0 + Σ_j y_{n,j} A_j tridiagonal
    (PAPER.md:672-690), given X = Y·A (row n: K diagonal then K-1
    off-diagonal perturbations, qmc_workloads.pde1d_uniform_matrix) and
    ĝ = (1, ..., 1) by default.  Each system is solved by
    LAPACK's banded solver (scipy.linalg.solve_banded); the mean per k is
    math.fsum over n."""
    from scipy.linalg import solve_banded
    N, t = X.shape
    K = (t + 1) // 2
    g = np.ones(K) if rhs is None else np.asarray(rhs, dtype=np.float64)
    U = np.empty((N, K))
    ab = np.zeros((3, K))
    for n in range(N):
        off = e0 + X[n, K:]
        ab[0, 1:] = off
        ab[1, :] = d0 + X[n, :K]
        ab[2, :-1] = off
        U[n] = solve_banded((1, 1), ab, g)
    return np.array([math.fsum(U[:, k]) / N for k in range(K)])


def pde1d_lognormal_fe_mean(Theta: np.ndarray, psi0: float, rhs: np.ndarray | None = None) -> np.ndarray:
    """Experiment 3: Θ = Y·Ψ at the M element
    midpoints (N × M), a_i = exp(ψ_0 + Θ[n, i]); the equal-weight quadrature
    (weight 1/M, reading R25) of b_{n,k,l} = ∫ a φ'_k φ'_l (Eq. def:b nkl)
    gives the tridiagonal B̂(y_n): diagonal M (a_{k-1} + a_k) for node k =
    1..M-1 (elements k-1 and k, 0-based), off-diagonal -M a_k between nodes
    k and k+1.  Solves B̂ û = ĝ (ĝ = 1) with LAPACK's banded solver; returns
    ū = (1/N) Σ_n û^{(n)} (fsum)."""
    from scipy.linalg import solve_banded
    N, M = Theta.shape
    K = M - 1
    g = np.ones(K) if rhs is None else np.asarray(rhs, dtype=np.float64)
    U = np.empty((N, K))
    ab = np.zeros((3, K))
    for n in range(N):
        a = np.exp(psi0 + Theta[n])
        off = -M * a[1:K]
        ab[0, 1:] = off
        ab[1, :] = M * (a[:K] + a[1:])
        ab[2, :-1] = off
        U[n] = solve_banded((1, 1), ab, g)
    return np.array([math.fsum(U[:, k]) / N for k in range(K)])


# ---------------------------------------------------------------- CBC
def cbc_criterion_table(N: int) -> np.ndarray:
    """B_2(i/N) = (i/N)^2 - i/N + 1/6, i = 0..N-1 (exact rationals, rounded once)."""
    return np.array([float(Fraction(i, N) ** 2 - Fraction(i, N) + Fraction(1, 6)) for i in range(N)])


def cbc_lattice(N: int, s: int, gamma) -> np.ndarray:
    """Component-by-component construction, plain form (no FFT): z_1 = 1; for
    d >= 2, z_d = argmin over z = 1..(N-1)/2 (first minimum) of
    Σ_{n>=1} B_2({n z/N}) p_n, with p_n = Π_{j<d} (1 + γ_j 2π² B_2({n z_j/N}))
    (shift-averaged worst-case error, weighted Korobov space, product
    weights; see libqmc's qmc_cbc_step)."""
    gam = np.broadcast_to(np.asarray(gamma, dtype=np.float64), (s,))
    B = cbc_criterion_table(N)
    n = np.arange(N, dtype=np.int64)
    p = np.ones(N)
    cand = np.arange(1, (N - 1) // 2 + 1, dtype=np.int64)
    z = np.zeros(s, dtype=np.int64)
    for d in range(s):
        if d == 0:
            zd = 1
        else:
            crit = B[(n[1:, None] * cand[None, :]) % N].T @ p[1:]
            zd = int(cand[np.argmin(crit)])
        z[d] = zd
        p = p * (1.0 + gam[d] * 2 * math.pi ** 2 * B[(n * zd) % N])
    return z


def cbc_error(N: int, z, gamma) -> float:
    """e²(z) = -1 + (1/N) Σ_n Π_j (1 + γ_j 2π² B_2({n z_j/N})) (fsum)."""
    z = np.asarray(z, dtype=np.int64)
    gam = np.broadcast_to(np.asarray(gamma, dtype=np.float64), (len(z),))
    B = cbc_criterion_table(N)
    n = np.arange(N, dtype=np.int64)
    p = np.ones(N)
    for j, zj in enumerate(z):
        p = p * (1.0 + gam[j] * 2 * math.pi ** 2 * B[(n * int(zj)) % N])
    return math.fsum(p) / N - 1.0
