"""Seeded synthetic inputs for the five BASELINE.json configs (and small
custom cases).  Shared by the oracle, the tests, bench.py and smoke().

This module holds NONE of the method's arithmetic: it only draws the
generating vector z (or q) and builds the matrix A.  Recipe (DESIGN.md
§Inputs; SURVEY.md §8(c) readings R12-R15, R20):

  rng = numpy.random.default_rng(seed), seed = config number 1..5;
  draw z (or q) first: rng.integers(1, m + 1, size=s)  (i.i.d. uniform on
  {1..m}, m = N-1 or 2^D-1); then, if A is random,
  rng.standard_normal((s, t)) in C order, then scale.
  A is returned column-major (Fortran order, lda = s) so a column of A is
  contiguous, which is the layout the C-ABI takes.

These stand in for the paper's synthetic workloads (random upper-triangular
A; analytic ODE coefficients);
no dataset is involved.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# ABI numbering of φ and of the fused f (restated; see include/qmc.h)
PHI_IDENTITY, PHI_SHIFT_HALF, PHI_TENT, PHI_INVNORM_MID, PHI_BERNOULLI2 = 0, 1, 2, 3, 4
F_IDENTITY, F_AFFINE, F_EXP, F_ROWMEAN_RELU = 0, 1, 2, 3

FAMILY_LATTICE = "lattice"
FAMILY_POLY = "poly"


@dataclass
class Workload:
    name: str
    family: str           # "lattice" | "poly"
    N: int                # number of points (prime, or 2^D)
    m: int                # circulant length N-1 (lattice) or 2^D-1 (poly)
    s: int
    t: int
    phi: int
    z: np.ndarray         # generating vector z_j (lattice) / q_j (poly), int64[s]
    A: np.ndarray         # s × t fp64, Fortran order
    D: int = 0            # poly degree
    p: int = 0            # primitive modulus (poly)
    f: int | None = None  # fused mean (None: X only)
    f_param: float = 0.0
    seed: int = 0
    extra: dict = field(default_factory=dict)

    @property
    def entries(self) -> int:
        return self.N * self.t


def _z(rng, m, s):
    return rng.integers(1, m + 1, size=s).astype(np.int64)


def ar1_upper_cholesky(s: int, ell: float) -> np.ndarray:
    """Upper factor A with AᵀA = Σ, Σ_ij = exp(-|i-j|/ell) (reading R15):
    ρ = exp(-1/ell); A[0,k] = ρ^k; A[j,k] = ρ^{k-j}·sqrt(1-ρ²) for 1<=j<=k."""
    rho = np.exp(-1.0 / ell)
    j = np.arange(s)[:, None]
    k = np.arange(s)[None, :]
    A = np.where(j <= k, rho ** np.maximum(k - j, 0).astype(np.float64), 0.0)
    A[1:, :] *= np.sqrt(1.0 - rho * rho)
    return np.asfortranarray(A)


def kl_sine_matrix(s: int, t: int, amp_pow: float, amp_scale: float,
                   cols=None) -> np.ndarray:
    """A_jk = amp_scale · j^{-amp_pow} · sin(j π x_k), j = 1..s, x_k = (k+0.5)/t
    (reading R12)."""
    kk = np.arange(t) if cols is None else np.asarray(cols)
    x = (kk + 0.5) / t
    j = np.arange(1, s + 1, dtype=np.float64)[:, None]
    A = np.empty((s, len(kk)), dtype=np.float64, order="F")
    B = 1024
    for c0 in range(0, len(kk), B):
        xs = x[c0:c0 + B][None, :]
        A[:, c0:c0 + B] = amp_scale * j ** (-amp_pow) * np.sin(j * np.pi * xs)
    return A


def config(c: int, t_override: int | None = None) -> Workload:
    """BASELINE.json configs[c-1] (c = 1..5), seeded with seed = c."""
    rng = np.random.default_rng(c)
    if c == 1:
        N, s, t = 257, 300, 64
        z = _z(rng, N - 1, s)
        t = t_override or t
        A = np.asfortranarray(rng.standard_normal((s, t)))
        return Workload("c1_lattice_N257_s300_t64", FAMILY_LATTICE, N, N - 1, s, t,
                        PHI_SHIFT_HALF, z, A, seed=c)
    if c == 2:
        N, s, t = 65537, 1024, 1024
        z = _z(rng, N - 1, s)
        A = ar1_upper_cholesky(s, 102.4)
        if t_override:
            A = np.asfortranarray(A[:, :t_override]); t = t_override
        return Workload("c2_lattice_N65537_s1024_t1024_invnorm_rowmeanrelu", FAMILY_LATTICE,
                        N, N - 1, s, t, PHI_INVNORM_MID, z, A, f=F_ROWMEAN_RELU, seed=c)
    if c == 3:
        N, s, t = 40961, 4096, 65536
        z = _z(rng, N - 1, s)
        tt = t_override or t
        A = kl_sine_matrix(s, t, 2.0, 1.0, cols=np.arange(tt))
        return Workload("c3_lattice_N40961_s4096_t65536_affine", FAMILY_LATTICE, N, N - 1,
                        s, tt, PHI_SHIFT_HALF, z, A, f=F_AFFINE, f_param=1.0, seed=c,
                        extra={"t_full": t})
    if c == 4:
        D, p, s, t = 16, 65581, 2000, 2000
        m = (1 << D) - 1
        q = _z(rng, m, s)
        A = rng.standard_normal((s, t)) / np.sqrt(s)
        if t_override:
            A = A[:, :t_override]; t = t_override
        return Workload("c4_poly_D16_p65581_s2000_t2000", FAMILY_POLY, 1 << D, m, s, t,
                        PHI_SHIFT_HALF, q, np.asfortranarray(A), D=D, p=p, seed=c)
    if c == 5:
        N, s, t = 786433, 8192, 8192
        z = _z(rng, N - 1, s)
        tt = t_override or t
        A = kl_sine_matrix(s, t, 1.0, np.sqrt(2.0), cols=np.arange(tt))
        return Workload("c5_lattice_N786433_s8192_t8192_exp", FAMILY_LATTICE, N, N - 1, s,
                        tt, PHI_INVNORM_MID, z, A, f=F_EXP, seed=c, extra={"t_full": t})
    raise ValueError("config must be 1..5")


def custom_lattice(N: int, s: int, t: int, phi: int, seed: int,
                   f: int | None = None, f_param: float = 0.0) -> Workload:
    """Small seeded lattice case (same draw order as the configs)."""
    rng = np.random.default_rng(seed)
    z = _z(rng, N - 1, s)
    A = np.asfortranarray(rng.standard_normal((s, t)))
    return Workload(f"lattice_N{N}_s{s}_t{t}_phi{phi}", FAMILY_LATTICE, N, N - 1, s, t, phi,
                    z, A, f=f, f_param=f_param, seed=seed)


def custom_poly(D: int, p: int, s: int, t: int, phi: int, seed: int,
                f: int | None = None, f_param: float = 0.0) -> Workload:
    rng = np.random.default_rng(seed)
    m = (1 << D) - 1
    q = _z(rng, m, s)
    A = np.asfortranarray(rng.standard_normal((s, t)))
    return Workload(f"poly_D{D}_p{p}_s{s}_t{t}_phi{phi}", FAMILY_POLY, 1 << D, m, s, t, phi,
                    q, A, D=D, p=p, f=f, f_param=f_param, seed=seed)


# ---------------------------------------------------------------- Experiment 2
def pde1d_uniform_matrix(M: int, s: int) -> tuple[np.ndarray, float, float]:
    """Stiffness coefficients of the paper's uniform 1-D ODE:
    -(a u')' = g on (0,1), a(x, y) = 2 + Σ_j y_j j^{-3/2} sin(2π j x), hat
    functions on x_k = k/M, K = M-1 unknowns.  Returns (A, d0, e0): A is the
    s × (2K-1) matrix (Fortran order) whose column c holds a_{j,k,l} for
    j = 1..s at the tridiagonal position c — c < K: (k, k), k = c+1; c >= K:
    (k, k+1), k = c-K+1 — and d0 = a_{0,k,k} = 4M, e0 = a_{0,k,k+1} = -2M.
    The closed forms are the paper's, restated."""
    K = M - 1
    j = np.arange(1, s + 1, dtype=np.float64)[:, None]
    amp = M * M / (np.pi * j ** 2.5)
    k = np.arange(1, K + 1, dtype=np.float64)[None, :]
    diag = amp * np.sin(2 * np.pi * j / M) * np.sin(2 * np.pi * j * k / M)
    ko = np.arange(1, K, dtype=np.float64)[None, :]
    off = -amp * np.sin(np.pi * j / M) * np.sin(np.pi * j * (2 * ko + 1) / M)
    A = np.asfortranarray(np.concatenate([diag, off], axis=1))
    return A, 4.0 * M, -2.0 * M


def pde1d_uniform(N: int, M: int, s: int, seed: int = 2) -> Workload:
    """Experiment 2 workload: lattice rule N (prime), random z (reading R19),
    φ(u) = u - 1/2, A from pde1d_uniform_matrix."""
    rng = np.random.default_rng(seed)
    z = _z(rng, N - 1, s)
    A, d0, e0 = pde1d_uniform_matrix(M, s)
    return Workload(f"exp2_pde1d_N{N}_M{M}_s{s}", FAMILY_LATTICE, N, N - 1, s, A.shape[1],
                    PHI_SHIFT_HALF, z, A, seed=seed, extra={"M": M, "K": M - 1, "d0": d0, "e0": e0})


# ---------------------------------------------------------------- Experiment 3
def pde1d_lognormal_matrix(M: int, s: int) -> tuple[np.ndarray, float]:
    """Log-normal ODE of Experiment 3: a(x, y) =
    exp(ψ_0 + Σ_j y_j ψ_j(x)), ψ_0 = 2, ψ_j(x) = j^{-3/2} sin(2π j x), with
    an equal-weight quadrature of I = M points (reading R25: the midpoint of
    each of the M elements, weight 1/M).  Returns (Ψ, ψ_0): Ψ is s × M
    (Fortran order), Ψ[j-1, i] = ψ_j((i + 1/2)/M), so that Θ = ψ_0 + Y·Ψ
    (Eq. fastB)."""
    j = np.arange(1, s + 1, dtype=np.float64)[:, None]
    x = (np.arange(M, dtype=np.float64)[None, :] + 0.5) / M
    return np.asfortranarray(j ** -1.5 * np.sin(2 * np.pi * j * x)), 2.0


def pde1d_lognormal(N: int, M: int, s: int, seed: int = 3) -> Workload:
    """Experiment 3 workload: lattice rule N, random z (R19), y_j ~ N(0,1) via
    φ(u) = Φ^{-1}(u + 1/(2N)) (reading R26), Ψ from pde1d_lognormal_matrix."""
    rng = np.random.default_rng(seed)
    z = _z(rng, N - 1, s)
    Psi, psi0 = pde1d_lognormal_matrix(M, s)
    return Workload(f"exp3_pde1d_lognormal_N{N}_M{M}_s{s}", FAMILY_LATTICE, N, N - 1, s, M,
                    PHI_INVNORM_MID, z, Psi, seed=seed, extra={"M": M, "K": M - 1, "psi0": psi0})
