"""Experiment 2 of the paper: the
mean finite-element solution of the uniform 1-D ODE

    -(a(x,y) u')' = g on (0,1),  a(x,y) = 2 + Σ_j y_j j^{-3/2} sin(2π j x),

over the N points of a rank-1 lattice rule (φ(u) = u - 1/2).  The stiffness
perturbations of all N samples are ONE fast product X = Y·A (PAPER.md:704-711:
"each matrix-vector multiplication Y a_{k,l} should be done using the approach
of the previous section"), with the row-major X holding sample n's K diagonal
and K-1 off-diagonal entries contiguously; the N tridiagonal solves and the
mean run in the library (qmc_tridiag_solve_mean).  Argument marshalling only.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _abi as abi
from .api import Plan, _stream, to_device_colmajor, x_empty


class UniformPDE1D:
    """Fast-QMC mean FE coefficients ū (K = M-1 values) of the uniform ODE.

    A, d0, e0 are the stiffness coefficients of qmc_workloads.pde1d_uniform_matrix
    (s × (2K-1), the paper's closed forms); z the lattice generating vector."""

    def __init__(self, N: int, z, A: np.ndarray, d0: float, e0: float, device=None):
        self.device = torch.device(device if device is not None else "cuda")
        self.plan = Plan.lattice(N, z, abi.QMC_PHI_SHIFT_HALF, device=self.device)
        self.N = N
        self.t = A.shape[1]
        self.K = (self.t + 1) // 2
        self.d0, self.e0 = float(d0), float(e0)
        self.A = to_device_colmajor(A, self.device)
        self.X = x_empty(N, self.t, self.device)
        self.mean = torch.empty(self.K, dtype=torch.float64, device=self.device)

    def solve_mean(self, A: torch.Tensor | None = None) -> torch.Tensor:
        """ū: X = Y·A (fast path), then N Thomas solves in place and the mean."""
        A = self.A if A is None else A
        self.plan.matmul(A, self.X)
        abi.qmc_tridiag_solve_mean(self.N, self.K, self.d0, self.e0, None, self.X, self.t, self.mean,
                                   _stream(self.device))
        return self.mean


class LognormalPDE1D:
    """Fast-QMC mean FE coefficients of the log-normal ODE of Experiment 3
    (PAPER.md:716-767, 924-940): Θ = Y·Ψ by the fast path (Ψ: s × M values of
    ψ_j at the element midpoints, qmc_workloads.pde1d_lognormal_matrix), then
    the on-the-fly exp / midpoint-rule assembly, the N tridiagonal solves and
    the mean in qmc_fe1d_lognormal_solve_mean.  φ defaults to Φ^{-1}(u +
    1/(2N)) (y_j ~ N(0,1), reading R26)."""

    def __init__(self, N: int, z, Psi: np.ndarray, psi0: float, phi: int = abi.QMC_PHI_INVNORM_MID,
                 device=None):
        self.device = torch.device(device if device is not None else "cuda")
        self.plan = Plan.lattice(N, z, phi, device=self.device)
        self.N = N
        self.M = Psi.shape[1]
        self.psi0 = float(psi0)
        self.Psi = to_device_colmajor(Psi, self.device)
        self.ldx = 2 * self.M - 2
        self.buf = torch.empty((N, self.ldx), dtype=torch.float64, device=self.device)
        self.mean = torch.empty(self.M - 1, dtype=torch.float64, device=self.device)

    def solve_mean(self) -> torch.Tensor:
        self.plan.matmul(self.Psi, self.buf[:, :self.M])      # Θ in the first M slots of each row
        abi.qmc_fe1d_lognormal_solve_mean(self.N, self.M, self.psi0, None, self.buf, self.ldx, self.mean,
                                          _stream(self.device))
        return self.mean
