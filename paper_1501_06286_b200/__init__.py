"""B200-native fast QMC matrix product X = Y·A (arXiv 1501.06286).

    from paper_1501_06286_b200 import Plan
    plan = Plan.lattice(N, z, phi)          # integer + spectral plan kernels
    X = plan.matmul(A)                      # X = Y·A, conventional row order
    out = plan.mean(A, f, f_param, X=X)     # fused f and QMC mean

The C ABI is include/qmc.h (libqmc.so, built by `build.py`); `_abi` is the
thin ctypes binding with the same names.  Importing this package loads the
shared library and fails loudly if it is missing: there is no CPU path.
"""
from . import _abi
from ._abi import (QMC_F_AFFINE, QMC_F_EXP, QMC_F_IDENTITY, QMC_F_NONE, QMC_F_ROWMEAN_RELU,
                   QMC_FAMILY_LATTICE, QMC_FAMILY_POLY, QMC_PHI_IDENTITY, QMC_PHI_INVNORM_MID,
                   QMC_PHI_SHIFT_HALF, QMC_PHI_TENT, QMC_PHI_BERNOULLI2, QMCError)
from .api import (KorobovPSet, Plan, ShiftedPlan, colmajor_empty, replicate_mean, shifted_means, to_device_colmajor,
                  x_empty)
from .cbc import cbc_lattice
from .pde import LognormalPDE1D, UniformPDE1D

__all__ = [
    "KorobovPSet", "LognormalPDE1D", "Plan", "QMCError", "UniformPDE1D", "cbc_lattice", "shifted_means", "ShiftedPlan", "replicate_mean", "colmajor_empty", "to_device_colmajor", "x_empty", "_abi",
    "QMC_FAMILY_LATTICE", "QMC_FAMILY_POLY", "QMC_PHI_IDENTITY", "QMC_PHI_SHIFT_HALF",
    "QMC_PHI_TENT", "QMC_PHI_INVNORM_MID", "QMC_F_NONE", "QMC_F_IDENTITY", "QMC_F_AFFINE",
    "QMC_F_EXP", "QMC_F_ROWMEAN_RELU",
]
