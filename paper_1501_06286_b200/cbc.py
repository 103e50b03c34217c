"""Fast component-by-component construction of a rank-1 lattice generating
vector on the GPU.  The paper cites the fast CBC
construction and notes that its circulant
structure is the same one the fast matrix product exploits: step d needs
Σ_n B_2({n z/N}) p_n for every candidate z, which is one fast product
X = Y_all·p with the lattice of generating vector (1, ..., N-1) and φ = B_2.
Argument marshalling only: the products, the selection and the update of p
run in libqmc (qmc_matmul, qmc_cbc_step)."""
from __future__ import annotations

import numpy as np
import torch

from . import _abi as abi
from .api import Plan, _stream, x_empty


def cbc_lattice(N: int, s: int, gamma, device=None) -> np.ndarray:
    """z (int64[s]) minimising, one component at a time, the shift-averaged
    worst-case error with product weights γ_j (z_1 = 1; candidates
    1..(N-1)/2)."""
    dev = torch.device(device if device is not None else "cuda")
    gam = np.broadcast_to(np.asarray(gamma, dtype=np.float64), (s,))
    plan = Plan.lattice(N, np.arange(1, N, dtype=np.int64), abi.QMC_PHI_BERNOULLI2, device=dev)
    p = torch.ones(N, dtype=torch.float64, device=dev)
    crit = x_empty(N, 1, dev)
    zs = torch.empty(s, dtype=torch.int64, device=dev)
    st = _stream(dev)
    for d in range(s):
        plan.matmul(p[1:].view(N - 1, 1), crit)
        abi.qmc_cbc_step(N, crit, 1 if d == 0 else (N - 1) // 2, float(gam[d]), p, zs, d, st)
    return zs.cpu().numpy()
