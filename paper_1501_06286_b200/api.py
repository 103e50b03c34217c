"""Python face of libqmc: a `Plan` that owns its device workspaces (torch
tensors — PyTorch supplies device memory and streams only) and forwards to
the C ABI.  Argument marshalling only; every step of X = Y·A runs in the
library's CUDA kernels.

Layouts (fp64 CUDA tensors): A is (s, t) column-major (``A.stride(0) == 1``,
column k contiguous); X is (N, t) row-major (``X.stride(1) == 1``, row n =
point n's t outputs contiguous, ``ldx = X.stride(0) >= t``).  A column slab of
either is a view.  ``to_device_colmajor`` / ``x_empty`` build such tensors.
"""
from __future__ import annotations

import sys

import numpy as np
import torch

from . import _abi as abi


def colmajor_empty(rows: int, cols: int, device, dtype=torch.float64) -> torch.Tensor:
    return torch.empty((cols, rows), dtype=dtype, device=device).t()


def to_device_colmajor(A: np.ndarray, device) -> torch.Tensor:
    """Host (s, t) array -> device (s, t) column-major fp64 tensor (same bits)."""
    At = np.ascontiguousarray(np.asarray(A, dtype=np.float64).T)
    return torch.from_numpy(At).to(device).t()


def x_empty(N: int, t: int, device, dtype=torch.float64) -> torch.Tensor:
    """Uninitialised (N, t) row-major X."""
    return torch.empty((N, t), dtype=dtype, device=device)


def _ld(x: torch.Tensor, rows: int) -> int:
    """Leading dimension of a column-major (rows, t) A."""
    if x.dtype != torch.float64:
        raise TypeError("fp64 tensors required")
    if x.dim() != 2 or x.shape[0] != rows:
        raise ValueError(f"expected ({rows}, t), got {tuple(x.shape)}")
    if x.shape[1] > 1 and x.stride(0) != 1:
        raise ValueError("column-major (stride(0) == 1) tensor required")
    return max(x.stride(1), rows) if x.shape[1] > 1 else rows


def _ldx(x: torch.Tensor, N: int, t: int) -> int:
    """Leading dimension of a row-major (N, t) X."""
    if x.dtype != torch.float64:
        raise TypeError("fp64 tensors required")
    if x.dim() != 2 or x.shape[0] != N or x.shape[1] != t:
        raise ValueError(f"expected X of shape ({N}, {t}), got {tuple(x.shape)}")
    if t > 1 and x.stride(1) != 1:
        raise ValueError("row-major (stride(1) == 1) X required")
    return max(x.stride(0), t, 1) if N > 1 else max(t, 1)


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(device) -> int:
    """The caller's current CUDA stream on `device` (raw handle)."""
    if _raw_stream is not None:
        return _raw_stream(device.index if device.index is not None else torch.cuda.current_device())
    return torch.cuda.current_stream(device).cuda_stream


class Plan:
    """Fast QMC point-matrix operator Y (N × s) for one device."""

    def __init__(self, family: int, N_or_D: int, z, phi: int, p: int = 0, device=None, delta: float = 0.0):
        if not torch.cuda.is_available():
            raise RuntimeError("libqmc needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device if device is not None else "cuda")
        z = np.asarray(z, dtype=np.int64)
        self.s = int(len(z))
        nbytes = abi.qmc_plan_workspace_size(family, N_or_D, self.s)
        self.plan_ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            st = _stream(self.device)
            if family == abi.QMC_FAMILY_LATTICE and delta:
                self.handle = abi.qmc_plan_create_shifted(N_or_D, self.s, z, phi, float(delta), self.plan_ws,
                                                          nbytes, st)
            elif family == abi.QMC_FAMILY_LATTICE:
                self.handle = abi.qmc_plan_create(N_or_D, self.s, z, phi, self.plan_ws, nbytes, st)
            else:
                self.handle = abi.qmc_plan_create_poly(N_or_D, p, self.s, z, phi, self.plan_ws, nbytes, st)
        self.info = abi.qmc_plan_info(self.handle)
        self.N, self.m, self.phi = self.info["N"], self.info["m"], phi
        self._ws = None
        self._ws_need = {}  # (t, f) -> call-workspace bytes (qmc_call_workspace_size)
        self._last_mm, self._last_mm_dims = None, None  # the last matmul's checked (A, X) layouts
        self._last_mean, self._last_mean_dims = None, None

    @classmethod
    def lattice(cls, N: int, z, phi: int, device=None, delta: float = 0.0) -> "Plan":
        """Rank-1 lattice plan; delta != 0: every point shifted by the equal shift Δ."""
        return cls(abi.QMC_FAMILY_LATTICE, N, z, phi, device=device, delta=delta)

    @classmethod
    def poly(cls, D: int, p: int, q, phi: int, device=None) -> "Plan":
        return cls(abi.QMC_FAMILY_POLY, D, q, phi, p=p, device=device)

    @classmethod
    def from_workload(cls, w, device=None) -> "Plan":
        if w.family == "poly":
            return cls.poly(w.D, w.p, w.z, w.phi, device)
        return cls.lattice(w.N, w.z, w.phi, device)

    def call_workspace(self, t: int, f: int = abi.QMC_F_NONE) -> torch.Tensor:
        key = (t, f)
        nbytes = self._ws_need.get(key)
        if nbytes is None:
            nbytes = self._ws_need[key] = abi.qmc_call_workspace_size(self.handle, t, f)
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        return self._ws

    def matmul(self, A: torch.Tensor, X: torch.Tensor | None = None) -> torch.Tensor:
        key = (A.data_ptr(), A.shape, A.stride(), None if X is None else (X.data_ptr(), X.shape, X.stride()))
        if X is not None and key == self._last_mm:   # same tensors as the last call: layouts already checked
            lda, t, ldx = self._last_mm_dims
        else:
            lda = _ld(A, self.s)
            t = A.shape[1]
            if X is None:
                X = x_empty(self.N, t, self.device)
            ldx = _ldx(X, self.N, t)
            if key[3] is not None:
                self._last_mm, self._last_mm_dims = key, (lda, t, ldx)
        ws = self.call_workspace(t)
        abi.qmc_matmul(self.handle, A, lda, t, X, ldx, ws, ws.numel(), _stream(self.device))
        return X

    def mean(self, A: torch.Tensor, f: int, f_param: float = 0.0, X: torch.Tensor | None = None,
             out: torch.Tensor | None = None) -> torch.Tensor:
        key = (A.data_ptr(), A.shape, A.stride(), None if X is None else (X.data_ptr(), X.shape, X.stride()))
        if key == self._last_mean:   # same tensors as the last call: layouts already checked
            lda, t, ldx = self._last_mean_dims
        else:
            lda = _ld(A, self.s)
            t = A.shape[1]
            ldx = _ldx(X, self.N, t) if X is not None else max(t, 1)
            self._last_mean, self._last_mean_dims = key, (lda, t, ldx)
        n_out = self.N if f == abi.QMC_F_ROWMEAN_RELU else t
        if out is None:
            out = torch.empty(max(n_out, 1), dtype=torch.float64, device=self.device)
        ws = self.call_workspace(t, f)
        abi.qmc_mean(self.handle, A, lda, t, f, f_param, out, X, ldx, ws, ws.numel(),
                     _stream(self.device))
        return out

    def finalize(self, f: int, reduced: torch.Tensor, t_total: int,
                 out: torch.Tensor | None = None) -> torch.Tensor:
        if out is None:
            out = torch.empty(1 if f == abi.QMC_F_ROWMEAN_RELU else t_total, dtype=torch.float64,
                              device=self.device)
        abi.qmc_mean_finalize(self.handle, f, reduced, t_total, out, _stream(self.device))
        return out

    def tables(self):
        return abi.qmc_plan_tables(self.handle, self.m, self.N, self.s)

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and not sys.is_finalizing():
            abi.qmc_plan_destroy(h)
            self.handle = None


class KorobovPSet:
    """The union of all Korobov lattice point sets (SURVEY
    §8(f) NEXT #1): N = (K-1)^2 points x_{n,g} = ({n g^j / K})_{j<s}, n, g =
    1..K-1, K prime, in the conventional order row = (g-1)(K-1) + (n-1)
    (reading R24).

    Block g is the Korobov rank-1 lattice z = (1, g, g^2, ...) mod K without
    its row n = 0; in the paper's reordering every block is Z·P_g with the
    same circulant Z.  So one lattice plan (N = K: one spectrum, one P/L) and
    one launch serve all blocks (qmc_pset_matmul: the block index is a grid
    dimension, the column map e_{g,j} = j·L[g] mod (K-1) is computed on the
    device).  Plans the batched kernel does not cover (K > 4097, i.e. rows
    longer than one row FFT, or s > 2048) run one lattice plan per block, each
    writing its K rows straight into X."""

    def __init__(self, K: int, s: int, phi: int, device=None):
        if not torch.cuda.is_available():
            raise RuntimeError("libqmc needs a CUDA device (no CPU fallback)")
        self.K, self.s, self.phi = int(K), int(s), int(phi)
        self.N = (self.K - 1) ** 2
        self.device = torch.device(device if device is not None else "cuda")
        # the shared plan (its generating vector is not used by qmc_pset_matmul)
        self.plan = Plan.lattice(self.K, np.ones(self.s, dtype=np.int64), self.phi, device=self.device)
        self.plans = None  # per-block plans, built on first use when the batched kernel does not apply
        self._ws = None

    def _block_plans(self):
        if self.plans is None:
            self.plans = []
            for g in range(1, self.K):
                z = np.array([pow(g, j, self.K) for j in range(self.s)], dtype=np.int64)
                self.plans.append(Plan.lattice(self.K, z, self.phi, device=self.device))
        return self.plans

    def matmul(self, A: torch.Tensor, per_block: bool = False) -> torch.Tensor:
        """X = Y·A for the p-set; A (s, t) column-major; returns X (N, t) row-major.
        per_block=True forces the one-plan-per-block path (comparison)."""
        lda = _ld(A, self.s)
        t = A.shape[1]
        st = _stream(self.device)
        if not per_block:
            X = torch.empty((self.N, t), dtype=torch.float64, device=self.device)
            with torch.cuda.device(self.device):
                rc = abi.qmc_pset_matmul(self.plan.handle, A, lda, t, X, max(t, 1), st)
            if rc == 0:
                return X
        plans = self._block_plans()
        buf = torch.empty((self.N + 1, t), dtype=torch.float64, device=self.device)
        ldx = max(t, 1)
        nbytes = max(abi.qmc_call_workspace_size(p.handle, t, abi.QMC_F_NONE) for p in plans)
        if self._ws is None or self._ws.numel() < nbytes:
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            # decreasing g: each block's row 0 lands on the row the next (lower)
            # block overwrites with its last row; X is a view of N+1 rows
            for g in range(self.K - 1, 0, -1):
                Xg = buf[(g - 1) * (self.K - 1):]          # rows n = 0..K-1 of block g
                abi.qmc_matmul(plans[g - 1].handle, A, lda, t, Xg, ldx, self._ws, self._ws.numel(), st)
        return buf[1:]


class ShiftedPlan(Plan):
    """A replicate of `base` with every point shifted by Δ (qmc_plan_shift):
    shares base's tables, owns only ζ, φ(x_0) and the spectrum (about
    8m + 16L bytes).  Keeps `base` alive."""

    def __init__(self, base: Plan, delta: float):
        self.base = base
        self.device = base.device
        self.s = base.s
        nbytes = abi.qmc_shift_workspace_size(base.handle)
        self.plan_ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        with torch.cuda.device(self.device):
            self.handle = abi.qmc_plan_shift(base.handle, float(delta), self.plan_ws, nbytes, _stream(self.device))
        self.info = abi.qmc_plan_info(self.handle)
        self.N, self.m, self.phi = self.info["N"], self.info["m"], base.phi
        self._ws = base._ws if base._ws is not None else None
        self._ws_need = base._ws_need
        self._last_mm, self._last_mm_dims = None, None
        self._last_mean, self._last_mean_dims = None, None


def replicate_mean(means: torch.Tensor, with_stderr: bool = True):
    """(R, t) replicate means -> (mean over r, standard error) by the library's
    fixed-order kernel (qmc_replicate_mean; reading R28)."""
    if means.dtype != torch.float64 or means.dim() != 2 or (means.shape[1] > 1 and means.stride(1) != 1):
        raise ValueError("(R, t) fp64 tensor with contiguous rows required")
    R, t = means.shape
    mean = torch.empty(t, dtype=torch.float64, device=means.device)
    err = torch.empty(t, dtype=torch.float64, device=means.device) if with_stderr else None
    abi.qmc_replicate_mean(means, R, t, max(means.stride(0), t), mean, err, _stream(means.device))
    return mean, err


def shifted_means(N: int, z, phi: int, A: torch.Tensor, f: int, f_param: float, deltas,
                  device=None, return_stderr: bool = False):
    """Randomised QMC: the fused means of f(X) over R
    equally shifted copies of the rule (Δ_r in `deltas`).
    Returns (per-replicate means R × t, their average over r[, the standard
    error]).  One lattice plan holds the tables; each replicate is a
    qmc_plan_shift view (only ζ and W are rebuilt) and one fused qmc_mean
    call writing its row of the R × t result; the average and standard error
    come from qmc_replicate_mean (fixed order r = 0..R-1)."""
    if f == abi.QMC_F_ROWMEAN_RELU:
        raise ValueError("shifted_means averages per-column means (f = IDENTITY / AFFINE / EXP)")
    deltas = [float(d) for d in deltas]
    base = Plan.lattice(N, z, phi, device=device)
    t = A.shape[1]
    out = torch.empty((len(deltas), max(t, 1)), dtype=torch.float64, device=base.device)
    rep = None
    for r, d in enumerate(deltas):
        rep = ShiftedPlan(base, d)
        rep.mean(A, f, f_param, out=out[r])
        base._ws = rep._ws  # one call workspace for all replicates
    R = out[:, :t]
    avg, err = replicate_mean(R, with_stderr=return_stderr)
    if return_stderr:
        return R, avg, err
    return R, avg
