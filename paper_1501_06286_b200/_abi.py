"""Thin ctypes binding of include/qmc.h (argument marshalling only).

Every function keeps the C name and order of arguments; device pointers are
taken from torch tensors (or raw ints), status codes become QMCError.  No
computation happens here: every step of the path runs in libqmc.so's
kernels.  If libqmc.so is missing this module raises at import — there is no
CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# QMC_LIB selects another build of the same sources (diagnostic variants, e.g.
# variants/libqmc_phase.so built with -DQMC_PHASE_TIMING); default: in-tree
LIB_PATH = os.environ.get("QMC_LIB") or os.path.join(_HERE, "libqmc.so")

QMC_FAMILY_LATTICE, QMC_FAMILY_POLY = 0, 1
QMC_PHI_IDENTITY, QMC_PHI_SHIFT_HALF, QMC_PHI_TENT, QMC_PHI_INVNORM_MID, QMC_PHI_BERNOULLI2 = 0, 1, 2, 3, 4
QMC_F_IDENTITY, QMC_F_AFFINE, QMC_F_EXP, QMC_F_ROWMEAN_RELU = 0, 1, 2, 3
QMC_F_NONE = -1  # workspace query for qmc_matmul

EXPORTS = [
    "qmc_plan_workspace_size", "qmc_call_workspace_size", "qmc_plan_create",
    "qmc_plan_create_poly", "qmc_matmul", "qmc_mean", "qmc_mean_finalize", "qmc_mean_host",
    "qmc_plan_info", "qmc_plan_tables", "qmc_launch_count", "qmc_plan_destroy", "qmc_strerror",
    "qmc_profile_enable", "qmc_profile_read", "qmc_profile_class_name", "qmc_tridiag_solve_mean",
    "qmc_fe1d_lognormal_solve_mean", "qmc_plan_create_shifted", "qmc_cbc_step", "qmc_pset_matmul", "qmc_build_flags",
    "qmc_shift_workspace_size", "qmc_plan_shift", "qmc_replicate_mean",
]
QMC_EUNSUPPORTED = -10


class QMCError(RuntimeError):
    def __init__(self, code: int, where: str):
        self.code = code
        super().__init__(f"{where}: {strerror(code)} (status {code})")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -m paper_1501_06286_b200.build` "
            "(no CPU fallback exists)")
    return C.CDLL(LIB_PATH)


_lib = _load()

_vp, _i64, _i32, _sz, _d = C.c_void_p, C.c_int64, C.c_int, C.c_size_t, C.c_double
_P64, _P32, _PD, _PSZ = C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_double), C.POINTER(C.c_size_t)

_sig = {
    "qmc_plan_workspace_size": (_i32, [_i32, _i64, _i64, _PSZ]),
    "qmc_call_workspace_size": (_i32, [_vp, _i64, _i32, _PSZ]),
    "qmc_plan_create": (_i32, [C.POINTER(_vp), _i64, _i64, _P64, _i32, _vp, _sz, _vp]),
    "qmc_plan_create_poly": (_i32, [C.POINTER(_vp), _i32, C.c_uint64, _i64, _P64, _i32, _vp, _sz, _vp]),
    "qmc_plan_create_shifted": (_i32, [C.POINTER(_vp), _i64, _i64, _P64, _i32, _d, _vp, _sz, _vp]),
    "qmc_shift_workspace_size": (_i32, [_vp, _PSZ]),
    "qmc_plan_shift": (_i32, [C.POINTER(_vp), _vp, _d, _vp, _sz, _vp]),
    "qmc_replicate_mean": (_i32, [_vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "qmc_matmul": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64, _vp, _sz, _vp]),
    "qmc_pset_matmul": (_i32, [_vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "qmc_mean": (_i32, [_vp, _vp, _i64, _i64, _i32, _d, _vp, _vp, _i64, _vp, _sz, _vp]),
    "qmc_mean_finalize": (_i32, [_vp, _i32, _vp, _i64, _vp, _vp]),
    "qmc_mean_host": (_i32, [_vp, _vp, _i64, _i64, _i32, _d, _vp, _vp, _vp, _i64, _vp, _vp, _sz, _vp]),
    "qmc_plan_info": (_i32, [_vp, _P64]),
    "qmc_tridiag_solve_mean": (_i32, [_i64, _i64, _d, _d, _vp, _vp, _i64, _vp, _vp]),
    "qmc_fe1d_lognormal_solve_mean": (_i32, [_i64, _i64, _d, _vp, _vp, _i64, _vp, _vp]),
    "qmc_cbc_step": (_i32, [_i64, _vp, _i64, _d, _vp, _vp, _i64, _vp]),
    "qmc_plan_tables": (_i32, [_vp, _P64, _P32, _P32, _P32, _PD]),
    "qmc_launch_count": (_i64, []),
    "qmc_build_flags": (_i32, []),
    "qmc_plan_destroy": (None, [_vp]),
    "qmc_strerror": (C.c_char_p, [_i32]),
    "qmc_profile_enable": (_i32, [_i32]),
    "qmc_profile_read": (_i32, [_P64, _PD, _i32]),
    "qmc_profile_class_name": (C.c_char_p, [_i32]),
}
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def qmc_build_flags() -> int:
    return int(_lib.qmc_build_flags())


def strerror(code: int) -> str:
    return _lib.qmc_strerror(int(code)).decode()


def _check(rc: int, where: str) -> None:
    if rc != 0:
        raise QMCError(rc, where)


def ptr(x) -> int | None:
    """Device/host address of a torch tensor or numpy array (or an int)."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if hasattr(x, "ctypes"):
        return x.ctypes.data
    raise TypeError(f"cannot take the address of {type(x)}")


def _i64arr(vals):
    import numpy as np
    a = np.ascontiguousarray(np.asarray(vals, dtype=np.int64))
    return a, a.ctypes.data_as(_P64)


# ----------------------------------------------------------------- C calls
def qmc_plan_workspace_size(family: int, N_or_D: int, s: int) -> int:
    out = C.c_size_t(0)
    _check(_lib.qmc_plan_workspace_size(family, N_or_D, s, C.byref(out)), "qmc_plan_workspace_size")
    return out.value


def qmc_call_workspace_size(plan, t: int, f: int = QMC_F_NONE) -> int:
    out = C.c_size_t(0)
    _check(_lib.qmc_call_workspace_size(plan, t, f, C.byref(out)), "qmc_call_workspace_size")
    return out.value


def qmc_plan_create(N: int, s: int, z, phi: int, plan_ws, plan_ws_bytes: int, stream=None):
    h = _vp()
    arr, p = _i64arr(z)
    assert len(arr) == s
    _check(_lib.qmc_plan_create(C.byref(h), N, s, p, phi, ptr(plan_ws), plan_ws_bytes, stream),
           "qmc_plan_create")
    return h


def qmc_plan_create_shifted(N: int, s: int, z, phi: int, delta: float, plan_ws, plan_ws_bytes: int,
                            stream=None):
    h = _vp()
    arr, p = _i64arr(z)
    assert len(arr) == s
    _check(_lib.qmc_plan_create_shifted(C.byref(h), N, s, p, phi, delta, ptr(plan_ws), plan_ws_bytes, stream),
           "qmc_plan_create_shifted")
    return h


def qmc_shift_workspace_size(base) -> int:
    out = C.c_size_t(0)
    _check(_lib.qmc_shift_workspace_size(base, C.byref(out)), "qmc_shift_workspace_size")
    return out.value


def qmc_plan_shift(base, delta: float, shift_ws, shift_ws_bytes: int, stream=None):
    h = _vp()
    _check(_lib.qmc_plan_shift(C.byref(h), base, delta, ptr(shift_ws), shift_ws_bytes, stream), "qmc_plan_shift")
    return h


def qmc_replicate_mean(means, R: int, t: int, ld: int, mean_out, stderr_out=None, stream=None):
    _check(_lib.qmc_replicate_mean(ptr(means), R, t, ld, ptr(mean_out), ptr(stderr_out), stream),
           "qmc_replicate_mean")


def qmc_plan_create_poly(D: int, p: int, s: int, q, phi: int, plan_ws, plan_ws_bytes: int, stream=None):
    h = _vp()
    arr, pq = _i64arr(q)
    assert len(arr) == s
    _check(_lib.qmc_plan_create_poly(C.byref(h), D, p, s, pq, phi, ptr(plan_ws), plan_ws_bytes, stream),
           "qmc_plan_create_poly")
    return h


def qmc_matmul(plan, A, lda: int, t: int, X, ldx: int, call_ws, call_ws_bytes: int, stream=None):
    _check(_lib.qmc_matmul(plan, ptr(A), lda, t, ptr(X), ldx, ptr(call_ws), call_ws_bytes, stream),
           "qmc_matmul")


def qmc_pset_matmul(plan, A, lda: int, t: int, X, ldx: int, stream=None) -> int:
    """Returns the status (QMC_OK or QMC_EUNSUPPORTED); raises on other errors."""
    rc = _lib.qmc_pset_matmul(plan, ptr(A), lda, t, ptr(X), ldx, stream)
    if rc != QMC_EUNSUPPORTED:
        _check(rc, "qmc_pset_matmul")
    return rc


def qmc_mean(plan, A, lda: int, t: int, f: int, f_param: float, out, X_or_null, ldx: int,
             call_ws, call_ws_bytes: int, stream=None):
    _check(_lib.qmc_mean(plan, ptr(A), lda, t, f, f_param, ptr(out), ptr(X_or_null), ldx,
                         ptr(call_ws), call_ws_bytes, stream), "qmc_mean")


def qmc_mean_finalize(plan, f: int, reduced, t_total: int, out, stream=None):
    _check(_lib.qmc_mean_finalize(plan, f, ptr(reduced), t_total, ptr(out), stream), "qmc_mean_finalize")


def qmc_mean_host(plan, A_host, lda: int, t: int, f: int, f_param: float, out_host, A_dev, X_dev,
                  ldx: int, out_dev, call_ws, call_ws_bytes: int, stream=None):
    _check(_lib.qmc_mean_host(plan, ptr(A_host), lda, t, f, f_param, ptr(out_host), ptr(A_dev),
                              ptr(X_dev), ldx, ptr(out_dev), ptr(call_ws), call_ws_bytes, stream),
           "qmc_mean_host")


def qmc_tridiag_solve_mean(N: int, K: int, d0: float, e0: float, rhs, X, ldx: int, mean_out, stream=None):
    _check(_lib.qmc_tridiag_solve_mean(N, K, d0, e0, ptr(rhs), ptr(X), ldx, ptr(mean_out), stream),
           "qmc_tridiag_solve_mean")


def qmc_fe1d_lognormal_solve_mean(N: int, M: int, psi0: float, rhs, X, ldx: int, mean_out, stream=None):
    _check(_lib.qmc_fe1d_lognormal_solve_mean(N, M, psi0, ptr(rhs), ptr(X), ldx, ptr(mean_out), stream),
           "qmc_fe1d_lognormal_solve_mean")


def qmc_cbc_step(N: int, crit, zmax: int, gamma: float, p, z_out, d: int, stream=None):
    _check(_lib.qmc_cbc_step(N, ptr(crit), zmax, gamma, ptr(p), ptr(z_out), d, stream), "qmc_cbc_step")


def qmc_plan_info(plan) -> dict:
    buf = (C.c_int64 * 18)()
    _check(_lib.qmc_plan_info(plan, buf), "qmc_plan_info")
    keys = ["family", "N", "m", "s", "phi", "gen", "L", "L1", "L2", "batch_pairs", "D", "p",
            "k1_order", "k1_slots", "k1_chunks", "k1_chunk_slots", "k1_staged_slots", "green_k2_sms"]
    return dict(zip(keys, list(buf)))


def qmc_plan_tables(plan, m: int, N: int, s: int):
    import numpy as np
    gen = C.c_int64(0)
    P = np.empty(m, dtype=np.int32)
    L = np.empty(N, dtype=np.int32)
    e = np.empty(s, dtype=np.int32)
    zeta = np.empty(m, dtype=np.float64)
    _check(_lib.qmc_plan_tables(plan, C.byref(gen), P.ctypes.data_as(_P32), L.ctypes.data_as(_P32),
                                e.ctypes.data_as(_P32), zeta.ctypes.data_as(_PD)), "qmc_plan_tables")
    return gen.value, P, L, e, zeta


def qmc_launch_count() -> int:
    return int(_lib.qmc_launch_count())


def qmc_plan_destroy(plan) -> None:
    _lib.qmc_plan_destroy(plan)


def qmc_strerror(code: int) -> str:
    return strerror(code)


N_KERNEL_CLASSES = 6


def qmc_profile_enable(on: bool) -> None:
    _check(_lib.qmc_profile_enable(1 if on else 0), "qmc_profile_enable")


def qmc_profile_read() -> dict:
    n = N_KERNEL_CLASSES
    launches = (C.c_int64 * n)()
    ms = (C.c_double * n)()
    _check(_lib.qmc_profile_read(launches, ms, n), "qmc_profile_read")
    return {qmc_profile_class_name(i): (int(launches[i]), float(ms[i])) for i in range(n)}


def qmc_profile_class_name(i: int) -> str:
    return _lib.qmc_profile_class_name(i).decode()
