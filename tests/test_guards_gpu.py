"""Guard zones around every buffer the library writes (compute-sanitizer is
closed on this GPU pool; this and the checked build, tools/check_build.sh,
stand in for memcheck): the plan workspace, the call workspace, X (with a
leading dimension wider than t, so the gaps between rows are guarded too),
out and A are carved out of larger buffers whose surroundings hold a NaN
bit pattern; after plan creation and the calls, every guard byte must be
unchanged, and X / the means must still match the oracle."""
import numpy as np
import pytest

import oracle as O
import qmc_workloads as W
from _ref import X_full, col_tolerance

pytestmark = pytest.mark.gpu

GUARD = 4096  # bytes on each side (256-byte aligned)
PATTERN = np.uint64(0x7FF8DEADBEEF1234)


@pytest.fixture(scope="module")
def abi():
    import torch
    assert torch.cuda.is_available(), "GPU tests need CUDA"
    from paper_1501_06286_b200 import _abi
    return _abi


def _guarded(nbytes):
    """A device buffer of nbytes with GUARD bytes of pattern on each side."""
    import torch
    n64 = (nbytes + 2 * GUARD + 7) // 8
    buf = torch.full((n64,), int(PATTERN.view(np.int64)), dtype=torch.int64, device="cuda")
    return buf, buf.data_ptr() + GUARD


def _guards_intact(buf, nbytes):
    h = buf.cpu().numpy().view(np.uint64)
    lo = h[: GUARD // 8]
    hi_start = (GUARD + nbytes + 7) // 8
    hi = h[hi_start:]
    return bool(np.all(lo == PATTERN) and np.all(hi == PATTERN))


CASES = [  # (name, workload factory, f)
    ("one_row_c1", lambda: W.config(1), None),
    ("pipe_k2_rowsum", lambda: W.custom_lattice(65537, 64, 64, W.PHI_INVNORM_MID, seed=3), W.F_ROWMEAN_RELU),
    ("two_stage_exp", lambda: W.custom_lattice(786433, 40, 34, W.PHI_INVNORM_MID, seed=4), W.F_EXP),
    ("padded_poly_affine", lambda: W.custom_poly(12, 4179, 300, 18, W.PHI_SHIFT_HALF, seed=5), W.F_AFFINE),
    ("multichunk_direct", lambda: W.custom_lattice(40961, 4096, 6, W.PHI_SHIFT_HALF, seed=6), W.F_IDENTITY),
    ("dense_first_pass", lambda: W.custom_lattice(7681, 15360, 4, W.PHI_SHIFT_HALF, seed=7), None),
]


@pytest.mark.parametrize("name,make,f", CASES, ids=[c[0] for c in CASES])
def test_no_write_outside_buffers(abi, name, make, f):
    import torch
    w = make()
    w.A = np.asfortranarray(w.A * 0.05)
    fam = abi.QMC_FAMILY_POLY if w.family == "poly" else abi.QMC_FAMILY_LATTICE
    nplan = abi.qmc_plan_workspace_size(fam, w.D if w.family == "poly" else w.N, w.s)
    pbuf, pws = _guarded(nplan)
    st = torch.cuda.current_stream().cuda_stream
    if w.family == "poly":
        h = abi.qmc_plan_create_poly(w.D, w.p, w.s, w.z, w.phi, pws, nplan, st)
    else:
        h = abi.qmc_plan_create(w.N, w.s, w.z, w.phi, pws, nplan, st)
    try:
        N, s, t = w.N, w.s, w.t
        lda, ldx = s + 3, t + 5                      # padded leading dimensions (odd ldx)
        abuf, Ap = _guarded(lda * t * 8)
        A_host = np.zeros((t, lda))
        A_host[:, :s] = w.A.T
        # A into its guarded slot: a float64 view of the int64 buffer
        abuf.view(torch.float64)[GUARD // 8: GUARD // 8 + lda * t] = torch.from_numpy(A_host.ravel()).cuda()
        xbuf, Xp = _guarded(N * ldx * 8)
        fcall = abi.QMC_F_NONE if f is None else f
        ncall = abi.qmc_call_workspace_size(h, t, fcall)
        cbuf, cws = _guarded(ncall)
        nout = N if f == W.F_ROWMEAN_RELU else t
        obuf, outp = _guarded(nout * 8)
        if f is None:
            abi.qmc_matmul(h, Ap, lda, t, Xp, ldx, cws, ncall, st)
        else:
            abi.qmc_mean(h, Ap, lda, t, f, 0.25, outp, Xp, ldx, cws, ncall, st)
        torch.cuda.synchronize()
        for buf, n in ((pbuf, nplan), (abuf, lda * t * 8), (xbuf, N * ldx * 8), (cbuf, ncall), (obuf, nout * 8)):
            assert _guards_intact(buf, n)
        # X itself is right, and the padding columns t..ldx-1 of every row are untouched
        Xall = xbuf.cpu().numpy().view(np.uint64)[GUARD // 8: GUARD // 8 + N * ldx].reshape(N, ldx)
        assert np.all(Xall[:, t:] == PATTERN)
        Xg = Xall[:, :t].view(np.float64)
        Xo = X_full(w)
        if f == W.F_AFFINE:
            Xg = Xg - 0.25
        assert np.all(np.abs(Xg - Xo).max(axis=0) <= col_tolerance(w))
    finally:
        abi.qmc_plan_destroy(h)


def test_report_build_flags(abi):
    """Which build ran this suite (bit 0: the checked build); printed for the
    evidence log of tools/check_build.sh."""
    f = abi.qmc_build_flags()
    print(f"libqmc build flags = {f} ({'checked' if f & 1 else 'product'} build)")
    assert f in (0, 1, 2, 3)


def test_plan_shift_guards(abi):
    """qmc_plan_shift writes only its own shift workspace (ζ, φ(x_0), W):
    the base plan's workspace is bitwise unchanged and the shift workspace's
    guards intact; bad requests are rejected with their status."""
    import torch
    w = W.custom_lattice(65537, 64, 6, W.PHI_INVNORM_MID, seed=11)
    nplan = abi.qmc_plan_workspace_size(abi.QMC_FAMILY_LATTICE, w.N, w.s)
    pbuf, pws = _guarded(nplan)
    st = torch.cuda.current_stream().cuda_stream
    h = abi.qmc_plan_create(w.N, w.s, w.z, w.phi, pws, nplan, st)
    hs = None
    try:
        before = pbuf.clone()
        nsh = abi.qmc_shift_workspace_size(h)
        assert nsh < nplan
        sbuf, sws = _guarded(nsh)
        hs = abi.qmc_plan_shift(h, 0.3, sws, nsh, st)
        torch.cuda.synchronize()
        assert torch.equal(pbuf, before)
        assert _guards_intact(sbuf, nsh)
        with pytest.raises(abi.QMCError) as e:
            abi.qmc_plan_shift(h, 1.0, sws, nsh, st)
        assert e.value.code == -5
        with pytest.raises(abi.QMCError) as e:
            abi.qmc_plan_shift(h, 0.3, sws, nsh - 8, st)
        assert e.value.code == -8
        D, p = 8, 285
        npoly = abi.qmc_plan_workspace_size(abi.QMC_FAMILY_POLY, D, 3)
        ppoly = torch.empty(npoly, dtype=torch.uint8, device="cuda")
        hp = abi.qmc_plan_create_poly(D, p, 3, [1, 2, 3], W.PHI_SHIFT_HALF, ppoly, npoly, st)
        try:
            with pytest.raises(abi.QMCError) as e:
                abi.qmc_plan_shift(hp, 0.3, sws, nsh, st)
            assert e.value.code == abi.QMC_EUNSUPPORTED
        finally:
            abi.qmc_plan_destroy(hp)
    finally:
        if hs is not None:
            abi.qmc_plan_destroy(hs)
        abi.qmc_plan_destroy(h)
