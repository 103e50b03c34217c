"""CPU-side checks of the C ABI (no GPU): the library builds, loads and
exports every symbol include/qmc.h declares; host-side validation returns the
documented status codes before anything touches CUDA."""
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def abi():
    import importlib.util
    spec = importlib.util.spec_from_file_location(
        "qmc_build", os.path.join(ROOT, "paper_1501_06286_b200", "build.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    mod.build()
    from paper_1501_06286_b200 import _abi
    return _abi


def declared_functions():
    txt = open(os.path.join(ROOT, "include", "qmc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(qmc_[a-z0-9_]+)\s*\(", txt)))


def test_exports_every_declared_symbol(abi):
    names = declared_functions()
    assert len(names) >= 13
    for n in names:
        assert hasattr(abi._lib, n), n
    assert sorted(abi.EXPORTS) == names


def test_strerror_and_counter(abi):
    assert abi.strerror(0) == "ok"
    for c in range(-9, 0):
        assert abi.strerror(c) != "unknown status"
    assert abi.qmc_launch_count() >= 0


def test_workspace_sizes_and_validation(abi):
    # configs: lattice 257, 65537, 40961, 786433; poly D=16
    for fam, n, s in [(0, 257, 300), (0, 65537, 1024), (0, 40961, 4096), (0, 786433, 8192), (1, 16, 2000)]:
        b = abi.qmc_plan_workspace_size(fam, n, s)
        assert b > 0 and b % 256 == 0
    for fam, n, s, code in [(0, 15, 3, -1), (0, 2, 3, -1), (0, 2 ** 31 + 11, 3, -1), (0, 257, 0, -4),
                            (1, 1, 3, -3), (1, 30, 3, -3), (7, 257, 3, -1)]:
        with pytest.raises(abi.QMCError) as e:
            abi.qmc_plan_workspace_size(fam, n, s)
        assert e.value.code == code


def test_plan_create_host_validation(abi):
    import ctypes as C
    for args, code in [((9, 2, [1, 2], 0), -1), ((13, 2, [0, 2], 0), -2), ((13, 2, [1, 13], 0), -2),
                       ((13, 2, [1, 2], 9), -5)]:
        N, s, z, phi = args
        with pytest.raises(abi.QMCError) as e:
            abi.qmc_plan_create(N, s, z, phi, 256, 1 << 20, None)
        assert e.value.code == code
    with pytest.raises(abi.QMCError) as e:        # p without bit D / even p
        abi.qmc_plan_create_poly(4, 0b1010, 2, [1, 2], 0, 256, 1 << 20, None)
    assert e.value.code == -3
    with pytest.raises(abi.QMCError) as e:        # workspace too small
        abi.qmc_plan_create(13, 2, [1, 2], 0, 256, 16, None)
    assert e.value.code == -8
    rc = abi._lib.qmc_plan_create(None, 13, 2, None, 0, None, 0, None)
    assert rc == -6
    assert abi._lib.qmc_matmul(None, None, 1, 1, None, 1, None, 0, None) == -6


def test_split_choices(abi):
    """FFT length chosen per DESIGN.md §Padding, checked via the workspace
    size formula (W holds L complex values)."""
    # m = 256 -> L = 256; m = 65535 (F_2, D = 16) -> padded L = 2^17
    small = abi.qmc_plan_workspace_size(0, 257, 1)
    big = abi.qmc_plan_workspace_size(1, 16, 1)
    assert big - 131072 * 16 > 0 and small < 64 * 1024
