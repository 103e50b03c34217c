"""Build libqmc.so in-tree with nvcc for sm_100a (B200).

    python -m paper_1501_06286_b200.build [--verbose]

Cross-compiles without a GPU.  The .so lands next to this file so that the
gpurun snapshot carries it to the B200 box.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libqmc.so")
SOURCES = ["plan.cu", "pipeline.cu", "pde.cu", "cbc.cu"]
HEADERS = ["fft.cuh", "qmc_internal.cuh", "rowcfg.cuh"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "qmc.h"))
    deps.append(os.path.abspath(__file__))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile_link(out: str, flags: list) -> str:
    """Each translation unit compiled on its own thread (no device code is
    shared between them), then one shared-library link; returns nvcc's
    stderr."""
    import concurrent.futures as cf
    import tempfile

    tmp = tempfile.mkdtemp(prefix="qmc_build_")
    objs = [os.path.join(tmp, f + ".o") for f in SOURCES]
    cflags = [f for f in NVCC_FLAGS if f != "-shared"] + flags
    cmds = [[_nvcc(), *cflags, "-c", "-o", o, os.path.join(CSRC, f)] for f, o in zip(SOURCES, objs)]
    with cf.ThreadPoolExecutor(len(cmds)) as ex:
        results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
    errs = "".join(r.stdout + r.stderr for r in results)
    if any(r.returncode != 0 for r in results):
        raise RuntimeError("nvcc failed:\n" + errs)
    res = subprocess.run([_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", out, *objs],
                         capture_output=True, text=True)
    for o in objs:
        os.remove(o)
    os.rmdir(tmp)
    if res.returncode != 0:
        raise RuntimeError("nvcc link failed:\n" + res.stdout + res.stderr)
    return errs


def build(force: bool = False, verbose: bool = False, out: str | None = None, extra: list | None = None) -> str:
    """Compile libqmc.so (or, with `out`, a variant build with `extra` flags)."""
    if out is not None:
        _compile_link(os.path.abspath(out), list(extra or []))
        return out
    if not force and not _stale():
        return LIB
    flags = os.environ.get("QMC_NVCC_EXTRA", "").split()
    if verbose:
        flags += ["-Xptxas", "-v"]
    errs = _compile_link(LIB + ".tmp", flags)
    if verbose:
        sys.stderr.write(errs)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose="--verbose" in sys.argv))
