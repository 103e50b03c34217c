"""CPU oracle for the fast QMC matrix product X = Y·A (arXiv 1501.06286).

TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the package
``paper_1501_06286_b200``) may import, call or execute anything in this
directory; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it.

The oracle is the *plain definition* of what the fast method reaches
("we want to have a fast method to compute YA = B"):
it forms Y explicitly from the conventional lattice points
{n·z_j/N} or the polynomial-lattice points over F_2,
applies φ element-wise and multiplies directly.
No primitive root, no reordering and no FFT are used to form X.

Independent of the CUDA path: no shared code, headers, tables or
constants; the only shared module is ``qmc_workloads`` (seeded input
generators, no arithmetic of the method).

Parity pins (see tests/test_oracle_pins.py and DESIGN.md §Oracle):
every function below is pinned by printed values of the paper's worked
example, closed forms, invariants or brute force.  The two fused
functionals have no closed form in general and are pinned by special
cases: ``rowmean_relu`` (config 2's scalar) by the worked example and the
no-clipping / all-clipped cases, the ``exp`` column mean (config 5) by
A = 0 and the geometric sum for equal z.
"""
from .qmc_oracle import *  # noqa: F401,F403
from .qmc_oracle import __all__  # noqa: F401
