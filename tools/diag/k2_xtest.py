"""K2 cost with and without the X write (is the scattered row-chunk write the
limiter?): config 2, one stream, per-class event times per step."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("QMC_ONE_STREAM", "1")
import torch  # noqa: E402

import paper_1501_06286_b200 as q  # noqa: E402
import qmc_workloads as W  # noqa: E402
from paper_1501_06286_b200 import _abi as abi  # noqa: E402

w = W.config(2)
plan = q.Plan.from_workload(w)
A = q.to_device_colmajor(w.A, "cuda")
X = q.x_empty(plan.N, w.t, "cuda")
for name, fn in [("matmul (X written)", lambda: plan.matmul(A, X)),
                 ("mean IDENTITY, no X", lambda: plan.mean(A, W.F_IDENTITY, 0.0)),
                 ("mean IDENTITY + X", lambda: plan.mean(A, W.F_IDENTITY, 0.0, X=X))]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    abi.qmc_profile_read()
    abi.qmc_profile_enable(True)
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    abi.qmc_profile_enable(False)
    prof = abi.qmc_profile_read()
    print(name, {k: round(v[1] / 10, 4) for k, v in prof.items() if v[0]})
