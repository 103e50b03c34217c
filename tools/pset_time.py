"""Korobov p-set timing: the one-plan batched launch (qmc_pset_matmul) against
one lattice plan per block (both write the same X); CUDA events, median of 10."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1501_06286_b200 as q  # noqa: E402

out = []
for K, s, t in [(257, 64, 16), (257, 256, 64), (1021, 64, 16), (1021, 256, 64)]:
    rng = np.random.default_rng(K)
    A = q.to_device_colmajor(rng.standard_normal((s, t)), "cuda")
    ps = q.KorobovPSet(K, s, q.QMC_PHI_SHIFT_HALF)
    res = {"K": K, "s": s, "t": t, "N": (K - 1) ** 2}
    for name, pb in (("batched_one_plan", False), ("per_block_plans", True)):
        for _ in range(3):
            ps.matmul(A, per_block=pb)
        ts = []
        for _ in range(10):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ps.matmul(A, per_block=pb)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        res[name + "_ms"] = sorted(ts)[len(ts) // 2]
    res["speedup"] = res["per_block_plans_ms"] / res["batched_one_plan_ms"]
    out.append(res)
    print(json.dumps(res), flush=True)
