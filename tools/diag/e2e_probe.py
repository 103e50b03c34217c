"""Where does the end-to-end (host buffers, synchronous) call spend its time?
Config 2: device-only steps back to back, device-only steps with a host sync
after each, and qmc_mean_host; all timed by CUDA events on the caller's stream."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1501_06286_b200 as q  # noqa: E402
import qmc_workloads as W  # noqa: E402
from paper_1501_06286_b200 import _abi as abi  # noqa: E402

w = W.config(int(os.environ.get("CFG", "2")))
plan = q.Plan.from_workload(w)
A = q.to_device_colmajor(w.A, "cuda")
X = q.x_empty(plan.N, w.t, "cuda")
st = torch.cuda.current_stream()
f = w.f if w.f is not None else W.F_IDENTITY


flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
FLUSH = os.environ.get("FLUSH") == "1"


def timed(fn, n=20, sync_each=False):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        if FLUSH:
            flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        if sync_each:
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
    torch.cuda.synchronize()
    if not sync_each:
        ts = [a.elapsed_time(b)]
    return sorted(ts)[len(ts) // 2]


def dev_step():
    out = plan.mean(A, f, w.f_param, X=X)
    if f == W.F_ROWMEAN_RELU:
        plan.finalize(f, out, w.t)


A_pin = torch.from_numpy(w.A.T.copy()).pin_memory()  # (t, s) rows = columns of A
A_dev2 = torch.empty_like(A_pin, device="cuda")
out_pin = torch.empty(max(plan.N, w.t), dtype=torch.float64).pin_memory()
out_dev = torch.empty(max(plan.N, w.t), dtype=torch.float64, device="cuda")
ws = plan.call_workspace(w.t, f)


def host_step():
    abi.qmc_mean_host(plan.handle, A_pin, w.s, w.t, f, w.f_param, out_pin, A_dev2, X, w.t, out_dev, ws, ws.numel(),
                      st.cuda_stream)


def copy_only():
    A_dev2.copy_(A_pin, non_blocking=True)


print("device step, sync each  ", round(timed(dev_step, sync_each=True), 4))
print("H2D copy of A only      ", round(timed(copy_only, sync_each=True), 4))
print("qmc_mean_host           ", round(timed(host_step, sync_each=True), 4))
