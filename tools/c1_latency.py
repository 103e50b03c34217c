"""Where config 1's step time goes: per-step CUDA events with L2 flushes of
256 MiB and 1 GiB before each step (the flush keeps the device busy while the
host enqueues the step), back-to-back calls, and the call captured in a CUDA
graph.  One JSON line per mode on stdout."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import paper_1501_06286_b200 as q  # noqa: E402
import qmc_workloads as W  # noqa: E402

dev = torch.device("cuda", 0)
w = W.config(1)
plan = q.Plan.from_workload(w, device=dev)
A = q.to_device_colmajor(w.A, dev)
X = q.x_empty(w.N, w.t, dev)
st = torch.cuda.current_stream(dev)
K = 200


def timed(fn, flush_bytes):
    flush = torch.empty(max(flush_bytes, 1), dtype=torch.uint8, device=dev)
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        if flush_bytes:
            flush.zero_()
        evs[k][0].record(st)
        fn()
        evs[k][1].record(st)
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in evs)
    return {"mean_us": 1e3 * sum(ts) / K, "median_us": 1e3 * ts[K // 2], "min_us": 1e3 * ts[0]}


def step():
    plan.matmul(A, X)


for fb in (256 << 20, 1 << 30):
    print(json.dumps({"mode": f"events_flush_{fb >> 20}MiB", **timed(step, fb)}))
# back to back: K calls between two events
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(st)
for _ in range(K):
    step()
e1.record(st)
torch.cuda.synchronize()
print(json.dumps({"mode": "back_to_back", "per_call_us": 1e3 * e0.elapsed_time(e1) / K}))
# CUDA graph of the call
try:
    s2 = torch.cuda.Stream(dev)
    s2.wait_stream(st)
    with torch.cuda.stream(s2):
        step()
    st.wait_stream(s2)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        step()
    Xref = X.clone()
    X.zero_()
    g.replay()
    torch.cuda.synchronize()
    same = bool(torch.equal(X, Xref))
    for fb in (256 << 20, 1 << 30):
        print(json.dumps({"mode": f"graph_flush_{fb >> 20}MiB", "bitwise_equal": same, **timed(g.replay, fb)}))
except Exception as e:  # noqa: BLE001
    print(json.dumps({"mode": "graph", "error": repr(e)[:300]}))
