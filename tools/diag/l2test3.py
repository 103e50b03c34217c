"""Does K2 hit L2 on U?  Variants: (a) t=128 X (N,128); (b) t=128 view of X (N,1024);
(c) t=128 plus an unused 600 MB allocation."""
import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1501_06286_b200 as q
import qmc_workloads as W
mode = sys.argv[1]
w = W.config(2, t_override=128)
plan = q.Plan.from_workload(w)
A = q.to_device_colmajor(w.A, "cuda")
if mode == "a":
    X = q.x_empty(plan.N, 128, "cuda")
elif mode == "b":
    X = q.x_empty(plan.N, 1024, "cuda")[:, :128]
elif mode == "c":
    X = q.x_empty(plan.N, 128, "cuda")
    junk = torch.empty(600 << 20, dtype=torch.uint8, device="cuda")
elif mode == "d":  # workspace first, then the big allocation
    plan.call_workspace(128)
    X = q.x_empty(plan.N, 128, "cuda")
    junk = torch.empty(600 << 20, dtype=torch.uint8, device="cuda")
else:  # e: big allocation freed before the workspace (caching allocator reuse)
    junk = torch.empty(600 << 20, dtype=torch.uint8, device="cuda")
    del junk
    X = q.x_empty(plan.N, 128, "cuda")
print("ws ptr", hex(plan.call_workspace(128).data_ptr()), "X", hex(X.data_ptr()))
for _ in range(2):
    plan.matmul(A, X)
torch.cuda.synchronize()
print("ok", mode)
