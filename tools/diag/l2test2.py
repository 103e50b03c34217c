import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1501_06286_b200 as q
import qmc_workloads as W
w = W.config(2, t_override=16)
plan = q.Plan.from_workload(w)
A = q.to_device_colmajor(w.A, "cuda")
X = q.x_empty(plan.N, w.t, "cuda")
for _ in range(2):
    plan.matmul(A, X)
    u = plan._ws[: 8 << 20].view(torch.float64)
    s1 = u.sum()
    s2 = u.sum()
torch.cuda.synchronize()
print("ok", float(s1), plan._ws.data_ptr() % 4096)
