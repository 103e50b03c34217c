import torch
n = (8 << 20) // 8
b = torch.empty(n, dtype=torch.float64, device="cuda")
c = torch.empty(n, dtype=torch.float64, device="cuda")
for it in range(3):
    b.fill_(1.0 + it)       # write 8 MB
    s = b.sum()             # read it back
    c.copy_(b)              # read b again + write c
    s2 = c.sum()
torch.cuda.synchronize()
print("ok", float(s), float(s2))
