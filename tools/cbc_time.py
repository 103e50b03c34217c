"""Time the GPU fast CBC construction: total for s
components (plan of all N-1 generators included) and, from the difference of
two lengths, the cost per component."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1501_06286_b200 as q  # noqa: E402


def run(N, s):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    z = q.cbc_lattice(N, s, 0.9)
    torch.cuda.synchronize()
    return time.perf_counter() - t0, z


for N, s1, s2 in [(65537, 8, 128), (786433, 4, 36)]:
    run(N, 2)  # warm-up
    a, _ = run(N, s1)
    b, z = run(N, s2)
    print(f"N={N}: s={s1} {a * 1e3:.1f} ms, s={s2} {b * 1e3:.1f} ms -> "
          f"{(b - a) / (s2 - s1) * 1e6:.1f} us per component, plan+setup ~{(a - s1 * (b - a) / (s2 - s1)) * 1e3:.1f} ms")
