"""Fused Adam update at 2^28 fp32 (BASELINE configs[1]'s Adam baseline):
mean ms per step over 10 blocks of 20 back-to-back steps after 5 warm-up
steps; with MG_LIB set, times that library build."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

n = 1 << 28
g = [torch.randn(n, device="cuda") for _ in range(2)]
pa, pb = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
upd = api.FusedAdamUpdate(n)
t = 0
for _ in range(5):
    upd.step(g[t % 2], pa, pb)
    pa, pb, t = pb, pa, t + 1
torch.cuda.synchronize()
ms = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        upd.step(g[t % 2], pa, pb)
        pa, pb, t = pb, pa, t + 1
    b.record()
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(b) / 20)
m = sum(ms) / len(ms)
print(f"adam 2^28 f32: {m:.4f} ms  {28 * n / m / 1e6:.1f} GB/s", flush=True)
