"""Fused meta update time vs parameter count and options (projection,
sparse gradients as in the mesh runs)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402


def run(n, project_lo=None, sparse=False, steps=20):
    g = torch.Generator(device="cuda").manual_seed(0)
    prop = torch.randn(n, device="cuda", generator=g)
    diff = 0.1 * torch.randn(n, device="cuda", generator=g)
    if sparse:
        prop[n // 4:] = 0
        diff[n // 4:] = 0
    p0 = torch.rand(n, device="cuda", generator=g)
    p1 = p0.clone()
    upd = api.FusedMetaUpdate(n, lr=0.01, project_lo=project_lo)
    for _ in range(3):
        upd.step(prop, diff, p0, p1)
        p0, p1 = p1, p0
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        upd.step(prop, diff, p0, p1)
        p0, p1 = p1, p0
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / steps
    gbs = 56 * n / ms / 1e6
    print(f"n {n:>10d} proj {project_lo} sparse {sparse}: {ms:.3f} ms  {gbs:.0f} GB/s", flush=True)


if __name__ == "__main__":
    for n in (1 << 24, 83886080, 1 << 27, 1 << 28):
        run(n)
    run(83886080, 0.0)
    run(83886080, 0.0, True)
    run(1 << 28, 0.0, True)
