"""Interleaved A/B of fused-update schedules in one process (same inputs,
same thermal state): blocks of 20 launches alternate between variants."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_15676_b200 import _lib, api  # noqa: E402

variants = [int(v) for v in (sys.argv[1:] or ["4", "6"])]
L = _lib.load()
n = 1 << 28
dt = torch.float64 if os.environ.get("AB_DTYPE") == "f64" else torch.float32
bpp = 112 if dt == torch.float64 else 56
props = [torch.randn(n, device="cuda", dtype=dt) for _ in range(4)]
diffs = [0.1 * torch.randn(n, device="cuda", dtype=dt) for _ in range(4)]
pa, pb = torch.zeros(n, device="cuda", dtype=dt), torch.zeros(n, device="cuda", dtype=dt)
upd = api.FusedMetaUpdate(n, dtype=dt)
res = {v: [] for v in variants}
t = 0
for rnd in range(int(os.environ.get("AB_ROUNDS", "8"))):
    for v in variants:
        L.mg_set_option(b"tma_variant", v)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(20):
            upd.step(props[t % 4], diffs[t % 4], pa, pb)
            pa, pb = pb, pa
            t += 1
        b.record()
        torch.cuda.synchronize()
        if rnd > 0:
            res[v].append(a.elapsed_time(b) / 20)
for v in variants:
    ms = np.mean(res[v])
    print(f"variant {v}: {ms:.4f} ms  {bpp * n / ms / 1e6:.1f} GB/s  (per block: "
          f"{' '.join(f'{x:.3f}' for x in res[v])})", flush=True)
