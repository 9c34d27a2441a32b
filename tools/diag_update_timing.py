"""Per-launch timing of the fused update over a long run (power/clock drift
diagnostic): prints the launch-time percentiles for pool sizes 2 and 4."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_15676_b200 import api  # noqa: E402

n = 1 << 28
for pool in (2, 4):
    props = [torch.randn(n, device="cuda") for _ in range(pool)]
    diffs = [0.1 * torch.randn(n, device="cuda") for _ in range(pool)]
    pa, pb = torch.zeros(n, device="cuda"), torch.zeros(n, device="cuda")
    upd = api.FusedMetaUpdate(n, dtype=torch.float32)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(120)]
    for t, (a, b) in enumerate(ev):
        a.record()
        upd.step(props[t % pool], diffs[t % pool], pa, pb)
        b.record()
        pa, pb = pb, pa
    torch.cuda.synchronize()
    ms = np.array([a.elapsed_time(b) for a, b in ev])
    print(f"pool={pool}: first10 {ms[:10].mean():.3f} ms, 20-60 {ms[20:60].mean():.3f}, "
          f"60-120 {ms[60:].mean():.3f}, p50 {np.median(ms):.3f}, min {ms.min():.3f}", flush=True)
    del props, diffs, pa, pb, upd
    torch.cuda.empty_cache()
