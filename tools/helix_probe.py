"""configs[2] iteration timing (fp32 / fp64)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

for dt in (torch.float32, torch.float64):
    prob = api.HelixProblem(256, 256, target_spp=16, dtype=dt)
    run = api.HelixRun(prob, "meta", lr=0.01)
    for _ in range(2):
        run.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        run.step()
    b.record()
    torch.cuda.synchronize()
    print(dt, "ms/it", round(a.elapsed_time(b) / 20, 4), flush=True)
