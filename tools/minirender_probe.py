"""Fused mini-render iteration at 16.7M pixels (philox, fp32) for ncu."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

run = api.MiniRenderRun(1 << 24, 2, gen_seed=1, lr=0.01, rng="philox", dtype=torch.float32)
for _ in range(6):
    run.step()
torch.cuda.synchronize()
