"""Fused mini-render iteration at 16.7M pixels with the exact mt19937_64 stream."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

run = api.MiniRenderRun(1 << 24, 2, gen_seed=1, lr=0.01, rng="mt64", dtype=torch.float32)
for _ in range(2):
    run.step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(32):
    run.step()
b.record()
torch.cuda.synchronize()
print("engines", run.rng.n, "K", run.block_iters, "ms/it", a.elapsed_time(b) / 32)
