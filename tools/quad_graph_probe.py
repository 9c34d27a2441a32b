"""configs[0] (64^2 quad, 32^2 RGB texture) optimisation loop: eager vs
CUDA-graph replay, ms per iteration (for ncu: the kernels of one replay)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

s = torch.cuda.Stream()
ctx = api.Context(0, stream=s)
with torch.cuda.stream(s):
    prob = api.QuadTextureProblem(64, 64, 32, target_spp=64, dtype=torch.float32, ctx=ctx)
    run = api.QuadTextureRun(prob, optimizer="meta", lr=0.01)
    run.run(3)
    run.run(4, graph=True)
    for mode in (False, True):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        run.run(200, graph=mode)
        b.record(s)
        torch.cuda.synchronize()
        print("graph" if mode else "eager", "ms/it", round(a.elapsed_time(b) / 200, 4), flush=True)
