"""configs[3] / configs[4] optimisation loops: eager vs CUDA-graph replay
(MeshTextureRun.run(k, graph=True)), ms per iteration."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

s = torch.cuda.Stream()
ctx = api.Context(0, stream=s)
with torch.cuda.stream(s):
    for name in sys.argv[1:] or ["configs3", "configs4"]:
        if name == "configs3":
            prob = api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4,
                                          dtype=torch.float32, ctx=ctx)
        else:
            prob = api.MeshLargeProblem(target_spp=2, ctx=ctx)
        run = api.MeshTextureRun(prob, "meta", lr=0.005)
        run.run(3)
        run.run(2, graph=True)
        for mode in (False, True, False, True):
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            run.run(20, graph=mode)
            b.record(s)
            torch.cuda.synchronize()
            print(name, "graph" if mode else "eager", "ms/it", round(a.elapsed_time(b) / 20, 4),
                  flush=True)
