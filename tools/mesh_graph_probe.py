"""Upper bound on what CUDA-graph capture of one mesh iteration would save:
eager iteration vs replay of a captured iteration (the replay reuses the
captured iteration number and buffers, so only its timing is meaningful)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402


def timed(fn, k):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(k):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / k


s = torch.cuda.Stream()
ctx = api.Context(0, stream=s)
for name in ("configs3", "configs4"):
    if name == "configs3":
        prob = api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4,
                                      dtype=torch.float32, ctx=ctx)
    else:
        prob = api.MeshLargeProblem(target_spp=2, ctx=ctx)
    run = api.MeshTextureRun(prob, "meta", lr=0.005)
    with torch.cuda.stream(s):
        for _ in range(3):
            run.step()
        torch.cuda.synchronize()
        eager = timed(run.step, 10)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            run.step()
        g.replay()
        torch.cuda.synchronize()
        graph = timed(g.replay, 10)
    print(name, "eager ms/it", round(eager, 4), "graph replay ms/it", round(graph, 4), flush=True)
