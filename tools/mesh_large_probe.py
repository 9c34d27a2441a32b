"""configs[4] full-scale iteration timing (1024^2, 16 objects / ~502k
triangles, 16 x 5 x 1024^2 = 83.9M parameters, depth 8, 1 FD + 4 prop spp)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

t0 = time.time()
prob = api.MeshLargeProblem(target_spp=2)
print("setup s", round(time.time() - t0, 2), prob.scene.info(), flush=True)
run = api.MeshTextureRun(prob, "meta", lr=0.005)
for _ in range(2):
    run.step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
K = 3
for _ in range(K):
    run.step()
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / K
print("ms/it", round(ms, 2), "paths/s", f"{prob.draws_per_sample() / (ms / 1e3):.3e}",
      "mem GB", round(torch.cuda.max_memory_allocated() / 1e9, 2), flush=True)
