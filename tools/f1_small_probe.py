"""configs[0] quad and configs[2] helix iterations (for ncu captures)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "quad"
if which == "quad":
    prob = api.QuadTextureProblem(1024, 1024, 512, target_spp=16, dtype=torch.float32)
    run = api.QuadTextureRun(prob, "meta", lr=0.01)
else:
    prob = api.HelixProblem(256, 256, target_spp=16, dtype=torch.float32)
    run = api.HelixRun(prob, "meta", lr=0.01)
for _ in range(5):
    run.step()
torch.cuda.synchronize()
