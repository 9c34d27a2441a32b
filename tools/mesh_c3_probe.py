"""configs[3] iteration timing (512^2, 3 objects / 22k triangles, 3.1M
texture parameters, depth 6, 1 FD + 2 prop spp; wavefront, fused update)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

prob = api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4, dtype=torch.float32)
run = api.MeshTextureRun(prob, optimizer="meta", lr=0.005)
for _ in range(3):
    run.step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    run.step()
b.record()
torch.cuda.synchronize()
print("ms/it", round(a.elapsed_time(b) / 5, 4), prob.scene.info(), flush=True)
