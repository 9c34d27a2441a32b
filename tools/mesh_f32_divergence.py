"""fp32 fast mode of the mesh renderer (fp32 traversal) vs the fp64 parity
mode: fraction of pixels whose 1-spp radiance differs by > 1e-3 relative
(path divergence), and the agreement of the gradient sample pair."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

prob = api.MeshTextureProblem(256, 256, 64, max_vertices=6, target_spp=4, dtype=torch.float64)
n = prob.dim()
th = torch.tensor(np.random.RandomState(0).uniform(0.2, 0.8, n), device="cuda")
i64 = prob.scene.render(th, 256, 256, 1, 77).cpu().numpy().reshape(3, -1)
i32 = prob.scene.render(th.float(), 256, 256, 1, 77).double().cpu().numpy().reshape(3, -1)
rel = np.abs(i32 - i64) / np.maximum(np.abs(i64), 1e-2)
print("pixel fraction diverged (1e-3 rel)", float(np.mean(rel.max(0) > 1e-3)),
      "median rel of the rest", float(np.median(rel.max(0)[rel.max(0) <= 1e-3])))
p64 = prob.sample_pair(th, th * 0.99, 3, key=5)
g64 = p64.prop.clone()
prob32 = api.MeshTextureProblem(256, 256, 64, max_vertices=6, target_spp=4, dtype=torch.float32)
prob32.target_img = prob.target_img.float()
g32 = prob32.sample_pair(th.float(), (th * 0.99).float(), 3, key=5).prop.double()
print("prop rel L2 err", float(torch.linalg.vector_norm(g32 - g64) / torch.linalg.vector_norm(g64)),
      "cos", float(torch.dot(g32, g64) / torch.linalg.vector_norm(g32) / torch.linalg.vector_norm(g64)))
