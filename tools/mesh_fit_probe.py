"""Diagnostic: configs[3]-style texture fit on a small mesh scene — texture
error (texels seen in the first 30 iterations) vs iteration for meta / Adam."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

W, H, R, iters = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
for opt, lr in [("meta", 0.005), ("meta", 0.01), ("meta", 0.02), ("adam", 0.01), ("adam", 0.03)]:
    prob = api.MeshTextureProblem(W, H, R, (12, 24), (24, 32), max_vertices=4, target_spp=16,
                                  dtype=torch.float32)
    run = api.MeshTextureRun(prob, opt, lr=lr)
    seen = torch.zeros(prob.dim(), dtype=torch.bool, device="cuda")
    p0 = run.params.clone()
    out = []
    for i in range(iters):
        pair = run.step()
        if i < 30:
            seen |= pair.prop != 0
        if i in (0, iters // 4, iters // 2, iters - 1):
            out.append((i, float(torch.linalg.vector_norm((run.params - prob.target_tex)[seen])),
                        run.loss_estimate()))
    e_init = float(torch.linalg.vector_norm((p0 - prob.target_tex)[seen]))
    print(opt, lr, "seen", int(seen.sum()), "init err", round(e_init, 3),
          [(i, round(e, 3), round(l, 2)) for i, e, l in out], flush=True)
