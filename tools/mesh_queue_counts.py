"""Per-depth wavefront queue sizes (paths entering isect, shadow rays) of
one configs[4] and one configs[3] sample pair, with the stage times of the
launch list beside them in DESIGN.md."""
import ctypes as C
import sys
sys.path.insert(0, ".")
import torch
from paper_2309_15676_b200 import api, _lib
L = _lib.load()
for name, make in (("configs4", lambda: api.MeshLargeProblem(target_spp=2)),
                   ("configs3", lambda: api.MeshTextureProblem(512, 512, 512, max_vertices=6,
                                                              target_spp=4, dtype=torch.float32))):
    prob = make()
    run = api.MeshTextureRun(prob, "meta", lr=0.005)
    for _ in range(3):
        run.step()
    out = (C.c_uint32 * 18)()
    assert L.mg_meshscene_queue_counts(prob.ctx.h, prob.scene.h, 18, out) == 0
    print(name, "paths per depth", list(out[:9]), "shadow rays", list(out[9:18]), flush=True)
