"""configs[3] mesh iteration timing, wavefront vs megakernel."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402
from paper_2309_15676_b200._lib import check, load  # noqa: E402

ctx = api.Context.default()
t0 = time.time()
mprob = api.MeshTextureProblem(512, 512, 512, max_vertices=6, target_spp=4, dtype=torch.float32,
                               ctx=ctx)
print("setup", round(time.time() - t0, 3), mprob.scene.info(), flush=True)
for mode in (0, 1, 0):
    check(load().mg_set_option(b"mesh_megakernel", mode))
    mrun = api.MeshTextureRun(mprob, optimizer="meta", lr=0.005)
    for _ in range(2):
        mrun.step()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5):
        mrun.step()
    b.record()
    torch.cuda.synchronize()
    print("megakernel" if mode else "wavefront", "ms/it", round(a.elapsed_time(b) / 5, 3),
          "loss", mrun.loss_estimate(), flush=True)
