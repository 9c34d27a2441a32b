"""Launch list probe for the mt64 (exact-stream) mini-render: three
iterations each of the IEEE kernel and four fast-kernel schedules, 16.7M
pixels, spp = argv[1].  Run under `ncu --metrics gpu__time_duration.sum` to
compare the render kernels; the mt_draw / mt_jump launches are the side
stream's block generation."""
import sys, os, torch
sys.path.insert(0, os.getcwd())
from paper_2309_15676_b200 import _lib, api
L = _lib.load()
spp = int(sys.argv[1])
run = api.MiniRenderRun(1 << 24, spp, gen_seed=1, lr=0.01, rng="mt64", dtype=torch.float32)
for fast, v in ((0, -1), (1, 0), (1, 3), (1, 10), (1, 12)):
    L.mg_set_option(b"render_fast", fast); L.mg_set_option(b"render_fast_variant", v)
    for _ in range(3): run.step()
    torch.cuda.synchronize()
