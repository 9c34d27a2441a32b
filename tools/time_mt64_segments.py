"""Breakdown of the segmented mt64 mode per iteration: draw / jump / render."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_15676_b200 import _lib, api  # noqa: E402

P, spp = 1 << 24, 2
D = P * spp
for gmax in (148, 296, 592, 1184):
    L = 312 * (-(-(-(-D // gmax)) // 312))
    G = -(-D // L)
    rng = api.Rng.split(12345, G, L)
    u = torch.empty(G * L, dtype=torch.float64, device="cuda")
    lib = _lib.load()
    rng.jump(D - L)  # warm the polynomial cache
    for name, fn in (("draw", lambda: lib.mg_mt64_draw(rng.ctx.h, rng.h, L, 1,
                                                         api._p(u))),
                     ("jump", lambda: rng.jump(D - L))):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        t0 = time.time()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            fn()
        e1.record()
        torch.cuda.synchronize()
        print(f"G={G} L={L} {name}: {e0.elapsed_time(e1) / 5:.3f} ms (wall {(time.time() - t0) / 5 * 1e3:.3f} ms)",
              flush=True)
