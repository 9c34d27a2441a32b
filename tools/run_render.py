"""Fused mini-render iterations at scale (profiling / timing helper)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_15676_b200 import api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pixels", type=int, default=1 << 24)
ap.add_argument("--spp", type=int, default=2)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--rng", default="philox")
ap.add_argument("--scalar", action="store_true", help="one pixel per thread (no 16B packs)")
a = ap.parse_args()
if a.scalar:
    from paper_2309_15676_b200 import _lib
    _lib.load().mg_set_option(b"render_vec", 0)
dt = torch.float32 if a.dtype == "f32" else torch.float64
run = api.MiniRenderRun(a.pixels, a.spp, gen_seed=1, lr=0.01, rng=a.rng, dtype=dt)
for _ in range(2):
    run.step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.iters):
    run.step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.iters
print(f"pixels={a.pixels} spp={a.spp} ms/iter={ms:.4f} pairs/s={a.pixels * a.spp / ms * 1e3:.4g} "
      f"loss={run.scalars().loss:.6g}")
