"""Times every schedule of the fused meta update (register-streaming kernel
and the TMA-pipeline variants of update.cu) at one size; prints GB/s.
Usage: python tools/sweep_update_variants.py [--n 268435456] [--dtype f32]"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_15676_b200 import _lib, api  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1 << 28)
ap.add_argument("--dtype", default="f32")
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
dt = torch.float32 if a.dtype == "f32" else torch.float64
L = _lib.load()
n = a.n
props = [torch.randn(n, device="cuda", dtype=dt) for _ in range(2)]
diffs = [0.1 * torch.randn(n, device="cuda", dtype=dt) for _ in range(2)]
pa, pb = torch.zeros(n, device="cuda", dtype=dt), torch.zeros(n, device="cuda", dtype=dt)
peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
bpp = 56 if a.dtype == "f32" else 112
res = {}
for name, opts in [("register", {"disable_tma": 1})] + [
        (f"tma{v}", {"disable_tma": 0, "tma_variant": v}) for v in range(10)]:
    for k, v in opts.items():
        L.mg_set_option(k.encode(), v)
    upd = api.FusedMetaUpdate(n, dtype=dt)
    for t in range(3):
        upd.step(props[t % 2], diffs[t % 2], pa, pb)
        pa, pb = pb, pa
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(a.reps):
        upd.step(props[t % 2], diffs[t % 2], pa, pb)
        pa, pb = pb, pa
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    gbs = bpp * n / ms / 1e6
    res[name] = {"ms": round(ms, 4), "gbs": round(gbs, 1), "frac": round(gbs / peak, 4)}
    print(name, res[name], flush=True)
    del upd
L.mg_set_option(b"disable_tma", 0)
L.mg_set_option(b"tma_variant", -1)
print(json.dumps(res))
