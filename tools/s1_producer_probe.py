"""The cluster runner's mt19937_64 producer alone (mg_mt_stream_probe): time
to stream the S1 run's 200 x 8192 raw engine words, and the tempered draws
against the sequential engine (Rng.stream(...).uniform) bit for bit."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2309_15676_b200 import _lib, api  # noqa: E402

L = _lib.load()
ctx = api.Context.default()
total = 200 * 8192
out = torch.empty(total, dtype=torch.float64, device="cuda")
prog = torch.zeros(1, dtype=torch.int64, device="cuda")
p = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
for _ in range(2):
    L.mg_mt_stream_probe(ctx.h, 0, 0, total, p(out), p(prog))
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    L.mg_mt_stream_probe(ctx.h, 0, 0, total, p(out), p(prog))
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 5
ref = api.Rng.stream(0, 0).uniform(4096)
# the producer streams raw engine words: temper + uniform() on the host
import numpy as np  # noqa: E402
z = out[:4096].view(torch.int64).cpu().numpy().view(np.uint64).copy()
z ^= (z >> np.uint64(29)) & np.uint64(0x5555555555555555)
z ^= (z << np.uint64(17)) & np.uint64(0x71d67fffeda60000)
z ^= (z << np.uint64(37)) & np.uint64(0xfff7eee000000000)
z ^= z >> np.uint64(43)
u = (z >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
same = bool(np.array_equal(u, ref.reshape(-1)[:4096].cpu().numpy()))
print(json.dumps({"draws": total, "ms": ms, "ns_per_draw": ms * 1e6 / total,
                  "us_per_s1_iteration": ms * 1e3 / 200, "matches_sequential_engine": same}))
