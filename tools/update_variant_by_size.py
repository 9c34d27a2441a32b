"""Fused meta update (fp32): TMA schedule variants by parameter count,
interleaved rounds of 100 state-carrying steps (eager launches, CUDA
events); min and median ms per step."""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import _lib, api  # noqa: E402

L = _lib.load()
dev = torch.device("cuda")
variants = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [8, 9, 2, 3]
for lg in (24, 25, 26, 27, 28):
    m = 1 << lg
    gen = torch.Generator(device=dev).manual_seed(7)
    mu = torch.rand(m, device=dev, generator=gen) * 2 - 1
    sg = torch.rand(m, device=dev, generator=gen) * 1.9 + 0.1
    pr = [mu + sg * torch.randn(m, device=dev, generator=gen) for _ in range(2)]
    df = [0.1 * sg * torch.randn(m, device=dev, generator=gen) for _ in range(2)]
    bufs = [torch.zeros(m, device=dev), torch.empty(m, device=dev)]
    ups = {}
    for v in variants:
        L.mg_set_option(b"tma_variant", v)
        ups[v] = api.FusedMetaUpdate(m, lr=0.01)
        for t in range(4):
            ups[v].step(pr[t % 2], df[t % 2], bufs[t % 2], bufs[(t + 1) % 2])
    res = {v: [] for v in variants}
    steps = 100 if lg <= 26 else 30
    for _ in range(6):
        for v in variants:
            L.mg_set_option(b"tma_variant", v)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for t in range(steps):
                ups[v].step(pr[t % 2], df[t % 2], bufs[t % 2], bufs[(t + 1) % 2])
            b.record()
            torch.cuda.synchronize()
            res[v].append(a.elapsed_time(b) / steps)
    print(json.dumps({"log2n": lg, "ms_min": {str(v): round(min(x), 4) for v, x in res.items()},
                      "ms_median": {str(v): round(statistics.median(x), 4) for v, x in res.items()},
                      "frac_of_6455": {str(v): round(56 * m / min(x) / 1e6 / 6455.6, 3)
                                       for v, x in res.items()}}), flush=True)
    del ups, pr, df, bufs
L.mg_set_option(b"tma_variant", -1)
