"""configs[1]'s smaller sizes (2^20, 2^24 fp32): the fused meta update per
TMA schedule variant and the register kernel, 100 state-carrying steps
replayed as one CUDA graph (us per step)."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import _lib, api  # noqa: E402

L = _lib.load()
dev = torch.device("cuda")
side = torch.cuda.Stream(device=dev)
ctx = api.Context(0, stream=side)
for m in (1 << 20, 1 << 22, 1 << 24):
    gen = torch.Generator(device=dev).manual_seed(7)
    mu = torch.rand(m, device=dev, generator=gen) * 2 - 1
    sg = torch.rand(m, device=dev, generator=gen) * 1.9 + 0.1
    pr = [mu + sg * torch.randn(m, device=dev, generator=gen) for _ in range(2)]
    df = [0.1 * sg * torch.randn(m, device=dev, generator=gen) for _ in range(2)]
    bufs = [torch.zeros(m, device=dev), torch.empty(m, device=dev)]
    res = {}
    for variant in list(range(10)) + ["reg"]:
        if variant == "reg":
            L.mg_set_option(b"disable_tma", 1)
        else:
            L.mg_set_option(b"disable_tma", 0)
            L.mg_set_option(b"tma_variant", variant)
        up = api.FusedMetaUpdate(m, lr=0.01, ctx=ctx)
        torch.cuda.synchronize()
        with torch.cuda.stream(side):
            for t in range(4):
                up.step(pr[t % 2], df[t % 2], bufs[t % 2], bufs[(t + 1) % 2])
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            up.reset()
            with torch.cuda.graph(g, stream=side):
                for t in range(100):
                    up.step(pr[t % 2], df[t % 2], bufs[t % 2], bufs[(t + 1) % 2])
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(side)
            for _ in range(5):
                g.replay()
            b.record(side)
            torch.cuda.synchronize()
        res[str(variant)] = round(a.elapsed_time(b) / 500 * 1e3, 2)
        del g, up
    print(json.dumps({"params": m, "us_per_step": res}), flush=True)
L.mg_set_option(b"disable_tma", 0)
L.mg_set_option(b"tma_variant", -1)
