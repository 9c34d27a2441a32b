"""In-process A/B of mg_set_option("helix_split") on configs[2] (256^2 helix,
fp32 and fp64): the sample pair of both settings on the same parameters must
be identical (fixed-point sums; the loss within 1e-12), then interleaved
timing of full iterations (sample pair + fused update), CUDA events."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2309_15676_b200 import _lib, api  # noqa: E402

L = _lib.load()
for dt in (torch.float32, torch.float64):
    prob = api.HelixProblem(256, 256, target_spp=16, dtype=dt)
    run = api.HelixRun(prob, "meta", lr=0.01)
    for _ in range(3):
        run.step()
    pairs = []
    for v in (0, 1):
        L.mg_set_option(b"helix_split", v)
        pr = prob.sample_pair(run.params, run.prev, 7, run.key)
        torch.cuda.synchronize()
        pairs.append((pr.prop.clone(), pr.diff.clone(), float(prob.loss_buf[0])))
    same = torch.equal(pairs[0][0], pairs[1][0]) and torch.equal(pairs[0][1], pairs[1][1])
    res = {0: [], 1: []}
    for _ in range(4):
        for v in (0, 1):
            L.mg_set_option(b"helix_split", v)
            run.step()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                run.step()
            b.record()
            torch.cuda.synchronize()
            res[v].append(a.elapsed_time(b) / 20)
    L.mg_set_option(b"helix_split", 1)
    print(json.dumps({"dtype": str(dt), "identical_pair": same,
                      "loss": [pairs[0][2], pairs[1][2]],
                      "ms": {"one_kernel": min(res[0]), "split": min(res[1])}}), flush=True)
