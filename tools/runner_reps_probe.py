"""Replicate-pool throughput of the per-CTA device runner (S1 shape:
mini-render P = 4096, spp 2, 200 iterations, meta) by replicate count:
run_experiment wall (median of 5) and replicate-iterations per second."""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

S1 = dict(problem="mini-render", pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0,
          problem_seed=1)
out = {}
for reps in (32, 148, 296, 592, 1184):
    cfg = api.ExperimentConfig(**S1, replicates=reps)
    api.run_experiment(cfg)
    walls = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        api.run_experiment(cfg)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    w = statistics.median(walls)
    out[reps] = {"wall_ms": round(w * 1e3, 2), "rep_iters_per_s": round(reps * 200 / w)}
print(json.dumps(out), flush=True)
