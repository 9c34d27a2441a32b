"""S1 single-replicate wall time inside a loaded process (as bench.py's
extras see it): ~16 GB of torch tensors resident and a configs[4] scene
built, stepped and freed first; pool release threshold 0 vs 512 MiB."""
import sys, time, statistics
sys.path.insert(0, ".")
import torch
from paper_2309_15676_b200 import api, _lib
lib = _lib.load()
S1 = dict(problem="mini-render", pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0, problem_seed=1)
ctx = api.Context(0)
cfg = api.ExperimentConfig(**S1, replicates=1)
def s1(tag):
    for keep in (0, 512 << 20):
        lib.mg_set_option(b"pool_keep_bytes", keep)
        api.run_experiment(cfg, ctx=ctx)
        w = []
        for _ in range(7):
            t = time.perf_counter(); api.run_experiment(cfg, ctx=ctx); w.append(time.perf_counter() - t)
        print(tag, f"keep={keep >> 20}MiB median {statistics.median(w)*1e3:.3f} ms min {min(w)*1e3:.3f}", flush=True)
s1("fresh")
big = [torch.empty(1 << 28, device="cuda") for _ in range(15)]
s1("16GB resident")
prob = api.MeshLargeProblem(target_spp=2, ctx=ctx)
run = api.MeshTextureRun(prob, optimizer="meta", lr=0.005)
for _ in range(3):
    run.step()
torch.cuda.synchronize()
s1("mesh scene live")
del run, prob
torch.cuda.empty_cache()
s1("after mesh freed")
