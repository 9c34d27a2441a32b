import os, sys, time, json
sys.path.insert(0, "/root/repo")
from paper_2309_15676_b200 import _lib, api, harness
L = _lib.load()
S1 = dict(problem="mini-render", pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0, problem_seed=1)
cfg = api.ExperimentConfig(**S1, replicates=1)
api.run_experiment(cfg)
for R in (1, 8):
    cfg = api.ExperimentConfig(**S1, replicates=R)
    w_dev, w_agg, w_all = [], [], []
    for _ in range(15):
        t0 = time.perf_counter()
        recs = harness._run_device(cfg, 0, R)
        t1 = time.perf_counter()
        harness.aggregate(cfg, recs)
        t2 = time.perf_counter()
        w_dev.append(t1 - t0); w_agg.append(t2 - t1)
        t0 = time.perf_counter(); api.run_experiment(cfg); w_all.append(time.perf_counter() - t0)
    print(json.dumps({"R": R, "dev_ms": sorted(round(x*1e3,2) for x in w_dev), "agg_ms": sorted(round(x*1e3,2) for x in w_agg), "all_ms": sorted(round(x*1e3,2) for x in w_all)}))
