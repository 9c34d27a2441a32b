import sys, time, statistics
sys.path.insert(0, ".")
from paper_2309_15676_b200 import api
S1 = dict(problem="mini-render", pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0, problem_seed=1)
for R in (1, 8, 1):
    cfg = api.ExperimentConfig(**S1, replicates=R)
    api.run_experiment(cfg)
    w = []
    for _ in range(15):
        t = time.perf_counter(); api.run_experiment(cfg); w.append(time.perf_counter() - t)
    print(R, "median ms", round(statistics.median(w) * 1e3, 3), "min", round(min(w) * 1e3, 3))
