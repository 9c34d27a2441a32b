"""S1 single-replicate wall time through run_experiment, split into the
device runner call (mg_run_replicates) and the host aggregation, with the
default pool's release threshold at 0 (CUDA default) and at 512 MiB."""
import sys, time, statistics
sys.path.insert(0, ".")
import torch
from paper_2309_15676_b200 import api, harness, _lib
S1 = dict(problem="mini-render", pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0, problem_seed=1)
lib = _lib.load()
cfg = api.ExperimentConfig(**S1, replicates=1)
for keep in (0, 512 << 20, 0, 512 << 20):
    lib.mg_set_option(b"pool_keep_bytes", keep)
    api.run_experiment(cfg)
    w, d, a = [], [], []
    for _ in range(15):
        t0 = time.perf_counter()
        recs = harness._run_device(cfg, 0, 1)
        t1 = time.perf_counter()
        harness.aggregate(cfg, recs)
        t2 = time.perf_counter()
        d.append(t1 - t0); a.append(t2 - t1); w.append(t2 - t0)
    med = lambda x: round(statistics.median(x) * 1e3, 3)
    print(f"keep={keep >> 20} MiB: wall {med(w)} ms (min {round(min(w)*1e3,3)}), runner call {med(d)} ms, aggregate {med(a)} ms", flush=True)
