"""SURVEY.md §8(d) CPU timing plan (iii): the reference's full run_experiment
for the configs[0] stand-in S1 (mini-render, 4096 pixels, spp 2, 200
iterations, meta, lr 0.01, seed 0, problem seed 1) on the host cores
(oracle/_ref/run_experiment: threads = 1 and threads = nproc with as many
replicates), against the device runs of the same configurations through
api.run_experiment (wall clock around the call, median of 9 after one warm-up): the
one-replicate-per-cluster runner (default for few replicates) and the
one-CTA-per-replicate runner (mg_set_option cluster_runner 0).  Prints one
JSON line per measurement."""
import json
import os
import statistics
import subprocess
import sys
import time

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2309_15676_b200 import _abi, _lib, api  # noqa: E402

S1 = dict(problem="mini-render", pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0,
          problem_seed=1)
REF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle", "_ref",
                   "run_experiment")
nproc = os.cpu_count() or 1
pairs = lambda r: r * 200 * 4096 * 2  # noqa: E731
L = _lib.load()
api.run_experiment(api.ExperimentConfig(**S1, replicates=1))  # warm-up (module load, context)
for runner in ("cluster", "cta"):
    L.mg_set_option(b"cluster_runner", 1 if runner == "cluster" else 0)
    for reps in (1, 8, nproc, 148):
        api.run_experiment(api.ExperimentConfig(**S1, replicates=reps))  # warm this shape
        walls = []
        for _ in range(9):
            t0 = time.time()
            rep = api.run_experiment(api.ExperimentConfig(**S1, replicates=reps))
            walls.append(time.time() - t0)
        wall = statistics.median(walls)
        print(json.dumps({"arm": "device", "runner": runner, "replicates": reps, "wall_s": wall,
                          "pairs_per_s": pairs(reps) / wall,
                          "final_param_err_mean": float(rep.stats["param_err"].mean[-1])}),
              flush=True)
L.mg_set_option(b"cluster_runner", 1)
# the reference last: its 16-thread runs perturb the host for a moment
if os.path.exists(REF):
    for reps, threads in ((1, 1), (nproc, nproc)):
        secs = []
        for _ in range(3):
            out = subprocess.run([REF, _abi.config_text(**S1, replicates=reps, threads=threads),
                                  "/tmp/s1_ref.csv"], capture_output=True, text=True, check=True)
            secs.append(float(out.stdout.split()[0]))
        sec = statistics.median(secs)
        print(json.dumps({"arm": "reference-cpu", "replicates": reps, "threads": threads,
                          "wall_s": sec, "pairs_per_s": pairs(reps) / sec}), flush=True)
