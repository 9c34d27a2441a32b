"""SURVEY.md §8(d) CPU timing plan (iii): the reference's full run_experiment
for the configs[1] stand-in S1 (mini-render, 4096 pixels, spp 2, 200
iterations, meta, lr 0.01, seed 0, problem seed 1) on the host cores
(oracle/_ref/run_experiment: threads = 1 and threads = nproc with as many
replicates), against the device runner on the same configurations.  Prints
one JSON line per measurement (profiles/r01_s1_compare.txt)."""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, ".")
from paper_2309_15676_b200 import _abi, api  # noqa: E402

S1 = dict(problem="mini-render", pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0,
          problem_seed=1)
REF = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "oracle", "_ref",
                   "run_experiment")
nproc = os.cpu_count() or 1
pairs = lambda r: r * 200 * 4096 * 2  # noqa: E731
for reps, threads in ((1, 1), (nproc, nproc)):
    out = subprocess.run([REF, _abi.config_text(**S1, replicates=reps, threads=threads),
                          "/tmp/s1_ref.csv"], capture_output=True, text=True, check=True)
    sec = float(out.stdout.split()[0])
    print(json.dumps({"arm": "reference-cpu", "replicates": reps, "threads": threads,
                      "wall_s": sec, "pairs_per_s": pairs(reps) / sec}), flush=True)
api.run_experiment(api.ExperimentConfig(**S1, replicates=1))  # warm-up (module load, context)
for reps in (1, nproc, 148, 1184):
    t0 = time.time()
    rep = api.run_experiment(api.ExperimentConfig(**S1, replicates=reps))
    wall = time.time() - t0
    print(json.dumps({"arm": "device", "replicates": reps, "wall_s": wall,
                      "pairs_per_s": pairs(reps) / wall,
                      "final_param_err_mean": float(rep.stats["param_err"].mean[-1])}),
          flush=True)
