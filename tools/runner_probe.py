"""One S1 replicate on the device runner (for ncu)."""
import sys

sys.path.insert(0, ".")
from paper_2309_15676_b200 import api  # noqa: E402

cfg = api.ExperimentConfig(problem="mini-render", pixel_count=4096, spp=2, iterations=200,
                           lr=0.01, seed=0, problem_seed=1, replicates=1)
api.run_experiment(cfg)
api.run_experiment(cfg)
