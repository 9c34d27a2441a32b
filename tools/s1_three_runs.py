import sys
sys.path.insert(0, ".")
from paper_2309_15676_b200 import api
S1 = dict(problem="mini-render", pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0, problem_seed=1)
for _ in range(3):
    api.run_experiment(api.ExperimentConfig(**S1, replicates=1))
