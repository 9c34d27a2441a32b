#!/bin/bash
# ncu launch durations of the S1 single-replicate run (cluster runner).
cat > /tmp/s1k.py <<'PY'
import sys
sys.path.insert(0, ".")
from paper_2309_15676_b200 import api
S1 = dict(problem="mini-render", pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0, problem_seed=1)
for _ in range(3):
    api.run_experiment(api.ExperimentConfig(**S1, replicates=1))
PY
ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:run_ --log-file /tmp/s1k.csv python /tmp/s1k.py > /dev/null 2>&1
python -c "import csv; [print(r[4][:40], r[-1]) for r in csv.reader(open('/tmp/s1k.csv')) if len(r) > 10 and 'run_' in r[4]]"
