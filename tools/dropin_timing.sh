#!/bin/bash
# The zero-patch drop-in route timed against the reference on the same box
# (VERDICT r01 #9): the reference's own run_experiment (S1: mini-render
# 4096 px, spp 2, 200 iterations, meta) and acceptance criterion 9, built
# (a) from the unmodified reference over its own estimators (oracle/_ref)
# and (b) over the B200-backed drop-in headers (tests/cpp/_build/dropin:
# every Moment2 / MetaEstimator / Adam call packs its operands, copies
# them to the GPU, launches, copies back).  Run ON THE GPU BOX; prints one
# line per measurement (median of 3).
S1=$(python -c "import sys; sys.path.insert(0,'.'); from paper_2309_15676_b200 import _abi; print(_abi.config_text(problem='mini-render', pixel_count=4096, spp=2, iterations=200, lr=0.01, seed=0, problem_seed=1, replicates=1, threads=1))")
for arm in oracle/_ref tests/cpp/_build/dropin; do
  for i in 1 2 3; do
    $arm/run_experiment "$S1" /tmp/dropin_s1.csv | awk -v a=$arm '{print "run_experiment S1", a, $1}'
  done | sort -k4 -n | sed -n 2p
  for i in 1 2 3; do
    $arm/acceptance 9 2>&1 | grep -o "([0-9.e+-]* s)" | tr -d '(s)' | awk -v a=$arm '{print "acceptance 9", a, $1}'
  done | sort -k4 -n | sed -n 2p
done
