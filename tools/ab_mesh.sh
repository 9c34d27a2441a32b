#!/bin/bash
# A/B timing of mesh builds on the GPU box: in-tree library ("new") against
# every ab/<variant>/libmgcuda.so; configs[4] and configs[3] iteration times.
# Optional first argument: pytest targets to run first (in-tree build).
mkdir -p gpurun_out
if [ -n "${1:-}" ]; then
  timeout 900 python -m pytest $1 -x -q > gpurun_out/ab_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/ab_tests.log
  tail -2 gpurun_out/ab_tests.log
fi
for i in 1 2; do
  for v in new $(ls ab 2>/dev/null); do
    if [ $v = new ]; then unset MG_LIB; else export MG_LIB=$PWD/ab/$v/libmgcuda.so; fi
    echo "$v c4 $(timeout 300 python tools/mesh_large_probe.py 2>&1 | grep ms/it)"
    echo "$v c3 $(timeout 300 python tools/mesh_bench_probe.py 2>&1 | grep wavefront | tail -1)"
  done
done
