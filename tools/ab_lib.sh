#!/bin/bash
# Interleaved A/B of the in-tree library against ab/<variant>/libmgcuda.so
# builds: configs[4] and configs[3] iteration times (mesh probes).
for i in 1 2; do
  for v in new $(ls ab 2>/dev/null); do
    if [ $v = new ]; then unset MG_LIB; else export MG_LIB=$PWD/ab/$v/libmgcuda.so; fi
    echo "$v c4 $(timeout 300 python tools/mesh_large_probe.py 2>&1 | grep ms/it)"
    echo "$v c3 $(timeout 300 python tools/mesh_bench_probe.py 2>&1 | grep wavefront | tail -1)"
  done
done
