#!/bin/bash
# A/B of ab/<variant>/libmgcuda.so builds on the S1 single replicate: wall
# through run_experiment (tools/s1_walls.py) and the cluster kernel's
# duration (ncu launch list), in-tree library first.
for v in new $(ls ab 2>/dev/null); do
  if [ $v = new ]; then unset MG_LIB; else export MG_LIB=$PWD/ab/$v/libmgcuda.so; fi
  echo "$v $(timeout 120 python tools/s1_walls.py 2>&1 | head -1) kernel_ns $(bash tools/s1_kernel_time.sh 2>&1 | tail -1)"
done
