#!/bin/bash
# A/B: in-tree library (fp64-exact --fmad=false everywhere but render_fast.cu)
# against ab/fma (every TU --fmad=true) on the fp32 F1 scenes.
for i in 1 2; do
  for v in new fma; do
    if [ $v = new ]; then unset MG_LIB; else export MG_LIB=$PWD/ab/fma/libmgcuda.so; fi
    echo "$v helix $(timeout 300 python tools/helix_probe.py 2>&1 | grep ms/it | head -1)"
    echo "$v c3 $(timeout 300 python tools/mesh_bench_probe.py 2>&1 | grep wavefront | tail -1)"
    echo "$v c4 $(timeout 300 python tools/mesh_large_probe.py 2>&1 | grep ms/it)"
    echo "$v quad $(timeout 300 python tools/quad_graph_probe.py 2>&1 | tail -1)"
  done
done
