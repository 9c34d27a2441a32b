#!/bin/bash
# Run ON THE GPU BOX: `--set full` captures of the configs[4] stage kernels
# at HEAD (depth-0 isect / shade / shadow, the tail, the scatter); details
# pages into gpurun_out/ph_*.txt.
set -u
mkdir -p gpurun_out
CMD="python tools/mesh_large_probe.py"
for k in wf_isect:16 wf_shade_kernel:16 wf_shadow:16 wf_tail:4 wf_scatter:4; do
  name=${k%%:*}; skip=${k##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$name -s $skip -c 1 \
    -o /tmp/ph_$name -f $CMD > gpurun_out/ph_ncu_$name.log 2>&1
  ncu -i /tmp/ph_$name.ncu-rep --page details > gpurun_out/ph_${name}_details.txt 2>&1
done
grep -H "Duration\|DRAM Throughput\|Issue Slots Busy\|Registers Per Thread\|Achieved Occupancy\|Avg. Active Threads Per Warp" gpurun_out/ph_*_details.txt
