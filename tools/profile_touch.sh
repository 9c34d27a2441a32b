#!/bin/bash
# Run ON THE GPU BOX: one `--set full` capture of the touch-map fused update
# inside a configs[4] iteration.
set -u
mkdir -p gpurun_out
CMD="python tools/mesh_large_probe.py"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:meta_update_fixed -s 3 -c 1 \
  -o /tmp/pt_update -f $CMD > gpurun_out/pt_ncu.log 2>&1
ncu -i /tmp/pt_update.ncu-rep --page details > gpurun_out/pt_update_details.txt 2>&1
ncu -i /tmp/pt_update.ncu-rep --page raw --csv --metrics \
  dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__registers_per_thread \
  > gpurun_out/pt_update_raw.csv 2>&1
cp /tmp/pt_update.ncu-rep gpurun_out/pt_update.ncu-rep
tail -3 gpurun_out/pt_update_raw.csv
