#!/bin/bash
# Run ON THE GPU BOX: configs[3] plain timing and per-launch metric list of
# the last iteration.
set -u
mkdir -p gpurun_out
CMD="python tools/mesh_c3_probe.py"
timeout 600 $CMD > gpurun_out/p3_plain.log 2>&1 || { cat gpurun_out/p3_plain.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 1200 ncu --metrics $M --clock-control none --csv -k regex:'wf_|mesh_|meta_update|tex_ilv' \
  --log-file gpurun_out/p3_launches.csv $CMD > /dev/null 2>&1
python tools/mesh_stage_table.py gpurun_out/p3_launches.csv > gpurun_out/p3_stage_table.md
python tools/launch_table.py gpurun_out/p3_launches.csv 14 > gpurun_out/p3_last_iteration.txt 2>&1
cat gpurun_out/p3_plain.log gpurun_out/p3_stage_table.md
