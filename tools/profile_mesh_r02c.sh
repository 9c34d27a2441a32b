#!/bin/bash
# Run ON THE GPU BOX: configs[4] after the per-vertex record layout — plain
# timing and the per-launch metric list over whole iterations (for
# tools/mesh_stage_table.py), per-launch rows of the last iteration.
set -u
mkdir -p gpurun_out
CMD="python tools/mesh_large_probe.py"
timeout 600 $CMD > gpurun_out/pc_plain.log 2>&1 || { cat gpurun_out/pc_plain.log; exit 1; }
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__thread_inst_executed_per_inst_executed.ratio,sm__warps_active.avg.pct_of_peak_sustained_active
timeout 1200 ncu --metrics $M --clock-control none --csv -k regex:'wf_|mesh_|meta_update|tex_ilv' \
  --log-file gpurun_out/pc_launches.csv $CMD > /dev/null 2>&1
python tools/mesh_stage_table.py gpurun_out/pc_launches.csv > gpurun_out/pc_stage_table.md
python tools/launch_table.py gpurun_out/pc_launches.csv 17 > gpurun_out/pc_last_iteration.txt 2>&1
cat gpurun_out/pc_plain.log gpurun_out/pc_stage_table.md
